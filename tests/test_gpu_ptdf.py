"""GPU parity of the dense-PTDF form (DCOPF_FORM_PTDF on DCOPF_PATH_DENSE;
SURVEY.md NEXT-4) against the numpy oracle oracle/ptdf.py, at the north_star
tolerances (1e-9 relative on the bound, reading A-17; 1e-8 normalised max-abs
on the multipliers, reading A-18).

Not bitwise: the GPU sums the PTDF products in DMMA tile order and builds H_a
by the cycle method, the oracle uses numpy's matmul and solve (reading A-30).
The library's H_a is also checked on its own against Kirchhoff's laws.
"""
from types import SimpleNamespace

import numpy as np
import pytest

import oracle
from oracle import ptdf as P
from paper_2406_13191_b200 import dual
from paper_2406_13191_b200 import instances as inst

from gpu_helpers import BOUND_RTOL, MULT_TOL, assert_parity, cost_scale, run_gpu

pytestmark = pytest.mark.gpu

ADAM = dict(variant=P.OPT_ADAM, beta1=0.9, beta2=0.999, eps=1e-8)
GDM = dict(variant=P.OPT_GDM, rho=0.9)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dual.load_library()


def _orc(net, loads, K, alpha, Ha=None, **kw):
    r = P.solve(net, loads, K, alpha, Ha=Ha, history=True, **kw)
    return SimpleNamespace(lam=r.lam[:, None], br=r.mu, bound=r.bound, best=r.best, status=r.status, hist=r.hist)


def _gpu(net, loads, K, alpha, **kw):
    return run_gpu(net, loads, K=K, alpha=alpha, form=dual.FORM_PTDF, path=dual.PATH_DENSE, history=True, **kw)


def _lib_ptdf(net):
    h = dual.DcopfDual(net, form=dual.FORM_PTDF, path=dual.PATH_DENSE)
    H = h.get_ptdf()
    h.close()
    return H


def _scaled_loads(net, B, seed):
    rng = np.random.default_rng(seed)
    return net.base_load[None, :] * rng.uniform(0.85, 1.15, (B, 1))


def _with_open_branch(net):
    b = net.br_b.copy()
    b[net.n_tree + 1] = 0.0   # a non-tree branch with b = 0 (open circuit)
    return inst.Network(**{**net.__dict__, "br_b": b})


# ---------------------------------------------------------------------------
# the PTDF matrix


@pytest.mark.parametrize("which", ["config0", "config1", "radial", "open_branch", "multi_gen"])
def test_ptdf_matrix(which):
    if which == "config0":
        net = inst.make_network(0)
    elif which == "config1":
        net = inst.make_network(1)
    elif which == "radial":
        net = inst.tiny_network(40, 39, 6, 3)
    elif which == "open_branch":
        net = _with_open_branch(inst.tiny_network(30, 50, 8, 5))
    else:
        net = inst.tiny_network(23, 40, 30, 9)
    H = _lib_ptdf(net)
    Ho = P.ptdf(net)
    assert np.max(np.abs(H - Ho)) <= 1e-11 * max(1.0, np.max(np.abs(Ho)))
    np.testing.assert_array_equal(H == 0.0, Ho == 0.0)  # the same structural zeros, exactly (reading A-30)
    # on its own: zero slack column, KCL (E^T H = I - e_ref 1^T over b > 0), KVL on the C oracle's cycles
    assert np.all(H[:, net.ref_bus] == 0.0)
    E = P.incidence(net) * (net.br_b > 0)[:, None]
    want = np.eye(net.n_bus)
    want[net.ref_bus, :] -= 1.0
    assert np.max(np.abs(E.T @ H - want)) <= 1e-10
    assert np.all(H[net.br_b == 0.0] == 0.0)
    _, cyc = oracle.cycles(net)
    for br, sg in cyc:
        if np.all(net.br_b[br] > 0):
            assert np.max(np.abs((sg[:, None] * H[br] / net.br_b[br][:, None]).sum(0))) <= 1e-11


# ---------------------------------------------------------------------------
# the iteration


@pytest.mark.parametrize("skinny,fused", [("1", "1"), ("1", "0"), ("0", "1")])
def test_config0_full_K(skinny, fused, monkeypatch):
    """B = 1: the single-read step (default), the two-pass matrix-vector
    kernels (skinny mode without it) and, forced, the GEMM kernels on a
    128-column tile."""
    monkeypatch.setenv("DCOPF_PTDF_SKINNY", skinny)
    monkeypatch.setenv("DCOPF_PTDF_FUSED", fused)
    net = inst.make_network(0)
    K = inst.ITERS[0]
    a = inst.alpha_schedule(K)
    gpu = _gpu(net, net.base_load[None], K, a)
    orc = _orc(net, net.base_load[None], K, a)
    assert_parity(net, gpu, orc)
    info = gpu["info"]
    assert info.path == dual.PATH_DENSE and info.form == dual.FORM_PTDF


@pytest.mark.parametrize("which", ["config3_gdm", "config3_plain", "config3_adam", "config3_adagrad",
                                   "config2_quadratic", "config1_warm"])
def test_single_read_step(which):
    """B = 1 on the single-read step (every step variant: AdaGrad / Adam on the
    branch-free fp64 division / square root since round 2): config 3's H_g
    (2 500 generator columns: two 20 KB rows per group, 148 CTAs of ~86
    lines) over several calls; the quadratic config-2 network; a warm start
    from random multipliers (Q_0 from the set nu) followed by the two-pass
    evaluate()."""
    import torch
    if which.startswith("config3"):
        net = inst.make_network(3)
        opt, alpha = {"config3_gdm": (GDM, 1e-3), "config3_plain": (None, 2e-3), "config3_adam": (ADAM, 0.5),
                      "config3_adagrad": (dict(variant=P.OPT_ADAGRAD, eps=1e-8), 0.5)}[which]
        K = 60
        a = inst.alpha_schedule(K, alpha)
        loads = net.base_load[None]
        gpu = _gpu(net, loads, K, a, opt=opt, split=25)
        orc = _orc(net, loads, K, a, opt=opt)
        assert gpu["info"].smem_bytes > 0  # the single-read kernels ran
        assert_parity(net, gpu, orc)
        return
    if which == "config2_quadratic":
        net = inst.make_network(2, quadratic=True)
        K, a = 300, inst.alpha_schedule(300)
        loads = _scaled_loads(net, 1, 6)
        gpu = _gpu(net, loads, K, a, split=110)
        orc = _orc(net, loads, K, a)
        assert_parity(net, gpu, orc)
        return
    net = inst.make_network(1)
    Ha = P.ptdf(net)
    rng = np.random.default_rng(9)
    loads = _scaled_loads(net, 1, 3)
    lam = rng.normal(0, 20, 1)
    mu = np.abs(rng.normal(0, 5, (1, 2 * net.n_branch))) * (rng.random((1, 2 * net.n_branch)) < 0.3)
    h = dual.DcopfDual(net, form=dual.FORM_PTDF)
    h.set_instance_batch(torch.from_numpy(np.ascontiguousarray(loads.T)).to(torch.device("cuda:0")))
    h.set_multipliers(np.ascontiguousarray(lam[None, :]), np.ascontiguousarray(mu.T))
    K = 80
    a = inst.alpha_schedule(K, 1e-3)
    h.set_optimizer(P.OPT_GDM, GDM["rho"])
    h.iterate(30, a[:30])
    h.iterate(K - 30, a[30:])
    bound, best, status, l2, b2 = h.results_numpy()
    val = np.empty(1)
    h.evaluate(val)  # the two-pass evaluate() after the single-read steps (nu_c kept current)
    h.close()
    r = P.solve(net, loads, K, a, Ha=Ha, lam0=lam, mu0=mu, opt=GDM)
    S = cost_scale(net)
    assert np.all(np.abs(bound - r.bound) <= BOUND_RTOL * np.maximum(np.abs(r.bound), S))
    assert np.all(np.abs(val - bound) <= BOUND_RTOL * np.maximum(np.abs(bound), S))
    y_g = np.concatenate([l2.T, b2.T], axis=1)
    y_o = np.concatenate([r.lam[:, None], r.mu], axis=1)
    assert np.max(np.abs(y_g - y_o) / np.maximum(1.0, np.abs(y_o).max(axis=1, keepdims=True))) <= MULT_TOL


def _no_flow_lines(net, Ha, loads):
    """Lines that carry no flow in any instance of the batch: a zero H_g row,
    zero load flow r = H_a d and a zero limit F -- exactly zero on both sides
    (structural zeros of H_a and literal zero limits, readings A-11 / A-30), so
    their gradient is exactly 0 and Adam / AdaGrad leave their mu at exactly 0."""
    Hg = Ha[:, net.gen_bus]
    r = np.abs(loads @ Ha.T).max(axis=0)
    m = (np.abs(Hg).max(axis=1) == 0.0) & (r == 0.0) & (net.br_fmax == 0.0)
    return np.r_[m, m]


@pytest.mark.parametrize("B", [1, 2, 3, 9])
def test_skinny_batches_config1_adam(B):
    """Skinny mode at every column count class (1, 2, 4 columns computed), and
    B = 9 on the split-K GEMMs, Adam."""
    net = inst.make_network(1)
    Ha = P.ptdf(net)
    K = 300
    a = inst.alpha_schedule(K, 0.1)
    loads = _scaled_loads(net, B, 17)
    gpu = _gpu(net, loads, K, a, opt=ADAM, split=120)
    orc = _orc(net, loads, K, a, Ha=Ha, opt=ADAM)
    noflow = _no_flow_lines(net, Ha, loads)
    assert 0 < noflow.sum() < 0.05 * noflow.size
    assert_parity(net, gpu, orc)  # every multiplier, the no-flow lines' included
    assert np.all(gpu["br"][:, noflow] == 0.0) and np.all(orc.br[:, noflow] == 0.0)


@pytest.mark.parametrize("B", [1, 130, 300])
def test_config1_batch_ragged(B):
    """Several 128-instance tiles and a ragged tail; M tiles over 3200 lines / 540 generators."""
    net = inst.make_network(1)
    Ha = P.ptdf(net)
    K = 200
    a = inst.alpha_schedule(K)
    loads = _scaled_loads(net, B, 11)
    gpu = _gpu(net, loads, K, a)
    idx = np.unique(np.r_[0, B - 1, np.linspace(0, B - 1, 6).astype(int)])
    orc = _orc(net, loads[idx], K, a, Ha=Ha)
    assert_parity(net, gpu, orc, idx=idx)


def test_quadratic_config2_network():
    """alpha = 1e-3 (reading A-9): the trajectory is well conditioned (a 1e-15
    perturbation of H_a stays at 1e-16 relative after 60 steps; at alpha = 0.05
    one instance amplifies it to 3e-7, reading A-30)."""
    net = inst.make_network(2, quadratic=True)
    K = 200
    a = inst.alpha_schedule(K)
    loads = _scaled_loads(net, 3, 5)
    gpu = _gpu(net, loads, K, a)
    orc = _orc(net, loads, K, a)
    assert_parity(net, gpu, orc)


@pytest.mark.parametrize("opt,alpha", [(ADAM, 0.05), (GDM, 1e-3),
                                       (dict(variant=P.OPT_GDM_CLASSIC, rho=0.5), 1e-3),
                                       (dict(variant=P.OPT_ADAGRAD, eps=1e-8), 0.5)])
def test_optimizers(opt, alpha):
    net = inst.tiny_network(60, 95, 14, 21)
    K = 400
    a = inst.alpha_schedule(K, alpha)
    loads = _scaled_loads(net, 140, 3)
    gpu = _gpu(net, loads, K, a, opt=opt, split=150)
    orc = _orc(net, loads, K, a, opt=opt)
    assert_parity(net, gpu, orc)


def test_divergence_and_stopping_rule():
    net = inst.tiny_network(14, 19, 5, 0)
    loads = _scaled_loads(net, 3, 1)
    K = 40
    a = np.full(K, 1e16)
    gpu = _gpu(net, loads, K, a)
    orc = _orc(net, loads, K, a)
    assert np.all(orc.status == P.DIVERGED)
    np.testing.assert_array_equal(gpu["status"], orc.status)
    np.testing.assert_array_equal(np.isfinite(gpu["best"]), np.isfinite(orc.best))
    # stopping rule: a tolerance between the smallest and the second smallest
    # per-instance min |g_k - g_{k-1}| fires for exactly one instance; no
    # difference lies within 1e-6 (relative) of it, far above the GPU/oracle gap
    K = 300
    a = inst.alpha_schedule(K)
    full = _orc(net, loads, K, a)
    d = np.abs(np.diff(full.hist, axis=1))
    m = np.sort(d.min(axis=1))
    tol = float(np.sqrt(m[0] * m[1]))
    assert m[1] / m[0] > 1.01 and np.min(np.abs(d / tol - 1.0)) > 1e-6
    gpu = _gpu(net, loads, K, a, tol=tol)
    orc = _orc(net, loads, K, a, tol=tol)
    assert np.sum(orc.status == P.CONVERGED) == 1
    assert_parity(net, gpu, orc, check_hist=False)


def test_evaluate_at_random_point_and_warm_start():
    import torch
    net = inst.make_network(1)
    Ha = P.ptdf(net)
    B = 5
    rng = np.random.default_rng(8)
    loads = _scaled_loads(net, B, 2)
    lam = rng.normal(0, 20, B)
    mu = np.abs(rng.normal(0, 5, (B, 2 * net.n_branch))) * (rng.random((B, 2 * net.n_branch)) < 0.3)
    h = dual.DcopfDual(net, form=dual.FORM_PTDF)
    dev = torch.device("cuda:0")
    h.set_instance_batch(torch.from_numpy(np.ascontiguousarray(loads.T)).to(dev))
    h.set_multipliers(np.ascontiguousarray(lam[None, :]), np.ascontiguousarray(mu.T))
    val = np.empty(B)
    gl = np.empty((1, B))
    gb = np.empty((2 * net.n_branch, B))
    h.evaluate(val, gl, gb)
    ev = P.evaluate(net, Ha, loads, lam, mu[:, :net.n_branch], mu[:, net.n_branch:])
    S = cost_scale(net)
    assert np.all(np.abs(val - ev.value) <= BOUND_RTOL * np.maximum(np.abs(ev.value), S))
    gmu = np.concatenate([ev.g_mup, ev.g_mum], axis=1)
    sc = max(1.0, np.max(np.abs(gmu)))
    assert np.max(np.abs(gb.T - gmu)) <= 1e-11 * sc
    assert np.max(np.abs(gl[0] - ev.g_lam)) <= 1e-11 * max(1.0, np.max(np.abs(ev.g_lam)))
    # warm start: 50 steps from that point
    K = 50
    a = inst.alpha_schedule(K)
    h.iterate(K, a)
    bound, best, status, l2, b2 = h.results_numpy()
    r = P.solve(net, loads, K, a, Ha=Ha, lam0=lam, mu0=mu)
    assert np.all(np.abs(bound - r.bound) <= BOUND_RTOL * np.maximum(np.abs(r.bound), S))
    y_g = np.concatenate([l2.T, b2.T], axis=1)
    y_o = np.concatenate([r.lam[:, None], r.mu], axis=1)
    assert np.max(np.abs(y_g - y_o) / np.maximum(1.0, np.abs(y_o).max(axis=1, keepdims=True))) <= MULT_TOL
    # mu < 0 in a warm start is rejected
    bad = mu.copy()
    bad[0, 3] = -1.0
    with pytest.raises(dual.DcopfError):
        h.set_multipliers(None, np.ascontiguousarray(bad.T))
    h.close()


def test_first_hit():
    import torch
    net = inst.make_network(0)
    K = 2000
    a = inst.alpha_schedule(K)
    orc = P.solve(net, net.base_load[None], K, a, history=True)
    run = np.maximum.accumulate(orc.hist[0])
    target = run[K // 2] - 1e-9 * abs(run[K // 2])
    want = int(np.argmax(run >= target))
    h = dual.DcopfDual(net, form=dual.FORM_PTDF)
    h.set_instance_batch(np.ascontiguousarray(net.base_load[:, None]))
    h.set_target(np.array([target]))
    h.iterate(700, a[:700])
    h.iterate(K - 700, a[700:])
    assert int(h.get_first_hit()[0]) == want
    h.close()


def test_edge_cases():
    # single bus (no branch), a radial network (no cycle), one instance
    one = inst.Network(n_bus=1, n_branch=0, n_gen=2, ref_bus=0, br_from=np.zeros(0, np.int32),
                       br_to=np.zeros(0, np.int32), br_b=np.zeros(0), br_fmax=np.zeros(0),
                       theta_max=np.zeros(1), gen_bus=np.zeros(2, np.int32), gen_pmin=np.zeros(2),
                       gen_pmax=np.array([1.0, 2.0]), gen_c=np.array([10.0, 20.0]), base_load=np.array([1.5]))
    for net in (one, inst.tiny_network(40, 39, 6, 3), _with_open_branch(inst.tiny_network(30, 50, 8, 5))):
        K = 300
        a = inst.alpha_schedule(K, 0.01)
        loads = _scaled_loads(net, 2, 4)
        gpu = _gpu(net, loads, K, a)
        orc = _orc(net, loads, K, a)
        assert_parity(net, gpu, orc)


def test_rejects_outages_and_wrong_path():
    net = inst.make_network(0)
    h = dual.DcopfDual(net, form=dual.FORM_PTDF)
    with pytest.raises(dual.DcopfError):
        h.set_instance_batch(np.ascontiguousarray(net.base_load[:, None]), np.array([[3]], np.int32))
    h.set_instance_batch(np.ascontiguousarray(net.base_load[:, None]), np.array([[-1]], np.int32))
    h.close()
    with pytest.raises(dual.DcopfError):
        dual.DcopfDual(net, form=dual.FORM_PTDF, path=dual.PATH_BATCHED)
    with pytest.raises(dual.DcopfError):
        dual.DcopfDual(net, form=dual.FORM_F2, path=dual.PATH_DENSE)


# ---------------------------------------------------------------------------
# the bench configuration: config 4b (8192 load scenarios of the 10 000-bus
# network, one factor each), sampled instances against the oracle


def test_config4b_full_size_sampled():
    """config 4b at its full size (8192 instances, the GEMM kernels) for 200
    steps, sampled instances against the oracle."""
    import torch
    net = inst.make_network(3)
    ids = np.arange(inst.CONFIG4_BATCH)
    batch = inst.config4_batch(net, ids, variant="4b")
    K = 200
    a = inst.alpha_schedule(K)
    gpu = _gpu(net, batch.load, K, a)
    idx = np.array([0, 1, 127, 128, 4095, 8191])
    orc = _orc(net, batch.load[idx], K, a)
    assert_parity(net, gpu, orc, idx=idx)
    assert gpu["info"].B_padded == inst.CONFIG4_BATCH


def test_decay_schedule_single_instance():
    """The schedule that gives the fastest time to gap on one instance (Adam,
    alpha_k = 5 / (1 + k/200)): skinny mode against the oracle."""
    net = inst.make_network(0)
    K = 2000
    a = inst.alpha_schedule(K, 5.0, "inv:200")
    loads = _scaled_loads(net, 2, 23)
    gpu = _gpu(net, loads, K, a, opt=ADAM, split=700)
    orc = _orc(net, loads, K, a, opt=ADAM)
    assert_parity(net, gpu, orc)


def test_evaluate_gemm_mode_and_rejections():
    """evaluate() on the GEMM kernels (B > 4) against the oracle; set_multipliers
    rejects NaN and mu < 0; compaction is not offered for the PTDF form."""
    import torch
    net = inst.make_network(0)
    Ha = P.ptdf(net)
    B = 40
    rng = np.random.default_rng(31)
    loads = _scaled_loads(net, B, 9)
    lam = rng.normal(0, 20, B)
    mu = np.abs(rng.normal(0, 5, (B, 2 * net.n_branch)))
    h = dual.DcopfDual(net, form=dual.FORM_PTDF)
    h.set_instance_batch(torch.from_numpy(np.ascontiguousarray(loads.T)).to("cuda:0"))
    h.set_multipliers(np.ascontiguousarray(lam[None, :]), np.ascontiguousarray(mu.T))
    val, gl, gb = np.empty(B), np.empty((1, B)), np.empty((2 * net.n_branch, B))
    h.evaluate(val, gl, gb)
    ev = P.evaluate(net, Ha, loads, lam, mu[:, :net.n_branch], mu[:, net.n_branch:])
    S = cost_scale(net)
    assert np.all(np.abs(val - ev.value) <= BOUND_RTOL * np.maximum(np.abs(ev.value), S))
    assert np.max(np.abs(gb.T - np.concatenate([ev.g_mup, ev.g_mum], axis=1))) <= 1e-11 * max(1.0, np.abs(gb).max())
    assert np.max(np.abs(gl[0] - ev.g_lam)) <= 1e-11 * max(1.0, np.abs(ev.g_lam).max())
    bad = mu.copy()
    bad[3, 2] = np.nan
    with pytest.raises(dual.DcopfError):
        h.set_multipliers(None, np.ascontiguousarray(bad.T))
    with pytest.raises(dual.DcopfError):
        h.compact()
    # the matrix into a device buffer equals the host copy
    Hd = torch.empty((net.n_branch, net.n_bus), dtype=torch.float64, device="cuda:0")
    h.get_ptdf(Hd)
    np.testing.assert_array_equal(Hd.cpu().numpy(), h.get_ptdf())
    h.close()
