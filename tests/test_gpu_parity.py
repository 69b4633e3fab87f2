"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on
identical seeded inputs, at the north_star tolerances (1e-9 relative on the
bound, 1e-8 normalised max-abs on the multipliers), plus the edge cases.

The per-entity arithmetic reproduces the oracle's operation order, so the
multipliers are expected to match bitwise; the tests that say so assert it.
"""
import numpy as np
import pytest

import oracle
from oracle import FORM_F1, FORM_F2
from paper_2406_13191_b200 import dual
from paper_2406_13191_b200 import instances as inst

from gpu_helpers import BOUND_RTOL, assert_parity, cost_scale, non_tree_switchable, run_gpu

pytestmark = pytest.mark.gpu

PATHS = [dual.PATH_SINGLE, dual.PATH_BATCHED, dual.PATH_CLUSTER]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dual.load_library()


# ---------------------------------------------------------------------------
# config 0 at its full K (BASELINE.json configs[0]), both forms, both paths


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
@pytest.mark.parametrize("path", PATHS)
def test_config0_full_K(form, path):
    net = inst.make_network(0)
    K = inst.ITERS[0]
    a = inst.alpha_schedule(K)
    orc = oracle.solve(net, net.base_load, K=K, alpha=a, form=form, history=True)
    gpu = run_gpu(net, net.base_load, K=K, alpha=a, form=form, path=path, history=True)
    assert_parity(net, gpu, orc, bitwise_multipliers=True)


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
@pytest.mark.parametrize("path", PATHS)
def test_config0_tuned_step(form, path):
    """alpha = 1e-2, theta = min(pi/3, implied): a trajectory that moves."""
    net = inst.make_network(0, theta_mode="min")
    K = 5000
    a = inst.alpha_schedule(K, 1e-2)
    orc = oracle.solve(net, net.base_load, K=K, alpha=a, form=form, history=True)
    gpu = run_gpu(net, net.base_load, K=K, alpha=a, form=form, path=path, history=True)
    assert_parity(net, gpu, orc, bitwise_multipliers=True)
    assert gpu["best"][0] > 0.0


# ---------------------------------------------------------------------------
# tiny random instances: QP, several generators per bus, ragged tiles


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("quad", [False, True])
def test_tiny_batch_ragged(form, path, quad):
    net = inst.tiny_network(23, 37, 30, seed=5, quadratic=quad)  # 30 gens on 23 buses
    rng = np.random.default_rng(9)
    B = 37  # two tiles, ragged tail
    loads = net.base_load[None, :] * rng.uniform(0.7, 1.3, (B, net.n_bus))
    outs = np.full((B, 3), -1, np.int32)
    non_tree = np.arange(net.n_tree, net.n_branch)
    for j in range(B):
        k = j % 4
        if k:
            outs[j, :k] = rng.choice(non_tree, k, replace=False)
    K = 700
    a = inst.alpha_schedule(K, 4e-3) * np.linspace(1.0, 0.2, K)  # non-constant schedule
    orc = oracle.solve(net, loads, outages=outs, K=K, alpha=a, form=form, history=True)
    gpu = run_gpu(net, loads, outages=outs, K=K, alpha=a, form=form, path=path, history=True)
    assert_parity(net, gpu, orc, bitwise_multipliers=True)


# ---------------------------------------------------------------------------
# the large single-instance configs (1, 2 QP, 3 LP/QP) at full K on the single
# path, and shortened on the batched path (B = 1)


@pytest.mark.parametrize("config,quad,form", [(1, False, FORM_F2), (1, False, FORM_F1), (2, True, FORM_F2),
                                              (2, True, FORM_F1), (3, False, FORM_F2), (3, True, FORM_F2),
                                              (3, False, FORM_F1)])
@pytest.mark.parametrize("path", [dual.PATH_SINGLE, dual.PATH_CLUSTER])
def test_large_single_instance_full_K(config, quad, form, path):
    net = inst.make_network(config, quadratic=quad)
    K = inst.ITERS[config]
    a = inst.alpha_schedule(K)
    orc = _oracle_full_K(config, quad, form)
    gpu = run_gpu(net, net.base_load, K=K, alpha=a, form=form, path=path, history=True)
    assert_parity(net, gpu, orc, bitwise_multipliers=(path == dual.PATH_CLUSTER))
    if path == dual.PATH_CLUSTER:
        assert gpu["info"].cluster_size >= (8 if config >= 2 else 2)


_ORC_CACHE = {}


def _oracle_full_K(config, quad, form):
    key = (config, quad, form)
    if key not in _ORC_CACHE:
        net = inst.make_network(config, quadratic=quad)
        K = inst.ITERS[config]
        _ORC_CACHE[key] = oracle.solve(net, net.base_load, K=K, alpha=inst.alpha_schedule(K), form=form,
                                       history=True)
    return _ORC_CACHE[key]


@pytest.mark.parametrize("C", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_cluster_sizes_bitwise(C, form):
    """Every cluster size (1..16 CTAs, the partition changes) gives the same
    bits: the per-entity order never depends on the partition."""
    net = inst.tiny_network(600, 900, 150, seed=3)  # fits one CTA (C = 1) as well
    K = 400
    a = inst.alpha_schedule(K, 1e-2)
    orc = oracle.solve(net, net.base_load, K=K, alpha=a, form=form, history=True)
    gpu = run_gpu(net, net.base_load, K=K, alpha=a, form=form, path=dual.PATH_CLUSTER, history=True, tile_parts=C)
    assert gpu["info"].cluster_size == C
    assert_parity(net, gpu, orc, bitwise_multipliers=True)


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_cluster_config4_instances_with_outages(form):
    """config-4 instances (per-bus load factors, 0-3 non-tree outages) on the
    cluster path: one cluster per instance, outages applied in shared memory."""
    net = inst.make_network(4)
    ids = [0, 1, 2, 3, 4097]
    batch = inst.config4_batch(net, ids)
    assert (batch.outages >= 0).any()
    K = 200
    a = inst.alpha_schedule(K)
    orc = oracle.solve(net, batch.load, outages=batch.outages, K=K, alpha=a, form=form, threads=4, history=True)
    gpu = run_gpu(net, batch.load, outages=batch.outages, K=K, alpha=a, form=form, path=dual.PATH_CLUSTER,
                  switchable=non_tree_switchable(net), history=True)
    assert gpu["info"].cluster_size == 16
    assert_parity(net, gpu, orc, bitwise_multipliers=True)


@pytest.mark.parametrize("config,form", [(1, FORM_F2), (3, FORM_F1)])
def test_large_network_batched_path(config, form):
    net = inst.make_network(config)
    K = 300
    a = inst.alpha_schedule(K)
    orc = oracle.solve(net, net.base_load, K=K, alpha=a, form=form, history=True)
    gpu = run_gpu(net, net.base_load, K=K, alpha=a, form=form, path=dual.PATH_BATCHED, history=True)
    assert_parity(net, gpu, orc, bitwise_multipliers=True)


# ---------------------------------------------------------------------------
# config 4: the bench's launch configuration (B = 8192, batched) at full K,
# checked on sampled instances; and a 64-instance cut checked everywhere


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_config4_full_batch_sampled(form):
    """config 4 at full K (5000) in the bench's launch configuration (8192
    instances, 147 tiles of 56), sampled instances vs the oracle."""
    net = inst.make_network(4)
    B = inst.CONFIG4_BATCH
    K = inst.ITERS[4]
    batch = inst.config4_batch(net, range(B))
    a = inst.alpha_schedule(K)
    gpu = run_gpu(net, batch.load, outages=batch.outages, K=K, alpha=a, form=form,
                  path=dual.PATH_BATCHED, switchable=non_tree_switchable(net))
    assert gpu["info"].grid * gpu["info"].tile_width >= B and gpu["info"].grid <= 148
    idx = np.array([0, 31, 4097, 8191])
    orc = oracle.solve(net, batch.load[idx], outages=batch.outages[idx], K=K, alpha=a, form=form,
                       threads=4)
    assert_parity(net, gpu, orc, idx=idx, bitwise_multipliers=True)


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_config4_cut_all_instances(form):
    net = inst.make_network(4)
    batch = inst.config4_batch(net, range(64))
    K = 150
    a = inst.alpha_schedule(K)
    orc = oracle.solve(net, batch.load, outages=batch.outages, K=K, alpha=a, form=form, history=True,
                       threads=8)
    # with and without the switchable declaration (outage test on every branch)
    sw = non_tree_switchable(net) if form == FORM_F2 else None
    gpu = run_gpu(net, batch.load, outages=batch.outages, K=K, alpha=a, form=form, path=dual.PATH_BATCHED,
                  history=True, switchable=sw)
    assert_parity(net, gpu, orc, bitwise_multipliers=True)


# ---------------------------------------------------------------------------
# evaluate-only kernel (value and gradient at given multipliers)


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
@pytest.mark.parametrize("path", PATHS)
def test_evaluate_at_random_points(form, path):
    import torch
    net = inst.tiny_network(40, 61, 12, seed=3, quadratic=True)
    rng = np.random.default_rng(1)
    B = 45
    loads = net.base_load[None, :] * rng.uniform(0.5, 1.5, (B, net.n_bus))
    lam, br = inst.random_multipliers(rng, net, B, form)
    val_o, gl_o, gb_o = oracle.evaluate(net, loads, lam, br, form=form)
    dev = torch.device("cuda:0")
    h = dual.DcopfDual(net, form=form, path=path)
    h.set_instance_batch(torch.from_numpy(loads.T.copy()).to(dev))
    h.set_multipliers(torch.from_numpy(lam.T.copy()).to(dev), torch.from_numpy(br.T.copy()).to(dev))
    val = torch.empty(B, dtype=torch.float64, device=dev)
    gl = torch.empty((net.n_bus, B), dtype=torch.float64, device=dev)
    gb = torch.empty((h.n_branch_mult, B), dtype=torch.float64, device=dev)
    h.evaluate(val, gl, gb)
    torch.cuda.synchronize()
    S = cost_scale(net)
    assert np.all(np.abs(val.cpu().numpy() - val_o) <= 1e-12 * np.maximum(np.abs(val_o), S))
    np.testing.assert_array_equal(gl.cpu().numpy().T, gl_o)
    np.testing.assert_array_equal(gb.cpu().numpy().T, gb_o)
    # evaluate does not move the state
    lam2 = np.empty((net.n_bus, B))
    h.get_multipliers(lam2, None)
    np.testing.assert_array_equal(lam2.T, lam)
    h.close()


# ---------------------------------------------------------------------------
# warm start, host buffers, invariants, edge cases


@pytest.mark.parametrize("path", PATHS)
def test_warm_start_and_host_buffers(path):
    net = inst.make_network(0)
    rng = np.random.default_rng(4)
    lam0, br0 = inst.random_multipliers(rng, net, 3, FORM_F1, scale=3.0)
    loads = np.tile(net.base_load, (3, 1))
    K = 400
    a = inst.alpha_schedule(K, 2e-3)
    orc = oracle.solve(net, loads, K=K, alpha=a, form=FORM_F1, lam0=lam0, br0=br0, history=True)
    # host (numpy) buffers straight through the ABI
    h = dual.DcopfDual(net, form=FORM_F1, path=path)
    h.set_instance_batch(np.ascontiguousarray(loads.T))
    h.set_multipliers(np.ascontiguousarray(lam0.T), np.ascontiguousarray(br0.T))
    hist = np.empty((K, 3))
    h.iterate(K, a, hist)
    bound, best, status, lam, br = h.results_numpy()
    gpu = dict(bound=bound, best=best, status=status, lam=lam.T, br=br.T, hist=hist.T)
    assert_parity(net, gpu, orc, bitwise_multipliers=True)
    # F1 rejects a negative mu
    bad = br0.copy()
    bad[1, 3] = -1.0
    with pytest.raises(dual.DcopfError):
        h.set_multipliers(np.ascontiguousarray(lam0.T), np.ascontiguousarray(bad.T))
    h.close()


@pytest.mark.parametrize("path", PATHS)
def test_divergence_isolated(path):
    net = inst.make_network(0)
    loads = np.stack([net.base_load, net.base_load * 1e14, net.base_load])
    K = 50
    a = inst.alpha_schedule(K)
    orc = oracle.solve(net, loads, K=K, alpha=a, history=True)
    gpu = run_gpu(net, loads, K=K, alpha=a, path=path, history=True)
    np.testing.assert_array_equal(gpu["status"], [0, 1, 0])
    np.testing.assert_array_equal(gpu["status"], orc.status)
    assert_parity(net, {k: (v[[0, 2]] if isinstance(v, np.ndarray) else v) for k, v in gpu.items()},
                  oracle.solve(net, loads[[0, 2]], K=K, alpha=a, history=True))
    # the diverged instance is frozen at the same y as the oracle's
    np.testing.assert_array_equal(gpu["lam"][1], orc.lam[1])


def test_sharding_invariance_and_determinism():
    """Instances never interact: 64 at once == 2 x 32 == 32 x 2 (multipliers and
    status bitwise; the dual value is a fixed-order sum per tiling, so across
    tilings it agrees to rounding order), and reruns are bitwise."""
    net = inst.make_network(4)
    batch = inst.config4_batch(net, range(64))
    K = 60
    a = inst.alpha_schedule(K, 1e-2)
    full = run_gpu(net, batch.load, outages=batch.outages, K=K, alpha=a, path=dual.PATH_BATCHED)
    again = run_gpu(net, batch.load, outages=batch.outages, K=K, alpha=a, path=dual.PATH_BATCHED)
    lo = run_gpu(net, batch.load[:32], outages=batch.outages[:32], K=K, alpha=a, path=dual.PATH_BATCHED)
    hi = run_gpu(net, batch.load[32:], outages=batch.outages[32:], K=K, alpha=a, path=dual.PATH_BATCHED)
    pairs = [run_gpu(net, batch.load[j:j + 2], outages=batch.outages[j:j + 2], K=K, alpha=a,
                     path=dual.PATH_BATCHED) for j in range(0, 64, 2)]
    for key in ("bound", "best", "lam", "br", "status"):
        np.testing.assert_array_equal(full[key], again[key])
    for parts in ([lo, hi], pairs):
        for key in ("lam", "br", "status"):
            np.testing.assert_array_equal(full[key], np.concatenate([p[key] for p in parts]))
        for key in ("bound", "best"):
            np.testing.assert_allclose(full[key], np.concatenate([p[key] for p in parts]), rtol=1e-12,
                                       atol=1e-12 * cost_scale(net))


@pytest.mark.parametrize("path", PATHS)
def test_single_bus_no_branches(path):
    """n_branch = 0 (SPEC 1-bus worked example): bound 250."""
    net = inst.Network(n_bus=1, n_branch=0, n_gen=1, ref_bus=0, br_from=np.zeros(0, np.int32),
                       br_to=np.zeros(0, np.int32), br_b=np.zeros(0), br_fmax=np.zeros(0),
                       theta_max=np.zeros(1), gen_bus=np.zeros(1, np.int32), gen_pmin=np.zeros(1),
                       gen_pmax=np.array([100.0]), gen_c=np.array([5.0]))
    gpu = run_gpu(net, np.array([[50.0]]), K=20, alpha=inst.alpha_schedule(20, 0.02), path=path)
    assert gpu["best"][0] == 250.0 and gpu["bound"][0] == 250.0
    if path != dual.PATH_SINGLE:  # KVL: no branches, no cycles
        gpu = run_gpu(net, np.array([[50.0]]), K=20, alpha=inst.alpha_schedule(20, 0.02), path=path,
                      form=dual.FORM_KVL)
        assert gpu["best"][0] == 250.0 and gpu["br"].shape[1] == 0


def test_implied_theta_box_matches_generator():
    """theta_max = NULL: the library computes the implied box (A-2) itself."""
    net = inst.make_network(1)
    K = 200
    a = inst.alpha_schedule(K, 1e-2)
    orc = oracle.solve(net, net.base_load, K=K, alpha=a, history=True)
    for path in (dual.PATH_SINGLE, dual.PATH_CLUSTER):
        gpu = run_gpu(net, net.base_load, K=K, alpha=a, path=path, history=True, implied_theta=True)
        assert_parity(net, gpu, orc)


def test_zero_iterations_evaluates_origin():
    net = inst.make_network(0)
    gpu = run_gpu(net, net.base_load, K=0, path=dual.PATH_BATCHED)
    assert gpu["bound"][0] == 0.0 and gpu["best"][0] == 0.0


# ---------------------------------------------------------------------------
# time to gap: the device-recorded first evaluation whose running best reaches
# a per-instance target equals the one read off the oracle's
# g(y_k) history; two iterate() calls continue the evaluation count


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
@pytest.mark.parametrize("path", PATHS)
def test_first_hit_matches_oracle_history(form, path):
    import torch
    net = inst.make_network(0, theta_mode="min")
    rng = np.random.default_rng(7)
    B = 5
    loads = net.base_load[None, :] * rng.uniform(0.8, 1.1, (B, 1))
    K1, K2 = 1200, 1800
    K = K1 + K2
    a = inst.alpha_schedule(K, 1e-2)
    orc = oracle.solve(net, loads, K=K, alpha=a, form=form, history=True)
    rb = np.maximum.accumulate(orc.hist, axis=1)   # running best over k = 0..K
    S = cost_scale(net)
    target = np.full(B, np.inf)
    expect = np.full(B, -1, dtype=np.int64)
    for b in range(B - 1):  # the last instance keeps an unreachable target
        # a target strictly between two running-best values far apart (robust
        # to the 1e-9 relative bound tolerance): the first big jump past 50%
        fin = rb[b, -1]
        ks = np.nonzero((rb[b] >= 0.5 * fin) & (np.diff(rb[b], prepend=-np.inf) > 1e-7 * S))[0]
        k = int(ks[0])
        target[b] = 0.5 * (rb[b, k - 1] + rb[b, k]) if k > 0 else rb[b, 0] - 1.0
        expect[b] = k
    dev = torch.device("cuda:0")
    h = dual.DcopfDual(net, form=form, path=path)
    h.set_instance_batch(torch.from_numpy(np.ascontiguousarray(loads.T)).to(dev))
    h.set_target(target)
    h.iterate(K1, a[:K1])
    h.iterate(K2, a[K1:])
    hit = h.get_first_hit()
    best = np.empty(B)
    h.get_bound(best=best)
    h.close()
    np.testing.assert_array_equal(hit, expect)
    assert np.all(np.abs(best - orc.best) <= BOUND_RTOL * np.maximum(np.abs(orc.best), S))


def test_first_hit_cleared_by_new_batch():
    import torch
    net = inst.make_network(0)
    dev = torch.device("cuda:0")
    h = dual.DcopfDual(net, path=dual.PATH_SINGLE)
    ld = torch.from_numpy(net.base_load[:, None].copy()).to(dev)
    h.set_instance_batch(ld)
    h.set_target(np.array([-1.0]))            # g(y_0) = 0 >= -1: hit at evaluation 0
    h.iterate(3, inst.alpha_schedule(3))
    assert h.get_first_hit()[0] == 0
    h.set_instance_batch(ld)                  # cleared: no target, no hit
    h.iterate(3, inst.alpha_schedule(3))
    assert h.get_first_hit()[0] == -1
    with pytest.raises(dual.DcopfError):
        h.set_target(np.array([np.nan]))
    h.close()


# ---------------------------------------------------------------------------
# gradient-based-optimisation variants (Algorithm 1) on the
# cluster path: bitwise multipliers against the oracle's variants

OPTS = {
    "gdm": (dict(variant=oracle.OPT_GDM, rho=0.9), 1e-3),
    "gdm_classic": (dict(variant=oracle.OPT_GDM_CLASSIC, rho=0.8), 3e-3),
    "adagrad": (dict(variant=oracle.OPT_ADAGRAD, eps=1e-8), 3.0),
    "adam": (dict(variant=oracle.OPT_ADAM, beta1=0.9, beta2=0.999, eps=1e-8), 0.1),
}


@pytest.mark.parametrize("name", sorted(OPTS))
@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_optimizer_variants_config0(name, form):
    opt, alpha = OPTS[name]
    net = inst.make_network(0, theta_mode="min")
    K = 3000
    a = inst.alpha_schedule(K, alpha)
    orc = oracle.solve(net, net.base_load, K=K, alpha=a, form=form, history=True, opt=opt)
    gpu = run_gpu(net, net.base_load, K=K, alpha=a, form=form, path=dual.PATH_CLUSTER, history=True, opt=opt,
                  split=1234)
    assert_parity(net, gpu, orc, bitwise_multipliers=True)


@pytest.mark.parametrize("name", sorted(OPTS))
def test_optimizer_variants_batch_with_outages(name):
    opt, alpha = OPTS[name]
    net = inst.tiny_network(23, 37, 30, seed=5)
    rng = np.random.default_rng(2)
    B = 6
    loads = net.base_load[None, :] * rng.uniform(0.7, 1.3, (B, net.n_bus))
    outs = np.full((B, 2), -1, np.int32)
    for j in range(B):
        if j % 3:
            outs[j, :j % 3] = rng.choice(np.arange(net.n_tree, net.n_branch), j % 3, replace=False)
    K = 1500
    a = inst.alpha_schedule(K, alpha) * np.linspace(1.0, 0.3, K)  # with a step decay
    for form in (FORM_F2, FORM_F1):
        orc = oracle.solve(net, loads, outages=outs, K=K, alpha=a, form=form, history=True, opt=opt)
        for path in (dual.PATH_CLUSTER, dual.PATH_BATCHED):
            gpu = run_gpu(net, loads, outages=outs, K=K, alpha=a, form=form, history=True, opt=opt, path=path,
                          split=600)
            assert gpu["info"].path == path
            assert_parity(net, gpu, orc, bitwise_multipliers=True)


def test_optimizer_adam_config3_cluster16():
    opt, alpha = OPTS["adam"]
    net = inst.make_network(3)
    K = 1000
    a = inst.alpha_schedule(K, alpha)
    orc = oracle.solve(net, net.base_load, K=K, alpha=a, history=True, opt=opt)
    gpu = run_gpu(net, net.base_load, K=K, alpha=a, path=dual.PATH_CLUSTER, history=True, opt=opt)
    assert gpu["info"].cluster_size == 16
    assert_parity(net, gpu, orc, bitwise_multipliers=True)


def test_optimizer_rejected_on_the_single_path():
    import torch
    net = inst.make_network(0)
    h = dual.DcopfDual(net, path=dual.PATH_SINGLE)
    h.set_instance_batch(torch.from_numpy(np.ascontiguousarray(np.tile(net.base_load[:, None], (1, 4)))).cuda())
    with pytest.raises(dual.DcopfError):
        h.set_optimizer(dual.OPT_ADAM, beta1=0.9, beta2=0.999, epsilon=1e-8)
    with pytest.raises(dual.DcopfError):
        h.set_optimizer(99)
    h.close()


# ---------------------------------------------------------------------------
# KVL (cycle-basis) form, on the cluster path


@pytest.mark.parametrize("name", ["plain"] + sorted(OPTS))
def test_kvl_config0(name):
    opt, alpha = OPTS[name] if name != "plain" else (None, 1e-2)
    net = inst.make_network(0)
    K = 3000
    a = inst.alpha_schedule(K, alpha)
    orc = oracle.solve(net, net.base_load, K=K, alpha=a, form=oracle.FORM_KVL, history=True, opt=opt)
    gpu = run_gpu(net, net.base_load, K=K, alpha=a, form=dual.FORM_KVL, history=True, opt=opt, split=777)
    assert gpu["info"].path == dual.PATH_CLUSTER
    assert_parity(net, gpu, orc, bitwise_multipliers=True)


@pytest.mark.parametrize("C", [1, 4, 16])
def test_kvl_cluster_sizes_and_outages(C):
    net = inst.tiny_network(600, 900, 150, seed=4)
    sw = non_tree_switchable(net)
    rng = np.random.default_rng(1)
    B = 4
    loads = net.base_load[None, :] * rng.uniform(0.8, 1.2, (B, net.n_bus))
    outs = np.full((B, 3), -1, np.int32)
    for j in range(1, B):
        outs[j, :j] = rng.choice(np.arange(net.n_tree, net.n_branch), j, replace=False)
    K = 500
    opt, alpha = OPTS["adam"]
    a = inst.alpha_schedule(K, alpha)
    orc = oracle.solve(net, loads, outages=outs, K=K, alpha=a, form=oracle.FORM_KVL, history=True, opt=opt,
                       switchable=sw)
    gpu = run_gpu(net, loads, outages=outs, K=K, alpha=a, form=dual.FORM_KVL, history=True, opt=opt,
                  switchable=sw, tile_parts=C)
    assert gpu["info"].cluster_size == C
    assert_parity(net, gpu, orc, bitwise_multipliers=True)


def test_kvl_config3_adam_and_evaluate():
    net = inst.make_network(3)
    K = 500
    opt, alpha = OPTS["adam"]
    a = inst.alpha_schedule(K, alpha)
    orc = oracle.solve(net, net.base_load, K=K, alpha=a, form=oracle.FORM_KVL, history=True, opt=opt)
    gpu = run_gpu(net, net.base_load, K=K, alpha=a, form=dual.FORM_KVL, history=True, opt=opt)
    assert gpu["info"].cluster_size == 16
    assert_parity(net, gpu, orc, bitwise_multipliers=True)
    # value and gradient at the reached point
    import torch
    dev = torch.device("cuda:0")
    h = dual.DcopfDual(net, form=dual.FORM_KVL)
    h.set_instance_batch(torch.from_numpy(net.base_load[:, None].copy()).to(dev))
    h.set_multipliers(torch.from_numpy(orc.lam.T.copy()).to(dev), torch.from_numpy(orc.br.T.copy()).to(dev))
    val = torch.empty(1, dtype=torch.float64, device=dev)
    gl = torch.empty((net.n_bus, 1), dtype=torch.float64, device=dev)
    gk = torch.empty((h.n_branch_mult, 1), dtype=torch.float64, device=dev)
    h.evaluate(val, gl, gk)
    ov, ogl, ogk, _, _ = oracle.evaluate_kvl(net, net.base_load, orc.lam, orc.br)
    assert abs(float(val.cpu()[0]) - ov[0]) <= BOUND_RTOL * max(abs(ov[0]), cost_scale(net))
    np.testing.assert_array_equal(gl.cpu().numpy()[:, 0], ogl[0])
    np.testing.assert_array_equal(gk.cpu().numpy()[:, 0], ogk[0])
    h.close()


def test_kvl_rejects_tree_outage_and_single_path():
    import torch
    net = inst.make_network(0)
    with pytest.raises(dual.DcopfError):
        h = dual.DcopfDual(net, form=dual.FORM_KVL, path=dual.PATH_SINGLE)
        h.set_instance_batch(torch.from_numpy(net.base_load[:, None].copy()).cuda())
    h = dual.DcopfDual(net, form=dual.FORM_KVL)   # no switchable mask: the tree may use any branch
    d, _ = oracle.cycles(net)
    tree = np.setdiff1d(np.arange(net.n_branch), d)
    with pytest.raises(dual.DcopfError):
        h.set_instance_batch(torch.from_numpy(net.base_load[:, None].copy()).cuda(),
                             torch.tensor([[int(tree[0])]], dtype=torch.int32).cuda())
    h.close()


# ---------------------------------------------------------------------------
# Algorithm 1's stopping rule per instance (reading A-29)


@pytest.mark.parametrize("path", PATHS)
def test_stopping_rule_per_instance(path):
    net = inst.tiny_network(23, 37, 30, seed=5)
    rng = np.random.default_rng(4)
    B = 9
    loads = net.base_load[None, :] * rng.uniform(0.7, 1.3, (B, net.n_bus))
    K = 2500
    a = inst.alpha_schedule(K, 3e-3)
    tol = 2e-3  # some instances stop, some do not
    orc = oracle.solve(net, loads, K=K, alpha=a, history=True, tol=tol)
    assert 0 < np.sum(orc.status == oracle.CONVERGED) < B
    gpu = run_gpu(net, loads, K=K, alpha=a, path=path, history=True, tol=tol)
    assert_parity(net, gpu, orc, bitwise_multipliers=True)
    # split calls: the rule looks only within a call (its first evaluation
    # re-evaluates the previous call's last point) -- same result here
    gpu2 = run_gpu(net, loads, K=K, alpha=a, path=path, history=True, tol=tol, split=997)
    np.testing.assert_array_equal(gpu2["status"], gpu["status"])


# KVL form on the batched path (sweep kernel)


def test_kvl_batched_tiny_ragged():
    net = inst.tiny_network(23, 37, 30, seed=5)
    sw = non_tree_switchable(net)
    rng = np.random.default_rng(9)
    B = 37  # two tiles, ragged tail
    loads = net.base_load[None, :] * rng.uniform(0.7, 1.3, (B, net.n_bus))
    outs = np.full((B, 3), -1, np.int32)
    for j in range(B):
        if j % 4:
            outs[j, :j % 4] = rng.choice(np.arange(net.n_tree, net.n_branch), j % 4, replace=False)
    K = 700
    a = inst.alpha_schedule(K, 4e-3) * np.linspace(1.0, 0.2, K)
    orc = oracle.solve(net, loads, outages=outs, K=K, alpha=a, form=oracle.FORM_KVL, history=True, switchable=sw)
    gpu = run_gpu(net, loads, outages=outs, K=K, alpha=a, form=dual.FORM_KVL, path=dual.PATH_BATCHED,
                  history=True, switchable=sw)
    assert gpu["info"].path == dual.PATH_BATCHED
    assert_parity(net, gpu, orc, bitwise_multipliers=True)


def test_kvl_batched_config4_sampled():
    """config 4 at its full K (5000) in the bench's launch configuration."""
    net = inst.make_network(4)
    sw = non_tree_switchable(net)
    B = inst.CONFIG4_BATCH
    K = inst.ITERS[4]
    batch = inst.config4_batch(net, range(B))
    a = inst.alpha_schedule(K)
    gpu = run_gpu(net, batch.load, outages=batch.outages, K=K, alpha=a, form=dual.FORM_KVL,
                  path=dual.PATH_BATCHED, switchable=sw)
    assert gpu["info"].grid * gpu["info"].tile_width >= B and gpu["info"].grid <= 148
    idx = np.array([0, 55, 4097, 8191])
    orc = oracle.solve(net, batch.load[idx], outages=batch.outages[idx], K=K, alpha=a, form=oracle.FORM_KVL,
                       switchable=sw, threads=4)
    assert_parity(net, gpu, orc, idx=idx, bitwise_multipliers=True)


def test_kvl_batched_evaluate_at_random_points():
    import torch
    net = inst.tiny_network(40, 70, 9, seed=3)
    sw = non_tree_switchable(net)
    rng = np.random.default_rng(2)
    B = 150
    nc = net.n_branch - net.n_bus + 1
    loads = net.base_load[None, :] * rng.uniform(0.8, 1.2, (B, net.n_bus))
    outs = np.full((B, 1), -1, np.int32)
    outs[::3, 0] = rng.choice(np.arange(net.n_tree, net.n_branch), len(outs[::3]))
    lam = rng.normal(-30, 10, (B, net.n_bus))
    kap = rng.normal(0, 20, (B, nc))
    d, _ = oracle.cycles(net, sw)
    for j in range(B):  # kappa of an inactive cycle must be 0 (set_multipliers checks it)
        if outs[j, 0] >= 0:
            kap[j, np.nonzero(d == outs[j, 0])[0]] = 0.0
    dev = torch.device("cuda:0")
    h = dual.DcopfDual(net, form=dual.FORM_KVL, path=dual.PATH_BATCHED, switchable=sw)
    h.set_instance_batch(torch.from_numpy(np.ascontiguousarray(loads.T)).to(dev), torch.from_numpy(outs).to(dev))
    h.set_multipliers(torch.from_numpy(np.ascontiguousarray(lam.T)).to(dev),
                      torch.from_numpy(np.ascontiguousarray(kap.T)).to(dev))
    val = torch.empty(B, dtype=torch.float64, device=dev)
    gl = torch.empty((net.n_bus, B), dtype=torch.float64, device=dev)
    gk = torch.empty((nc, B), dtype=torch.float64, device=dev)
    h.evaluate(val, gl, gk)
    ov, ogl, ogk, _, _ = oracle.evaluate_kvl(net, loads, lam, kap, outages=outs, switchable=sw)
    S = cost_scale(net)
    assert np.all(np.abs(val.cpu().numpy() - ov) <= BOUND_RTOL * np.maximum(np.abs(ov), S))
    np.testing.assert_array_equal(gl.cpu().numpy().T, ogl)
    np.testing.assert_array_equal(gk.cpu().numpy().T, ogk)
    bad = kap.copy()
    j = int(np.nonzero(outs[:, 0] >= 0)[0][0])
    bad[j, np.nonzero(d == outs[j, 0])[0]] = 1.0
    with pytest.raises(dual.DcopfError):
        h.set_multipliers(None, torch.from_numpy(np.ascontiguousarray(bad.T)).to(dev))
    h.close()


@pytest.mark.parametrize("form", [FORM_F2, oracle.FORM_KVL])
def test_batched_more_tiles_than_sms(form):
    """B = 10 000 on the 2000-bus network: 64-wide tiles, 157 tiles on 148
    SMs (a second wave of persistent CTAs); sampled instances vs the oracle."""
    net = inst.make_network(1)
    sw = non_tree_switchable(net)
    B = 10000
    batch = inst.config4_batch(net, range(B), total=B)
    K = 60
    a = inst.alpha_schedule(K, 1e-2)
    gpu = run_gpu(net, batch.load, outages=batch.outages, K=K, alpha=a, form=form, path=dual.PATH_BATCHED,
                  switchable=sw, tile_parts=1, lane_instances=2)
    assert gpu["info"].tile_width == 64 and gpu["info"].grid > 148
    idx = np.array([0, 63, 64, 9407, 9999])
    orc = oracle.solve(net, batch.load[idx], outages=batch.outages[idx], K=K, alpha=a, form=form, switchable=sw,
                       threads=4)
    assert_parity(net, gpu, orc, idx=idx, bitwise_multipliers=True)


@pytest.mark.parametrize("name", ["adam", "gdm"])
def test_optimizer_batched_config4_kvl_sampled(name):
    """KVL + an optimiser variant on the config-4 batch (variant 4b: feasible,
    one load factor per instance), the bench's launch configuration."""
    opt, alpha = OPTS[name]
    net = inst.make_network(4)
    sw = non_tree_switchable(net)
    B = inst.CONFIG4_BATCH
    batch = inst.config4_batch(net, range(B), variant="4b")
    K = 300
    a = inst.alpha_schedule(K, alpha if name == "adam" else 1e-3)
    gpu = run_gpu(net, batch.load, K=K, alpha=a, form=dual.FORM_KVL, path=dual.PATH_BATCHED, switchable=sw,
                  opt=opt)
    idx = np.array([0, 77, 8191])
    orc = oracle.solve(net, batch.load[idx], K=K, alpha=a, form=oracle.FORM_KVL, switchable=sw, opt=opt, threads=3)
    assert_parity(net, gpu, orc, idx=idx, bitwise_multipliers=True)


# ---------------------------------------------------------------------------
# split tiles (split_schedule.cpp): a tile swept by C CTAs, V instances per
# lane; every (V, C) gives the oracle's multipliers bitwise


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1, oracle.FORM_KVL])
@pytest.mark.parametrize("V,C", [(2, 1), (4, 1), (2, 3), (4, 2), (4, 7), (4, 16)])
def test_split_tiles_bitwise(form, V, C):
    """2000-bus network, 150 config-4-style instances (per-bus load factors,
    0-3 non-tree outages, ragged last tile) at every tiling: owned items, halo
    recomputation and the once-per-sweep meeting of the parts."""
    if form == FORM_F1 and V == 4:
        pytest.skip("F1 runs 2 instances per lane")
    net = inst.make_network(1)
    sw = non_tree_switchable(net)
    B = 150
    batch = inst.config4_batch(net, range(B), total=B)
    K = 120
    a = inst.alpha_schedule(K, 1e-2) * np.linspace(1.0, 0.3, K)
    gpu = run_gpu(net, batch.load, outages=batch.outages, K=K, alpha=a, form=form, path=dual.PATH_BATCHED,
                  switchable=sw, history=True, tile_parts=C, lane_instances=V)
    info = gpu["info"]
    assert (info.tile_parts, info.lane_instances) == (C, V)
    assert info.grid == C * -(-B // info.tile_width)
    orc = oracle.solve(net, batch.load, outages=batch.outages, K=K, alpha=a, form=form, switchable=sw,
                       history=True, threads=8)
    assert_parity(net, gpu, orc, bitwise_multipliers=True)


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1, oracle.FORM_KVL])
@pytest.mark.parametrize("B", [1024, 2048, 4096])
def test_strong_scaling_shards_sampled(form, B):
    """The per-GPU shards of the literal config-4 split (8192 over 8 / 4 / 2
    GPUs) in the library's own tiling (split tiles, the parts chosen by the
    chunk-aware model: e.g. F2 9 / 4 / 2 parts), full K = 5000, sampled
    instances vs the oracle."""
    net = inst.make_network(4)
    sw = non_tree_switchable(net)
    K = inst.ITERS[4]
    batch = inst.config4_batch(net, range(B))
    a = inst.alpha_schedule(K)
    gpu = run_gpu(net, batch.load, outages=batch.outages, K=K, alpha=a, form=form, path=dual.PATH_BATCHED,
                  switchable=sw)
    info = gpu["info"]
    assert info.grid <= 148 and info.tile_parts > 1
    idx = np.array([0, 1, B // 2 + 3, B - 1])
    orc = oracle.solve(net, batch.load[idx], outages=batch.outages[idx], K=K, alpha=a, form=form, switchable=sw,
                       threads=4)
    assert_parity(net, gpu, orc, idx=idx, bitwise_multipliers=True)


@pytest.mark.parametrize("V,C", [(4, 2), (4, 16)])
def test_split_tiles_optimizer_and_evaluate(V, C):
    """Adam on split tiles (state rows of owned entities only) and the
    evaluate-only kernel (gradients written by the owning part)."""
    import torch
    net = inst.make_network(1)
    sw = non_tree_switchable(net)
    B = 64
    batch = inst.config4_batch(net, range(B), total=B)
    K = 150
    opt, alpha = OPTS["adam"]
    a = inst.alpha_schedule(K, alpha)
    gpu = run_gpu(net, batch.load, outages=batch.outages, K=K, alpha=a, path=dual.PATH_BATCHED, switchable=sw,
                  opt=opt, history=True, tile_parts=C, lane_instances=V)
    orc = oracle.solve(net, batch.load, outages=batch.outages, K=K, alpha=a, switchable=sw, opt=opt, history=True,
                       threads=8)
    assert_parity(net, gpu, orc, bitwise_multipliers=True)
    # evaluate at the oracle's final multipliers, on a handle with Adam set (the
    # evaluate kernel runs on the optimiser variant's schedule / warp count)
    dev = torch.device("cuda:0")
    h = dual.DcopfDual(net, path=dual.PATH_BATCHED, switchable=sw, tile_parts=C, lane_instances=V)
    h.set_instance_batch(torch.from_numpy(np.ascontiguousarray(batch.load.T)).to(dev),
                         torch.from_numpy(batch.outages).to(dev))
    h.set_optimizer(opt["variant"], 0.0, opt["beta1"], opt["beta2"], opt["eps"])
    h.set_multipliers(torch.from_numpy(np.ascontiguousarray(orc.lam.T)).to(dev),
                      torch.from_numpy(np.ascontiguousarray(orc.br.T)).to(dev))
    val = torch.empty(B, dtype=torch.float64, device=dev)
    gl = torch.empty((net.n_bus, B), dtype=torch.float64, device=dev)
    gb = torch.empty((net.n_branch, B), dtype=torch.float64, device=dev)
    h.evaluate(val, gl, gb)
    ov, ogl, ogb = oracle.evaluate(net, batch.load, orc.lam, orc.br, outages=batch.outages)[:3]
    S = cost_scale(net)
    assert np.all(np.abs(val.cpu().numpy() - ov) <= BOUND_RTOL * np.maximum(np.abs(ov), S))
    np.testing.assert_array_equal(gl.cpu().numpy().T, ogl)
    np.testing.assert_array_equal(gb.cpu().numpy().T, ogb)
    h.close()


def test_forced_split_tiling_beyond_one_wave_rejected():
    """A split tile is a cooperative launch (its parts meet every sweep): a
    forced tiling needing more CTAs than SMs is rejected at set_instance_batch
    with EINVAL, leaving no batch loaded."""
    import torch
    net = inst.make_network(4)
    sw = non_tree_switchable(net)
    B = 1024
    batch = inst.config4_batch(net, range(B))
    dev = torch.device("cuda:0")
    h = dual.DcopfDual(net, path=dual.PATH_BATCHED, switchable=sw, tile_parts=12, lane_instances=2)
    with pytest.raises(dual.DcopfError, match="EINVAL"):
        h.set_instance_batch(torch.from_numpy(np.ascontiguousarray(batch.load.T)).to(dev),
                             torch.from_numpy(batch.outages).to(dev))
