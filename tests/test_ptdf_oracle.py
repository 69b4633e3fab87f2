"""Pins of the dense-PTDF oracle (oracle/ptdf.py) against
what the paper and the mathematics fix -- none of them re-types the oracle's
own formulas:

* the PTDF matrix: the SPEC 2-bus example, closed-form path flows on a radial
  network, the zero slack column, Kirchhoff's current law
  E^T H_a = I - e_ref 1^T and Kirchhoff's voltage law on the cycle basis of
  the C oracle (an independent implementation) -- KCL + KVL fix H uniquely;
* the dual function: brute force over the generator box vertices (linear
  cost) and a bounded numerical minimiser (quadratic cost) of the Lagrangian
  Eq. 4, central finite differences for the gradient,
  economic dispatch (merit order) when no flow limit binds;
* the loop: weak duality against the exact LP optimum of Eq. 1 (HiGHS on the
  B-theta model with no angle box, which never touches H), convergence to it,
  divergence freeze and the stopping rule (readings A-23, A-29).
"""
import dataclasses
import math

import numpy as np
import pytest

import oracle
from oracle import ptdf as P
from paper_2406_13191_b200 import instances as inst


def _net(n_bus, n_branch, n_gen, seed, quadratic=False):
    return inst.tiny_network(n_bus, n_branch, n_gen, seed, quadratic=quadratic)


def _no_angle_box(net):
    th = np.full(net.n_bus, 1e6)
    th[net.ref_bus] = 0.0
    return dataclasses.replace(net, theta_max=th)


def test_two_bus_spec_example():
    # 2-bus, one line bus1 -> bus2, b = 10, slack = bus1 -> h_a = [0, -1]
    net = inst.Network(n_bus=2, n_branch=1, n_gen=1, ref_bus=0, br_from=np.array([0], np.int32),
                       br_to=np.array([1], np.int32), br_b=np.array([10.0]), br_fmax=np.array([1.0]),
                       theta_max=np.array([0.0, 1.0]), gen_bus=np.array([0], np.int32),
                       gen_pmin=np.zeros(1), gen_pmax=np.ones(1), gen_c=np.ones(1))
    np.testing.assert_array_equal(P.ptdf(net), [[0.0, -1.0]])


def _tree_flows(net):
    """Closed form on a radial network: a unit injected at bus i and withdrawn
    at the reference flows along the unique path i -> ref."""
    adj = [[] for _ in range(net.n_bus)]
    for l in range(net.n_branch):
        adj[net.br_from[l]].append(l)
        adj[net.br_to[l]].append(l)
    parent = [-1] * net.n_bus
    pbr = [-1] * net.n_bus
    seen = [False] * net.n_bus
    seen[net.ref_bus] = True
    stack = [net.ref_bus]
    while stack:
        u = stack.pop()
        for l in adj[u]:
            v = net.br_to[l] if net.br_from[l] == u else net.br_from[l]
            if not seen[v]:
                seen[v] = True
                parent[v], pbr[v] = u, l
                stack.append(v)
    H = np.zeros((net.n_branch, net.n_bus))
    for i in range(net.n_bus):
        u = i
        while u != net.ref_bus:
            l = pbr[u]
            H[l, i] = 1.0 if net.br_from[l] == u else -1.0   # traversed child -> parent
            u = parent[u]
    return H


@pytest.mark.parametrize("n_bus,seed", [(7, 1), (25, 2), (60, 3)])
def test_radial_network_path_flows(n_bus, seed):
    net = _net(n_bus, n_bus - 1, 3, seed)
    np.testing.assert_allclose(P.ptdf(net), _tree_flows(net), atol=1e-12, rtol=0)


@pytest.mark.parametrize("n_bus,seed", [(7, 1), (25, 2), (60, 3)])
def test_radial_structural_zeros_are_exact(n_bus, seed):
    """A radial line carries flow for an injection at bus i iff it lies on the
    path from i to the slack: every other entry is an exact zero (the solve's
    rounding residues are snapped, reading A-30)."""
    net = _net(n_bus, n_bus - 1, 3, seed)
    np.testing.assert_array_equal(P.ptdf(net) == 0.0, _tree_flows(net) == 0.0)


def test_injection_free_part_carries_exactly_no_flow():
    """Config 1's lines into parts of the network with no load and no
    generator (literal zero limits, reading A-11): zero H_g rows, zero load
    flow and F = 0 -- all exactly, so the dual gradient on them is exactly 0."""
    net = inst.make_network(1)
    Ha = P.ptdf(net)
    d = net.base_load
    noflow = (np.abs(Ha[:, net.gen_bus]).max(axis=1) == 0.0) & (Ha @ d == 0.0)
    assert noflow.sum() >= 20
    assert np.all(net.br_fmax[noflow] == 0.0)
    rng = np.random.default_rng(0)
    mup = np.abs(rng.normal(size=(1, net.n_branch)))
    ev = P.evaluate(net, Ha, d[None], np.full(1, -40.0), mup, mup[:, ::-1].copy())
    assert np.all(ev.g_mup[0][noflow] == 0.0) and np.all(ev.g_mum[0][noflow] == 0.0)


@pytest.mark.parametrize("shape", [(14, 19, 5, 0), (30, 52, 9, 4), (80, 130, 20, 7)])
def test_kirchhoff_current_and_voltage_laws(shape):
    n, nl, ng, seed = shape
    net = _net(n, nl, ng, seed)
    Ha = P.ptdf(net)
    # zero slack column
    assert np.all(Ha[:, net.ref_bus] == 0.0)
    # KCL: the flows of "inject 1 at i, withdraw at ref" leave bus i with net 1
    E = P.incidence(net)
    want = np.eye(n)
    want[net.ref_bus, :] -= 1.0
    np.testing.assert_allclose(E.T @ Ha, want, atol=1e-11, rtol=0)
    # KVL on every fundamental cycle of the C oracle's basis (reading A-28)
    dfn, cyc = oracle.cycles(net)
    assert len(cyc) == nl - n + 1
    for br, sg in cyc:
        s = (sg[:, None] * Ha[br, :] / net.br_b[br][:, None]).sum(axis=0)
        np.testing.assert_allclose(s, 0.0, atol=1e-12)


def _lagrangian(net, Ha, d, lam, mup, mum, p):
    """Eq. 4 for Eq. 1 written out: c'p (+ a p^2) + lambda (1'p - 1'd)
    + mu+ (H_a (G p - d) - F) + mu- (-H_a (G p - d) - F)."""
    inj = -d.copy()
    np.add.at(inj, net.gen_bus, p)
    f = Ha @ inj
    obj = net.gen_c @ p + (0.0 if net.gen_a is None else net.gen_a @ (p * p))
    return obj + lam * (p.sum() - d.sum()) + mup @ (f - net.br_fmax) + mum @ (-f - net.br_fmax)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_inner_minimum_brute_force_vertices(seed):
    net = _net(10, 15, 6, seed)
    Ha = P.ptdf(net)
    rng = np.random.default_rng(100 + seed)
    d = net.base_load
    for _ in range(5):
        lam = rng.normal(0, 20)
        mup = np.abs(rng.normal(0, 20, net.n_branch)) * (rng.random(net.n_branch) < 0.5)
        mum = np.abs(rng.normal(0, 20, net.n_branch)) * (rng.random(net.n_branch) < 0.5)
        ev = P.evaluate(net, Ha, d[None], [lam], mup[None], mum[None])
        best = math.inf
        for bits in range(1 << net.n_gen):
            p = np.where([(bits >> g) & 1 for g in range(net.n_gen)], net.gen_pmax, net.gen_pmin)
            best = min(best, _lagrangian(net, Ha, d, lam, mup, mum, p))
        assert abs(ev.value[0] - best) <= 1e-9 * max(1.0, abs(best))
        # the minimiser attains it
        assert abs(_lagrangian(net, Ha, d, lam, mup, mum, ev.p[0]) - best) <= 1e-9 * max(1.0, abs(best))


def test_inner_minimum_quadratic_numerical():
    from scipy.optimize import minimize
    net = _net(10, 15, 6, 5, quadratic=True)
    Ha = P.ptdf(net)
    rng = np.random.default_rng(7)
    d = net.base_load
    for _ in range(4):
        lam = rng.normal(0, 5)
        mup = np.abs(rng.normal(0, 1, net.n_branch))
        mum = np.abs(rng.normal(0, 1, net.n_branch))
        ev = P.evaluate(net, Ha, d[None], [lam], mup[None], mum[None])
        res = minimize(lambda p: _lagrangian(net, Ha, d, lam, mup, mum, p),
                       0.5 * (net.gen_pmin + net.gen_pmax), method="L-BFGS-B",
                       bounds=list(zip(net.gen_pmin, net.gen_pmax)), options=dict(ftol=1e-15, gtol=1e-12))
        assert ev.value[0] <= res.fun + 1e-9 * max(1.0, abs(res.fun))
        assert ev.value[0] >= res.fun - 1e-6 * max(1.0, abs(res.fun))


@pytest.mark.parametrize("quadratic", [False, True])
def test_gradient_central_differences(quadratic):
    net = _net(12, 20, 5, 11, quadratic=quadratic)
    Ha = P.ptdf(net)
    rng = np.random.default_rng(3)
    d = net.base_load[None]
    lam = np.array([rng.normal(0, 10)])
    mup = np.abs(rng.normal(0, 10, (1, net.n_branch)))
    mum = np.abs(rng.normal(0, 10, (1, net.n_branch)))
    ev = P.evaluate(net, Ha, d, lam, mup, mum)
    h = 1e-6
    val = lambda l, a, b: P.evaluate(net, Ha, d, l, a, b).value[0]
    fd = (val(lam + h, mup, mum) - val(lam - h, mup, mum)) / (2 * h)
    assert abs(fd - ev.g_lam[0]) <= 1e-5 * max(1.0, abs(fd))
    for l in rng.choice(net.n_branch, 6, replace=False):
        e = np.zeros_like(mup)
        e[0, l] = h
        fdp = (val(lam, mup + e, mum) - val(lam, mup - e, mum)) / (2 * h)
        fdm = (val(lam, mup, mum + e) - val(lam, mup, mum - e)) / (2 * h)
        assert abs(fdp - ev.g_mup[0, l]) <= 1e-5 * max(1.0, abs(fdp))
        assert abs(fdm - ev.g_mum[0, l]) <= 1e-5 * max(1.0, abs(fdm))


def test_economic_dispatch_when_no_limit_binds():
    """With mu = 0 the dual is max over the scalar lambda of the merit-order
    relaxation; at lambda = -(marginal cost) it equals the economic-dispatch
    cost (fill the load in order of cost) -- a textbook closed form."""
    net = _net(20, 30, 8, 4)
    Ha = P.ptdf(net)
    d = net.base_load
    order = np.argsort(net.gen_c)
    left, cost, marg = d.sum(), 0.0, None
    for g in order:
        take = min(left, net.gen_pmax[g])
        cost += net.gen_c[g] * take
        left -= take
        if left <= 0:
            marg = net.gen_c[g]
            break
    ev = P.evaluate(net, Ha, d[None], [-marg], np.zeros((1, net.n_branch)), np.zeros((1, net.n_branch)))
    assert abs(ev.value[0] - cost) <= 1e-10 * cost


def test_weak_duality_and_convergence_to_lp_optimum():
    net = _net(14, 19, 5, 0)
    st, opt = inst.primal_lp(_no_angle_box(net), net.base_load)
    assert st == 0
    Ha = P.ptdf(net)
    K = 20000
    r = P.solve(net, net.base_load[None], K, np.full(K, 0.05), Ha=Ha, history=True,
                opt=dict(variant=P.OPT_ADAM, beta1=0.9, beta2=0.999, eps=1e-8))
    assert np.all(r.hist <= opt + 1e-9 * abs(opt))          # every iterate is a valid lower bound
    assert r.best[0] >= opt - 1e-4 * abs(opt)                 # and the ascent gets there
    assert np.all(r.mu >= 0.0)
    # same problem, plain step: still below, and best is the running max of the history
    r2 = P.solve(net, net.base_load[None], 2000, np.full(2000, 1e-3), Ha=Ha, history=True)
    assert np.all(r2.hist <= opt + 1e-9 * abs(opt))
    assert r2.best[0] == r2.hist[0].max()
    assert r2.bound[0] == r2.hist[0, -1]


def test_quadratic_weak_duality():
    net = _net(14, 19, 5, 1, quadratic=True)
    st, lo, hi = inst.primal_qp(_no_angle_box(net), net.base_load)
    assert st == 0
    K = 5000
    r = P.solve(net, net.base_load[None], K, np.full(K, 0.05), history=True,
                opt=dict(variant=P.OPT_ADAM, beta1=0.9, beta2=0.999, eps=1e-8))
    assert np.all(r.hist <= hi + 1e-9 * abs(hi))
    assert r.best[0] >= lo - 1e-3 * abs(lo)


def test_divergence_freeze_and_stopping_rule():
    net = _net(14, 19, 5, 0)
    Ha = P.ptdf(net)
    d = np.stack([net.base_load, 0.5 * net.base_load])
    # a huge step drives |g| past 1e15 (reading A-23): the detecting step is taken, later ones skipped
    K = 40
    r = P.solve(net, d, K, np.full(K, 1e16), Ha=Ha, history=True)
    assert np.all(r.status == P.DIVERGED)
    k0 = int(np.argmax(~np.isfinite(r.hist[0]) | (np.abs(r.hist[0]) > 1e15)))
    r0 = P.solve(net, d, k0 + 1, np.full(k0 + 1, 1e16), Ha=Ha)
    np.testing.assert_array_equal(r0.lam[0], r.lam[0])
    np.testing.assert_array_equal(r0.mu[0], r.mu[0])
    # stopping rule (A-29): a loose tolerance fires at k = 1 for the first instance only if
    # |g_1 - g_0| < tol; the frozen multipliers are those after the step of iteration 1
    K = 50
    full = P.solve(net, d, K, np.full(K, 1e-3), Ha=Ha, history=True)
    tol = float(np.abs(np.diff(full.hist[0]))[5]) * 1.0000001
    rs = P.solve(net, d, K, np.full(K, 1e-3), Ha=Ha, tol=tol, history=True)
    first = [int(np.argmax(np.abs(np.diff(full.hist[j])) < tol)) + 1 for j in range(2)]
    for j in range(2):
        if np.any(np.abs(np.diff(full.hist[j])) < tol):
            assert rs.status[j] == P.CONVERGED
            ref = P.solve(net, d[j:j + 1], first[j] + 1, np.full(first[j] + 1, 1e-3), Ha=Ha)
            np.testing.assert_array_equal(rs.mu[j], ref.mu[0])
            np.testing.assert_array_equal(rs.lam[j], ref.lam[0])
