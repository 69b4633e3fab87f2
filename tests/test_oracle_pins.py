"""Pins of the fp64 CPU oracle against what the paper and the mathematics fix
(SURVEY.md §8(c) P-1 ... P-9).  None of these re-types the oracle's closed
form: each compares it with a different computation (the plain Lagrangian of
Eq. 3 at enumerated box vertices, an LP solver, finite differences, textbook
closed forms, the paper's own Eq. 15 s-form, worked examples from SPEC.md).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.optimize import minimize_scalar

import oracle
from oracle import FORM_F1, FORM_F2
from paper_2406_13191_b200 import instances as inst

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _incidence(net, b=None):
    nl = net.n_branch
    li = np.arange(nl)
    A = sp.csr_matrix((np.r_[np.ones(nl), -np.ones(nl)], (np.r_[li, li], np.r_[net.br_from, net.br_to])),
                      shape=(nl, net.n_bus)).toarray()
    G = np.zeros((net.n_bus, net.n_gen))
    G[net.gen_bus, np.arange(net.n_gen)] = 1.0
    return A, G


def lagrangian_f2(net, d, lam, nu, P, Fl, Th, b):
    """Eq. 3 for the B-theta F2 form, evaluated at many
    points (rows of P, Fl, Th): cost + lam^T(Gp - A^T f - d) + nu^T(f - diag(b) A theta)."""
    A, G = _incidence(net)
    cost = P @ net.gen_c
    if net.gen_a is not None:
        cost = cost + (P * P) @ net.gen_a
    kcl = P @ G.T - Fl @ A - d[None, :]
    kvl = Fl - Th @ (np.diag(b) @ A).T
    return cost + kcl @ lam + kvl @ nu, kcl, kvl


def lagrangian_f1(net, d, lam, mup, mum, P, Th, b, F):
    """Eq. 3 for F1: flow limits +-diag(b)A theta <= F as the C x <= d rows."""
    A, G = _incidence(net)
    cost = P @ net.gen_c
    if net.gen_a is not None:
        cost = cost + (P * P) @ net.gen_a
    phi = Th @ (np.diag(b) @ A).T
    kcl = P @ G.T - phi @ A - d[None, :]
    return cost + kcl @ lam + (phi - F) @ mup + (-phi - F) @ mum, kcl, phi


def _vertices(lo, hi):
    n = len(lo)
    bits = np.array(list(itertools.product([0, 1], repeat=n)), dtype=float) if n else np.zeros((1, 0))
    return lo[None, :] + bits * (hi - lo)[None, :]


# ---------------------------------------------------------------------------
# P-1  inner minimiser vs brute force over all box vertices (LP)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_f2_value_equals_vertex_minimum(seed):
    net = inst.tiny_network(4, 5, 2, seed)  # 2 + 5 + 3 = 10 box coordinates
    rng = np.random.default_rng(100 + seed)
    lam, nu = inst.random_multipliers(rng, net, 4, FORM_F2)
    d = net.base_load
    lo = np.r_[net.gen_pmin, -net.br_fmax, -net.theta_max[1:]]
    hi = np.r_[net.gen_pmax, net.br_fmax, net.theta_max[1:]]
    V = _vertices(lo, hi)
    ng, nl = net.n_gen, net.n_branch
    P, Fl = V[:, :ng], V[:, ng:ng + nl]
    Th = np.c_[np.zeros(len(V)), V[:, ng + nl:]]
    val, gl, gb = oracle.evaluate(net, np.tile(d, (4, 1)), lam, nu)
    for j in range(4):
        L, _, _ = lagrangian_f2(net, d, lam[j], nu[j], P, Fl, Th, net.br_b)
        assert val[j] == pytest.approx(L.min(), rel=1e-13, abs=1e-11)
        # gradient = constraint residual at the minimising vertex (Danskin)
        k = int(np.argmin(L))
        _, kcl, kvl = lagrangian_f2(net, d, lam[j], nu[j], P[k:k + 1], Fl[k:k + 1], Th[k:k + 1], net.br_b)
        np.testing.assert_allclose(gl[j], kcl[0], rtol=0, atol=1e-12)
        np.testing.assert_allclose(gb[j], kvl[0], rtol=0, atol=1e-12)


@pytest.mark.parametrize("seed", [4, 5])
def test_f1_value_equals_vertex_minimum(seed):
    net = inst.tiny_network(6, 8, 3, seed)  # 3 + 5 coordinates
    rng = np.random.default_rng(200 + seed)
    lam, mu = inst.random_multipliers(rng, net, 3, FORM_F1)
    d = net.base_load
    lo = np.r_[net.gen_pmin, -net.theta_max[1:]]
    hi = np.r_[net.gen_pmax, net.theta_max[1:]]
    V = _vertices(lo, hi)
    P = V[:, :net.n_gen]
    Th = np.c_[np.zeros(len(V)), V[:, net.n_gen:]]
    val, gl, gb = oracle.evaluate(net, np.tile(d, (3, 1)), lam, mu, form=FORM_F1)
    nl = net.n_branch
    for j in range(3):
        L, _, _ = lagrangian_f1(net, d, lam[j], mu[j, :nl], mu[j, nl:], P, Th, net.br_b, net.br_fmax)
        assert val[j] == pytest.approx(L.min(), rel=1e-13, abs=1e-11)
        k = int(np.argmin(L))
        _, kcl, phi = lagrangian_f1(net, d, lam[j], mu[j, :nl], mu[j, nl:], P[k:k + 1], Th[k:k + 1],
                                    net.br_b, net.br_fmax)
        np.testing.assert_allclose(gl[j], kcl[0], atol=1e-12)
        np.testing.assert_allclose(gb[j, :nl], phi[0] - net.br_fmax, atol=1e-12)
        np.testing.assert_allclose(gb[j, nl:], -phi[0] - net.br_fmax, atol=1e-12)


def test_f1_config0_full_vertex_enumeration():
    """SURVEY P-1: F1 at config 0 has 5 + 13 = 18 coordinates, 262 144 vertices."""
    net = inst.make_network(0)
    rng = np.random.default_rng(7)
    lam, mu = inst.random_multipliers(rng, net, 1, FORM_F1, scale=10.0)
    d = net.base_load
    lo = np.r_[net.gen_pmin, -net.theta_max[1:]]
    hi = np.r_[net.gen_pmax, net.theta_max[1:]]
    V = _vertices(lo, hi)
    P = V[:, :net.n_gen]
    Th = np.c_[np.zeros(len(V)), V[:, net.n_gen:]]
    nl = net.n_branch
    L, _, _ = lagrangian_f1(net, d, lam[0], mu[0, :nl], mu[0, nl:], P, Th, net.br_b, net.br_fmax)
    val, _, _ = oracle.evaluate(net, d, lam, mu, form=FORM_F1)
    assert val[0] == pytest.approx(L.min(), rel=1e-13)


def test_dual_norm_identity():
    """App. A2: min over [lo,hi] of r.x = r.mid - |r|.half,
    i.e. max over the unit inf-ball of x^T y is ||y||_1, attained at sign(y).
    Checked through a 1-bus network whose dual value is sum_g min_p r_g p - lam d."""
    rng = np.random.default_rng(11)
    ng = 7
    net = inst.Network(n_bus=1, n_branch=0, n_gen=ng, ref_bus=0, br_from=np.zeros(0, np.int32),
                       br_to=np.zeros(0, np.int32), br_b=np.zeros(0), br_fmax=np.zeros(0),
                       theta_max=np.zeros(1), gen_bus=np.zeros(ng, np.int32),
                       gen_pmin=rng.uniform(-2, 0, ng), gen_pmax=rng.uniform(0, 3, ng),
                       gen_c=rng.normal(0, 5, ng))
    for lamv in rng.normal(0, 5, 20):
        val, _, _ = oracle.evaluate(net, np.array([0.0]), np.array([[lamv]]), np.zeros((1, 0)))
        r = net.gen_c + lamv
        mid = 0.5 * (net.gen_pmin + net.gen_pmax)
        half = 0.5 * (net.gen_pmax - net.gen_pmin)
        assert val[0] == pytest.approx(np.sum(r * mid) - np.sum(np.abs(r) * half), rel=1e-14, abs=1e-13)
        xs = rng.uniform(-1, 1, (1000, ng))  # random points of the ball never beat the bound
        assert np.all(xs @ (r * half) <= np.sum(np.abs(r * half)) + 1e-12)


# ---------------------------------------------------------------------------
# QP: coordinate-wise optimality of the clip minimiser + paper's Eq. 15


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_qp_minimiser_is_coordinatewise_optimal(form):
    net = inst.tiny_network(5, 6, 4, 9, quadratic=True)
    rng = np.random.default_rng(31)
    lam, br = inst.random_multipliers(rng, net, 2, form)
    # put r_g = c_g + lam_{beta(g)} inside (-2 a pmax, 0) so p* is interior for instance 0
    lam[0, net.gen_bus] = -net.gen_c - rng.uniform(0.1, 0.9, net.n_gen) * 2 * net.gen_a * net.gen_pmax
    d = net.base_load
    P, Fl, Th = oracle.minimiser(net, np.tile(d, (2, 1)), lam, br, form=form)
    val, _, _ = oracle.evaluate(net, np.tile(d, (2, 1)), lam, br, form=form)
    nl = net.n_branch
    interior = 0
    for j in range(2):
        def L(Pm, Fm, Tm):
            if form == FORM_F2:
                return lagrangian_f2(net, d, lam[j], br[j], Pm, Fm, Tm, net.br_b)[0]
            return lagrangian_f1(net, d, lam[j], br[j, :nl], br[j, nl:], Pm, Tm, net.br_b, net.br_fmax)[0]
        L0 = L(P[j:j + 1], Fl[j:j + 1], Th[j:j + 1])[0]
        assert val[j] == pytest.approx(L0, rel=1e-13)
        for g in range(net.n_gen):
            grid = np.linspace(net.gen_pmin[g], net.gen_pmax[g], 4001)
            Pm = np.repeat(P[j:j + 1], len(grid), 0)
            Pm[:, g] = grid
            Lg = L(Pm, np.repeat(Fl[j:j + 1], len(grid), 0), np.repeat(Th[j:j + 1], len(grid), 0))
            assert Lg.min() >= L0 - 1e-12
            interior += net.gen_pmin[g] < P[j, g] < net.gen_pmax[g]
    assert interior > 0


def _eq15_term(a, r, lo, hi, s):
    """Paper's final QP dual (Eq. 15) for one generator in the
    normalised coordinates of App. A1: x = m + sig*xt,
    cost a x^2 + r x = M xt^2 + ct xt + off with M = a sig^2, ct = (2 a m + r) sig,
    off = a m^2 + r m; the dual term is -|ct - s sqrt(M)| - 0.25 s^2 + off."""
    m, sig = 0.5 * (lo + hi), 0.5 * (hi - lo)
    M = a * sig * sig
    ct = (2 * a * m + r) * sig
    off = a * m * m + r * m
    return -abs(ct - s * math.sqrt(M)) - 0.25 * s * s + off


def test_eq15_equals_clip():
    """P-6 / PAPER.md:236 ('objective solutions of (9) and (15) exactly agree'):
    the oracle's clip-form dual value equals Eq. 15 maximised over s, exactly
    at s* = -2 sqrt(M) xt*, and to 1e-8 by a 1-D search."""
    rng = np.random.default_rng(5)
    for trial in range(300):
        a = rng.uniform(0.001, 0.5)
        lo = rng.uniform(-1, 1)
        hi = lo + rng.uniform(0.1, 3)
        c = rng.uniform(-5, 5)
        lamv = rng.normal(0, 2)
        d = rng.uniform(lo, hi)
        net = inst.Network(n_bus=1, n_branch=0, n_gen=1, ref_bus=0, br_from=np.zeros(0, np.int32),
                           br_to=np.zeros(0, np.int32), br_b=np.zeros(0), br_fmax=np.zeros(0),
                           theta_max=np.zeros(1), gen_bus=np.zeros(1, np.int32), gen_pmin=np.array([lo]),
                           gen_pmax=np.array([hi]), gen_c=np.array([c]), gen_a=np.array([a]))
        val, _, _ = oracle.evaluate(net, np.array([d]), np.array([[lamv]]), np.zeros((1, 0)))
        P, _, _ = oracle.minimiser(net, np.array([d]), np.array([[lamv]]), np.zeros((1, 0)))
        r = c + lamv
        m, sig = 0.5 * (lo + hi), 0.5 * (hi - lo)
        xt = (P[0, 0] - m) / sig
        s_star = -2.0 * math.sqrt(a * sig * sig) * xt
        ref = _eq15_term(a, r, lo, hi, s_star) - lamv * d
        assert val[0] == pytest.approx(ref, rel=1e-12, abs=1e-12)
        res = minimize_scalar(lambda s: -_eq15_term(a, r, lo, hi, s), bounds=(-50, 50), method="bounded",
                              options={"xatol": 1e-12})
        assert val[0] == pytest.approx(-res.fun - lamv * d, rel=1e-8, abs=1e-8)
        # weak duality of Eq. 15 at any s (Remark 2)
        for s in rng.normal(0, 3, 5):
            assert _eq15_term(a, r, lo, hi, s) - lamv * d <= val[0] + 1e-12


# ---------------------------------------------------------------------------
# P-3 gradient vs central finite differences


@pytest.mark.parametrize("form,quad", [(FORM_F2, False), (FORM_F2, True), (FORM_F1, False), (FORM_F1, True)])
def test_gradient_central_differences(form, quad):
    net = inst.tiny_network(8, 11, 4, 21, quadratic=quad)
    rng = np.random.default_rng(42)
    lam, br = inst.random_multipliers(rng, net, 1, form, scale=5.0)
    if form == FORM_F1:
        br = br + 1.0  # keep mu > 0 under the perturbation
    d = net.base_load
    val, gl, gb = oracle.evaluate(net, d, lam, br, form=form)
    h = 1e-6
    y = np.r_[lam[0], br[0]]
    grad = np.r_[gl[0], gb[0]]
    nb = net.n_bus
    fd = np.zeros_like(y)
    for k in range(len(y)):
        yp, ym = y.copy(), y.copy()
        yp[k] += h
        ym[k] -= h
        vp, _, _ = oracle.evaluate(net, d, yp[None, :nb], yp[None, nb:], form=form)
        vm, _, _ = oracle.evaluate(net, d, ym[None, :nb], ym[None, nb:], form=form)
        fd[k] = (vp[0] - vm[0]) / (2 * h)
    np.testing.assert_allclose(grad, fd, rtol=0, atol=2e-6)


# ---------------------------------------------------------------------------
# P-2 weak duality vs an exact LP solver (HiGHS) and the oracle trajectory


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_weak_duality_random_points_config0(form):
    net = inst.make_network(0)
    status, opt = inst.primal_lp(net, net.base_load)
    assert status == 0 and opt == pytest.approx(77.578167948, rel=1e-10)  # SURVEY P-1 value
    rng = np.random.default_rng(3)
    lam, br = inst.random_multipliers(rng, net, 1000, form, scale=30.0)
    val, _, _ = oracle.evaluate(net, np.tile(net.base_load, (1000, 1)), lam, br, form=form)
    assert np.all(val <= opt + 1e-9 * abs(opt))


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_weak_duality_every_iterate(form):
    net = inst.make_network(0, theta_mode="min")
    status, opt = inst.primal_lp(net, net.base_load)
    assert status == 0
    r = oracle.solve(net, net.base_load, K=3000, alpha=inst.alpha_schedule(3000, 1e-2), form=form,
                     history=True)
    assert np.all(r.hist <= opt + 1e-9 * abs(opt))
    assert r.best[0] <= opt


def test_weak_duality_qp_tiny():
    net = inst.tiny_network(6, 8, 4, 17, quadratic=True)
    st, lower, upper = inst.primal_qp(net, net.base_load)
    assert st == 0
    rng = np.random.default_rng(8)
    for form in (FORM_F2, FORM_F1):
        lam, br = inst.random_multipliers(rng, net, 500, form, scale=30.0)
        val, _, _ = oracle.evaluate(net, np.tile(net.base_load, (500, 1)), lam, br, form=form)
        assert np.all(val <= upper + 1e-9 * abs(upper))
        r = oracle.solve(net, net.base_load, K=4000, alpha=inst.alpha_schedule(4000, 1e-2), form=form,
                         history=True)
        assert np.all(r.hist <= upper + 1e-9 * abs(upper))


# ---------------------------------------------------------------------------
# P-4 first iterates in closed form (exact in fp64)


def test_first_iterates_f2_closed_form():
    net = inst.make_network(0)
    d = net.base_load
    a = 1e-3
    assert np.all(net.gen_c > a * d[net.gen_bus])  # precondition of the closed form
    r = oracle.solve(net, d, K=1, alpha=inst.alpha_schedule(1, a), history=True)
    assert r.hist[0, 0] == 0.0  # g(y_0) = sum_g c_g pmin_g = 0
    np.testing.assert_array_equal(r.lam[0], -a * d)  # y_1 = (-alpha d, 0): grad_lam(y_0) = -d
    np.testing.assert_array_equal(r.br[0], 0.0)
    closed = a * (d @ d - np.sum(net.br_fmax * np.abs(d[net.br_from] - d[net.br_to])))
    assert r.hist[0, 1] == pytest.approx(closed, rel=1e-13)
    assert r.hist[0, 1] == pytest.approx(-0.0014577610775518, abs=1e-16)  # SURVEY Appendix P-6 value


def test_first_iterates_f1_closed_form():
    net = inst.make_network(0)
    d = net.base_load
    a = 1e-3
    r = oracle.solve(net, d, K=1, alpha=inst.alpha_schedule(1, a), form=FORM_F1, history=True)
    assert r.hist[0, 0] == 0.0
    np.testing.assert_array_equal(r.lam[0], -a * d)
    np.testing.assert_array_equal(r.br[0], 0.0)  # projection active at y_0: mu stays 0
    A, _ = _incidence(net)
    Ld = A.T @ np.diag(net.br_b) @ A @ d
    closed = a * (d @ d) - a * np.sum(net.theta_max[1:] * np.abs(Ld[1:]))
    assert r.hist[0, 1] == pytest.approx(closed, rel=1e-12)


# ---------------------------------------------------------------------------
# P-5 single-bus economic dispatch (n_branch = 0) and the SPEC worked examples


def test_spec_1bus_golden():
    g = json.load(open(os.path.join(GOLDEN, "spec_1bus.json")))
    net = inst.Network(n_bus=1, n_branch=0, n_gen=1, ref_bus=0, br_from=np.zeros(0, np.int32),
                       br_to=np.zeros(0, np.int32), br_b=np.zeros(0), br_fmax=np.zeros(0),
                       theta_max=np.array(g["theta_max"]), gen_bus=np.array(g["gen_bus"], np.int32),
                       gen_pmin=np.array(g["gen_pmin"]), gen_pmax=np.array(g["gen_pmax"]),
                       gen_c=np.array(g["gen_c"]))
    r = oracle.solve(net, np.array(g["load"]), K=g["K"], alpha=inst.alpha_schedule(g["K"], g["alpha"]))
    assert r.best[0] == g["expected_bound"]
    assert r.bound[0] == g["expected_bound"]


def test_spec_2bus_golden_strong_duality():
    g = json.load(open(os.path.join(GOLDEN, "spec_2bus.json")))
    net = inst.Network(n_bus=2, n_branch=1, n_gen=1, ref_bus=0, br_from=np.array(g["br_from"], np.int32),
                       br_to=np.array(g["br_to"], np.int32), br_b=np.array(g["br_b"]),
                       br_fmax=np.array(g["br_fmax"]), theta_max=np.array(g["theta_max"]),
                       gen_bus=np.array(g["gen_bus"], np.int32), gen_pmin=np.array(g["gen_pmin"]),
                       gen_pmax=np.array(g["gen_pmax"]), gen_c=np.array(g["gen_c"]))
    st, opt = inst.primal_lp(net, np.array(g["load"]))
    assert st == 0 and opt == pytest.approx(g["expected_optimum"], rel=1e-12)
    # A dual optimum: lambda = -c at both buses (r = 0, p* = any; the KCL residual
    # vanishes at the midpoint 100), nu = 0 -> g = -lambda^T d = 5 * 100.
    for form in (FORM_F2, FORM_F1):
        nbr = 1 if form == FORM_F2 else 2
        val, _, _ = oracle.evaluate(net, np.array(g["load"]), np.array([[-5.0, -5.0]]), np.zeros((1, nbr)),
                                    form=form)
        assert val[0] == g["expected_optimum"]


def test_single_bus_merit_order():
    rng = np.random.default_rng(13)
    ng = 9
    pmax = rng.uniform(0.5, 3, ng)
    c = rng.uniform(10, 50, ng)
    net = inst.Network(n_bus=1, n_branch=0, n_gen=ng, ref_bus=0, br_from=np.zeros(0, np.int32),
                       br_to=np.zeros(0, np.int32), br_b=np.zeros(0), br_fmax=np.zeros(0),
                       theta_max=np.zeros(1), gen_bus=np.zeros(ng, np.int32), gen_pmin=np.zeros(ng),
                       gen_pmax=pmax, gen_c=c)
    d = 0.55 * pmax.sum()
    # textbook merit order: fill cheapest first
    order = np.argsort(c)
    rem, cost, marg = d, 0.0, None
    for g in order:
        take = min(rem, pmax[g])
        cost += c[g] * take
        rem -= take
        if rem <= 0:
            marg = c[g]
            break
    val, _, _ = oracle.evaluate(net, np.array([d]), np.array([[-marg]]), np.zeros((1, 0)))
    assert val[0] == pytest.approx(cost, rel=1e-13)
    # and no other lambda does better (concave 1-D dual)
    grid = np.linspace(-60, 0, 2001)
    vals, _, _ = oracle.evaluate(net, np.full((len(grid), 1), d), grid[:, None], np.zeros((len(grid), 0)))
    assert vals.max() <= cost + 1e-9


def test_single_bus_qp_equal_incremental_cost():
    """QP economic dispatch: max_lambda g = min cost, found by bisection on the
    equal-incremental-cost condition sum_g clip((lam-c)/(2a)) = d."""
    rng = np.random.default_rng(14)
    ng = 6
    pmax = rng.uniform(0.5, 3, ng)
    c = rng.uniform(10, 50, ng)
    a = rng.uniform(0.5, 5, ng)
    net = inst.Network(n_bus=1, n_branch=0, n_gen=ng, ref_bus=0, br_from=np.zeros(0, np.int32),
                       br_to=np.zeros(0, np.int32), br_b=np.zeros(0), br_fmax=np.zeros(0),
                       theta_max=np.zeros(1), gen_bus=np.zeros(ng, np.int32), gen_pmin=np.zeros(ng),
                       gen_pmax=pmax, gen_c=c, gen_a=a)
    d = 0.5 * pmax.sum()
    lo, hi = 0.0, 200.0
    for _ in range(200):
        mc = 0.5 * (lo + hi)
        if np.clip((mc - c) / (2 * a), 0, pmax).sum() < d:
            lo = mc
        else:
            hi = mc
    p = np.clip((mc - c) / (2 * a), 0, pmax)
    cost = c @ p + a @ (p * p)
    val, _, _ = oracle.evaluate(net, np.array([d]), np.array([[-mc]]), np.zeros((1, 0)))
    assert val[0] == pytest.approx(cost, rel=1e-10)


# ---------------------------------------------------------------------------
# P-7 invariants


def test_best_is_running_max_and_projection_keeps_mu_nonnegative():
    net = inst.make_network(0)
    r = oracle.solve(net, net.base_load, K=500, alpha=inst.alpha_schedule(500, 5e-3), form=FORM_F1,
                     history=True)
    assert r.best[0] == r.hist[0].max()
    assert np.all(r.br >= 0.0)
    assert r.bound[0] == r.hist[0, -1]


def test_determinism_and_batch_isolation():
    net = inst.make_network(0)
    rng = np.random.default_rng(0)
    loads = net.base_load[None, :] * rng.uniform(0.8, 1.2, (8, net.n_bus))
    a = inst.alpha_schedule(300, 3e-3)
    r1 = oracle.solve(net, loads, K=300, alpha=a, history=True, threads=4)
    r2 = oracle.solve(net, loads, K=300, alpha=a, history=True, threads=1)
    np.testing.assert_array_equal(r1.lam, r2.lam)
    np.testing.assert_array_equal(r1.hist, r2.hist)
    for j in range(8):
        rj = oracle.solve(net, loads[j], K=300, alpha=a, history=True)
        np.testing.assert_array_equal(rj.lam[0], r1.lam[j])
        np.testing.assert_array_equal(rj.br[0], r1.br[j])
        np.testing.assert_array_equal(rj.hist[0], r1.hist[j])


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_outage_equals_branch_removed(form):
    """Reading A-16: an outaged branch (b = F = 0) behaves exactly like a
    network without it; its multipliers stay at 0."""
    net = inst.make_network(0)
    l_out = 15  # a non-tree branch (tree = first 13)
    assert l_out >= net.n_tree
    keep = np.array([l for l in range(net.n_branch) if l != l_out])
    import copy
    red = copy.copy(net)
    red.n_branch = len(keep)
    red.br_from, red.br_to = net.br_from[keep], net.br_to[keep]
    red.br_b, red.br_fmax = net.br_b[keep], net.br_fmax[keep]
    a = inst.alpha_schedule(400, 4e-3)
    r_full = oracle.solve(net, net.base_load, outages=np.array([[l_out, -1]]), K=400, alpha=a, form=form,
                          history=True)
    r_red = oracle.solve(red, net.base_load, K=400, alpha=a, form=form, history=True)
    np.testing.assert_array_equal(r_full.lam, r_red.lam)
    np.testing.assert_array_equal(r_full.hist, r_red.hist)
    nl = net.n_branch
    if form == FORM_F2:
        assert r_full.br[0, l_out] == 0.0
        np.testing.assert_array_equal(r_full.br[0, keep], r_red.br[0])
    else:
        assert r_full.br[0, l_out] == 0.0 and r_full.br[0, nl + l_out] == 0.0


def test_divergence_freezes_instance():
    """SPEC.md:320/360 and reading A-23: |g| > 1e15 marks DIVERGED, y frozen
    after the step of that iteration, best keeps only valid values; other
    instances in the batch are unaffected."""
    net = inst.make_network(0)
    loads = np.stack([net.base_load, net.base_load * 1e14])
    a = inst.alpha_schedule(50, 1e-3)
    r = oracle.solve(net, loads, K=50, alpha=a, history=True)
    assert r.status[0] == 0 and r.status[1] == oracle.DIVERGED
    ok = oracle.solve(net, loads[:1], K=50, alpha=a, history=True)
    np.testing.assert_array_equal(ok.hist[0], r.hist[0])
    h = r.hist[1]
    k = int(np.argmax(~((np.abs(h) <= 1e15) & np.isfinite(h))))
    assert np.all(h[k + 1:] == h[k + 1])  # frozen at y_{k+1}
    valid = h[:k][np.isfinite(h[:k])]
    assert r.best[1] == (valid.max() if len(valid) else -np.inf)


# ---------------------------------------------------------------------------
# P-9 strong duality (loose sanity): a tuned plain ascent gets close on config 0


@pytest.mark.parametrize("form,tol", [(FORM_F2, 0.03), (FORM_F1, 0.06)])
def test_strong_duality_loose(form, tol):
    net = inst.make_network(0, theta_mode="min")
    st, opt = inst.primal_lp(net, net.base_load)
    r = oracle.solve(net, net.base_load, K=20000, alpha=inst.alpha_schedule(20000, 1e-2), form=form)
    assert r.best[0] <= opt
    assert (opt - r.best[0]) / opt < tol


def test_literal_config0_pi3_box_is_not_binding():
    """SURVEY F-2: at seed 0 the pi/3 box does not bind (same LP optimum)."""
    a = inst.make_network(0)
    b = inst.make_network(0, theta_mode="implied")
    assert inst.primal_lp(a, a.base_load)[1] == pytest.approx(inst.primal_lp(b, b.base_load)[1], rel=1e-12)


# ---------------------------------------------------------------------------
# gradient-based-optimisation variants (Algorithm 1 247-272;
# SPEC.md:326-328): pins from special cases, closed-form first steps, weak
# duality along every trajectory and convergence to the LP optimum

ADAM = dict(variant=oracle.OPT_ADAM, beta1=0.9, beta2=0.999, eps=1e-8)
ADAGRAD = dict(variant=oracle.OPT_ADAGRAD, eps=1e-8)
GDM = dict(variant=oracle.OPT_GDM, rho=0.9)
GDM_C = dict(variant=oracle.OPT_GDM_CLASSIC, rho=0.9)


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_gdm_classic_without_momentum_is_the_plain_step(form):
    """rho = 0: v = 0 v + a g = a g exactly, y + v = y + a g: bitwise plain."""
    net = inst.make_network(0, theta_mode="min")
    K = 800
    a = inst.alpha_schedule(K, 1e-2)
    p = oracle.solve(net, net.base_load, K=K, alpha=a, form=form, history=True)
    q = oracle.solve(net, net.base_load, K=K, alpha=a, form=form, history=True,
                     opt=dict(variant=oracle.OPT_GDM_CLASSIC, rho=0.0))
    np.testing.assert_array_equal(p.lam, q.lam)
    np.testing.assert_array_equal(p.br, q.br)
    np.testing.assert_array_equal(p.hist, q.hist)


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
def test_gdm_first_step_is_a_double_plain_step(form):
    """Algorithm 1 from y_0 = v_0 = 0: v_1 = a g_0, y = a g_0 (velocity
    update) then y = a g_0 + a g_0 (gradient update) = (2a) g_0 exactly: the
    plain step with 2a (then mu <- max(mu, 0) on both sides)."""
    net = inst.make_network(0, theta_mode="min")
    a = 7e-3
    g = oracle.solve(net, net.base_load, K=1, alpha=np.array([a]), form=form, opt=dict(GDM, rho=0.37))
    p = oracle.solve(net, net.base_load, K=1, alpha=np.array([2 * a]), form=form)
    np.testing.assert_array_equal(g.lam, p.lam)
    np.testing.assert_array_equal(g.br, p.br)


@pytest.mark.parametrize("opt", [ADAM, ADAGRAD, dict(ADAM, beta1=0.0, beta2=0.0)])
def test_adaptive_first_step_is_a_normalised_sign_step(opt):
    """Adam (Kingma & Ba) and AdaGrad from zero state: the first step is
    a g_0 / (|g_0| + eps) per coordinate (bias corrections cancel)."""
    net = inst.make_network(0, theta_mode="min")
    a = 0.05
    _, g0l, g0b = oracle.evaluate(net, net.base_load, np.zeros((1, net.n_bus)), np.zeros((1, net.n_branch)))
    r = oracle.solve(net, net.base_load, K=1, alpha=np.array([a]), opt=opt)
    g0 = np.r_[g0l[0], g0b[0]]
    y1 = np.r_[r.lam[0], r.br[0]]
    expect = a * g0 / (np.abs(g0) + opt["eps"])
    assert np.max(np.abs(y1 - expect)) <= 1e-15 * a * 4
    nz = np.abs(g0) > 1e-3
    assert np.allclose(np.abs(y1[nz]), a, rtol=1e-5)   # magnitude ~ a wherever |g| >> eps


@pytest.mark.parametrize("form", [FORM_F2, FORM_F1])
@pytest.mark.parametrize("opt,alpha", [(ADAM, 0.1), (ADAGRAD, 3.0), (GDM, 1e-3), (GDM_C, 3e-3)])
def test_variants_weak_duality_and_convergence(form, opt, alpha):
    """Every iterate of every variant is a valid lower bound (PAPER.md:135:
    any lambda, nu and mu >= 0), and with a reasonable step each reaches the
    HiGHS LP optimum of config 0 within 2% (Tables 1-3 report gaps
    of 1e-4 .. 1% for the tuned IEEE runs; this is a sanity bar)."""
    net = inst.make_network(0, theta_mode="min")
    _, opt_val = inst.primal_lp(net, net.base_load)
    K = 20000
    r = oracle.solve(net, net.base_load, K=K, alpha=inst.alpha_schedule(K, alpha), form=form, history=True,
                     opt=opt)
    assert r.status[0] == 0
    assert np.all(r.hist[0] <= opt_val + 1e-9 * abs(opt_val))
    assert r.best[0] >= (0.98 if form == FORM_F2 else 0.95) * opt_val, r.best[0]
    if form == FORM_F1:
        assert np.all(r.br >= 0.0)


# ---------------------------------------------------------------------------
# KVL (cycle-basis) form, reading A-28: the sparse twin of the
# paper's PTDF constraint (Eq. 1) with no angles


def _cycle_matrix(net, switchable=None):
    d, cyc = oracle.cycles(net, switchable)
    C = np.zeros((len(d), net.n_branch))
    for k, (bs, ss) in enumerate(cyc):
        C[k, bs] = ss
    return d, C


@pytest.mark.parametrize("config", [0, 1])
def test_kvl_cycle_basis_is_a_basis_of_closed_loops(config):
    """n_l - n_b + 1 independent cycles; each is a closed walk (C A = 0: the
    signed incidence around a loop cancels at every bus); its defining
    non-tree branch appears with +1 and no other non-tree branch appears."""
    net = inst.make_network(config)
    d, C = _cycle_matrix(net)
    A, _ = _incidence(net)
    assert C.shape[0] == net.n_branch - net.n_bus + 1
    assert np.all(C @ A == 0)
    assert np.linalg.matrix_rank(C) == C.shape[0]
    nontree = np.zeros(net.n_branch, bool)
    nontree[d] = True
    for k in range(len(d)):
        assert C[k, d[k]] == 1
        assert np.count_nonzero(C[k, nontree]) == 1


def test_kvl_annihilates_dc_power_flow():
    """DC power-flow flows f = diag(b) A theta satisfy sum_l C_kl f_l / b_l = 0
    on every cycle (Kirchhoff's voltage law), and any vector in the null space
    of C diag(1/b) with KCL is such a flow (dimension count)."""
    net = inst.make_network(1)
    _, C = _cycle_matrix(net)
    inj = np.zeros(net.n_bus)
    np.add.at(inj, net.gen_bus, net.gen_pmax * net.base_load.sum() / net.gen_pmax.sum())
    inj -= net.base_load
    f = inst.dc_flows(net.n_bus, net.ref_bus, net.br_from, net.br_to, net.br_b, inj)
    assert np.max(np.abs(C @ (f / net.br_b))) <= 1e-9 * np.max(np.abs(f / net.br_b))


def lagrangian_kvl(net, d, lam, kap, P, Fl, C, x):
    """Eq. 3 for the KVL form: cost + lam^T(Gp - A^T f - d) + kap^T C diag(x) f."""
    A, G = _incidence(net)
    cost = P @ net.gen_c
    if net.gen_a is not None:
        cost = cost + (P * P) @ net.gen_a
    kcl = P @ G.T - Fl @ A - d[None, :]
    kvl = Fl @ (C @ np.diag(x)).T
    return cost + kcl @ lam + kvl @ kap, kcl, kvl


@pytest.mark.parametrize("seed", range(4))
def test_kvl_value_equals_vertex_minimum(seed):
    """The dual function = min of the Lagrangian over ALL vertices of the
    p and f boxes (brute force, dense matrices); gradient = residuals there."""
    net = inst.tiny_network(5, 8, 2, seed=seed)
    _, C = _cycle_matrix(net)
    x = 1.0 / net.br_b
    rng = np.random.default_rng(seed + 10)
    lam = rng.normal(0, 20, net.n_bus)
    kap = rng.normal(0, 3, C.shape[0])
    val, gl, gk, p, f = oracle.evaluate_kvl(net, net.base_load, lam, kap)
    V = _vertices(np.r_[net.gen_pmin, -net.br_fmax], np.r_[net.gen_pmax, net.br_fmax])
    L, kcl, kvl = lagrangian_kvl(net, net.base_load, lam, kap, V[:, :net.n_gen], V[:, net.n_gen:], C, x)
    j = int(np.argmin(L))
    assert abs(val[0] - L[j]) <= 1e-9 * max(1.0, abs(L[j]))
    np.testing.assert_allclose(gl[0], kcl[j], atol=1e-9)
    np.testing.assert_allclose(gk[0], kvl[j], atol=1e-9)


def test_kvl_gradient_central_differences():
    net = inst.make_network(0)
    _, C = _cycle_matrix(net)
    rng = np.random.default_rng(3)
    lam = rng.normal(-30, 10, net.n_bus)
    kap = rng.normal(0, 50, C.shape[0])
    _, gl, gk, _, _ = oracle.evaluate_kvl(net, net.base_load, lam, kap)
    h = 1e-6
    for i in range(net.n_bus):
        e = np.zeros(net.n_bus)
        e[i] = h
        fd = (oracle.evaluate_kvl(net, net.base_load, lam + e, kap)[0][0] -
              oracle.evaluate_kvl(net, net.base_load, lam - e, kap)[0][0]) / (2 * h)
        assert abs(fd - gl[0, i]) <= 1e-6
    for k in range(C.shape[0]):
        e = np.zeros(C.shape[0])
        e[k] = h
        fd = (oracle.evaluate_kvl(net, net.base_load, lam, kap + e)[0][0] -
              oracle.evaluate_kvl(net, net.base_load, lam, kap - e)[0][0]) / (2 * h)
        assert abs(fd - gk[0, k]) <= 1e-6


@pytest.mark.parametrize("opt,alpha,tol", [(None, 1e-2, 0.01), (ADAM, 0.1, 0.01), (GDM, 1e-3, 0.01)])
def test_kvl_weak_and_strong_duality_config0(opt, alpha, tol):
    """Every iterate <= the LP optimum (no angle box in this form: the primal
    is the paper's Eq. 1); Adam / GDM get within 1% (survey P-4: KVL is the
    best-converging form)."""
    net = inst.make_network(0)
    _, opt_val = inst.primal_lp(net, net.base_load)
    K = 20000
    r = oracle.solve(net, net.base_load, K=K, alpha=inst.alpha_schedule(K, alpha), form=oracle.FORM_KVL,
                     history=True, opt=opt)
    assert np.all(r.hist[0] <= opt_val + 1e-9 * abs(opt_val))
    assert r.best[0] >= (1 - tol) * opt_val, r.best[0]


def test_kvl_outage_equals_branch_removed():
    """An outaged (switchable, hence non-tree) branch drops its own cycle:
    the run equals the network without that branch, bitwise."""
    net = inst.make_network(1)
    sw = np.zeros(net.n_branch, np.uint8)
    sw[net.n_tree:] = 1
    l = net.n_tree + 17
    K = 300
    a = inst.alpha_schedule(K, 0.05)
    r = oracle.solve(net, net.base_load, outages=np.array([[l]]), K=K, alpha=a, form=oracle.FORM_KVL,
                     switchable=sw, opt=ADAM)
    keep = np.r_[0:l, l + 1:net.n_branch]
    sub = inst.Network(**{**net.__dict__, "n_branch": net.n_branch - 1, "br_from": net.br_from[keep],
                          "br_to": net.br_to[keep], "br_b": net.br_b[keep], "br_fmax": net.br_fmax[keep]})
    r2 = oracle.solve(sub, net.base_load, K=K, alpha=a, form=oracle.FORM_KVL, switchable=sw[keep], opt=ADAM)
    d, _ = _cycle_matrix(net, sw)
    k = int(np.nonzero(d == l)[0][0])
    assert r.br[0, k] == 0.0
    np.testing.assert_array_equal(r.lam, r2.lam)
    np.testing.assert_array_equal(np.delete(r.br[0], k), r2.br[0])
    assert r.best[0] == r2.best[0]


# ---------------------------------------------------------------------------
# Algorithm 1's stopping rule, reading A-29


def test_stopping_rule_oracle():
    """The instance stops at the first k >= 1 with |g_k - g_{k-1}| < tol (the
    step of that iteration is still taken, A-29): its multipliers equal a run
    of exactly k+1 steps, no earlier consecutive pair is within tol, and
    tol = 0 changes nothing."""
    net = inst.make_network(0, theta_mode="min")
    K = 20000
    a = inst.alpha_schedule(K, 0.1)
    tol = 1e-4
    r = oracle.solve(net, net.base_load, K=K, alpha=a, opt=ADAM, tol=tol, history=True)
    full = oracle.solve(net, net.base_load, K=K, alpha=a, opt=ADAM, history=True)
    assert r.status[0] == oracle.CONVERGED
    d = np.abs(np.diff(full.hist[0]))
    k = int(np.nonzero(d < tol)[0][0]) + 1
    np.testing.assert_array_equal(r.hist[0, :k + 1], full.hist[0, :k + 1])
    again = oracle.solve(net, net.base_load, K=k + 1, alpha=a, opt=ADAM)
    np.testing.assert_array_equal(r.lam, again.lam)
    np.testing.assert_array_equal(r.br, again.br)
    assert np.all(r.hist[0, k + 1:] == r.hist[0, k + 1])      # frozen afterwards
    z = oracle.solve(net, net.base_load, K=3000, alpha=a, opt=ADAM, tol=0.0)
    z0 = oracle.solve(net, net.base_load, K=3000, alpha=a, opt=ADAM)
    np.testing.assert_array_equal(z.lam, z0.lam)
    assert z.status[0] == 0


def test_alpha_schedule_decays():
    """The explicit step arrays (reading A-9) with the paper's step decay
    (PAPER.md:348): constant, alpha/(1 + k/T), alpha F^floor(k/N)."""
    a = inst.alpha_schedule(6, 2.0)
    assert np.all(a == 2.0)
    a = inst.alpha_schedule(5, 5.0, "inv:200")
    np.testing.assert_allclose(a, 5.0 / (1.0 + np.arange(5) / 200.0), rtol=0, atol=0)
    a = inst.alpha_schedule(7, 2.0, "step:0.5:3")
    np.testing.assert_array_equal(a, [2, 2, 2, 1, 1, 1, 0.5])
    with pytest.raises(ValueError):
        inst.alpha_schedule(3, 1.0, "cosine:1")
