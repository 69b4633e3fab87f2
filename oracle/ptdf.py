"""Dense-PTDF form of the dual, plain numpy fp64.

TEST INFRASTRUCTURE ONLY, like the rest of oracle/: tests/, the smoke check and
bench.py's cpu_baseline / `--impl reference` legs are the only callers; the
product path never imports it.

This is the paper's problem literally (Eq. 1):

    min_p  sum_g a_g p_g^2 + c_g p_g
    s.t.   1^T p - 1^T d = 0                         : lambda (scalar, free)
           H_a (G p - d) - F <= 0                     : mu+ >= 0   (n_l rows)
          -H_a (G p - d) - F <= 0                     : mu- >= 0   (n_l rows)
           pmin <= p <= pmax

with H = Omega E (E^T Omega E)^{-1} the PTDF matrix and H_a its slack-augmented
version, G the generator-to-bus map (reading A-22: several
generators per bus), -F / +F the flow limits p_f bounds of Eq. 1c.  In the
paper's canonical notation (Eq. 2) the equality row is
A x - b = 0 and the 2 n_l flow rows are C x - d <= 0; the dual function
(Eq. 4-5) is, with r = H_a d and H_g = H_a G,

    q      = c + lambda 1 + H_g^T (mu+ - mu-)                 (cost vector)
    p*     = argmin over the box of a p^2 + q p                (Eq. 7b / 15)
    g      = sum_g (a p*^2 + q p*) - lambda 1^T d
             - mu+^T (r + F) + mu-^T (r - F)                   (the bound)
    dg/dlambda = 1^T p* - 1^T d,   dg/dmu+ = H_g p* - r - F,   dg/dmu- = r - H_g p* - F

and the ascent step y <- y + alpha_k grad, mu <- max(mu, 0) (
Alg. 1).  The linear-cost minimiser is the dual-norm bound
selection (sign(0) -> box midpoint, reading A-4); the quadratic one is
per-generator clipping (reading A-6).  Step variants, divergence and stopping
rule follow readings A-23, A-25, A-26, A-29 exactly as oracle/dcopf_oracle.c
does for the sparse forms.

Everything is numpy matrix algebra in fp64 (a library matmul / solve is a
step, no blocking or reordering).  Pinned in tests/test_ptdf_oracle.py against
the SPEC 2-bus example, the closed-form flows of a radial network, Kirchhoff's
current and voltage laws, brute force over box vertices, finite differences,
economic dispatch, and the exact LP optimum (weak duality and convergence).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

OPT_PLAIN, OPT_GDM, OPT_GDM_CLASSIC, OPT_ADAGRAD, OPT_ADAM = 0, 1, 2, 3, 4
DIVERGED = 1
CONVERGED = 2


def incidence(net) -> np.ndarray:
    """Dense branch-bus incidence E [n_l][n_b]: +1 at the from-bus, -1 at the
    to-bus (SPEC.md:111 orientation), so f = diag(b) E theta."""
    E = np.zeros((net.n_branch, net.n_bus))
    li = np.arange(net.n_branch)
    E[li, net.br_from] = 1.0
    E[li, net.br_to] = -1.0
    return E


def ptdf(net) -> np.ndarray:
    """H_a [n_l][n_b] = Omega E_r (E_r^T Omega E_r)^{-1} with the slack column
    set to zero (solve, do not invert).  E_r is
    E without the reference bus column; a branch with b = 0 carries no flow.
    Raises numpy.linalg.LinAlgError when E^T Omega E is singular
    (disconnected over b > 0)."""
    E = incidence(net)
    keep = np.array([i for i in range(net.n_bus) if i != net.ref_bus], dtype=np.int64)
    Er = E[:, keep]
    Om = np.diag(np.asarray(net.br_b, dtype=np.float64))
    Bred = Er.T @ Om @ Er                       # reduced nodal susceptance matrix
    X = np.linalg.solve(Bred, (Om @ Er).T)      # (E^T Omega E) X = (Omega E)^T, X = H^T
    Ha = np.zeros((net.n_branch, net.n_bus))
    Ha[:, keep] = X.T
    # PTDF entries are flow fractions (|H| <= 1); below 1e-12 an entry is the
    # solve's rounding residue of a structural zero -- no path from the bus to
    # the slack runs through the line -- and is set to that exact 0 (reading A-30)
    Ha[np.abs(Ha) < 1e-12] = 0.0
    return Ha


def _gen_a(net):
    return None if net.gen_a is None else np.asarray(net.gen_a, dtype=np.float64)


def minimiser(net, q: np.ndarray) -> np.ndarray:
    """p* [B][n_g] minimising a p^2 + q p over [pmin, pmax] per generator:
    clip(-q / (2a)) where a > 0, else bound selection with sign(0) -> midpoint
    (PAPER.md:157-160 dual norm; App. A2; readings A-4, A-6)."""
    lo = np.broadcast_to(net.gen_pmin, q.shape)
    hi = np.broadcast_to(net.gen_pmax, q.shape)
    p = np.where(q > 0.0, lo, np.where(q < 0.0, hi, 0.5 * (lo + hi)))
    a = _gen_a(net)
    if a is not None:
        quad = np.broadcast_to(a > 0.0, q.shape)
        with np.errstate(divide="ignore", invalid="ignore"):
            x = -q / (2.0 * np.where(a > 0.0, a, 1.0))
        p = np.where(quad, np.clip(x, lo, hi), p)
    return p


@dataclass
class PtdfEval:
    value: np.ndarray     # [B]
    g_lam: np.ndarray     # [B]
    g_mup: np.ndarray     # [B][n_l]
    g_mum: np.ndarray     # [B][n_l]
    p: np.ndarray         # [B][n_g]


def evaluate(net, Ha, load, lam, mup, mum, _pre=None) -> PtdfEval:
    """Dual value and gradient at (lambda[B], mu+[B][n_l], mu-[B][n_l]).
    _pre: (H_g, 1^T d, H_a d) already formed for this net and load (solve()
    forms them once; the same expressions, so the same values)."""
    load = np.atleast_2d(np.asarray(load, dtype=np.float64))
    lam = np.asarray(lam, dtype=np.float64).reshape(-1)
    mup = np.atleast_2d(np.asarray(mup, dtype=np.float64))
    mum = np.atleast_2d(np.asarray(mum, dtype=np.float64))
    if _pre is None:
        _pre = _constants(net, Ha, load)
    Hg, D, r = _pre                             # H_a G [n_l][n_g], 1^T d [B], H_a d [B][n_l]
    F = np.asarray(net.br_fmax, dtype=np.float64)
    q = net.gen_c[None, :] + lam[:, None] + (mup - mum) @ Hg
    p = minimiser(net, q)
    a = _gen_a(net)
    obj = q * p if a is None else a[None, :] * p * p + q * p
    value = obj.sum(axis=1) - lam * D - (mup * (r + F)).sum(axis=1) + (mum * (r - F)).sum(axis=1)
    y = p @ Hg.T                                # H_g p*  [B][n_l]
    return PtdfEval(value, p.sum(axis=1) - D, y - r - F, r - y - F, p)


def _constants(net, Ha, load):
    """The parts of the dual function that do not depend on the multipliers."""
    return Ha[:, net.gen_bus], load.sum(axis=1), load @ Ha.T


def _valid(g):
    return np.isfinite(g) & (np.abs(g) <= 1e15)


def _opt_step(o, y, g, a, s1, s2, b1t, b2t):
    """One coordinate-wise step of the chosen variant (readings A-25, A-26;
    the same formulas as oracle/dcopf_oracle.c opt_step).  Updates s1/s2 in
    place where the variant has state."""
    v = o["variant"]
    if v == OPT_GDM:
        s1[...] = o["rho"] * s1 + a * g
        y = y + s1
        return y + a * g
    if v == OPT_GDM_CLASSIC:
        s1[...] = o["rho"] * s1 + a * g
        return y + s1
    if v == OPT_ADAGRAD:
        s1[...] = s1 + g * g
        return y + (a * g) / (np.sqrt(s1) + o["eps"])
    if v == OPT_ADAM:
        s1[...] = o["beta1"] * s1 + (1.0 - o["beta1"]) * g
        s2[...] = o["beta2"] * s2 + (1.0 - o["beta2"]) * (g * g)
        mh = s1 / (1.0 - b1t)
        vh = s2 / (1.0 - b2t)
        return y + (a * mh) / (np.sqrt(vh) + o["eps"])
    return y + a * g


@dataclass
class PtdfResult:
    lam: np.ndarray       # [B]
    mu: np.ndarray        # [B][2 n_l]: mu+ then mu-
    bound: np.ndarray     # [B] g at the last evaluation
    best: np.ndarray      # [B] running max of valid g
    status: np.ndarray    # [B]
    hist: Optional[np.ndarray]  # [B][K+1]


def solve(net, load, K, alpha, Ha=None, lam0=None, mu0=None, opt=None, tol=0.0,
          history=False) -> PtdfResult:
    """K projected ascent steps from y_0 = 0 (or the warm start), then one more
    evaluation: k = 0..K, best = running max of valid g, Jacobi steps (every
    coordinate's step reads y_k).  Per instance: a non-finite or |g| > 1e15
    value marks it DIVERGED (A-23), |g_k - g_{k-1}| < tol for k >= 1 marks it
    CONVERGED (A-29); in both cases that iteration's step is still taken and
    every later one skipped."""
    if Ha is None:
        Ha = ptdf(net)
    load = np.atleast_2d(np.asarray(load, dtype=np.float64))
    B, nl = load.shape[0], net.n_branch
    alpha = np.asarray(alpha, dtype=np.float64)
    assert alpha.shape[0] >= K
    o = dict(variant=OPT_PLAIN, rho=0.0, beta1=0.0, beta2=0.0, eps=0.0)
    o.update(opt or {})
    if o["variant"] in (OPT_ADAGRAD, OPT_ADAM) and not o["eps"] > 0.0:
        raise ValueError("AdaGrad / Adam need eps > 0 (SPEC.md:359: 1e-8): the state starts at 0")
    lam = np.zeros(B) if lam0 is None else np.array(lam0, dtype=np.float64).reshape(B)
    mu = np.zeros((B, 2 * nl)) if mu0 is None else np.array(mu0, dtype=np.float64).reshape(B, 2 * nl)
    sl1, sl2 = np.zeros(B), np.zeros(B)               # optimiser state (lambda)
    sm1, sm2 = np.zeros((B, 2 * nl)), np.zeros((B, 2 * nl))
    b1t = b2t = 1.0
    best = np.full(B, -np.inf)
    status = np.zeros(B, dtype=np.int32)
    frozen = np.zeros(B, dtype=bool)
    gprev = np.zeros(B)
    hist = np.zeros((B, K + 1)) if history else None
    bound = np.zeros(B)
    pre = _constants(net, Ha, load)
    for k in range(K + 1):
        ev = evaluate(net, Ha, load, lam, mu[:, :nl], mu[:, nl:], _pre=pre)
        g = ev.value
        if hist is not None:
            hist[:, k] = g
        was_frozen = frozen.copy()
        ok = _valid(g)
        live = ~was_frozen
        upd = live & ok & (g > best)
        best[upd] = g[upd]
        if tol > 0.0 and k > 0:
            conv = live & ok & (np.abs(g - gprev) < tol)
            status[conv] = CONVERGED
            frozen |= conv
        div = live & ~ok
        status[div] = DIVERGED
        frozen |= div
        gprev = g
        if k == K:
            bound = g
            break
        a = alpha[k]
        if o["variant"] == OPT_ADAM:
            b1t = b1t * o["beta1"]
            b2t = b2t * o["beta2"]
        step = ~was_frozen
        t1, t2 = sl1.copy(), sl2.copy()
        nlam = _opt_step(o, lam, ev.g_lam, a, t1, t2, b1t, b2t)
        gmu = np.concatenate([ev.g_mup, ev.g_mum], axis=1)
        s1, s2 = sm1.copy(), sm2.copy()
        v = _opt_step(o, mu, gmu, a, s1, s2, b1t, b2t)
        nmu = np.where(v > 0.0, v, 0.0)                 # mu <- max(mu, 0)
        # frozen instances keep multipliers and state
        lam = np.where(step, nlam, lam)
        sl1 = np.where(step, t1, sl1)
        sl2 = np.where(step, t2, sl2)
        mu = np.where(step[:, None], nmu, mu)
        sm1 = np.where(step[:, None], s1, sm1)
        sm2 = np.where(step[:, None], s2, sm2)
    return PtdfResult(lam, mu, bound, best, status, hist)
