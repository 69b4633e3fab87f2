"""Seeded synthetic DCOPF instances for BASELINE.json configs 0-4 (and variant 4b).

This module is the ONE place shared by the CUDA path's tests/bench and by the
oracle's tests: it draws inputs and holds none of the dual method's arithmetic
(no multipliers, no inner minimiser, no gradient).  Everything it produces is
plain problem data in the caller-visible *original* numbering:

    network : n_bus, n_branch, n_gen, ref_bus, br_from, br_to, br_b, br_fmax,
              theta_max, gen_bus, gen_pmin, gen_pmax, gen_c, gen_a (or None)
    batch   : load[B][n_bus]  (instance-major here; the C-ABI takes [n_bus][B])
              outages[B][max_out] int32 branch ids, -1 padded (or None)

Draw order is pinned so a rerun,
the oracle and the GPU see bit-identical data:

  * config 0 (14/19/5): tree j=rng.integers(0,i); extra edges u,v uniform;
    b~U[5,20], F~U[0.5,2], gen_bus=choice(n,5), pmax~U[.5,3], c~U[10,50],
    d~U[0,.6] rescaled to 0.6*sum(pmax); Theta = pi/3 (BASELINE.json configs[0]).
  * configs 1-3: tree as above; extra edges by a 2-or-3-step random walk on the
    current adjacency (reading A-12 of the "biased to graph distance <= 3" text);
    b~U[5,20]; gen_bus; load mask Bernoulli(0.7) (A-13), d~lognormal(-1,0.8);
    pmax~lognormal(0,1) rescaled to 1.4*sum(d); c~U[5,80]; a~U[0.001,0.05]
    drawn last (A-14); F = 1.3 |flows of the uniform-dispatch B-theta solution|
    (A-11); Theta = implied box dist_{F/b}(ref, i) (A-2).
  * config 4: config-3 network; instance j draws from
    default_rng(SeedSequence(seed).spawn(8192)[j]): per-bus factors
    U[0.85,1.15], k=integers(0,4) outages among non-tree branches (A-15/16);
    Theta from tree-only distances.  Variant 4b: one factor per instance, no
    outages (feasible by construction).

PAPER.md:94-102 (Eq. 1) is the problem these stand in for; PAPER.md:277 names
the IEEE 2000/4601/10000-bus cases (not available here) whose sizes configs
1-3 copy.
"""
from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

# (n_bus, n_branch, n_gen) for BASELINE.json configs 0..4
SHAPES = {
    0: (14, 19, 5),
    1: (2000, 3200, 540),
    2: (4601, 7200, 1000),
    3: (10000, 12700, 2500),
    4: (10000, 12700, 2500),
}
# K and step of BASELINE.json configs (alpha: reading A-9)
ITERS = {0: 2000, 1: 20000, 2: 20000, 3: 50000, 4: 5000}
ALPHA = 1e-3
CONFIG4_BATCH = 8192


@dataclass
class Network:
    n_bus: int
    n_branch: int
    n_gen: int
    ref_bus: int
    br_from: np.ndarray      # int32 [n_branch]
    br_to: np.ndarray        # int32 [n_branch]
    br_b: np.ndarray         # f64 [n_branch]
    br_fmax: np.ndarray      # f64 [n_branch]
    theta_max: np.ndarray    # f64 [n_bus]
    gen_bus: np.ndarray      # int32 [n_gen]
    gen_pmin: np.ndarray     # f64 [n_gen]
    gen_pmax: np.ndarray     # f64 [n_gen]
    gen_c: np.ndarray        # f64 [n_gen]
    gen_a: Optional[np.ndarray] = None   # f64 [n_gen] or None (linear cost)
    n_tree: int = 0          # branches [0, n_tree) form the spanning tree
    base_load: Optional[np.ndarray] = None  # f64 [n_bus]

    _a_draw: Optional[np.ndarray] = field(default=None, repr=False)


@dataclass
class Batch:
    load: np.ndarray                 # f64 [B][n_bus], instance-major
    outages: Optional[np.ndarray]    # int32 [B][max_out] or None
    instance_ids: np.ndarray         # int64 [B] global ids (for sharding)

    @property
    def B(self) -> int:
        return int(self.load.shape[0])

    @property
    def max_out(self) -> int:
        return 0 if self.outages is None else int(self.outages.shape[1])


# ----------------------------------------------------------------------------
# topology


def _tree(rng, n):
    frm, to = [], []
    adj = [[] for _ in range(n)]
    for i in range(1, n):
        j = int(rng.integers(0, i))
        frm.append(j)
        to.append(i)
        adj[j].append(i)
        adj[i].append(j)
    return frm, to, adj


def _extra_uniform(rng, n, n_l, frm, to, adj):
    seen = {(min(a, b), max(a, b)) for a, b in zip(frm, to)}
    while len(frm) < n_l:
        u = int(rng.integers(0, n))
        v = int(rng.integers(0, n))
        key = (min(u, v), max(u, v))
        if u == v or key in seen:
            continue
        seen.add(key)
        frm.append(u)
        to.append(v)
        adj[u].append(v)
        adj[v].append(u)


def _extra_walk(rng, n, n_l, frm, to, adj):
    """Reading A-12: u uniform, 2 or 3 uniform steps on the current adjacency."""
    seen = {(min(a, b), max(a, b)) for a, b in zip(frm, to)}
    while len(frm) < n_l:
        u = int(rng.integers(0, n))
        steps = int(rng.integers(2, 4))
        v = u
        for _ in range(steps):
            nb = adj[v]
            v = nb[int(rng.integers(0, len(nb)))]
        key = (min(u, v), max(u, v))
        if u == v or key in seen:
            continue
        seen.add(key)
        frm.append(u)
        to.append(v)
        adj[u].append(v)
        adj[v].append(u)


def dc_flows(n_bus, ref, br_from, br_to, br_b, injection):
    """B-theta power flow: solve L_rr theta_r = P_r (theta_ref = 0), return
    branch flows b_l (theta_s - theta_t).  Used only to derive flow limits
    (reading A-11), never on the dual path."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    n_l = len(br_from)
    rows = np.concatenate([np.arange(n_l), np.arange(n_l)])
    cols = np.concatenate([br_from, br_to])
    vals = np.concatenate([np.ones(n_l), -np.ones(n_l)])
    A = sp.csr_matrix((vals, (rows, cols)), shape=(n_l, n_bus))
    L = (A.T @ sp.diags(br_b) @ A).tocsc()
    keep = np.array([i for i in range(n_bus) if i != ref])
    theta = np.zeros(n_bus)
    theta[keep] = spla.spsolve(L[keep][:, keep], injection[keep])
    return br_b * (A @ theta)


def implied_theta_box(n_bus, ref, br_from, br_to, br_b, br_fmax, use=None):
    """Reading A-2: Theta_i = shortest-path distance from ref with branch
    weights F_l / b_l over the branches in `use` (default: all with b > 0).
    Valid because |theta_i| <= sum over any ref-i path of |dtheta_l| <= sum F_l/b_l.
    Zero weights are legal (F = 0), so this is a plain heap Dijkstra."""
    adj = [[] for _ in range(n_bus)]
    idx = range(len(br_from)) if use is None else use
    for l in idx:
        if br_b[l] <= 0:
            continue
        wgt = br_fmax[l] / br_b[l]
        s, t = int(br_from[l]), int(br_to[l])
        adj[s].append((t, wgt))
        adj[t].append((s, wgt))
    dist = np.full(n_bus, np.inf)
    dist[ref] = 0.0
    pq = [(0.0, ref)]
    while pq:
        dv, v = heapq.heappop(pq)
        if dv > dist[v]:
            continue
        for u, wgt in adj[v]:
            nd = dv + wgt
            if nd < dist[u]:
                dist[u] = nd
                heapq.heappush(pq, (nd, u))
    if not np.all(np.isfinite(dist)):
        raise ValueError("graph over the chosen branches is disconnected")
    return dist


# ----------------------------------------------------------------------------
# networks


def make_network(config: int, seed: int = 0, quadratic: Optional[bool] = None,
                 theta_mode: Optional[str] = None) -> Network:
    """Build the network of BASELINE.json configs[config] (0..4).

    quadratic: default True for config 2, False otherwise (config 3 has both).
    theta_mode: 'pi3' (literal |theta| <= pi/3), 'implied' (A-2), 'min'
                (min(pi/3, implied)).  Default: 'pi3' for config 0, 'implied'
                for 1-3, 'implied-tree' for 4.
    """
    n, n_l, n_g = SHAPES[config]
    rng = np.random.default_rng(seed)
    frm, to, adj = _tree(rng, n)
    n_tree = len(frm)
    if config == 0:
        _extra_uniform(rng, n, n_l, frm, to, adj)
    else:
        _extra_walk(rng, n, n_l, frm, to, adj)
    br_from = np.asarray(frm, dtype=np.int32)
    br_to = np.asarray(to, dtype=np.int32)
    a_draw = None
    if config == 0:
        br_b = rng.uniform(5, 20, n_l)
        br_fmax = rng.uniform(0.5, 2.0, n_l)
        gen_bus = rng.choice(n, n_g, replace=False).astype(np.int32)
        pmax = rng.uniform(0.5, 3.0, n_g)
        c = rng.uniform(10, 50, n_g)
        d = rng.uniform(0, 0.6, n)
        d = d * (0.6 * pmax.sum() / d.sum())
    else:
        br_b = rng.uniform(5, 20, n_l)
        gen_bus = rng.choice(n, n_g, replace=False).astype(np.int32)
        mask = rng.random(n) < 0.7
        d = np.where(mask, rng.lognormal(-1.0, 0.8, n), 0.0)
        pmax = rng.lognormal(0.0, 1.0, n_g)
        pmax = pmax * (1.4 * d.sum() / pmax.sum())
        c = rng.uniform(5, 80, n_g)
        a_draw = rng.uniform(0.001, 0.05, n_g)
        # A-11: uniform dispatch (equal fraction of capacity), B-theta flows
        pg = pmax * (d.sum() / pmax.sum())
        inj = -d.copy()
        np.add.at(inj, gen_bus, pg)
        f_u = dc_flows(n, 0, br_from, br_to, br_b, inj)
        # A-11: a structurally zero flow (a line into a part of the network with
        # no load and no generator) is a literal zero limit; the sparse solve
        # leaves rounding residues < 1e-12 there, against flows >= 3e-5 elsewhere
        f_u[np.abs(f_u) < 1e-9 * np.abs(f_u).max()] = 0.0
        br_fmax = 1.3 * np.abs(f_u)
    pmin = np.zeros(n_g)
    if theta_mode is None:
        theta_mode = "pi3" if config == 0 else ("implied-tree" if config == 4 else "implied")
    if theta_mode == "pi3":
        theta = np.full(n, math.pi / 3)
    elif theta_mode == "implied":
        theta = implied_theta_box(n, 0, br_from, br_to, br_b, br_fmax)
    elif theta_mode == "implied-tree":
        theta = implied_theta_box(n, 0, br_from, br_to, br_b, br_fmax, use=range(n_tree))
    elif theta_mode == "min":
        theta = np.minimum(math.pi / 3, implied_theta_box(n, 0, br_from, br_to, br_b, br_fmax))
    else:
        raise ValueError(theta_mode)
    theta[0] = 0.0  # ref bus: theta_0 == 0 (A-3); the value is never used
    if quadratic is None:
        quadratic = config == 2
    net = Network(n_bus=n, n_branch=n_l, n_gen=n_g, ref_bus=0, br_from=br_from, br_to=br_to,
                  br_b=br_b, br_fmax=br_fmax, theta_max=theta, gen_bus=gen_bus, gen_pmin=pmin,
                  gen_pmax=pmax, gen_c=c, gen_a=(a_draw if quadratic else None), n_tree=n_tree,
                  base_load=d)
    net._a_draw = a_draw
    return net


def single_batch(net: Network) -> Batch:
    return Batch(load=net.base_load[None, :].copy(), outages=None,
                 instance_ids=np.zeros(1, dtype=np.int64))


def config4_batch(net: Network, ids, seed: int = 0, variant: str = "4",
                  total: int = CONFIG4_BATCH) -> Batch:
    """Instances `ids` (global indices into the `total`-instance sweep) of
    config 4 (variant '4': per-bus factors + 0-3 non-tree outages; '4b': one
    factor per instance, no outages).  Drawing only a shard's ids gives the
    same data as drawing all and slicing (sharding invariance)."""
    ids = np.asarray(list(ids), dtype=np.int64)
    children = np.random.SeedSequence(seed).spawn(total)
    non_tree = np.arange(net.n_tree, net.n_branch, dtype=np.int32)
    load = np.empty((len(ids), net.n_bus))
    outs = np.full((len(ids), 3), -1, dtype=np.int32)
    for r, j in enumerate(ids):
        rj = np.random.default_rng(children[int(j)])
        if variant == "4":
            load[r] = net.base_load * rj.uniform(0.85, 1.15, net.n_bus)
            k = int(rj.integers(0, 4))
            if k:
                outs[r, :k] = rj.choice(non_tree, k, replace=False)
        elif variant == "4b":
            load[r] = net.base_load * rj.uniform(0.85, 1.15)
        else:
            raise ValueError(variant)
    return Batch(load=load, outages=(outs if variant == "4" else None), instance_ids=ids)


def alpha_schedule(K: int, alpha: float = ALPHA, decay: Optional[str] = None) -> np.ndarray:
    """Explicit step array (reading A-9): both sides consume identical values.
    decay (the paper's step decay; reading A-26): None = constant,
    "inv:T" = alpha / (1 + k/T), "step:F:N" = alpha * F^floor(k/N)."""
    k = np.arange(int(K), dtype=np.float64)
    if not decay:
        return np.full(int(K), float(alpha), dtype=np.float64)
    kind, *par = decay.split(":")
    if kind == "inv":
        return float(alpha) / (1.0 + k / float(par[0]))
    if kind == "step":
        return float(alpha) * float(par[0]) ** np.floor(k / float(par[1]))
    raise ValueError(f"unknown decay {decay!r}")


# ----------------------------------------------------------------------------
# the primal problem being bounded (test/bench side: weak-duality pins, gap)


def primal_lp(net: Network, load: np.ndarray, outages=None):
    """Exact optimum of the B-theta DCOPF (SURVEY §8 'Primal problem being
    bounded' = PAPER.md:94-101 Eq. 1 with the angle box), linear cost, via
    scipy HiGHS.  Variables [p (n_g), f (n_l), theta (n_b)].
    Returns (status, objective) with status 0 = optimal, 2 = infeasible."""
    import scipy.sparse as sp
    from scipy.optimize import linprog
    n, nl, ng = net.n_bus, net.n_branch, net.n_gen
    b = net.br_b.copy()
    F = net.br_fmax.copy()
    if outages is not None:
        for l in outages:
            if l >= 0:
                b[l] = 0.0
                F[l] = 0.0
    s, t = net.br_from, net.br_to
    li = np.arange(nl)
    # KCL: G p - A^T f = d
    G = sp.csr_matrix((np.ones(ng), (net.gen_bus, np.arange(ng))), shape=(n, ng))
    A = sp.csr_matrix((np.r_[np.ones(nl), -np.ones(nl)], (np.r_[li, li], np.r_[s, t])), shape=(nl, n))
    kcl = sp.hstack([G, -A.T, sp.csr_matrix((n, n))])
    # Kirchhoff: f - diag(b) A theta = 0
    kvl = sp.hstack([sp.csr_matrix((nl, ng)), sp.eye(nl), -sp.diags(b) @ A])
    Aeq = sp.vstack([kcl, kvl]).tocsc()
    beq = np.r_[load, np.zeros(nl)]
    th = net.theta_max.copy()
    bounds = ([(lo, hi) for lo, hi in zip(net.gen_pmin, net.gen_pmax)]
              + [(-x, x) for x in F]
              + [((0.0, 0.0) if i == net.ref_bus else (-th[i], th[i])) for i in range(n)])
    cost = np.r_[net.gen_c, np.zeros(nl + n)]
    res = linprog(cost, A_eq=Aeq, b_eq=beq, bounds=bounds, method="highs")
    return res.status, (res.fun if res.status == 0 else None)


def primal_qp(net: Network, load: np.ndarray, outages=None, tol=1e-10, max_rounds=60):
    """Quadratic-cost optimum by Kelley cutting planes on HiGHS (SURVEY P-2):
    epigraph t_g >= a_g p_g^2 replaced by tangent cuts; stop when the LP value
    (a lower bound) meets the true cost at the LP point (an upper bound).
    Returns (status, lower, upper)."""
    import scipy.sparse as sp
    from scipy.optimize import linprog
    assert net.gen_a is not None
    n, nl, ng = net.n_bus, net.n_branch, net.n_gen
    b = net.br_b.copy()
    F = net.br_fmax.copy()
    if outages is not None:
        for l in outages:
            if l >= 0:
                b[l] = 0.0
                F[l] = 0.0
    s, t = net.br_from, net.br_to
    li = np.arange(nl)
    G = sp.csr_matrix((np.ones(ng), (net.gen_bus, np.arange(ng))), shape=(n, ng))
    A = sp.csr_matrix((np.r_[np.ones(nl), -np.ones(nl)], (np.r_[li, li], np.r_[s, t])), shape=(nl, n))
    Z = lambda r, c: sp.csr_matrix((r, c))
    kcl = sp.hstack([G, -A.T, Z(n, n), Z(n, ng)])
    kvl = sp.hstack([Z(nl, ng), sp.eye(nl), -sp.diags(b) @ A, Z(nl, ng)])
    Aeq = sp.vstack([kcl, kvl]).tocsc()
    beq = np.r_[load, np.zeros(nl)]
    th = net.theta_max
    a = net.gen_a
    bounds = ([(lo, hi) for lo, hi in zip(net.gen_pmin, net.gen_pmax)]
              + [(-x, x) for x in F]
              + [((0.0, 0.0) if i == net.ref_bus else (-th[i], th[i])) for i in range(n)]
              + [(0.0, None)] * ng)
    cost = np.r_[net.gen_c, np.zeros(nl + n), np.ones(ng)]
    pts = [net.gen_pmin.copy(), net.gen_pmax.copy(), 0.5 * (net.gen_pmin + net.gen_pmax)]
    rows, rhs = [], []

    def add_cuts(ph):
        # t_g >= a (2 ph p - ph^2)  <=>  2 a ph p - t <= a ph^2
        for g in range(ng):
            rows.append((g, 2 * a[g] * ph[g]))
            rhs.append(a[g] * ph[g] ** 2)

    for ph in pts:
        add_cuts(ph)
    lower = upper = None
    for _ in range(max_rounds):
        m = len(rows)
        r_idx = np.arange(m)
        gcol = np.array([g for g, _ in rows])
        coef = np.array([cf for _, cf in rows])
        Aub = sp.csr_matrix((np.r_[coef, -np.ones(m)], (np.r_[r_idx, r_idx], np.r_[gcol, ng + nl + n + gcol])),
                            shape=(m, ng + nl + n + ng))
        res = linprog(cost, A_ub=Aub, b_ub=np.asarray(rhs), A_eq=Aeq, b_eq=beq, bounds=bounds, method="highs")
        if res.status != 0:
            return res.status, None, None
        p = res.x[:ng]
        lower = res.fun
        upper = float(net.gen_c @ p + a @ (p * p))
        if upper - lower <= tol * max(1.0, abs(upper)):
            break
        add_cuts(p)
    return 0, lower, upper


def tiny_network(n_bus: int, n_branch: int, n_gen: int, seed: int, quadratic: bool = False,
                 theta: float = math.pi / 3, load_frac: float = 0.6) -> Network:
    """Small random instance for brute-force / parity tests: config-0 recipe
    with arbitrary sizes (random tree + uniform extra edges, b~U[5,20],
    F~U[0.5,2], pmax~U[0.5,3], c~U[10,50], a~U[0.001,0.05] if quadratic,
    loads rescaled to load_frac*sum(pmax)).  n_gen may exceed n_bus (several
    generators per bus, reading A-22)."""
    rng = np.random.default_rng(seed)
    frm, to, adj = _tree(rng, n_bus)
    n_tree = len(frm)
    _extra_uniform(rng, n_bus, n_branch, frm, to, adj)
    br_b = rng.uniform(5, 20, n_branch)
    br_fmax = rng.uniform(0.5, 2.0, n_branch)
    if n_gen <= n_bus:
        gen_bus = rng.choice(n_bus, n_gen, replace=False).astype(np.int32)
    else:
        gen_bus = rng.integers(0, n_bus, n_gen).astype(np.int32)
    pmax = rng.uniform(0.5, 3.0, n_gen)
    c = rng.uniform(10, 50, n_gen)
    a = rng.uniform(0.001, 0.05, n_gen)
    d = rng.uniform(0, 0.6, n_bus)
    d = d * (load_frac * pmax.sum() / d.sum())
    th = np.full(n_bus, float(theta))
    th[0] = 0.0
    return Network(n_bus=n_bus, n_branch=n_branch, n_gen=n_gen, ref_bus=0,
                   br_from=np.asarray(frm, np.int32), br_to=np.asarray(to, np.int32), br_b=br_b,
                   br_fmax=br_fmax, theta_max=th, gen_bus=gen_bus, gen_pmin=np.zeros(n_gen),
                   gen_pmax=pmax, gen_c=c, gen_a=(a if quadratic else None), n_tree=n_tree,
                   base_load=d)


def random_multipliers(rng, net: Network, B: int, form: int, scale: float = 20.0):
    """Random dual points (lambda free, nu free; mu >= 0 for form 1)."""
    lam = rng.normal(0.0, scale, (B, net.n_bus))
    if form == 1:
        br = np.abs(rng.normal(0.0, scale, (B, 2 * net.n_branch)))
    else:
        br = rng.normal(0.0, scale, (B, net.n_branch))
    return lam, br
