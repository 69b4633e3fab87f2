"""ctypes wrapper of the fp64 CPU oracle (oracle/dcopf_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs are the only callers.  The product path
(paper_2406_13191_b200) never imports this package.

Arrays here are instance-major ([B][n_bus]) in the caller's original
numbering; the oracle has no reordering, tiling or batching of its own.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dcopf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# gradient-based-optimisation variants (Algorithm 1)
OPT_PLAIN, OPT_GDM, OPT_GDM_CLASSIC, OPT_ADAGRAD, OPT_ADAM = 0, 1, 2, 3, 4

FORM_F2 = 0  # flow box (lambda, nu)
FORM_F1 = 1  # limit rows (lambda, mu+, mu-)
FORM_KVL = 2  # cycle basis (lambda, kappa), no angles
DIVERGED = 1
CONVERGED = 2  # the stopping rule |g_k - g_{k-1}| < tol fired (Alg. 1)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: -O2, no fast-math, no FMA contraction
    (reading A-19), OpenMP across instances only."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
               "-fopenmp", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int
        L = ctypes.c_long
        net = [I, I, I, I, P, P, P, P, P, P, P, P, P, P]
        lib.oracle_solve.argtypes = net + [I, L, P, P, I, L, P, P, P, P, P, P, P, I, I]
        lib.oracle_solve.restype = I
        D = ctypes.c_double
        lib.oracle_solve_opt.argtypes = net + [I, L, P, P, I, L, P, P, P, P, P, P, P, I, I, I, D, D, D, D, P, D]
        lib.oracle_evaluate_kvl.argtypes = net + [P, L, P, P, I, P, P, P, P, P, P, P]
        lib.oracle_evaluate_kvl.restype = I
        lib.oracle_cycles.argtypes = net + [P, P, P, P, P, P, L]
        lib.oracle_cycles.restype = I
        lib.oracle_solve_opt.restype = I
        lib.oracle_evaluate.argtypes = net + [I, L, P, P, I, P, P, P, P, P]
        lib.oracle_evaluate.restype = I
        lib.oracle_minimiser.argtypes = net + [I, L, P, P, I, P, P, P, P, P]
        lib.oracle_minimiser.restype = I
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _net_args(net, keep):
    f = lambda x, dt: keep.append(np.ascontiguousarray(x, dtype=dt)) or keep[-1]
    a = None if net.gen_a is None else f(net.gen_a, np.float64)
    return [net.n_bus, net.n_branch, net.n_gen, net.ref_bus,
            _p(f(net.br_from, np.int32)), _p(f(net.br_to, np.int32)),
            _p(f(net.br_b, np.float64)), _p(f(net.br_fmax, np.float64)),
            _p(f(net.theta_max, np.float64)), _p(f(net.gen_bus, np.int32)),
            _p(f(net.gen_pmin, np.float64)), _p(f(net.gen_pmax, np.float64)),
            _p(f(net.gen_c, np.float64)), _p(a)]


def n_branch_mult(net, form):
    if form == FORM_KVL:
        return net.n_branch - net.n_bus + 1
    return net.n_branch * (2 if form == FORM_F1 else 1)


def _sw(switchable):
    return None if switchable is None else np.ascontiguousarray(switchable, dtype=np.uint8)


@dataclass
class OracleResult:
    lam: np.ndarray      # [B][n_bus]
    br: np.ndarray       # [B][nbr]
    bound: np.ndarray    # [B]
    best: np.ndarray     # [B]
    status: np.ndarray   # [B]
    hist: Optional[np.ndarray]  # [B][K+1]


def solve(net, load, outages=None, K=0, alpha=None, form=FORM_F2, lam0=None, br0=None,
          history=False, threads=1, opt=None, switchable=None, tol=0.0) -> OracleResult:
    """K projected ascent steps from y_0 = 0 (or the given warm start).
    opt: None (plain step) or dict(variant=OPT_*, rho=, beta1=, beta2=, eps=)."""
    lib = _load()
    load = np.ascontiguousarray(np.atleast_2d(load), dtype=np.float64)
    B = load.shape[0]
    nbr = n_branch_mult(net, form)
    alpha = np.ascontiguousarray(alpha if alpha is not None else np.zeros(0), dtype=np.float64)
    assert alpha.shape[0] >= K
    warm = lam0 is not None
    lam = np.zeros((B, net.n_bus)) if lam0 is None else np.array(lam0, dtype=np.float64, order="C").reshape(B, net.n_bus)
    br = np.zeros((B, nbr)) if br0 is None else np.array(br0, dtype=np.float64, order="C").reshape(B, nbr)
    outs = None
    max_out = 0
    if outages is not None:
        outs = np.ascontiguousarray(np.atleast_2d(outages), dtype=np.int32)
        max_out = outs.shape[1]
    bound = np.zeros(B)
    best = np.zeros(B)
    status = np.zeros(B, dtype=np.int32)
    hist = np.zeros((B, K + 1)) if history else None
    keep = []
    o = dict(variant=OPT_PLAIN, rho=0.0, beta1=0.0, beta2=0.0, eps=0.0)
    o.update(opt or {})
    rc = lib.oracle_solve_opt(*_net_args(net, keep), form, B, _p(load), _p(outs), max_out, K, _p(alpha),
                              _p(lam), _p(br), _p(bound), _p(best), _p(status), _p(hist), int(warm),
                              int(threads), int(o["variant"]), float(o["rho"]), float(o["beta1"]),
                              float(o["beta2"]), float(o["eps"]), _p(_sw(switchable)), float(tol))
    if rc != 0:
        raise ValueError("oracle_solve rejected its arguments")
    return OracleResult(lam, br, bound, best, status, hist)


def evaluate(net, load, lam, br, outages=None, form=FORM_F2):
    """(value[B], grad_lam[B][n_bus], grad_br[B][nbr]) at the given multipliers."""
    lib = _load()
    load = np.ascontiguousarray(np.atleast_2d(load), dtype=np.float64)
    B = load.shape[0]
    nbr = n_branch_mult(net, form)
    lam = np.ascontiguousarray(np.reshape(lam, (B, net.n_bus)), dtype=np.float64)
    br = np.ascontiguousarray(np.reshape(br, (B, nbr)), dtype=np.float64)
    outs = None
    max_out = 0
    if outages is not None:
        outs = np.ascontiguousarray(np.atleast_2d(outages), dtype=np.int32)
        max_out = outs.shape[1]
    val = np.zeros(B)
    gl = np.zeros((B, net.n_bus))
    gb = np.zeros((B, nbr))
    keep = []
    rc = lib.oracle_evaluate(*_net_args(net, keep), form, B, _p(load), _p(outs), max_out, _p(lam),
                             _p(br), _p(val), _p(gl), _p(gb))
    if rc != 0:
        raise ValueError("oracle_evaluate rejected its arguments")
    return val, gl, gb


def minimiser(net, load, lam, br, outages=None, form=FORM_F2):
    """Inner minimiser (p*[B][n_gen], flow[B][n_branch], theta*[B][n_bus])."""
    lib = _load()
    load = np.ascontiguousarray(np.atleast_2d(load), dtype=np.float64)
    B = load.shape[0]
    nbr = n_branch_mult(net, form)
    lam = np.ascontiguousarray(np.reshape(lam, (B, net.n_bus)), dtype=np.float64)
    br = np.ascontiguousarray(np.reshape(br, (B, nbr)), dtype=np.float64)
    outs = None
    max_out = 0
    if outages is not None:
        outs = np.ascontiguousarray(np.atleast_2d(outages), dtype=np.int32)
        max_out = outs.shape[1]
    p = np.zeros((B, net.n_gen))
    fl = np.zeros((B, net.n_branch))
    th = np.zeros((B, net.n_bus))
    keep = []
    rc = lib.oracle_minimiser(*_net_args(net, keep), form, B, _p(load), _p(outs), max_out, _p(lam),
                              _p(br), _p(p), _p(fl), _p(th))
    if rc != 0:
        raise ValueError("oracle_minimiser rejected its arguments")
    return p, fl, th


def evaluate_kvl(net, load, lam, kap, outages=None, switchable=None):
    """KVL form at given multipliers: (value[B], grad_lam[B][n_bus], grad_kap[B][nc], p[B][n_gen], f[B][n_l])."""
    lib = _load()
    load = np.ascontiguousarray(np.atleast_2d(load), dtype=np.float64)
    B = load.shape[0]
    nc = n_branch_mult(net, FORM_KVL)
    lam = np.ascontiguousarray(np.atleast_2d(lam), dtype=np.float64)
    kap = np.ascontiguousarray(np.atleast_2d(kap), dtype=np.float64).reshape(B, nc)
    outs, max_out = None, 0
    if outages is not None:
        outs = np.ascontiguousarray(np.atleast_2d(outages), dtype=np.int32)
        max_out = outs.shape[1]
    val, gl, gk = np.zeros(B), np.zeros((B, net.n_bus)), np.zeros((B, nc))
    p, f = np.zeros((B, net.n_gen)), np.zeros((B, net.n_branch))
    keep = []
    rc = lib.oracle_evaluate_kvl(*_net_args(net, keep), _p(_sw(switchable)), B, _p(load), _p(outs), max_out,
                                 _p(lam), _p(kap), _p(val), _p(gl), _p(gk), _p(p), _p(f))
    if rc != 0:
        raise ValueError("oracle_evaluate_kvl rejected its arguments")
    return val, gl, gk, p, f


def cycles(net, switchable=None):
    """The fundamental cycle basis (reading A-28): (def[nc], list of (branch ids, signs) per cycle)."""
    lib = _load()
    keep = []
    nc = ctypes.c_int(0)
    sw = _sw(switchable)
    tot = lib.oracle_cycles(*_net_args(net, keep), _p(sw), ctypes.byref(nc), None, None, None, None, 0)
    if tot < 0:
        raise ValueError("network disconnected over never-switched branches")
    d = np.zeros(nc.value, np.int32)
    cp = np.zeros(nc.value + 1, np.int32)
    cb = np.zeros(max(tot, 1), np.int32)
    cs = np.zeros(max(tot, 1), np.int32)
    lib.oracle_cycles(*_net_args(net, keep), _p(sw), ctypes.byref(nc), _p(d), _p(cp), _p(cb), _p(cs), tot)
    return d, [(cb[cp[k]:cp[k + 1]], cs[cp[k]:cp[k + 1]]) for k in range(nc.value)]
