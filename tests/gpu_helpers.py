"""Shared helpers for the -m gpu parity tests: run the CUDA path through the
C-ABI binding with torch device buffers, run the oracle on the same seeded
inputs, and compare at the north_star tolerances."""
import numpy as np

import oracle
from paper_2406_13191_b200 import dual
from paper_2406_13191_b200 import instances as inst

BOUND_RTOL = 1e-9   # north_star: relative 1e-9 on the dual bound (scale: reading A-17)
MULT_TOL = 1e-8     # north_star: 1e-8 max-abs, normalised (reading A-18)


def cost_scale(net):
    """S = sum_g c_g pmax_g (+ a_g pmax_g^2): the bound's scale when g ~ 0 (A-17)."""
    s = float(np.sum(np.abs(net.gen_c) * np.abs(net.gen_pmax)))
    if net.gen_a is not None:
        s += float(np.sum(net.gen_a * net.gen_pmax ** 2))
    return max(s, 1.0)


def run_gpu(net, loads, outages=None, K=0, alpha=None, form=0, path=dual.PATH_AUTO, history=False,
            lam0=None, br0=None, implied_theta=False, switchable=None, opt=None, split=None, tol=0.0,
            tile_parts=0, lane_instances=0):
    """loads [B][n_bus] (instance-major, like the oracle); returns instance-major results.
    tile_parts / lane_instances: dcopf_options (batched path: CTAs per tile and
    instances per lane; cluster path: CTAs per cluster); 0 = the library's choice."""
    import torch
    dev = torch.device("cuda:0")
    loads = np.atleast_2d(loads)
    B = loads.shape[0]
    h = dual.DcopfDual(net, form=form, path=path, implied_theta=implied_theta, switchable=switchable,
                       tile_parts=tile_parts, lane_instances=lane_instances)
    if tol:
        h.set_stop(tol)
    if opt is not None:  # oracle-style dict(variant=, rho=, beta1=, beta2=, eps=)
        h.set_optimizer(opt.get("variant", 0), opt.get("rho", 0.0), opt.get("beta1", 0.0), opt.get("beta2", 0.0),
                        opt.get("eps", 0.0))
    ld = torch.from_numpy(np.ascontiguousarray(loads.T)).to(dev)
    out = None if outages is None else torch.from_numpy(np.ascontiguousarray(outages, dtype=np.int32)).to(dev)
    h.set_instance_batch(ld, out)
    nbr = h.n_branch_mult
    if lam0 is not None:
        h.set_multipliers(torch.from_numpy(np.ascontiguousarray(np.atleast_2d(lam0).T)).to(dev),
                          torch.from_numpy(np.ascontiguousarray(np.atleast_2d(br0).T)).to(dev))
    hist = torch.empty((K, B), dtype=torch.float64, device=dev) if history else None
    a = alpha if alpha is not None else np.zeros(0)
    if split:  # K steps as two iterate() calls (state and counters must carry over)
        h.iterate(split, a[:split], None if hist is None else hist[:split])
        h.iterate(K - split, a[split:], None if hist is None else hist[split:])
    else:
        h.iterate(K, a, hist)
    bound = torch.empty(B, dtype=torch.float64, device=dev)
    best = torch.empty(B, dtype=torch.float64, device=dev)
    status = torch.empty(B, dtype=torch.int32, device=dev)
    lam = torch.empty((h.n_lambda, B), dtype=torch.float64, device=dev)
    br = torch.empty((nbr, B), dtype=torch.float64, device=dev)
    h.get_bound(bound, best, status)
    h.get_multipliers(lam, br)
    torch.cuda.synchronize()
    res = dict(bound=bound.cpu().numpy(), best=best.cpu().numpy(), status=status.cpu().numpy(),
               lam=lam.cpu().numpy().T.copy(), br=br.cpu().numpy().T.copy(),
               hist=None if hist is None else hist.cpu().numpy().T.copy(), info=h.info())
    h.close()
    return res


def non_tree_switchable(net):
    """config 4: only non-tree branches are ever taken out"""
    sw = np.zeros(net.n_branch, np.uint8)
    sw[net.n_tree:] = 1
    return sw


def assert_parity(net, gpu, orc, idx=None, check_hist=True, bitwise_multipliers=False):
    """Compare a GPU result with an oracle result (optionally on instance subset
    idx): every multiplier coordinate, the bound, best, status and history."""
    sel = slice(None) if idx is None else idx
    S = cost_scale(net)
    ob, obest = orc.bound, orc.best
    gb, gbest = gpu["bound"][sel], gpu["best"][sel]
    scale = np.maximum(np.abs(ob), S)
    assert np.all(np.abs(gb - ob) <= BOUND_RTOL * scale), (gb, ob)
    fin = np.isfinite(obest)
    assert np.array_equal(np.isfinite(gbest), fin)
    assert np.all(np.abs(gbest[fin] - obest[fin]) <= BOUND_RTOL * np.maximum(np.abs(obest[fin]), S))
    np.testing.assert_array_equal(gpu["status"][sel], orc.status)
    gbr, obr = gpu["br"][sel], orc.br
    y_g = np.concatenate([gpu["lam"][sel], gbr], axis=1)
    y_o = np.concatenate([orc.lam, obr], axis=1)
    err = np.max(np.abs(y_g - y_o), axis=1) / np.maximum(1.0, np.max(np.abs(y_o), axis=1))
    assert np.all(err <= MULT_TOL), err.max()
    if bitwise_multipliers:
        np.testing.assert_array_equal(y_g, y_o)
    if check_hist and gpu["hist"] is not None and orc.hist is not None:
        K = gpu["hist"].shape[1]
        oh = orc.hist[:, :K]
        assert np.all(np.abs(gpu["hist"][sel] - oh) <= BOUND_RTOL * np.maximum(np.abs(oh), S))
    return float(err.max())
