"""Batch compaction (dcopf_dual_compact): after some
instances freeze (stopping rule, reading A-29), dropping them and iterating
the packed batch must give the kept instances bitwise the results of an
uncompacted run -- multipliers, optimiser state, best, status and first hit."""
import numpy as np
import pytest

from paper_2406_13191_b200 import dual
from paper_2406_13191_b200 import instances as inst

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dual.load_library()


def _run(net, loads, form, path, K1, K2, alpha, tol, opt, compact, target):
    h = dual.DcopfDual(net, form=form, path=path)
    if opt:
        h.set_optimizer(dual.OPT_ADAM, beta1=0.9, beta2=0.999, epsilon=1e-8)
    h.set_stop(tol)
    h.set_instance_batch(np.ascontiguousarray(loads.T))
    h.set_target(target)
    h.iterate(K1, alpha[:K1])
    kept = np.arange(loads.shape[0])
    if compact:
        kept = h.compact()
        assert h.info().B == len(kept)
    h.iterate(K2, alpha[K1:K1 + K2])
    bound, best, status, lam, br = h.results_numpy()
    hit = h.get_first_hit()
    h.close()
    return kept, dict(bound=bound, best=best, status=status, lam=lam, br=br, hit=hit)


@pytest.mark.parametrize("form,path,opt", [(dual.FORM_F2, dual.PATH_BATCHED, False),
                                           (dual.FORM_F2, dual.PATH_BATCHED, True),
                                           (dual.FORM_KVL, dual.PATH_BATCHED, False),
                                           (dual.FORM_F1, dual.PATH_CLUSTER, False),
                                           (dual.FORM_F2, dual.PATH_SINGLE, False)])
def test_compaction_matches_uncompacted_run(form, path, opt):
    net = inst.make_network(0)
    B = 300 if path == dual.PATH_BATCHED else 40
    rng = np.random.default_rng(5)
    loads = net.base_load[None, :] * rng.uniform(0.7, 1.3, (B, 1))
    K1, K2 = 400, 300
    alpha = inst.alpha_schedule(K1 + K2, 0.05 if opt else 1e-3)
    # a tolerance that freezes part of the batch during the first call
    probe = dual.DcopfDual(net, form=form, path=path)
    if opt:
        probe.set_optimizer(dual.OPT_ADAM, beta1=0.9, beta2=0.999, epsilon=1e-8)
    probe.set_instance_batch(np.ascontiguousarray(loads.T))
    hist = np.empty((K1, B))
    probe.iterate(K1, alpha[:K1], hist)
    probe.close()
    d = np.abs(np.diff(hist, axis=0)).min(axis=0)
    tol = float(np.quantile(d, 0.4))
    target = hist[-1] - 1e-6 * np.abs(hist[-1])        # some instances reach it only after compaction
    _, ref = _run(net, loads, form, path, K1, K2, alpha, tol, opt, False, target)
    kept, got = _run(net, loads, form, path, K1, K2, alpha, tol, opt, True, target)
    assert 0 < len(kept) < B
    for k in ("bound", "best", "status", "hit"):
        np.testing.assert_array_equal(got[k], ref[k][kept], err_msg=k)
    np.testing.assert_array_equal(got["lam"], ref["lam"][:, kept])
    np.testing.assert_array_equal(got["br"], ref["br"][:, kept])


def test_compaction_no_op_cases():
    net = inst.make_network(0)
    loads = np.tile(net.base_load, (10, 1))
    h = dual.DcopfDual(net, path=dual.PATH_BATCHED)
    h.set_instance_batch(np.ascontiguousarray(loads.T))
    h.iterate(5, inst.alpha_schedule(5))
    kept = h.compact()           # nothing frozen: unchanged
    np.testing.assert_array_equal(kept, np.arange(10))
    assert h.info().B == 10
    h.set_stop(1e300)            # everything converges at the second evaluation
    h.iterate(5, inst.alpha_schedule(5))
    kept = h.compact()           # nothing left: the batch stays, n_kept = 0
    assert len(kept) == 0 and h.info().B == 10
    h.close()


@pytest.mark.parametrize("form", [dual.FORM_F2, dual.FORM_KVL])
def test_compaction_retiles_split_batch(form):
    """A branch-and-bound-style shrink on the 10k-bus network: 2048 instances
    (4 per lane, 8 parts per tile) compacted to about half are re-tiled (the
    library picks 16 parts per tile for the smaller batch), so the kept
    instances still fill the SMs.  Multipliers, status and first hits stay
    bitwise those of the uncompacted run; the dual value is a fixed-order sum
    per tiling, so across the re-tiling bound / best agree to rounding order."""
    net = inst.make_network(4)
    sw = np.zeros(net.n_branch, np.uint8)
    sw[net.n_tree:] = 1
    B = 2048
    batch = inst.config4_batch(net, range(B), variant="4b")
    K1, K2 = 40, 30
    alpha = inst.alpha_schedule(K1 + K2, 1e-2)
    probe = dual.DcopfDual(net, form=form, path=dual.PATH_BATCHED, switchable=sw)
    probe.set_instance_batch(np.ascontiguousarray(batch.load.T))
    hist = np.empty((K1, B))
    probe.iterate(K1, alpha[:K1], hist)
    info0 = probe.info()
    probe.close()
    d = np.abs(np.diff(hist, axis=0)).min(axis=0)
    tol = float(np.quantile(d, 0.5))

    def run(compact):
        h = dual.DcopfDual(net, form=form, path=dual.PATH_BATCHED, switchable=sw)
        h.set_stop(tol)
        h.set_instance_batch(np.ascontiguousarray(batch.load.T))
        h.iterate(K1, alpha[:K1])
        kept = np.arange(B)
        info = h.info()
        if compact:
            kept = h.compact()
            info = h.info()
        h.iterate(K2, alpha[K1:])
        bound, best, status, lam, br = h.results_numpy()
        hit = h.get_first_hit()
        h.close()
        return kept, info, dict(bound=bound, best=best, status=status, lam=lam, br=br, hit=hit)

    _, _, ref = run(False)
    kept, info, got = run(True)
    assert 0 < len(kept) < B
    # re-tiled as a fresh batch of the kept size would be, filling the SMs again
    fresh = dual.DcopfDual(net, form=form, path=dual.PATH_BATCHED, switchable=sw)
    fresh.set_instance_batch(np.ascontiguousarray(batch.load[kept].T))
    fi = fresh.info()
    fresh.close()
    assert (info.lane_instances, info.tile_parts, info.tile_width, info.grid) == (
        fi.lane_instances, fi.tile_parts, fi.tile_width, fi.grid)
    assert (info.tile_width, info.grid) != (info0.tile_width, info0.grid)
    assert info.grid > 148 // 2, "the compacted batch should still fill most SMs"
    for k in ("status", "hit"):
        np.testing.assert_array_equal(got[k], ref[k][kept], err_msg=k)
    np.testing.assert_array_equal(got["lam"], ref["lam"][:, kept])
    np.testing.assert_array_equal(got["br"], ref["br"][:, kept])
    for k in ("bound", "best"):
        np.testing.assert_allclose(got[k], ref[k][kept], rtol=1e-12, atol=1e-9, err_msg=k)
