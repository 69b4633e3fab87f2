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
