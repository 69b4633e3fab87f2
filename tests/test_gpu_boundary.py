"""Boundary contracts of the C ABI (include/dcopf_dual.h) that the round-1
advisor found broken, each pinned on the GPU:

* handles are independent: a second handle with a smaller shared-memory plan
  does not break launches of the first (the per-function dynamic shared-memory
  limit is set before every launch);
* a rejected set_instance_batch leaves the loaded batch as it was;
* an outage under an angle box implied over ALL branches is rejected (the box
  would not be a valid relaxation for that instance, reading A-2);
* AdaGrad / Adam with epsilon = 0 are rejected (0 / 0 at y0);
* set_optimizer on a loaded KVL cluster batch keeps the multipliers (the
  cycle storage order depends on the cluster size, cluster.cpp).
"""
import numpy as np
import pytest

import oracle
from paper_2406_13191_b200 import dual
from paper_2406_13191_b200 import instances as inst

from gpu_helpers import assert_parity, non_tree_switchable, run_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dual.load_library()


def _dev():
    import torch
    return torch.device("cuda:0")


def _to_dev(a, dtype=None):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a if dtype is None else a.astype(dtype))).to(_dev())


def _results(h, B):
    import torch
    bound = torch.empty(B, dtype=torch.float64, device=_dev())
    best = torch.empty(B, dtype=torch.float64, device=_dev())
    status = torch.empty(B, dtype=torch.int32, device=_dev())
    lam = torch.empty((h.n_lambda, B), dtype=torch.float64, device=_dev())
    br = torch.empty((h.n_branch_mult, B), dtype=torch.float64, device=_dev())
    h.get_bound(bound, best, status)
    h.get_multipliers(lam, br)
    torch.cuda.synchronize()
    return dict(bound=bound.cpu().numpy(), best=best.cpu().numpy(), status=status.cpu().numpy(),
                lam=lam.cpu().numpy().T.copy(), br=br.cpu().numpy().T.copy(), hist=None, info=h.info())


@pytest.mark.parametrize("path", [dual.PATH_BATCHED, dual.PATH_CLUSTER])
def test_handles_independent_shared_memory(path):
    """Handle A (config 1, larger plan) keeps working after handle B (config 0,
    smaller plan of the same kernel instantiation) is configured."""
    net_a = inst.make_network(1)
    net_b = inst.make_network(0)
    sw = non_tree_switchable(net_a)
    B = 64 if path == dual.PATH_BATCHED else 4
    batch = inst.config4_batch(net_a, range(B), total=B)
    K = 40
    a = inst.alpha_schedule(K)
    ha = dual.DcopfDual(net_a, path=path, switchable=sw)
    ha.set_instance_batch(_to_dev(batch.load.T), _to_dev(batch.outages))
    ha.iterate(K // 2, a[:K // 2])
    hb = dual.DcopfDual(net_b, path=path)
    hb.set_instance_batch(_to_dev(np.tile(net_b.base_load[:, None], (1, B))))
    hb.iterate(5, inst.alpha_schedule(5))
    ha.iterate(K - K // 2, a[K // 2:])  # failed with ECUDA before the fix
    gpu = _results(ha, B)
    hb.close()
    ha.close()
    orc = oracle.solve(net_a, batch.load, outages=batch.outages, K=K, alpha=a, switchable=sw, threads=8)
    assert_parity(net_a, gpu, orc, check_hist=False, bitwise_multipliers=True)


def test_rejected_batch_leaves_loaded_batch():
    """A set_instance_batch rejected for a bad outage id (with a batch size that
    would need another schedule) changes nothing: the loaded batch continues
    bitwise as if the call had not been made."""
    net = inst.make_network(1)
    sw = non_tree_switchable(net)
    B = 64
    batch = inst.config4_batch(net, range(B), total=B)
    K = 40
    a = inst.alpha_schedule(K)
    h = dual.DcopfDual(net, path=dual.PATH_BATCHED, switchable=sw)
    h.set_instance_batch(_to_dev(batch.load.T), _to_dev(batch.outages))
    h.iterate(K // 2, a[:K // 2])
    B2 = 200
    bad = np.full((B2, 1), -1, np.int32)
    bad[7, 0] = net.n_branch  # out of range
    with pytest.raises(dual.DcopfError, match="EINVAL"):
        h.set_instance_batch(_to_dev(np.tile(net.base_load[:, None], (1, B2))), _to_dev(bad))
    tree = np.full((B2, 1), -1, np.int32)
    tree[3, 0] = 0  # a never-switchable branch
    with pytest.raises(dual.DcopfError, match="EINVAL"):
        h.set_instance_batch(_to_dev(np.tile(net.base_load[:, None], (1, B2))), _to_dev(tree))
    h.iterate(K - K // 2, a[K // 2:])
    gpu = _results(h, B)
    h.close()
    orc = oracle.solve(net, batch.load, outages=batch.outages, K=K, alpha=a, switchable=sw, threads=8)
    assert_parity(net, gpu, orc, check_hist=False, bitwise_multipliers=True)


@pytest.mark.parametrize("form", [oracle.FORM_F2, oracle.FORM_F1])
def test_outage_under_all_branch_implied_box_rejected(form):
    """theta_max and br_switchable NULL: the implied box is a shortest path over
    every branch, so no outage may be accepted; with the switchable set
    declared (box over never-switched branches, reading A-2) it is."""
    net = inst.make_network(0)
    outs = np.array([[net.n_branch - 1]], np.int32)
    ld = _to_dev(net.base_load[:, None])
    h = dual.DcopfDual(net, form=form, path=dual.PATH_BATCHED, implied_theta=True)
    with pytest.raises(dual.DcopfError, match="EINVAL"):
        h.set_instance_batch(ld, _to_dev(outs))
    h.set_instance_batch(ld)  # no outage: fine
    h.close()
    sw = np.zeros(net.n_branch, np.uint8)
    sw[net.n_branch - 1] = 1
    h = dual.DcopfDual(net, form=form, path=dual.PATH_BATCHED, implied_theta=True, switchable=sw)
    h.set_instance_batch(ld, _to_dev(outs))
    h.close()


@pytest.mark.parametrize("variant", [dual.OPT_ADAGRAD, dual.OPT_ADAM])
def test_adaptive_step_needs_positive_epsilon(variant):
    net = inst.make_network(0)
    h = dual.DcopfDual(net, path=dual.PATH_BATCHED)
    with pytest.raises(dual.DcopfError, match="EINVAL"):
        h.set_optimizer(variant, 0.0, 0.9, 0.999, 0.0)
    h.set_optimizer(variant, 0.0, 0.9, 0.999, 1e-8)
    h.close()


def test_kvl_cluster_set_optimizer_keeps_multipliers():
    """Switching a loaded KVL cluster batch to Adam rebuilds the shared-memory
    plan at the batch's cluster size: kappa read back unchanged."""
    net = inst.make_network(1)
    sw = non_tree_switchable(net)
    B = 3
    batch = inst.config4_batch(net, range(B), total=B)
    h = dual.DcopfDual(net, form=dual.FORM_KVL, path=dual.PATH_CLUSTER, switchable=sw)
    h.set_instance_batch(_to_dev(batch.load.T), _to_dev(batch.outages))
    h.iterate(30, inst.alpha_schedule(30))
    before = _results(h, B)
    h.set_optimizer(dual.OPT_ADAM, 0.0, 0.9, 0.999, 1e-8)
    after = _results(h, B)
    assert before["info"].cluster_size == after["info"].cluster_size
    np.testing.assert_array_equal(before["lam"], after["lam"])
    np.testing.assert_array_equal(before["br"], after["br"])
    h.close()
