"""Multi-rank host logic on CPU (world size 2, gloo): the config-4 batch is
sharded contiguously, each rank solves only its instances (here with the
oracle, the only solver available without a GPU), the per-instance results are
gathered once, and the gathered vector equals the unsharded solve bitwise --
instances never interact (SURVEY §8(e) sharding invariance)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2406_13191_b200.distributed import shard, shard_sizes


def test_shard_covers_exactly():
    for B in (1, 7, 8192, 8191):
        for world in (1, 2, 3, 8):
            spans = [shard(B, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(shard_sizes(B, world)) - min(shard_sizes(B, world)) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, K, out_path):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2406_13191_b200 import instances as inst
    from paper_2406_13191_b200.distributed import gather_instance_results, shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    net = inst.make_network(0)
    lo, hi = shard(B, rank, world)
    # a config-4-style sweep on the small network: per-instance load factors
    rng = np.random.default_rng(5)
    factors = rng.uniform(0.85, 1.15, (B, net.n_bus))
    loads = net.base_load[None, :] * factors[lo:hi]
    r = oracle.solve(net, loads, K=K, alpha=inst.alpha_schedule(K, 3e-3))
    g = gather_instance_results([torch.from_numpy(r.bound), torch.from_numpy(r.best),
                                 torch.from_numpy(r.status.astype(np.float64))], B)
    if rank == 0:
        np.save(out_path, g.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_gather_equals_unsharded(tmp_path):
    import oracle
    from paper_2406_13191_b200 import instances as inst

    B, K = 9, 200
    out = str(tmp_path / "g.npy")
    mp.spawn(_worker, args=(2, _free_port(), B, K, out), nprocs=2, join=True)
    g = np.load(out)
    net = inst.make_network(0)
    rng = np.random.default_rng(5)
    loads = net.base_load[None, :] * rng.uniform(0.85, 1.15, (B, net.n_bus))
    ref = oracle.solve(net, loads, K=K, alpha=inst.alpha_schedule(K, 3e-3))
    np.testing.assert_array_equal(g[0], ref.bound)
    np.testing.assert_array_equal(g[1], ref.best)
    np.testing.assert_array_equal(g[2], ref.status)


def _worker_weak(rank, world, port, B, K, out_path):
    """weak scaling: every rank its own B-instance batch = instances
    [rank B, (rank+1) B) of the seeded config-4 sweep (bench.py --scaling weak)"""
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2406_13191_b200 import instances as inst
    from paper_2406_13191_b200.distributed import gather_instance_results

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    net = inst.tiny_network(40, 60, 8, seed=1)
    lo, hi = rank * B, (rank + 1) * B
    batch = inst.config4_batch(net, range(lo, hi), total=world * B)
    r = oracle.solve(net, batch.load, outages=batch.outages, K=K, alpha=inst.alpha_schedule(K, 3e-3))
    g = gather_instance_results([torch.from_numpy(r.bound), torch.from_numpy(r.best)], world * B,
                                sizes=[B] * world)
    if rank == 0:
        np.save(out_path, g.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_weak_scaling_gather(tmp_path):
    """Each rank draws only its own instances; the gathered results equal one
    process solving all 2B instances (instance data depend only on the id)."""
    import oracle
    from paper_2406_13191_b200 import instances as inst

    B, K = 5, 150
    out = str(tmp_path / "w.npy")
    mp.spawn(_worker_weak, args=(2, _free_port(), B, K, out), nprocs=2, join=True)
    g = np.load(out)
    net = inst.tiny_network(40, 60, 8, seed=1)
    batch = inst.config4_batch(net, range(2 * B))
    ref = oracle.solve(net, batch.load, outages=batch.outages, K=K, alpha=inst.alpha_schedule(K, 3e-3))
    np.testing.assert_array_equal(g[0], ref.bound)
    np.testing.assert_array_equal(g[1], ref.best)
