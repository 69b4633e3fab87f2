"""CPU check of the batched path's host-compiled sweep schedule (the slot
allocator behind the TMA pipeline): tests/sched_check.cpp replays every
part's producer/consumer order of k_sweep with worst-case (instant) copy
landing and asserts every shared-memory slot read holds the expected row /
code, codes are read only after the step writing them, and the owned items
cover every bus, branch and cycle once per phase.  Shares schedule.cpp /
split_schedule.cpp with the library (host logic, no GPU, no oracle)."""
import os
import subprocess

import numpy as np
import pytest

from paper_2406_13191_b200 import instances as inst

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = "/tmp/dcopf_sched_check"


@pytest.fixture(scope="module")
def checker():
    src = [os.path.join(ROOT, "tests", "sched_check.cpp"),
           os.path.join(ROOT, "paper_2406_13191_b200", "csrc", "schedule.cpp"),
           os.path.join(ROOT, "paper_2406_13191_b200", "csrc", "split_schedule.cpp"),
           os.path.join(ROOT, "paper_2406_13191_b200", "csrc", "cluster.cpp")]
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-o", EXE] + src)
    return EXE


def run(checker, net, form, CH, P, order="dfs", W=32, life=4, V=None, C=None, gap=3):
    lines = [f"{net.n_bus} {net.n_branch} {net.ref_bus} {form} {CH} {P}"]
    lines += [f"{a} {b}" for a, b in zip(net.br_from, net.br_to)]
    args = [checker, order, str(W), str(life)]
    if V is not None:  # the split-tile compiler (V instances per lane, C parts per tile)
        args += [str(gap), str(V), str(C)]
    res = subprocess.run(args, input="\n".join(lines) + "\n", capture_output=True, text=True)
    return res.returncode, res.stdout


@pytest.mark.parametrize("config", [0, 1, 3])
@pytest.mark.parametrize("form", [0, 1, 2])
@pytest.mark.parametrize("CH,P,W,life", [(32, 2, 56, 4), (8, 1, 2, 0), (64, 3, 64, 6), (16, 2, 56, 2)])
def test_schedule_slots_valid(checker, config, form, CH, P, W, life):
    net = inst.make_network(config)
    rc, out = run(checker, net, form, CH, P, W=W, life=life)
    assert rc == 0, out


@pytest.mark.parametrize("seed", range(6))
def test_schedule_random_small(checker, seed):
    rng = np.random.default_rng(seed)
    nb = int(rng.integers(1, 60))
    nl = int(rng.integers(nb - 1, 3 * nb)) if nb > 1 else 0
    net = inst.tiny_network(nb, max(nl, nb - 1), 3, seed=seed) if nb > 1 else None
    if net is None:
        return
    for form in (0, 1, 2):
        for CH, P, life in ((1, 1, 0), (3, 2, 2), (16, 1, 6)):
            rc, out = run(checker, net, form, CH, P, life=life)
            assert rc == 0, out
            rc, out = run(checker, net, form, CH, P, order="rcm", life=life)
            assert rc == 0, out


def test_dfs_order_keeps_smem_small(checker):
    """The DFS tree order is what makes the window fit: config-3 network with
    56-instance tiles (the config-4 bench tiling) fits one CTA's shared memory
    (F2 at CH=16, F1 at CH=8, ring life 2) with ~10x fewer bulk copies than
    rows; with RCM order it does not come close."""
    net = inst.make_network(3)
    for form, ch, factor in ((0, 16, 8), (1, 8, 3)):
        rc, out = run(checker, net, form, ch, 2, W=56, life=2)
        smem = int(out.split("smem ")[1].split()[0])
        copies = int(out.split("copies ")[1].split()[0])
        assert rc == 0 and smem <= 220 * 1024 and copies * factor < net.n_bus * 2 + net.n_branch, out
    rc, out = run(checker, net, 0, 16, 2, order="rcm", W=56, life=2)
    assert int(out.split("smem ")[1].split()[0]) > 227 * 1024, out


# ---- split tiles (split_schedule.cpp): forms F2 (0) and KVL (2) -------------
@pytest.mark.parametrize("config", [0, 1, 3])
@pytest.mark.parametrize("form", [0, 1, 2])
@pytest.mark.parametrize("CH,P,W,life,V,C", [(26, 2, 56, 2, 2, 1), (10, 2, 112, 2, 4, 2), (10, 2, 112, 2, 4, 4),
                                             (24, 2, 58, 2, 2, 8), (10, 1, 116, 2, 4, 16), (3, 2, 8, 0, 4, 3)])
def test_split_schedule_valid(checker, config, form, CH, P, W, life, V, C):
    """Every part's slot reads see the expected row / code, codes are read only
    in a later step than the one writing them and rewritten only pool_gap steps
    after their last read, and the owned items of the parts cover every bus,
    branch and cycle exactly once (halo items recompute the rest)."""
    net = inst.make_network(config)
    if C > net.n_bus:
        pytest.skip("more parts than buses")
    if form == 1 and V == 4:
        V, W = 2, W // 2  # F1 runs 2 instances per lane
    rc, out = run(checker, net, form, CH, P, W=W, life=life, V=V, C=C)
    assert rc == 0 and " bad 0" in out, out


@pytest.mark.parametrize("seed", range(6))
def test_split_schedule_random_small(checker, seed):
    rng = np.random.default_rng(100 + seed)
    nb = int(rng.integers(2, 60))
    nl = int(rng.integers(nb - 1, 3 * nb))
    net = inst.tiny_network(nb, max(nl, nb - 1), 3, seed=seed)
    for form in (0, 1, 2):
        for CH, P, life, V, C in ((1, 1, 0, 2, 2), (3, 2, 2, 4, 3), (16, 1, 6, 4, min(nb, 7))):
            V = 2 if form == 1 else V
            rc, out = run(checker, net, form, CH, P, life=life, W=8 * V, V=V, C=C)
            assert rc == 0 and " bad 0" in out, out


def test_split_halo_is_small_and_fits(checker):
    """Config-3 network at the config-4 tilings the library picks (8192 instances:
    4 per lane, 112-instance tiles over 2 parts; 1024: 116 over 16 parts): the
    shared memory fits and the recomputed halo items are a few percent of the
    ~32 700 items of a sweep."""
    exe = checker
    net = inst.make_network(3)
    for form, CH, P, W, V, C, max_halo in ((0, 10, 2, 112, 4, 2, 40), (0, 10, 2, 116, 4, 16, 400),
                                           (2, 22, 1, 112, 4, 2, 40), (2, 22, 1, 116, 4, 16, 400)):
        rc, out = run(exe, net, form, CH, P, W=W, life=2, V=V, C=C)
        smem = int(out.split("smem ")[1].split()[0])
        halo = int(out.split("halo ")[1].split()[0])
        assert rc == 0 and smem <= 227 * 1024 and halo <= max_halo, out
