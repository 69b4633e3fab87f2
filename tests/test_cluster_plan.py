"""CPU check of the cluster path's host-built shared-memory plan
(paper_2406_13191_b200/csrc/cluster.cpp): tests/cluster_check.cpp decodes
every distributed-shared-memory address of every CTA's blob and checks it names
the right bus / branch / cycle value, that ownership is a partition, and (KVL
form) that the library's canonical cycle basis is made of closed loops whose
only non-tree branch is the defining one -- and, against the ORACLE's
independent implementation of the same definition (reading A-28), that the
two bases are identical.  Host logic only; no GPU."""
import os
import subprocess

import numpy as np
import pytest

import oracle
from paper_2406_13191_b200 import instances as inst

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = "/tmp/dcopf_cluster_check"


@pytest.fixture(scope="module")
def checker():
    src = [os.path.join(ROOT, "tests", "cluster_check.cpp"),
           os.path.join(ROOT, "paper_2406_13191_b200", "csrc", "cluster.cpp"),
           os.path.join(ROOT, "paper_2406_13191_b200", "csrc", "schedule.cpp")]
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-o", EXE] + src)
    return EXE


def run(checker, net, form, C, sw=None):
    sw = np.zeros(net.n_branch, np.uint8) if sw is None else sw
    lines = [f"{net.n_bus} {net.n_branch} {net.ref_bus} {form} {C}"]
    lines += [f"{a} {b} {float(x)!r} {float(F)!r} {s}" for a, b, x, F, s in zip(net.br_from, net.br_to, net.br_b, net.br_fmax, sw)]
    r = subprocess.run([checker], input="\n".join(lines) + "\n", capture_output=True, text=True)
    return r.returncode, r.stdout


@pytest.mark.parametrize("config", [0, 1, 3])
@pytest.mark.parametrize("form", [0, 1, 2])
@pytest.mark.parametrize("C", [1, 2, 4, 16])
def test_cluster_plan_addresses(checker, config, form, C):
    net = inst.make_network(config)
    sw = np.zeros(net.n_branch, np.uint8)
    sw[net.n_tree:] = 1
    rc, out = run(checker, net, form, C, sw)
    if "does not fit" in out:  # the library then picks a larger cluster (config 3: 16 CTAs)
        assert C < 16
        pytest.skip(out)
    assert rc == 0, out


def test_cluster_plan_zero_susceptance_branch(checker):
    """A b = 0 branch is never a tree branch; in the KVL form its cycle is inactive."""
    net = inst.tiny_network(30, 50, 4, seed=2)
    net.br_b[net.n_tree + 3] = 0.0
    rc, out = run(checker, net, 2, 4)
    assert rc == 0, out


@pytest.mark.parametrize("config,all_switchable", [(0, False), (1, True), (3, True)])
def test_library_and_oracle_cycle_bases_agree(checker, config, all_switchable):
    """The oracle (C) and the library (C++) build the canonical basis from the
    same written definition (reading A-28), independently: identical cycles."""
    net = inst.make_network(config)
    sw = np.zeros(net.n_branch, np.uint8)
    if all_switchable:
        sw[net.n_tree:] = 1
    lines = [f"{net.n_bus} {net.n_branch} {net.ref_bus} 2 16"]
    lines += [f"{a} {b} {float(x)!r} {float(F)!r} {s}" for a, b, x, F, s in
              zip(net.br_from, net.br_to, net.br_b, net.br_fmax, sw)]
    r = subprocess.run([checker], input="\n".join(lines) + "\n", capture_output=True, text=True,
                       env={**os.environ, "DUMP_BASIS": "1"})
    lib = [list(map(int, ln.split()[1:])) for ln in r.stdout.splitlines() if ln.startswith("cycle ")]
    d, cyc = oracle.cycles(net, sw if all_switchable else None)
    assert len(lib) == len(d) == net.n_branch - net.n_bus + 1
    for k, row in enumerate(lib):
        assert row[0] == d[k]
        n = row[1]
        assert np.array_equal(np.array(row[2::2][:n]), cyc[k][0])
        assert np.array_equal(np.array(row[3::2][:n]), cyc[k][1])
