"""CPU-side checks of the C ABI boundary: the library builds for sm_100a,
loads without a GPU, exports every symbol include/dcopf_dual.h declares, and
its host-side validation (SPEC.md:30-50 rules) rejects malformed networks
before touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2406_13191_b200 import _build, dual
from paper_2406_13191_b200 import instances as inst

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return dual.load_library()


def test_header_symbols_exported(lib):
    hdr = open(os.path.join(ROOT, "include", "dcopf_dual.h")).read()
    declared = set(re.findall(r"\b(dcopf_dual_\w+)\s*\(", hdr))
    assert {"dcopf_dual_create", "dcopf_dual_set_instance_batch", "dcopf_dual_iterate", "dcopf_dual_get_bound",
            "dcopf_dual_get_multipliers"} <= declared
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(dual.SYMBOLS)


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _err(net, **kw):
    with pytest.raises(dual.DcopfError) as e:
        dual.DcopfDual(net, **kw)
    return e.value


def test_validation_errors(lib):
    net = inst.make_network(0)
    import copy
    bad = copy.deepcopy(net)
    bad.br_to = bad.br_to.copy()
    bad.br_to[3] = bad.br_from[3]
    assert _err(bad).code == -1 and "self loop" in str(_err(bad))
    bad = copy.deepcopy(net)
    bad.gen_pmin = bad.gen_pmax + 1
    assert _err(bad).code == -1
    bad = copy.deepcopy(net)
    bad.br_b = bad.br_b.copy()
    bad.br_b[2] = -1.0
    assert _err(bad).code == -1
    bad = copy.deepcopy(net)
    bad.ref_bus = 99
    assert _err(bad).code == -1
    # disconnect bus 13: zero susceptance on all its branches
    bad = copy.deepcopy(net)
    bad.br_b = bad.br_b.copy()
    bad.br_b[(bad.br_from == 13) | (bad.br_to == 13)] = 0.0
    assert _err(bad).code == -2
    # never-switchable part must connect the network
    sw = np.zeros(net.n_branch, np.uint8)
    sw[: net.n_tree] = 1
    assert _err(net, switchable=sw).code == -2
    assert _err(net, form=7).code == -1


def test_last_error_null_handle(lib):
    msg = lib.dcopf_dual_last_error(None)
    assert isinstance(msg, bytes)
