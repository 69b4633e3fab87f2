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


def test_binding_constants_match_header():
    """The ctypes binding's enum values and struct layouts are the header's."""
    hdr = open(os.path.join(ROOT, "include", "dcopf_dual.h")).read()
    vals = {k: int(v) for k, v in re.findall(r"\b(DCOPF_[A-Z_0-9]+)\s*=\s*(-?\d+)", hdr)}
    assert vals["DCOPF_FORM_FLOW_BOX"] == dual.FORM_F2
    assert vals["DCOPF_FORM_LIMIT_ROWS"] == dual.FORM_F1
    assert vals["DCOPF_FORM_CYCLE"] == dual.FORM_KVL
    assert vals["DCOPF_FORM_PTDF"] == dual.FORM_PTDF
    assert (vals["DCOPF_PATH_AUTO"], vals["DCOPF_PATH_BATCHED"], vals["DCOPF_PATH_SINGLE"], vals["DCOPF_PATH_CLUSTER"],
            vals["DCOPF_PATH_DENSE"]) == (dual.PATH_AUTO, dual.PATH_BATCHED, dual.PATH_SINGLE, dual.PATH_CLUSTER,
                                          dual.PATH_DENSE)
    assert (vals["DCOPF_INST_OK"], vals["DCOPF_INST_DIVERGED"], vals["DCOPF_INST_CONVERGED"]) == (
        dual.INST_OK, dual.INST_DIVERGED, dual.INST_CONVERGED)
    assert (vals["DCOPF_OPT_PLAIN"], vals["DCOPF_OPT_GDM"], vals["DCOPF_OPT_GDM_CLASSIC"], vals["DCOPF_OPT_ADAGRAD"],
            vals["DCOPF_OPT_ADAM"]) == (dual.OPT_PLAIN, dual.OPT_GDM, dual.OPT_GDM_CLASSIC, dual.OPT_ADAGRAD,
                                        dual.OPT_ADAM)
    for k, v in vals.items():
        if k in ("DCOPF_OK", "DCOPF_EINVAL", "DCOPF_ETOPOLOGY", "DCOPF_ECUDA", "DCOPF_ENOMEM", "DCOPF_ESTATE"):
            assert v == 0 or dual.ERRORS[v] == k[len("DCOPF_"):]


def test_binding_struct_sizes_match_c(tmp_path):
    """sizeof of every ABI struct as the C compiler lays it out == the ctypes mirror."""
    import subprocess
    src = tmp_path / "sizes.c"
    src.write_text('#include <stdio.h>\n#include "dcopf_dual.h"\nint main(void){printf("%zu %zu %zu %zu",'
                   'sizeof(dcopf_network_desc),sizeof(dcopf_options),sizeof(dcopf_optimizer),sizeof(dcopf_info));'
                   'return 0;}\n')
    exe = tmp_path / "sizes"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(dual.NetworkDesc), ctypes.sizeof(dual.Options), ctypes.sizeof(dual.Optimizer),
                   ctypes.sizeof(dual.Info)]
