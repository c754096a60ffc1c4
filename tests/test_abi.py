"""The C-ABI engine library builds, loads without a GPU, and exports every
entry point include/ps_b200.h declares (no compute calls here)."""

import ctypes
import os
import re

from paper_1405_2636_b200 import _abi, _native

HEADER = os.path.join(_native.INCLUDE, "ps_b200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("ps_plan_create", "ps_factor", "ps_factor_status", "ps_assemble",
                 "ps_run_factor_task", "ps_run_update_task", "ps_plan_destroy",
                 "ps_last_error"):
        assert must in names


def test_engine_library_exports_every_declared_symbol():
    path = _native.build_engine()
    lib = ctypes.CDLL(path)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_table_matches_header():
    assert sorted(_abi.EXPORTS) == declared()


def test_engine_loads_through_package():
    lib = _native.engine_lib()
    assert lib.ps_last_error() is not None


def test_host_library_exports():
    lib = _native.host_lib()
    for n in ("psh_nested_dissection", "psh_etree", "psh_postorder", "psh_symbolic"):
        assert hasattr(lib, n)
