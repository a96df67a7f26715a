"""C-ABI library: loads, exports every symbol include/tnl.h declares (CPU-only)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2602_01613_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols(name="tnl.h"):
    text = open(os.path.join(ROOT, "include", name)).read()
    return sorted(set(re.findall(r"TNL_API\s+[\w\s\*]+?\b(tnl_\w+)\s*\(", text)))


def all_symbols():
    return sorted(set(header_symbols("tnl.h")) | set(header_symbols("tnl_stack.h")))


def test_header_and_binding_agree():
    syms = header_symbols()
    assert len(syms) == 13  # the reference boundary: plan lifecycle, forward, reconstruct, Jacobi SVD
    assert sorted(N.EXPORTED) == syms
    assert sorted(N.EXPORTED_STACK) == header_symbols("tnl_stack.h")


def test_library_exports_every_symbol():
    assert os.path.exists(N.lib_path()), "build libtnl.so first (python -m paper_2602_01613_b200.build)"
    out = subprocess.run(["nm", "-D", "--defined-only", N.lib_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tnl_\w+)", out))
    missing = set(all_symbols()) - exported
    assert not missing, missing


def test_library_loads_and_reports_abi():
    lib = N.load()
    assert lib.tnl_abi_version() == 1
    assert isinstance(lib.tnl_last_error(), bytes)
    for s in all_symbols():
        assert hasattr(lib, s)


def test_struct_layout_matches_header():
    # tnl_layer_desc: 4 x int32, 6 x int64, 7 x int64, 7 x pointer
    assert ctypes.sizeof(N.LayerDesc) == 16 + 8 * 6 + 8 * 7 + 8 * 7
    assert ctypes.sizeof(N.PlanInfo) == 8 * 9 + 4 * 4 + 8 * 2


def test_validation_errors_without_gpu():
    # validation happens before any CUDA call -> same ShapeError on a CPU box
    from paper_2602_01613_b200.errors import ShapeError

    lib = N.load()
    desc = N.LayerDesc()
    desc.family = N.FAMILY_CODE["tt"]
    desc.ndim = 2
    desc.row_mode_count = 2  # invalid: must be < d
    desc.mode_shape[0] = desc.mode_shape[1] = 4
    h = ctypes.c_void_p()
    st = lib.tnl_plan_create(ctypes.byref(desc), N.TNL_BF16, 0, 0, ctypes.byref(h))
    with pytest.raises(ShapeError, match="row_mode_count 2 invalid for 2 modes"):
        N.check(st)
