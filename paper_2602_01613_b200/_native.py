"""ctypes binding of libtnl.so (include/tnl.h) — the only route to compute.

There is no CPU fallback: if the library or a GPU is missing, every compute
entry point raises ``DeviceError``. Loading the library itself needs only the
CUDA runtime, so CPU-only test boxes can check the exported symbols.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DeviceError, NumericsError, RankError, ShapeError, UnsupportedError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtnl.so")

TNL_OK, TNL_ERR_SHAPE, TNL_ERR_RANK, TNL_ERR_NUMERICS, TNL_ERR_CUDA, TNL_ERR_UNSUPPORTED, TNL_ERR_ARG = range(7)
FAMILY_CODE = {"dense": 0, "tucker": 1, "tt": 2, "tr": 3}
TNL_F64, TNL_F32, TNL_BF16 = 0, 1, 2
PLAN_AUTO, PLAN_CUT, PLAN_CHAIN, PLAN_GENERIC, PLAN_NO_DECODE, PLAN_GEMV = 0, 1, 2, 4, 8, 16
PLAN_NAMES = {PLAN_CUT: "cut", PLAN_CHAIN: "chain", PLAN_GENERIC: "generic", 0: "none"}
MAX_MODES = 6

# Every symbol include/tnl.h declares: the drop-in boundary of the reference layer
# (checked by tests/test_abi.py).
EXPORTED = (
    "tnl_abi_version",
    "tnl_last_error",
    "tnl_plan_create",
    "tnl_plan_create_rows",
    "tnl_plan_destroy",
    "tnl_plan_query",
    "tnl_workspace_size",
    "tnl_forward",
    "tnl_forward_host",
    "tnl_reconstruct",
    "tnl_jacobi_sweeps",
    "tnl_jacobi_sweeps_parallel",
    "tnl_svd_finish",
)
# include/tnl_stack.h: decoder-stack extensions (no reference counterpart; the Qwen3 stack driver).
EXPORTED_STACK = (
    "tnl_rms_stats",
    "tnl_forward_ex",
    "tnl_stack_workspace_size",
    "tnl_stack_forward",
    "tnl_stack_forward_host",
    "tnl_mlp_create",
    "tnl_mlp_destroy",
    "tnl_mlp_is_fused",
    "tnl_mlp_workspace_size",
    "tnl_mlp_forward",
    "tnl_mlp_forward_ex",
    "tnl_add_rmsnorm",
    "tnl_copy_async",
    "tnl_launch_count",
    "tnl_plan_set_trace",
    "tnl_group_create",
    "tnl_group_destroy",
    "tnl_group_workspace_size",
    "tnl_group_forward_ex",
)


class FwdOpts(ctypes.Structure):
    """tnl_fwd_opts (include/tnl.h): folded residual add / RMSNorm of a decoder stack (prefill)."""

    _fields_ = [
        ("accumulate", ctypes.c_int32),
        ("ss_in", ctypes.c_void_p),
        ("rms_n", ctypes.c_int32),
        ("rms_eps", ctypes.c_float),
        ("rms_fused", ctypes.c_int32),
    ]


class LayerDesc(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_int32),
        ("ndim", ctypes.c_int32),
        ("row_mode_count", ctypes.c_int32),
        ("src_dtype", ctypes.c_int32),
        ("mode_shape", ctypes.c_int64 * MAX_MODES),
        ("ranks", ctypes.c_int64 * (MAX_MODES + 1)),
        ("arrays", ctypes.c_void_p * (MAX_MODES + 1)),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("r_cut", ctypes.c_int64),
        ("param_count", ctypes.c_int64),
        ("chain_flops_per_token", ctypes.c_int64),
        ("cut_flops_per_token", ctypes.c_int64),
        ("dense_flops_per_token", ctypes.c_int64),
        ("weight_bytes", ctypes.c_int64),
        ("decode_weight_bytes", ctypes.c_int64),
        ("compute_dtype", ctypes.c_int32),
        ("plan_large", ctypes.c_int32),
        ("plan_small", ctypes.c_int32),
        ("decode_max_m", ctypes.c_int32),
        ("row_begin", ctypes.c_int64),
        ("row_end", ctypes.c_int64),
    ]


_lib = None
_lock = threading.Lock()


def lib_path() -> str:
    # TNL_LIB_AB: load an alternative in-tree build (A/B measurements of compile-time variants)
    return os.environ.get("TNL_LIB_AB") or LIB_PATH


def load():
    """Load libtnl.so once; raises DeviceError (no fallback) when it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if not os.path.exists(path):
            raise DeviceError(
                f"{path} is missing: build it with `python -m paper_2602_01613_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(path)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        lib.tnl_abi_version.restype = ctypes.c_int
        lib.tnl_last_error.restype = ctypes.c_char_p
        lib.tnl_plan_create.argtypes = [ctypes.POINTER(LayerDesc), ctypes.c_int32, i64, ctypes.c_int32, ctypes.POINTER(P)]
        lib.tnl_plan_create_rows.argtypes = [
            ctypes.POINTER(LayerDesc), ctypes.c_int32, i64, ctypes.c_int32, i64, i64, ctypes.POINTER(P)]
        lib.tnl_plan_destroy.argtypes = [P]
        lib.tnl_plan_query.argtypes = [P, ctypes.POINTER(PlanInfo)]
        lib.tnl_workspace_size.argtypes = [P, i64, ctypes.POINTER(ctypes.c_size_t)]
        lib.tnl_forward.argtypes = [P, P, i64, i64, P, i64, P, ctypes.c_size_t, P]
        lib.tnl_forward_host.argtypes = [P, P, i64, P, P]
        lib.tnl_reconstruct.argtypes = [P, P, i64, ctypes.c_int32, P]
        lib.tnl_stack_workspace_size.argtypes = [ctypes.POINTER(P), ctypes.c_int32, i64,
                                                 ctypes.POINTER(ctypes.c_size_t)]
        lib.tnl_stack_workspace_size.restype = ctypes.c_int
        lib.tnl_stack_forward.argtypes = [ctypes.POINTER(P), ctypes.c_int32, P, i64, i64, P, i64, P,
                                          ctypes.c_size_t, P]
        lib.tnl_stack_forward.restype = ctypes.c_int
        lib.tnl_mlp_create.argtypes = [P, P, P, ctypes.c_int32, ctypes.POINTER(P)]
        lib.tnl_mlp_create.restype = ctypes.c_int
        lib.tnl_mlp_destroy.argtypes = [P]
        lib.tnl_mlp_destroy.restype = ctypes.c_int
        lib.tnl_mlp_is_fused.argtypes = [P]
        lib.tnl_mlp_is_fused.restype = ctypes.c_int32
        lib.tnl_mlp_workspace_size.argtypes = [P, i64, ctypes.POINTER(ctypes.c_size_t)]
        lib.tnl_mlp_workspace_size.restype = ctypes.c_int
        lib.tnl_mlp_forward.argtypes = [P, P, i64, i64, P, i64, P, ctypes.c_size_t, P]
        lib.tnl_mlp_forward.restype = ctypes.c_int
        lib.tnl_plan_set_trace.argtypes = [P, P]
        lib.tnl_plan_set_trace.restype = ctypes.c_int
        lib.tnl_jacobi_sweeps.argtypes = [P, P, i64, i64, i64, i64, ctypes.c_double, ctypes.c_int32, P, P]
        lib.tnl_jacobi_sweeps.restype = ctypes.c_int
        lib.tnl_group_create.argtypes = [ctypes.POINTER(P), ctypes.c_int32, ctypes.POINTER(P)]
        lib.tnl_group_create.restype = ctypes.c_int
        lib.tnl_group_destroy.argtypes = [P]
        lib.tnl_group_destroy.restype = ctypes.c_int
        lib.tnl_group_workspace_size.argtypes = [P, i64, ctypes.POINTER(ctypes.c_size_t)]
        lib.tnl_group_workspace_size.restype = ctypes.c_int
        lib.tnl_group_forward_ex.argtypes = [P, P, i64, i64, ctypes.POINTER(P), ctypes.POINTER(i64), P, ctypes.c_size_t,
                                             P, P]
        lib.tnl_group_forward_ex.restype = ctypes.c_int
        lib.tnl_jacobi_sweeps_parallel.argtypes = [P, P, i64, i64, i64, ctypes.c_double, ctypes.c_int32, P, P]
        lib.tnl_jacobi_sweeps_parallel.restype = ctypes.c_int
        lib.tnl_svd_finish.argtypes = [P, P, i64, i64, i64, P, P, P, P, P]
        lib.tnl_svd_finish.restype = ctypes.c_int
        lib.tnl_add_rmsnorm.argtypes = [P, i64, P, i64, P, i64, i64, i64, ctypes.c_float, P]
        lib.tnl_add_rmsnorm.restype = ctypes.c_int
        lib.tnl_copy_async.argtypes = [P, P, ctypes.c_size_t, P]
        lib.tnl_copy_async.restype = ctypes.c_int
        lib.tnl_stack_forward_host.argtypes = [ctypes.POINTER(P), ctypes.c_int32, P, i64, i64, P, i64, P,
                                               ctypes.c_size_t, P]
        lib.tnl_stack_forward_host.restype = ctypes.c_int
        OP = ctypes.POINTER(FwdOpts)
        lib.tnl_forward_ex.argtypes = [P, P, i64, i64, P, i64, P, ctypes.c_size_t, OP, P]
        lib.tnl_forward_ex.restype = ctypes.c_int
        lib.tnl_mlp_forward_ex.argtypes = [P, P, i64, i64, P, i64, P, ctypes.c_size_t, OP, P]
        lib.tnl_mlp_forward_ex.restype = ctypes.c_int
        lib.tnl_rms_stats.argtypes = [P, i64, i64, i64, P, P]
        lib.tnl_rms_stats.restype = ctypes.c_int
        lib.tnl_launch_count.argtypes = [ctypes.c_int32]
        lib.tnl_launch_count.restype = i64
        for name in ("tnl_plan_create", "tnl_plan_create_rows", "tnl_plan_destroy", "tnl_plan_query",
                     "tnl_workspace_size", "tnl_forward", "tnl_forward_host", "tnl_reconstruct"):
            getattr(lib, name).restype = ctypes.c_int
        if lib.tnl_abi_version() != 1:
            raise DeviceError(f"libtnl ABI {lib.tnl_abi_version()} != 1")
        _lib = lib
        return lib


def check(status: int) -> None:
    """Map a tnl_status onto the reference exception classes (errors.py:8-21)."""
    if status == TNL_OK:
        return
    msg = (load().tnl_last_error() or b"").decode(errors="replace")
    if status == TNL_ERR_SHAPE:
        raise ShapeError(msg)
    if status == TNL_ERR_RANK:
        raise RankError(msg)
    if status == TNL_ERR_NUMERICS:
        raise NumericsError(msg)
    if status == TNL_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    if status == TNL_ERR_ARG:
        raise ValueError(msg)
    raise DeviceError(msg)


def launch_count(reset: bool = False) -> int:
    return int(load().tnl_launch_count(1 if reset else 0))
