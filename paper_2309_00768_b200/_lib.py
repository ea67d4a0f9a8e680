"""ctypes binding of the C-ABI in include/stmhd_b200.h.

The native library is the only compute path: if it cannot be loaded (or
built from the in-tree sources), every operator raises instead of falling
back to a CPU implementation.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors

_lock = threading.Lock()
_lib = None

c_i64, c_int, c_dbl, c_vp = C.c_int64, C.c_int, C.c_double, C.c_void_p
P = C.c_void_p  # device/host pointers are passed as integers

_SIGS = {
    "stmhd_abi_version": (c_int, []),
    "stmhd_launch_count": (c_i64, []),
    "stmhd_last_error": (C.c_char_p, []),
    "stmhd_last_block": (C.c_char_p, []),
    "stmhd_device_fault": (c_int, [P]),
    "stmhd_disc_create": (c_int, [C.POINTER(c_vp)]),
    "stmhd_disc_destroy": (c_int, [c_vp]),
    "stmhd_disc_set_int": (c_int, [c_vp, C.c_char_p, c_i64]),
    "stmhd_disc_set_real": (c_int, [c_vp, C.c_char_p, c_dbl]),
    "stmhd_disc_upload": (c_int, [c_vp, C.c_char_p, P, c_i64, c_int]),
    "stmhd_disc_finalize": (c_int, [c_vp, P]),
    "stmhd_disc_device_bytes": (c_i64, [c_vp]),
    "stmhd_assemble": (c_int, [c_vp, P, P, P, P, P, P, P, P]),
    "stmhd_jac_apply": (c_int, [c_vp, P, P, P, P]),
    "stmhd_pc_create": (c_int, [c_vp, P, P, P, P, c_int, C.POINTER(c_vp)]),
    "stmhd_pc_destroy": (c_int, [c_vp]),
    "stmhd_pc_apply": (c_int, [c_vp, P, c_int, P, P]),
    "stmhd_pc_op": (c_int, [c_vp, P, c_int, P, P]),
    "stmhd_pc_export": (c_int, [c_vp, P, c_int, P]),
    "stmhd_gs_work_size": (c_i64, [c_i64, c_int]),
    "stmhd_gs_dots": (c_int, [P, P, c_i64, c_int, P, c_i64, P, P]),
    "stmhd_gs_update": (c_int, [P, P, c_i64, c_int, P, P, c_i64, P, P, P]),
    "stmhd_gs_normalize": (c_int, [P, P, P, c_i64, P]),
    "stmhd_gs_combine": (c_int, [P, P, c_i64, c_int, P, P, c_i64]),
    "stmhd_axpby": (c_int, [P, c_dbl, P, c_dbl, P, P, c_i64, P, P]),
    "stmhd_lu_create": (c_int, [c_i64, P, P, P, P, c_int, c_int, C.POINTER(c_vp)]),
    "stmhd_lu_destroy": (c_int, [c_vp]),
    "stmhd_lu_factor": (c_int, [c_vp, P, P, c_i64, P]),
    "stmhd_lu_solve": (c_int, [c_vp, P, P, c_i64, P, c_i64, c_int]),
    "stmhd_lu_info": (c_int, [c_vp, P]),
    "stmhd_lu_sweep": (c_int, [c_vp, P, P, c_i64, P, c_i64, c_int, P, P, P, c_dbl]),
    "stmhd_c5_values": (c_int, [P, c_i64, c_int, P, P, P, P, P, c_i64, P, P, P]),
    "stmhd_c5_velocity": (c_int, [P, c_i64, c_int, P, P, P]),
    "stmhd_bidiag_spmv": (c_int, [P, c_i64, c_int, P, P, P, c_i64, P, P, P, c_dbl, P, P]),
    "stmhd_nd_plan_info": (c_int, [c_i64, P, P, P, P, c_int, P]),
    "stmhd_spmv_create": (c_int, [c_i64, P, P, P, P, P, C.c_int32, P, C.POINTER(c_vp)]),
    "stmhd_spmv_destroy": (c_int, [c_vp]),
    "stmhd_spmv_sell_size": (c_i64, [c_vp]),
    "stmhd_spmv_relayout": (c_int, [c_vp, P, c_int, P, c_i64, P]),
    "stmhd_spmv_apply": (c_int, [c_vp, P, c_int, P, c_dbl, c_dbl, P, P]),
    "stmhd_const_assemble": (c_int, [P, c_i64, c_int, c_int, c_i64, P, P, P, P, P, P, P, c_i64, P]),
    "stmhd_jac_sell_size": (c_i64, [c_vp, P]),
    "stmhd_jac_relayout": (c_int, [c_vp, P, P, P]),
    "stmhd_jac_apply_sell": (c_int, [c_vp, P, P, P, P]),
}

EXPORTS = tuple(_SIGS)
# must equal stmhd_abi_version() of the loaded library (include/stmhd_b200.h)
ABI_VERSION = 3


def lib_path() -> str:
    from . import _build

    return _build.OUT


def load(build_if_needed: bool = True):
    """Load (building first if the in-tree .so is missing or stale)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        from . import _build

        path = _build.OUT
        if build_if_needed and _build.needs_build():
            try:
                _build.build()
            except Exception as exc:  # pragma: no cover - depends on toolchain
                # never run a stale library against newer sources: the ctypes
                # signatures below follow the sources, not the old binary
                raise ImportError(f"stmhd_b200 native library is missing or stale and the rebuild "
                                  f"failed: {exc}") from exc
        if not os.path.exists(path):
            raise ImportError(f"stmhd_b200 native library not found at {path}; run __graft_entry__.build()")
        lib = C.CDLL(path)
        lib.stmhd_abi_version.restype = c_int
        got = lib.stmhd_abi_version()
        if got != ABI_VERSION:
            raise ImportError(f"stmhd_b200 native library {path} has ABI version {got}, "
                              f"the bindings expect {ABI_VERSION}; rebuild it (__graft_entry__.build())")
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int, block: str | None = None):
    """Raise the stmhd exception matching a C-ABI status code."""
    if status == errors.STATUS_OK:
        return
    lib = load()
    msg = (lib.stmhd_last_error() or b"").decode()
    blk = (lib.stmhd_last_block() or b"").decode() or block
    if status == errors.STATUS_SINGULAR:
        if blk:
            raise errors.PreconditionerError(blk, msg)
        raise errors.SingularMatrixError(msg)
    if status == errors.STATUS_NONFINITE:
        raise errors.BreakdownError(msg)
    if status in (errors.STATUS_CONFIG, errors.STATUS_MISSING):
        raise errors.ConfigurationError(msg)
    raise errors.CudaError(msg or f"native call failed with status {status}")


def ptr(t) -> int:
    """Raw pointer of a torch tensor or numpy array (None -> 0)."""
    if t is None:
        return 0
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
