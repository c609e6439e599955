"""ctypes binding of libbsgpu.so (include/blocksolve_b200.h).

The library is built in-tree (``paper_2009_12638_b200/_lib/libbsgpu.so``,
see ``build.py``).  There is no CPU fallback: if the library is missing or a
CUDA device is absent, every solver entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigurationError, DeviceError, ProtocolError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BS_LIB") or os.path.join(HERE, "_lib", "libbsgpu.so")

NDIR = 6
STOP_NAMES = {0: "none", 1: "tolerance_met", 2: "max_iterations", 3: "breakdown", 4: "stalled"}
BASIS = {"rhs": 0, "initial": 1}
VEC_WORK = 512  # BS_VEC_WORK


class BlockDesc(ctypes.Structure):
    _fields_ = [
        ("global_dims", ctypes.c_int32 * 3),
        ("owned_lo", ctypes.c_int32 * 3),
        ("owned_hi", ctypes.c_int32 * 3),
        ("overlap", ctypes.c_int32),
        ("x", ctypes.c_void_p),
        ("r", ctypes.c_void_p),
        ("p0", ctypes.c_void_p),
        ("p1", ctypes.c_void_p),
        ("b", ctypes.c_void_p),
        ("ghost", ctypes.c_void_p * NDIR),
        ("history", ctypes.c_void_p),
        ("history_cap", ctypes.c_int32),
        ("remote", ctypes.c_int32),
    ]


class GmresDesc(ctypes.Structure):
    _fields_ = [("V", ctypes.c_void_p), ("vstride", ctypes.c_int64), ("W", ctypes.c_void_p)]


class BlockReport(ctypes.Structure):
    _fields_ = [
        ("phase", ctypes.c_int32),
        ("stop_reason", ctypes.c_int32),
        ("iterations_used", ctypes.c_int32),
        ("pending_flush", ctypes.c_int32),
        ("final_relative_residual", ctypes.c_double),
        ("rhs_sq", ctypes.c_double),
        ("r_sq", ctypes.c_double),
        ("r_owned_sq", ctypes.c_double),
        ("rglob_owned_sq", ctypes.c_double),
        ("scale", ctypes.c_double),
        ("last_iterations", ctypes.c_int32),
        ("last_stop_reason", ctypes.c_int32),
    ]


_P = ctypes.c_void_p
_I = ctypes.c_int
_SIGS = {
    "bs_abi_version": ([], _I),
    "bs_last_error": ([], ctypes.c_char_p),
    "bs_ctx_create": ([_I, _I, ctypes.POINTER(BlockDesc), _I, ctypes.POINTER(_P)], _I),
    "bs_ctx_destroy": ([_P], _I),
    "bs_ctx_num_ctas": ([_P], _I),
    "bs_ctx_run_path": ([_P], _I),
    "bs_block_pitch": ([_P, _I], _I),
    "bs_stencil_apply": ([_P, _I, _P, _P, _P], _I),
    "bs_cg_begin": ([_P, _I, ctypes.c_double, _I, _P, _P], _I),
    "bs_jacobi_begin": ([_P, _I, ctypes.c_double, _I, _P, _P], _I),
    "bs_async_post_slot": ([_P, _I, _I, _P, _P, _P, _I, ctypes.c_uint64, ctypes.c_int64, _P], _I),
    "bs_async_receive_at": ([_P, _I, _I, _P, _P, _P, _I, ctypes.c_int64, _P, _P, _P, _P], _I),
    "bs_vec_nrm2": ([_P, ctypes.c_int64, _P, _P], _I),
    "bs_vec_scale": ([_P, ctypes.c_int64, ctypes.c_double, _P, _P], _I),
    "bs_sweep_resid": ([_P, _P], _I),
    "bs_cancel": ([_P, _P, _P], _I),
    "bs_run": ([_P, _I, _I, _P, ctypes.POINTER(ctypes.c_int64)], _I),
    "bs_residual": ([_P, _P, _P], _I),
    "bs_flush": ([_P, _P], _I),
    "bs_halo_pack": ([_P, _I, _P, _P], _I),
    "bs_read_reports": ([_P, ctypes.POINTER(BlockReport), _P], _I),
    "bs_launch_count": ([], ctypes.c_ulonglong),
    "bs_overlap_merge": ([_P, _P], _I),
    "bs_ipc_export": ([_P, _P, ctypes.POINTER(ctypes.c_uint64)], _I),
    "bs_ipc_open": ([_P, ctypes.c_uint64, ctypes.POINTER(_P)], _I),
    "bs_ipc_close": ([_P], _I),
    "bs_uniform_pcg64": ([_P, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                          ctypes.c_double, ctypes.c_double, _P], _I),
    "bs_async_post": ([_P, _I, _I, _P, _P, _I, ctypes.c_uint64, _P], _I),
    "bs_async_receive": ([_P, _I, _I, _P, _P, _I, _P, _P, _P, _P], _I),
    "bs_owner_residual": ([_P, _P], _I),
    "bs_gmres_setup": ([_P, _I, ctypes.POINTER(GmresDesc)], _I),
    "bs_gmres_begin": ([_P, _I, ctypes.c_double, _I, _P, _P], _I),
    "bs_gmres_run": ([_P, _I, _P, ctypes.POINTER(ctypes.c_int64)], _I),
    "bs_overlap_snapshot": ([_P, _P], _I),
    "bs_overlap_combine": ([_P, _P], _I),
    "bs_gmres_run_block": ([_P, _I, _I, _P, ctypes.POINTER(ctypes.c_int64)], _I),
    "bs_timing": ([_P, _I, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_longlong)], _I),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the engine; raise DeviceError (never fall back) if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"CUDA engine not built: {LIB_PATH} missing (run `python -m "
            "paper_2009_12638_b200.build` or __graft_entry__.build())"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.bs_abi_version() != 2:
        raise DeviceError("libbsgpu.so ABI version mismatch")
    _lib = lib
    return lib


def check(code: int) -> None:
    """Map a C status code onto the reference's exception types."""
    if code == 0:
        return
    msg = (_lib.bs_last_error() or b"").decode(errors="replace")
    if code == -1:
        raise ConfigurationError(msg)
    if code == -3:
        raise ProtocolError(msg)
    raise DeviceError(msg)
