"""ctypes binding of the C ABI in include/striped_attn.h.

The product path has no fallback: if ``libstriped_attn.so`` is missing or a CUDA
device is unavailable, every op raises.  Tensors are passed as raw device pointers
(``tensor.data_ptr()``) plus the current torch stream handle.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SA_LIB_PATH") or os.path.join(_HERE, "libstriped_attn.so")

_lib = None

# name -> (restype, argtypes); must match include/striped_attn.h exactly.
_P, _I32, _I64, _F32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
SIGNATURES = {
    "sa_abi_version": (ctypes.c_int, []),
    "sa_last_error": (ctypes.c_char_p, []),
    "sa_launch_count": (_I64, []),
    "sa_permute": (ctypes.c_int, [_P, _P, _I64, _I32, _I64, _I32, _I32, _I32, _P]),
    "sa_fwd_block": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _F32, _I32,
                                    _I32, _I32, _P, _P]),
    "sa_bwd_preprocess": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I32, _I32, _P]),
    "sa_bwd_block": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32,
                                    _F32, _I32, _P]),
    "sa_bwd_block_range": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I32, _I32,
                                          _I32, _F32, _I32, _I32, _I32, _P]),
    "sa_bwd_block_final": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I32, _I32,
                                          _I32, _F32, _I32, _P]),
    "sa_bwd_block_ex": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I32,
                                       _I32, _I32, _F32, _I32, _I32, _I32, _P, _P]),
    "sa_cast_f32_bf16": (ctypes.c_int, [_P, _P, _I64, _P]),
    "sa_memcpy2d_async": (ctypes.c_int, [_P, _I64, _P, _I64, _I64, _I64, _P]),
    "sa_memcpy_async": (ctypes.c_int, [_P, _P, _I64, _P]),
    "sa_ipc_mem_handle": (ctypes.c_int, [_P, _P, ctypes.POINTER(_I64)]),
    "sa_ipc_mem_open": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "sa_ipc_mem_close": (ctypes.c_int, [_P]),
    "sa_ipc_event_create": (ctypes.c_int, [ctypes.POINTER(_P), _P]),
    "sa_ipc_event_open": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "sa_event_record": (ctypes.c_int, [_P, _P]),
    "sa_stream_wait_event": (ctypes.c_int, [_P, _P]),
    "sa_event_destroy": (ctypes.c_int, [_P]),
}


class StripedAttnError(RuntimeError):
    pass


def lib():
    """Load the shared library once (CDLL with the exact signatures)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise StripedAttnError(
                f"{LIB_PATH} is missing: run `python -m paper_2311_09431_b200.build` "
                "(there is no CPU fallback)")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().sa_last_error().decode(errors="replace")
        kind = ValueError if status > 0 else StripedAttnError
        raise kind(f"{what} failed (status {status}): {msg}")


def launch_count() -> int:
    return int(lib().sa_launch_count())
