"""ctypes binding of the TEST-ONLY probe library tests/csrc/libsa_probe.so (tcgen05 / TMA
operand-layout probes used by test_gpu_primitives.py).  Not part of the product."""

import ctypes

import torch

_P = ctypes.c_void_p
_lib = None


def lib():
    global _lib
    if _lib is None:
        from paper_2311_09431_b200 import build
        path = build.build_probe()
        h = ctypes.CDLL(path)
        for name in ("sa_probe_umma", "sa_probe_pair"):
            fn = getattr(h, name)
            fn.restype = ctypes.c_int
            fn.argtypes = [_P] * 7
        h.sa_probe_last_error.restype = ctypes.c_char_p
        _lib = h
    return _lib


def _check(status, what):
    if status != 0:
        raise RuntimeError(f"{what} failed ({status}): {lib().sa_probe_last_error().decode()}")


def _stream(t):
    return torch.cuda.current_stream(t.device).cuda_stream


def probe_umma(a, b, v):
    """(s, o, y) = (a b^T, bf16(s) v, b^T v) computed with tcgen05 on one 128^3 tile."""
    s, o, y = (torch.empty(128, 128, device=a.device, dtype=torch.float32) for _ in range(3))
    _check(lib().sa_probe_umma(a.data_ptr(), b.data_ptr(), v.data_ptr(), s.data_ptr(),
                               o.data_ptr(), y.data_ptr(), _stream(a)), "sa_probe_umma")
    return s, o, y


def probe_pair(a, b, v):
    """CTA-pair layouts: a [256,128], b [128,128], v [128,128] bf16 ->
    (s, o, s2) = (a b^T, bf16(s) v, a b^T with A staged in TMEM)."""
    s, o, s2 = (torch.empty(256, 128, device=a.device, dtype=torch.float32) for _ in range(3))
    _check(lib().sa_probe_pair(a.data_ptr(), b.data_ptr(), v.data_ptr(), s.data_ptr(),
                               o.data_ptr(), s2.data_ptr(), _stream(a)), "sa_probe_pair")
    return s, o, s2
