"""torch-facing wrappers of the C ABI (device buffers in, device buffers out).

Each wrapper validates dtype / device / contiguity, then calls the CUDA library on
the current torch stream.  No CPU fallback exists: CPU tensors or a missing library
raise.
"""

from __future__ import annotations

import torch

from . import _lib
from .masks import CAUSAL_EXCLUSIVE, CAUSAL_INCLUSIVE, FULLY_MASKED, FULLY_UNMASKED  # noqa: F401

CONTIGUOUS, STRIPED = 0, 1
PARTITION, GATHER = 0, 1


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _need_cuda(name: str, t: torch.Tensor, dtype=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _ptr(t):
    return None if t is None else t.data_ptr()


def _on(t: torch.Tensor):
    """The CUDA runtime launches on the CURRENT device: make it the tensor's."""
    return torch.cuda.device(t.device)


def permute(src: torch.Tensor, dst: torch.Tensor, n_dev: int, scheme: int, direction: int,
            device: int = -1) -> torch.Tensor:
    """K1: Layout.partition / Layout.gather (layout.py:81-117) of whole rows, bit-exact."""
    _need_cuda("src", src)
    _need_cuda("dst", dst)
    if direction == PARTITION:
        n_seq = src.shape[0]
    else:
        n_seq = dst.shape[0]
    row_bytes = src[0].numel() * src.element_size() if src.dim() > 1 else src.element_size()
    with _on(src):
        _lib.check(_lib.lib().sa_permute(src.data_ptr(), dst.data_ptr(), n_seq, n_dev, row_bytes,
                                         scheme, direction, device, _stream(src)), "sa_permute")
    return dst


def fwd_block(q, k, v, o_acc, lse, out, softmax_scale: float, mask_kind: int, first_step: bool,
              last_step: bool, tiles_computed=None):
    """K2+K3: one ring step of the forward (see include/striped_attn.h)."""
    for n, t in (("q", q), ("k", k), ("v", v)):
        _need_cuda(n, t, torch.bfloat16)
    _need_cuda("lse", lse, torch.float32)
    if o_acc is not None:
        _need_cuda("o_acc", o_acc, torch.float32)
    if out is not None:
        _need_cuda("out", out, torch.bfloat16)
    c, hq, d = q.shape
    hkv = k.shape[1]
    if k.shape != (c, hkv, d) or v.shape != (c, hkv, d):
        raise ValueError(f"k/v must be [{c}, hkv, {d}], got {tuple(k.shape)} / {tuple(v.shape)}")
    with _on(q):
        _lib.check(_lib.lib().sa_fwd_block(
            q.data_ptr(), k.data_ptr(), v.data_ptr(), _ptr(o_acc), lse.data_ptr(), _ptr(out), c, hq,
            hkv, d, float(softmax_scale), int(mask_kind), int(first_step), int(last_step),
            _ptr(tiles_computed), _stream(q)), "sa_fwd_block")


def bwd_preprocess(out, dout, dsum, dq_acc):
    _need_cuda("out", out, torch.bfloat16)
    _need_cuda("dout", dout, torch.bfloat16)
    _need_cuda("dsum", dsum, torch.float32)
    _need_cuda("dq_acc", dq_acc, torch.float32)
    c, hq, d = out.shape
    with _on(out):
        _lib.check(_lib.lib().sa_bwd_preprocess(out.data_ptr(), dout.data_ptr(), dsum.data_ptr(),
                                                dq_acc.data_ptr(), c, hq, d, _stream(out)),
                   "sa_bwd_preprocess")


def _sem_ptr(dq_sem, hq, c):
    if dq_sem is None:
        return None
    if not (isinstance(dq_sem, torch.Tensor) and dq_sem.is_cuda and dq_sem.dtype == torch.int32):
        raise ValueError("dq_sem must be a CUDA int32 tensor")
    if dq_sem.numel() < hq * ((c + 63) // 64):
        raise ValueError(f"dq_sem needs hq * ceil(c / 64) = {hq * ((c + 63) // 64)} entries")
    return dq_sem.data_ptr()


def bwd_block(q, k, v, dout, lse, dsum, dq_acc, dk_acc, dv_acc, softmax_scale: float,
              mask_kind: int, key_rows=None, dq_sem=None):
    """K5: one ring step of the backward (accumulates into dq_acc / dk_acc / dv_acc);
    ``key_rows=(r0, r1)`` restricts it to those held-stripe keys (sa_bwd_block_range);
    ``dq_sem`` (zeroed int32 [hq * ceil(c/64)]) makes the dQ reduction deterministic."""
    for n, t in (("q", q), ("k", k), ("v", v), ("dout", dout)):
        _need_cuda(n, t, torch.bfloat16)
    for n, t in (("lse", lse), ("dsum", dsum), ("dq_acc", dq_acc), ("dk_acc", dk_acc),
                 ("dv_acc", dv_acc)):
        _need_cuda(n, t, torch.float32)
    c, hq, d = q.shape
    hkv = k.shape[1]
    with _on(q):
        if dq_sem is not None:
            r0, r1 = key_rows if key_rows is not None else (0, c)
            _lib.check(_lib.lib().sa_bwd_block_ex(
                q.data_ptr(), k.data_ptr(), v.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                dsum.data_ptr(), dq_acc.data_ptr(), dk_acc.data_ptr(), dv_acc.data_ptr(), None,
                None, c, hq, hkv, d, float(softmax_scale), int(mask_kind), int(r0), int(r1),
                _sem_ptr(dq_sem, hq, c), _stream(q)), "sa_bwd_block_ex")
        elif key_rows is None:
            _lib.check(_lib.lib().sa_bwd_block(
                q.data_ptr(), k.data_ptr(), v.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                dsum.data_ptr(), dq_acc.data_ptr(), dk_acc.data_ptr(), dv_acc.data_ptr(), c, hq,
                hkv, d, float(softmax_scale), int(mask_kind), _stream(q)), "sa_bwd_block")
        else:
            _lib.check(_lib.lib().sa_bwd_block_range(
                q.data_ptr(), k.data_ptr(), v.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                dsum.data_ptr(), dq_acc.data_ptr(), dk_acc.data_ptr(), dv_acc.data_ptr(), c, hq,
                hkv, d, float(softmax_scale), int(mask_kind), int(key_rows[0]),
                int(key_rows[1]), _stream(q)), "sa_bwd_block_range")


def bwd_block_final(q, k, v, dout, lse, dsum, dq_acc, dk, dv, softmax_scale: float,
                    mask_kind: int, dq_sem=None):
    """K5 for a block that is the only contribution to dK / dV: dk / dv (bf16 [c, Hkv, D])
    are written, not accumulated (sa_bwd_block_final; sa_bwd_block_ex with ``dq_sem``)."""
    for n, t in (("q", q), ("k", k), ("v", v), ("dout", dout), ("dk", dk), ("dv", dv)):
        _need_cuda(n, t, torch.bfloat16)
    for n, t in (("lse", lse), ("dsum", dsum), ("dq_acc", dq_acc)):
        _need_cuda(n, t, torch.float32)
    c, hq, d = q.shape
    hkv = k.shape[1]
    with _on(q):
        if dq_sem is not None:
            _lib.check(_lib.lib().sa_bwd_block_ex(
                q.data_ptr(), k.data_ptr(), v.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                dsum.data_ptr(), dq_acc.data_ptr(), None, None, dk.data_ptr(), dv.data_ptr(), c,
                hq, hkv, d, float(softmax_scale), int(mask_kind), 0, int(c),
                _sem_ptr(dq_sem, hq, c), _stream(q)), "sa_bwd_block_ex")
            return
        _lib.check(_lib.lib().sa_bwd_block_final(
            q.data_ptr(), k.data_ptr(), v.data_ptr(), dout.data_ptr(), lse.data_ptr(),
            dsum.data_ptr(), dq_acc.data_ptr(), dk.data_ptr(), dv.data_ptr(), c, hq, hkv, d,
            float(softmax_scale), int(mask_kind), _stream(q)), "sa_bwd_block_final")


def cast_f32_bf16(src: torch.Tensor, dst: torch.Tensor) -> torch.Tensor:
    _need_cuda("src", src, torch.float32)
    _need_cuda("dst", dst, torch.bfloat16)
    if src.numel() != dst.numel():
        raise ValueError("cast size mismatch")
    with _on(src):
        _lib.check(_lib.lib().sa_cast_f32_bf16(src.data_ptr(), dst.data_ptr(), src.numel(),
                                               _stream(src)), "sa_cast_f32_bf16")
    return dst
