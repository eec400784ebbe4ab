"""Public API: striped / ring causal attention forward + backward on sharded Q/K/V.

The drop-in for the reference's hot path (ringsim: simulate / run_schedule,
simulator.py:237-277, 358-368).  Each rank passes its local stripe (rows already in
the layout's order -- see ``stripe_permute``) and gets back O and LSE for those rows,
and dQ/dK/dV in the backward.  bf16 in/out, fp32 accumulation, CUDA only.

    out, lse = striped_attn_forward(q, k, v, group=pg, layout="striped")
    dq, dk, dv = striped_attn_backward(dout, q, k, v, out, lse, group=pg)
    out = striped_attention(q, k, v, group=pg)          # autograd

Shapes: q [c, Hq, D], k/v [c, Hkv, D] (Hq % Hkv == 0, D in {64, 128}); an optional
leading batch dim is looped.  lse is [Hq, c] fp32 natural-log.  ``softmax_scale``
defaults to 1/sqrt(D) (the reference's ``scale=True``, attention.py:137-138).
"""

from __future__ import annotations

import math

import torch
import torch.distributed as dist

from . import ring
from .layout import Layout, Scheme

LAYOUTS = ("striped", "ring")


def _check(q, k, v, layout):
    if layout not in LAYOUTS:
        raise ValueError(f"layout must be one of {LAYOUTS}, got {layout!r}")
    for name, t in (("q", q), ("k", k), ("v", v)):
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (there is no CPU fallback)")
        if t.dtype != torch.bfloat16:
            raise ValueError(f"{name} must be bfloat16, got {t.dtype}")
    if q.dim() != k.dim() or q.dim() not in (3, 4):
        raise ValueError("q/k/v must be [c, H, D] or [B, c, H, D]")
    if k.shape != v.shape or q.shape[:-2] != k.shape[:-2] or q.shape[-1] != k.shape[-1]:
        raise ValueError(f"shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)}")
    if q.shape[-2] % k.shape[-2]:
        raise ValueError("Hq must be a multiple of Hkv")


def _scale(q, softmax_scale):
    return 1.0 / math.sqrt(q.shape[-1]) if softmax_scale is None else float(softmax_scale)


def striped_attn_forward(q, k, v, *, group=None, layout: str = "striped", softmax_scale=None,
                         comm=None):
    """Forward over the ring of ``group`` (default: the world, or one GPU when
    torch.distributed is not initialised).  ``comm``: the ring hop backend
    (``ring.NcclComm`` by default, ``ipc.IpcComm``, ``ring.LocalComm``).  Returns (out, lse)."""
    _check(q, k, v, layout)
    scale = _scale(q, softmax_scale)
    if q.dim() == 4:
        res = [striped_attn_forward(q[b], k[b], v[b], group=group, layout=layout,
                                    softmax_scale=scale, comm=comm) for b in range(q.shape[0])]
        return torch.stack([r[0] for r in res]), torch.stack([r[1] for r in res])
    return ring.ring_forward(q.contiguous(), k.contiguous(), v.contiguous(), group=group,
                             layout=layout, softmax_scale=scale, comm=comm)


def striped_attn_backward(dout, q, k, v, out, lse, *, group=None, layout: str = "striped",
                          softmax_scale=None, deterministic: bool = False, comm=None,
                          fused_dkv: bool = False):
    """Backward -> (dq, dk, dv), bf16, same layout as the inputs.  ``deterministic``:
    bit-identical reruns (ordered dQ reduction; slower).  ``fused_dkv`` (peer-memory comms
    only): no dK/dV hops, every rank's kernel adds into the held stripe's home buffer."""
    _check(q, k, v, layout)
    scale = _scale(q, softmax_scale)
    if q.dim() == 4:
        res = [striped_attn_backward(dout[b], q[b], k[b], v[b], out[b], lse[b], group=group,
                                     layout=layout, softmax_scale=scale,
                                     deterministic=deterministic, comm=comm,
                                     fused_dkv=fused_dkv)
               for b in range(q.shape[0])]
        return tuple(torch.stack([r[i] for r in res]) for i in range(3))
    return ring.ring_backward(dout.contiguous(), q.contiguous(), k.contiguous(), v.contiguous(),
                              out.contiguous(), lse.contiguous(), group=group, layout=layout,
                              softmax_scale=scale, deterministic=deterministic, comm=comm,
                              fused_dkv=fused_dkv)


class StripedAttnFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, group, layout, softmax_scale, deterministic=False, comm=None,
                fused_dkv=False):
        out, lse = striped_attn_forward(q, k, v, group=group, layout=layout,
                                        softmax_scale=softmax_scale, comm=comm)
        ctx.save_for_backward(q, k, v, out, lse)
        ctx.group, ctx.layout, ctx.softmax_scale = group, layout, softmax_scale
        ctx.deterministic, ctx.comm, ctx.fused_dkv = deterministic, comm, fused_dkv
        return out

    @staticmethod
    def backward(ctx, dout):
        q, k, v, out, lse = ctx.saved_tensors
        dq, dk, dv = striped_attn_backward(dout.contiguous(), q, k, v, out, lse, group=ctx.group,
                                           layout=ctx.layout, softmax_scale=ctx.softmax_scale,
                                           deterministic=ctx.deterministic, comm=ctx.comm,
                                           fused_dkv=ctx.fused_dkv)
        return dq, dk, dv, None, None, None, None, None, None


def striped_attention(q, k, v, group=None, layout: str = "striped", softmax_scale=None,
                      deterministic: bool = False, comm=None, fused_dkv: bool = False):
    """Autograd entry point: returns O for this rank's stripe."""
    return StripedAttnFunction.apply(q, k, v, group, layout, softmax_scale, deterministic, comm,
                                     fused_dkv)


def ring_attention(q, k, v, group=None, softmax_scale=None, comm=None):
    """Contiguous-layout baseline (the ring the paper compares against)."""
    return StripedAttnFunction.apply(q, k, v, group, "ring", softmax_scale, False, comm, False)


def stripe_permute(x: torch.Tensor, n_devices: int, layout: str = "striped",
                   device: int | None = None) -> torch.Tensor:
    """Token order -> stripe order (Layout.partition, layout.py:81-101), applied once
    before the first layer.  ``device`` selects one rank's shard."""
    lay = Layout(Scheme.STRIPED if layout == "striped" else Scheme.CONTIGUOUS, x.shape[0],
                 n_devices)
    return lay.permute(x) if device is None else lay.shard(x, device)


def stripe_unpermute(x: torch.Tensor, n_devices: int, layout: str = "striped") -> torch.Tensor:
    """Exact inverse of ``stripe_permute`` (Layout.gather, layout.py:103-117)."""
    lay = Layout(Scheme.STRIPED if layout == "striped" else Scheme.CONTIGUOUS, x.shape[0],
                 n_devices)
    return lay.unpermute(x)


def world_info(group=None):
    if dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1
