"""Host-resident tensors through the GPU path: head groups streamed with copy/compute overlap.

``attention_fwd_bwd_host`` takes this rank's stripe as pinned HOST tensors (token-major
``[c, H, D]`` bf16, exactly what the device API takes) and returns O, LSE and dQ/dK/dV in
caller-provided pinned host buffers.  Heads are independent, so the work is split into
head groups: the host->device copy of group g+1 and the device->host copy of group g-1
run on their own streams (the two PCIe directions and the copy engines work in parallel)
while the kernels of group g run on the compute stream.  One group's strided slice of a
token-major tensor is moved with a single 2-D DMA (``sa_memcpy2d_async``), no host gather.

The kernels, ring driver and numerics are the same as ``api.striped_attn_forward`` /
``striped_attn_backward`` (called per group, so a ring runs per group under
torch.distributed).
"""

from __future__ import annotations

import math

import torch

from . import _lib, ring


def _copy2d(dst: torch.Tensor, src: torch.Tensor, heads: slice, to_device: bool,
            stream: torch.cuda.Stream):
    """dst[:, :, :] <-> src[:, heads, :] (to_device) or dst[:, heads, :] <- src (to host)."""
    if to_device:
        c, h_all, d = src.shape
        esz = src.element_size()
        width = (heads.stop - heads.start) * d * esz
        src_ptr = src.data_ptr() + heads.start * d * esz
        _lib.check(_lib.lib().sa_memcpy2d_async(dst.data_ptr(), width, src_ptr, h_all * d * esz,
                                                width, c, stream.cuda_stream), "sa_memcpy2d_async")
    else:
        c, h_all, d = dst.shape
        esz = dst.element_size()
        width = (heads.stop - heads.start) * d * esz
        dst_ptr = dst.data_ptr() + heads.start * d * esz
        _lib.check(_lib.lib().sa_memcpy2d_async(dst_ptr, h_all * d * esz, src.data_ptr(), width,
                                                width, c, stream.cuda_stream), "sa_memcpy2d_async")


def attention_fwd_bwd_host(q, k, v, dout, out, lse, dq, dk, dv, *, group=None,
                           layout: str = "striped", softmax_scale=None, head_groups: int = 4,
                           device=None):
    """Forward + backward of this rank's stripe from/to pinned host memory.

    q, dout, out, dq: [c, Hq, D] bf16 pinned; k, v, dk, dv: [c, Hkv, D] bf16 pinned;
    lse: [Hq, c] fp32 pinned.  Returns an event recorded when every result is in host
    memory (the caller synchronises on it)."""
    for name, t in (("q", q), ("k", k), ("v", v), ("dout", dout), ("out", out), ("dq", dq),
                    ("dk", dk), ("dv", dv), ("lse", lse)):
        if t.is_cuda or not t.is_pinned() or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous pinned host tensor")
    c, hq, d = q.shape
    hkv = k.shape[1]
    if hq % head_groups or hkv % head_groups:
        raise ValueError(f"head_groups={head_groups} must divide Hq={hq} and Hkv={hkv}")
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else float(softmax_scale)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    gq, gk = hq // head_groups, hkv // head_groups
    compute = torch.cuda.current_stream(dev)
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def slot():
        mk = lambda h: torch.empty(c, h, d, device=dev, dtype=torch.bfloat16)
        return {"q": mk(gq), "k": mk(gk), "v": mk(gk), "do": mk(gq)}

    slots = [slot(), slot()]
    freed = [None, None]  # event: the slot's inputs are no longer read by compute
    results = []
    for g in range(head_groups):
        s = slots[g % 2]
        hs_q = slice(g * gq, (g + 1) * gq)
        hs_k = slice(g * gk, (g + 1) * gk)
        if freed[g % 2] is not None:
            h2d.wait_event(freed[g % 2])
        _copy2d(s["q"], q, hs_q, True, h2d)
        _copy2d(s["k"], k, hs_k, True, h2d)
        _copy2d(s["v"], v, hs_k, True, h2d)
        _copy2d(s["do"], dout, hs_q, True, h2d)
        loaded = torch.cuda.Event()
        loaded.record(h2d)
        compute.wait_event(loaded)
        o_g, lse_g = ring.ring_forward(s["q"], s["k"], s["v"], group=group, layout=layout,
                                       softmax_scale=scale)
        dq_g, dk_g, dv_g = ring.ring_backward(s["do"], s["q"], s["k"], s["v"], o_g, lse_g,
                                              group=group, layout=layout, softmax_scale=scale)
        done = torch.cuda.Event()
        done.record(compute)
        freed[g % 2] = done
        d2h.wait_event(done)
        _copy2d(out, o_g, hs_q, False, d2h)
        _copy2d(dq, dq_g, hs_q, False, d2h)
        _copy2d(dk, dk_g, hs_k, False, d2h)
        _copy2d(dv, dv_g, hs_k, False, d2h)
        with torch.cuda.stream(d2h):
            lse[hs_q].copy_(lse_g, non_blocking=True)  # [gq, c] rows are contiguous
        # keep the group's device results alive until their copies are issued/finished
        for t in (o_g, lse_g, dq_g, dk_g, dv_g):
            t.record_stream(d2h)
        results.append((o_g, lse_g, dq_g, dk_g, dv_g))
    finished = torch.cuda.Event()
    finished.record(d2h)
    for sl in slots:
        for t in sl.values():
            t.record_stream(h2d)
    return finished
