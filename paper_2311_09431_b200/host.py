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


def ramp_groups(hq: int, hkv: int, max_groups: int = 16) -> list:
    """Head-group sizes (q heads) for streaming: small groups first and last, so only a
    small H2D before the first kernel and a small D2H after the last one are exposed,
    large groups in the middle.  Every size is a multiple of Hq/Hkv (whole kv heads)."""
    r = hq // hkv
    units = hkv  # in kv heads
    lo, hi, step = [], [], 1
    while units >= 2 * step and len(lo) + len(hi) + 2 <= max_groups:
        lo.append(step)
        hi.append(step)
        units -= 2 * step
        step *= 2
    if units:
        if lo:
            lo[-1] += units
        else:
            lo = [units]
    sizes = lo + hi[::-1]
    return [x * r for x in sizes]


def attention_fwd_bwd_host(q, k, v, dout, out, lse, dq, dk, dv, *, group=None,
                           layout: str = "striped", softmax_scale=None, head_groups=4,
                           device=None, comm=None):
    """Forward + backward of this rank's stripe from/to pinned host memory.

    q, dout, out, dq: [c, Hq, D] bf16 pinned; k, v, dk, dv: [c, Hkv, D] bf16 pinned;
    lse: [Hq, c] fp32 pinned.  ``head_groups``: an int (equal groups) or a list of q-head
    counts per group (each a multiple of Hq/Hkv, summing to Hq; see ``ramp_groups``).
    Returns an event recorded when every result is in host memory (the caller
    synchronises on it)."""
    for name, t in (("q", q), ("k", k), ("v", v), ("dout", dout), ("out", out), ("dq", dq),
                    ("dk", dk), ("dv", dv), ("lse", lse)):
        if t.is_cuda or not t.is_pinned() or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous pinned host tensor")
    c, hq, d = q.shape
    hkv = k.shape[1]
    r = hq // hkv
    if isinstance(head_groups, int):
        if head_groups < 1 or hq % head_groups or hkv % head_groups:
            raise ValueError(f"head_groups={head_groups} must divide Hq={hq} and Hkv={hkv}")
        sizes = [hq // head_groups] * head_groups
    else:
        sizes = [int(x) for x in head_groups]
        if sum(sizes) != hq or any(x <= 0 or x % r for x in sizes):
            raise ValueError(f"head group sizes {sizes} must be multiples of Hq/Hkv={r} "
                             f"summing to Hq={hq}")
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else float(softmax_scale)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else \
        torch.device(device)
    with torch.cuda.device(dev):  # copies and kernels go to the current device
        return _stream_groups(q, k, v, dout, out, lse, dq, dk, dv, sizes, r, c, d, scale, dev,
                              group, layout, comm)


def _stream_groups(q, k, v, dout, out, lse, dq, dk, dv, sizes, r, c, d, scale, dev, group,
                   layout, comm=None):
    st = _streamer(dev)
    compute = torch.cuda.current_stream(dev)
    h2d, d2h = st.h2d, st.d2h
    q0 = 0
    for g, gq in enumerate(sizes):
        b = g % 2
        gk = gq // r
        hs_q = slice(q0, q0 + gq)
        hs_k = slice(q0 // r, q0 // r + gk)
        q0 += gq
        # slot b's inputs were last read by the compute of group g-2 (or the previous call)
        if st.freed[b] is not None:
            h2d.wait_event(st.freed[b])
        sl = st.slots[b]
        s = {"q": sl.get("q", (c, gq, d), torch.bfloat16, dev),
             "k": sl.get("k", (c, gk, d), torch.bfloat16, dev),
             "v": sl.get("v", (c, gk, d), torch.bfloat16, dev),
             "do": sl.get("do", (c, gq, d), torch.bfloat16, dev)}
        # forward inputs first: the forward starts while dO is still on the wire
        _copy2d(s["q"], q, hs_q, True, h2d)
        _copy2d(s["k"], k, hs_k, True, h2d)
        _copy2d(s["v"], v, hs_k, True, h2d)
        fwd_in = torch.cuda.Event()
        fwd_in.record(h2d)
        _copy2d(s["do"], dout, hs_q, True, h2d)
        bwd_in = torch.cuda.Event()
        bwd_in.record(h2d)
        compute.wait_event(fwd_in)
        # workspace b's results were last read by the D2H copies of group g-2
        if st.copied[b] is not None:
            compute.wait_event(st.copied[b])
        ws = st.work[b]
        o_g, lse_g = ring.ring_forward(s["q"], s["k"], s["v"], group=group, layout=layout,
                                       softmax_scale=scale, workspace=ws, comm=comm)
        fwd_done = torch.cuda.Event()
        fwd_done.record(compute)
        compute.wait_event(bwd_in)
        dq_g, dk_g, dv_g = ring.ring_backward(s["do"], s["q"], s["k"], s["v"], o_g, lse_g,
                                              group=group, layout=layout, softmax_scale=scale,
                                              workspace=ws, comm=comm)
        done = torch.cuda.Event()
        done.record(compute)
        st.freed[b] = done
        # O and LSE leave while the backward runs; the gradients once it is done
        d2h.wait_event(fwd_done)
        _copy2d(out, o_g, hs_q, False, d2h)
        with torch.cuda.stream(d2h):
            lse[hs_q].copy_(lse_g, non_blocking=True)  # [gq, c] rows are contiguous
        d2h.wait_event(done)
        _copy2d(dq, dq_g, hs_q, False, d2h)
        _copy2d(dk, dk_g, hs_k, False, d2h)
        _copy2d(dv, dv_g, hs_k, False, d2h)
        copied = torch.cuda.Event()
        copied.record(d2h)
        st.copied[b] = copied
    finished = torch.cuda.Event()
    finished.record(d2h)
    return finished


class _Streamer:
    """Per-device state the streaming API keeps across calls: the two copy streams, two
    input slots and two ring workspaces (allocated once, grown on demand: no per-call
    device allocation, hence no allocator synchronisation), and the events ordering
    their reuse across groups and across calls."""

    def __init__(self, dev):
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.slots = [ring.Workspace(), ring.Workspace()]
        self.work = [ring.Workspace(), ring.Workspace()]
        self.freed = [None, None]   # compute finished reading slot b
        self.copied = [None, None]  # D2H finished reading workspace b


_STREAMERS: dict = {}


def _streamer(dev) -> _Streamer:
    key = torch.device(dev).index if torch.device(dev).index is not None else torch.cuda.current_device()
    if key not in _STREAMERS:
        _STREAMERS[key] = _Streamer(dev)
    return _STREAMERS[key]
