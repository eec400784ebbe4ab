"""Ring driver: the N-round rotation of Algorithm 1 over real ranks (or one device).

Mirrors the reference's schedule (simulator.py:189-234): every rank keeps its query
stripe resident, runs the block op against the key/value stripe it holds -- held index
``(j - i) mod N`` at round i (simulator.py:115-117) -- then forwards that stripe to
``j + 1`` and receives from ``j - 1``.  The reference swaps Python references
(_run_serial, 194-197) or passes them through ordered queues (_run_threads, 211-215);
here the hop is a point-to-point transfer over NVLink issued on a side stream and
double-buffered, so round i+1's K/V arrive while round i computes.

Backward (no reference counterpart): fp32 dK/dV accumulators ride with their K/V
stripe and arrive home after N hops; dQ accumulates locally.

Block ops are pluggable (``BlockOps``): the default is the CUDA library
(``ops.py``); CPU tests inject an oracle-backed implementation to test this host logic
over ``gloo`` without a GPU.
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from . import masks


class BlockOps:
    """Per-step compute used by the driver (CUDA library by default)."""

    def __init__(self):
        from . import ops as _ops
        self._ops = _ops

    def fwd_block(self, q, k, v, o_acc, lse, out, scale, kind, first, last, tiles=None):
        self._ops.fwd_block(q, k, v, o_acc, lse, out, scale, kind, first, last, tiles)

    def bwd_preprocess(self, out, dout, dsum, dq_acc):
        self._ops.bwd_preprocess(out, dout, dsum, dq_acc)

    def bwd_block(self, q, k, v, dout, lse, dsum, dq_acc, dk_acc, dv_acc, scale, kind,
                  key_rows=None):
        self._ops.bwd_block(q, k, v, dout, lse, dsum, dq_acc, dk_acc, dv_acc, scale, kind,
                            key_rows)

    def bwd_block_final(self, q, k, v, dout, lse, dsum, dq_acc, dk, dv, scale, kind):
        """Single-step backward: bf16 dK / dV written directly (no accumulators / casts)."""
        self._ops.bwd_block_final(q, k, v, dout, lse, dsum, dq_acc, dk, dv, scale, kind)

    def cast(self, src, dst):
        self._ops.cast_f32_bf16(src, dst)


@dataclass
class StepRecord:
    """Per-(rank, round) telemetry: block held, mask kind, tiles, CUDA-event times."""
    round: int
    block_index: int
    mask_kind: int
    tiles_computed: int = 0
    compute_ms: float = 0.0


@dataclass
class RingStats:
    rank: int
    rounds: list = field(default_factory=list)


class _Comm:
    """Point-to-point neighbour exchange for one ring hop (torch.distributed P2P)."""

    def __init__(self, group):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.next = dist.get_global_rank(group, (self.rank + 1) % self.world) if group is not None \
            else (self.rank + 1) % self.world
        self.prev = dist.get_global_rank(group, (self.rank - 1) % self.world) if group is not None \
            else (self.rank - 1) % self.world

    def exchange(self, send, recv):
        ops = []
        for s, r in zip(send, recv):
            ops.append(dist.P2POp(dist.isend, s, self.next, self.group))
            ops.append(dist.P2POp(dist.irecv, r, self.prev, self.group))
        # even ranks send first, odd ranks receive first (deadlock-free on any backend)
        if self.rank % 2:
            ops = [o for pair in zip(ops[1::2], ops[0::2]) for o in pair]
        return dist.batch_isend_irecv(ops)


def _is_cuda(t):
    return t.is_cuda


class _Streams:
    """Compute on the current stream, hops on a side stream (CUDA); no-ops on CPU."""

    def __init__(self, ref: torch.Tensor):
        self.cuda = _is_cuda(ref)
        if self.cuda:
            self.compute = torch.cuda.current_stream(ref.device)
            self.comm = torch.cuda.Stream(device=ref.device)

    def on_comm(self):
        return torch.cuda.stream(self.comm) if self.cuda else contextlib.nullcontext()

    def comm_after_compute(self):
        if self.cuda:
            self.comm.wait_stream(self.compute)

    def compute_after_comm(self):
        if self.cuda:
            self.compute.wait_stream(self.comm)

    def _event(self, stream):
        if not self.cuda:
            return None
        e = torch.cuda.Event()
        e.record(stream)
        return e

    def compute_event(self):
        return self._event(self.compute) if self.cuda else None

    def comm_event(self):
        return self._event(self.comm) if self.cuda else None

    def compute_waits(self, ev):
        if ev is not None:
            self.compute.wait_event(ev)

    def comm_waits(self, ev):
        if ev is not None:
            self.comm.wait_event(ev)


def kv_parts(c: int, tile: int = 128) -> list:
    """Row ranges of the held stripe's keys, in launch order, for the backward's
    pipelined dK/dV hop: the upper half first (cheapest per row under a causal mask), then
    the next quarter, the lowest quarter last, so the exposed hop is a quarter of the rows.
    Blocks of fewer than 4 key tiles run in one part."""
    nt = -(-c // tile)
    if nt < 4:
        return [(0, c)]
    b1, b2 = nt // 4, nt // 2
    rows = lambda t: min(c, t * tile)
    return [(rows(b2), c), (rows(b1), rows(b2)), (0, rows(b1))]


class Workspace:
    """Reusable device buffers for ring_forward / ring_backward: with a workspace the
    calls allocate nothing (outputs are views into it, valid until the next call that
    uses the same workspace)."""

    def __init__(self):
        self._bufs = {}

    def get(self, name, shape, dtype, device, zero=False):
        n = 1
        for x in shape:
            n *= int(x)
        t = self._bufs.get(name)
        if t is None or t.numel() < n or t.dtype != dtype or t.device != torch.device(device):
            if t is not None and t.is_cuda:
                # growing: the old buffer may still be in use on any stream
                torch.cuda.synchronize(t.device)
            t = torch.empty(max(n, 1), dtype=dtype, device=device)
            self._bufs[name] = t
        v = t[:n].view(*shape)
        if zero:
            v.zero_()
        return v


def _alloc(ws, name, shape, dtype, device, zero=False):
    if ws is not None:
        return ws.get(name, shape, dtype, device, zero)
    return (torch.zeros if zero else torch.empty)(*shape, dtype=dtype, device=device)


class _StepTimer:
    """CUDA-event time of each round's block kernel on the compute stream (telemetry)."""

    def __init__(self, ref: torch.Tensor, enabled: bool):
        self.on = enabled and _is_cuda(ref)
        self.events = []

    def start(self):
        if self.on:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.events.append([e, None])

    def stop(self):
        if self.on:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.events[-1][1] = e

    def fill(self, records):
        """Write the measured ms into the last len(events) StepRecords."""
        if not self.on or not self.events:
            return
        self.events[-1][1].synchronize()
        for rec, (a, b) in zip(records[-len(self.events):], self.events):
            rec.compute_ms = a.elapsed_time(b)


def ring_forward(q, k, v, *, group=None, layout: str = "striped", softmax_scale: float,
                 block_ops: BlockOps | None = None, stats: RingStats | None = None,
                 count_tiles: bool = False, workspace: Workspace | None = None):
    """Forward for this rank's stripe.  q [c,Hq,D], k/v [c,Hkv,D] (bf16 on GPU).

    Returns (out [c,Hq,D] bf16, lse [Hq,c] fp32) in local (permuted) order, like
    run_schedule's outputs (simulator.py:237-277)."""
    bops = block_ops or BlockOps()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    c, hq, d = q.shape
    ws = workspace
    out = _alloc(ws, "out", (c, hq, d), q.dtype, q.device)
    lse = _alloc(ws, "lse", (hq, c), torch.float32, q.device)
    o_acc = None if world == 1 else _alloc(ws, "o_acc", (c, hq, d), torch.float32, q.device)
    tiles = torch.zeros(1, device=q.device, dtype=torch.int64) if count_tiles else None
    timer = _StepTimer(q, stats is not None)
    if world == 1:
        kind = masks.block_mask(layout, 0, 0, 1)
        timer.start()
        bops.fwd_block(q, k, v, None, lse, out, softmax_scale, kind, True, True, tiles)
        timer.stop()
        if stats is not None:
            stats.rounds.append(StepRecord(0, 0, int(kind),
                                           int(tiles.item()) if tiles is not None else 0))
            timer.fill(stats.rounds)
        return out, lse
    comm = _Comm(group)
    st = _Streams(q)
    bufs = [(_alloc(ws, f"kbuf{b}", k.shape, k.dtype, k.device),
             _alloc(ws, f"vbuf{b}", v.shape, v.dtype, v.device)) for b in range(2)]
    cur = (k, v)
    for i in range(world):
        held = (rank - i) % world
        pending = None
        nxt = bufs[i % 2]
        if i < world - 1:
            st.comm_after_compute()  # nxt's previous reader (round i-1) has finished
            with st.on_comm():
                pending = comm.exchange(list(cur), list(nxt))
        kind = masks.block_mask(layout, rank, held, world)
        before = int(tiles.item()) if (tiles is not None and stats is not None) else 0
        timer.start()
        bops.fwd_block(q, cur[0], cur[1], o_acc, lse, out, softmax_scale, kind, i == 0,
                       i == world - 1, tiles)
        timer.stop()
        if stats is not None:
            after = int(tiles.item()) if tiles is not None else 0
            stats.rounds.append(StepRecord(i, held, int(kind), after - before))
        if pending is not None:
            with st.on_comm():
                for w in pending:
                    w.wait()
            st.compute_after_comm()
            cur = nxt
    if stats is not None:
        timer.fill(stats.rounds)
    return out, lse


def ring_backward(dout, q, k, v, out, lse, *, group=None, layout: str = "striped",
                  softmax_scale: float, block_ops: BlockOps | None = None,
                  stats: RingStats | None = None, workspace: Workspace | None = None):
    """Backward for this rank's stripe -> (dq, dk, dv) bf16 in local order.

    K/V hop one rank per round (prefetched on the side stream); the fp32 dK/dV
    accumulators of the held stripe hop after each round's compute and are home
    after N hops."""
    bops = block_ops or BlockOps()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    c, hq, d = q.shape
    hkv = k.shape[1]
    dev = q.device
    ws = workspace
    dsum = _alloc(ws, "dsum", (hq, c), torch.float32, dev)
    dq_acc = _alloc(ws, "dq_acc", (c, hq, d), torch.float32, dev)
    bops.bwd_preprocess(out, dout, dsum, dq_acc)
    timer = _StepTimer(q, stats is not None)
    if world == 1 and hasattr(bops, "bwd_block_final"):
        # one step: dK / dV come out of the kernel as bf16 (no fp32 accumulators / casts)
        kind = masks.block_mask(layout, 0, 0, 1)
        dk = _alloc(ws, "dk", k.shape, k.dtype, dev)
        dv = _alloc(ws, "dv", v.shape, v.dtype, dev)
        timer.start()
        bops.bwd_block_final(q, k, v, dout, lse, dsum, dq_acc, dk, dv, softmax_scale, kind)
        timer.stop()
        if stats is not None:
            stats.rounds.append(StepRecord(0, 0, int(kind)))
            timer.fill(stats.rounds)
        dq = _alloc(ws, "dq", q.shape, q.dtype, dev)
        bops.cast(dq_acc, dq)
        return dq, dk, dv
    dk_acc = _alloc(ws, "dk_acc", (c, hkv, d), torch.float32, dev, zero=True)
    dv_acc = _alloc(ws, "dv_acc", (c, hkv, d), torch.float32, dev, zero=True)
    if world == 1:
        kind = masks.block_mask(layout, 0, 0, 1)
        timer.start()
        bops.bwd_block(q, k, v, dout, lse, dsum, dq_acc, dk_acc, dv_acc, softmax_scale, kind)
        timer.stop()
        if stats is not None:
            stats.rounds.append(StepRecord(0, 0, int(kind)))
    else:
        comm = _Comm(group)
        st = _Streams(q)
        kv_bufs = [(_alloc(ws, f"bkbuf{b}", k.shape, k.dtype, dev),
                    _alloc(ws, f"bvbuf{b}", v.shape, v.dtype, dev)) for b in range(2)]
        dkv_bufs = [(_alloc(ws, "dk_spare", dk_acc.shape, torch.float32, dev),
                     _alloc(ws, "dv_spare", dv_acc.shape, torch.float32, dev))]
        cur = (k, v)
        dcur = (dk_acc, dv_acc)
        dspare = dkv_bufs[0]
        # the block runs in parts over the held stripe's keys; each part's dK/dV rows hop
        # to the next rank while the later parts compute (the last, smallest part's hop is
        # the only one between rounds)
        parts = kv_parts(c)
        arrived = [None] * len(parts)  # comm-stream events: part p of dcur has arrived
        for i in range(world):
            held = (rank - i) % world
            pending = None
            nxt = kv_bufs[i % 2]
            kv_ready = None
            if i < world - 1:
                st.comm_after_compute()  # nxt's previous reader (round i-1) has finished
                with st.on_comm():
                    pending = comm.exchange(list(cur), list(nxt))
                    for w in pending:
                        w.wait()
                kv_ready = st.comm_event()
            kind = masks.block_mask(layout, rank, held, world)
            timer.start()
            sent = [None] * len(parts)
            for pi, (r0, r1) in enumerate(parts):
                st.compute_waits(arrived[pi])  # this part's accumulator rows are here
                bops.bwd_block(q, cur[0], cur[1], dout, lse, dsum, dq_acc, dcur[0], dcur[1],
                               softmax_scale, kind, key_rows=(r0, r1))
                done = st.compute_event()
                with st.on_comm():
                    st.comm_waits(done)
                    works = comm.exchange([dcur[0][r0:r1], dcur[1][r0:r1]],
                                          [dspare[0][r0:r1], dspare[1][r0:r1]])
                    for w in works:
                        w.wait()
                sent[pi] = st.comm_event()
            timer.stop()
            if stats is not None:
                stats.rounds.append(StepRecord(i, held, int(kind)))
            arrived = sent
            dcur, dspare = dspare, dcur
            st.compute_waits(kv_ready)
            if pending is not None:
                cur = nxt
        for ev in arrived:  # the accumulators are home after the N-th hop
            st.compute_waits(ev)
        dk_acc, dv_acc = dcur
    if stats is not None:
        timer.fill(stats.rounds)
    dq = _alloc(ws, "dq", q.shape, q.dtype, dev)
    dk = _alloc(ws, "dk", k.shape, k.dtype, dev)
    dv = _alloc(ws, "dv", v.shape, v.dtype, dev)
    bops.cast(dq_acc, dq)
    bops.cast(dk_acc, dk)
    bops.cast(dv_acc, dv)
    return dq, dk, dv


def virtual_ring_forward(qs, ks, vs, *, layout: str = "striped", softmax_scale: float,
                         block_ops: BlockOps | None = None, count_tiles: bool = False):
    """All N ranks' stripes on ONE device, rounds in order (the reference's serial
    executor, simulator.py:189-198).  Same kernels and merge as the distributed path."""
    bops = block_ops or BlockOps()
    n = len(qs)
    c, hq, d = qs[0].shape
    outs = [torch.empty_like(x) for x in qs]
    lses = [torch.empty(hq, c, device=x.device, dtype=torch.float32) for x in qs]
    accs = [None if n == 1 else torch.empty(c, hq, d, device=x.device, dtype=torch.float32)
            for x in qs]
    stats = [RingStats(j) for j in range(n)]
    tiles = torch.zeros(1, device=qs[0].device, dtype=torch.int64) if count_tiles else None
    for i in range(n):
        for j in range(n):
            held = (j - i) % n
            kind = masks.block_mask(layout, j, held, n)
            before = int(tiles.item()) if tiles is not None else 0
            bops.fwd_block(qs[j], ks[held], vs[held], accs[j], lses[j], outs[j], softmax_scale,
                           kind, i == 0, i == n - 1, tiles)
            after = int(tiles.item()) if tiles is not None else 0
            stats[j].rounds.append(StepRecord(i, held, int(kind), after - before))
    return outs, lses, stats


def virtual_ring_backward(douts, qs, ks, vs, outs, lses, *, layout: str = "striped",
                          softmax_scale: float, block_ops: BlockOps | None = None):
    """Backward over all N stripes on one device; dK/dV accumulators stay with their
    stripe (index ``held``), exactly what the travelling buffers compute."""
    bops = block_ops or BlockOps()
    n = len(qs)
    c, hq, d = qs[0].shape
    dev = qs[0].device
    dsums = [torch.empty(hq, c, device=dev, dtype=torch.float32) for _ in range(n)]
    dqs = [torch.empty(c, hq, d, device=dev, dtype=torch.float32) for _ in range(n)]
    for j in range(n):
        bops.bwd_preprocess(outs[j], douts[j], dsums[j], dqs[j])
    dks = [torch.zeros(k.shape, device=dev, dtype=torch.float32) for k in ks]
    dvs = [torch.zeros(v.shape, device=dev, dtype=torch.float32) for v in vs]
    for i in range(n):
        for j in range(n):
            held = (j - i) % n
            kind = masks.block_mask(layout, j, held, n)
            bops.bwd_block(qs[j], ks[held], vs[held], douts[j], lses[j], dsums[j], dqs[j],
                           dks[held], dvs[held], softmax_scale, kind)
    res = []
    for acc, like in ((dqs, qs), (dks, ks), (dvs, vs)):
        outl = []
        for a, x in zip(acc, like):
            o = torch.empty_like(x)
            bops.cast(a, o)
            outl.append(o)
        res.append(outl)
    return tuple(res)
