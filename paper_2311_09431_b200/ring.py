"""Ring driver: the N-round rotation of Algorithm 1 over real ranks (or one device).

Mirrors the reference's schedule (simulator.py:189-234): every rank keeps its query
stripe resident, runs the block op against the key/value stripe it holds -- held index
``(j - i) mod N`` at round i (simulator.py:115-117) -- then forwards that stripe to
``j + 1`` and receives from ``j - 1``.  The reference swaps Python references
(_run_serial, 194-197) or passes them through ordered queues (_run_threads, 211-215);
here the hop is a point-to-point transfer issued on a side stream and double-buffered,
so round i+1's K/V arrive while round i computes.

The hop itself is pluggable (``Comm``):

* ``NcclComm``  -- torch.distributed P2P (NCCL over NVLink between processes; gloo for
  CPU tensors in the host-logic tests);
* ``LocalComm`` -- ranks as threads of ONE process (several GPUs of a node, or virtual
  ranks sharing one GPU): a copy-engine ``cudaMemcpyAsync`` into the next rank's receive
  buffer, ordered by CUDA events handed over through per-rank FIFO inboxes -- the
  reference's threaded executor (one inbox per device written only by its predecessor,
  30 s stall timeout, simulator.py:201-234) with device buffers instead of references;
* ``IpcComm`` (``ipc.py``) -- one process per GPU, the same protocol over CUDA IPC
  memory / event handles: copy engines instead of NCCL kernels on the SMs.

Backward (no reference counterpart): fp32 dK/dV accumulators ride with their K/V
stripe and arrive home after N hops; dQ accumulates locally.  Each round runs in three
key parts (``kv_parts``: upper half, lower half) and each part's dK/dV rows leave as soon
as that part retires.

Block ops are pluggable (``BlockOps``): the default is the CUDA library (``ops.py``);
CPU tests inject an oracle-backed implementation to test this host logic over ``gloo``
or ``LocalComm`` threads without a GPU.
"""

from __future__ import annotations

import contextlib
import queue
import threading
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from . import masks

STALL_TIMEOUT_S = 30.0  # simulator.py:40 (ring channel stalled)


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
                  key_rows=None, dq_sem=None):
        self._ops.bwd_block(q, k, v, dout, lse, dsum, dq_acc, dk_acc, dv_acc, scale, kind,
                            key_rows, dq_sem)

    def bwd_block_final(self, q, k, v, dout, lse, dsum, dq_acc, dk, dv, scale, kind,
                        dq_sem=None):
        """Single-step backward: bf16 dK / dV written directly (no accumulators / casts)."""
        self._ops.bwd_block_final(q, k, v, dout, lse, dsum, dq_acc, dk, dv, scale, kind,
                                  dq_sem)

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
class HopRecord:
    """One ring hop on a side stream: what moved, how many bytes, its CUDA-event time
    (from the hop's issue on the comm stream to its completion, waits included)."""
    round: int
    what: str  # "kv" | "dkv"
    nbytes: int
    ms: float = 0.0


@dataclass
class RingStats:
    rank: int
    rounds: list = field(default_factory=list)
    hops: list = field(default_factory=list)


# ----------------------------------------------------------------------------- comms
class Comm:
    """Neighbour exchange of one ring hop.  ``exchange(send, recv)``: ``send[i]`` goes to
    the next rank's ``recv[i]`` and ``recv[i]`` is filled from the previous rank's
    ``send[i]``.  For CUDA tensors the transfer is enqueued on the CURRENT stream (its
    completion is stream-ordered, the call does not block on the GPU); CPU tensors are
    exchanged before the call returns."""

    rank: int = 0
    world: int = 1
    name: str = "comm"
    # backends whose ranks can address each other's device memory (LocalComm threads,
    # IpcComm processes) also provide peer_views / sync_all, used by the fused backward
    peer_memory: bool = False

    def exchange(self, send, recv):  # pragma: no cover - interface
        raise NotImplementedError

    def peer_views(self, t: torch.Tensor) -> list:  # pragma: no cover - interface
        """Every rank's tensor ``t`` (same shape / dtype on all ranks), addressable here."""
        raise NotImplementedError

    def sync_all(self, ref: torch.Tensor) -> None:  # pragma: no cover - interface
        """Stream-level barrier: work every rank enqueued before the call precedes work
        any rank enqueues after it (on the current streams)."""
        raise NotImplementedError


class NcclComm(Comm):
    """torch.distributed point-to-point (NCCL between GPUs, gloo for CPU tensors)."""

    name = "nccl"

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        glob = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
        self.next = glob((self.rank + 1) % self.world)
        self.prev = glob((self.rank - 1) % self.world)

    def exchange(self, send, recv):
        ops = []
        for s, r in zip(send, recv):
            ops.append(dist.P2POp(dist.isend, s, self.next, self.group))
            ops.append(dist.P2POp(dist.irecv, r, self.prev, self.group))
        # even ranks send first, odd ranks receive first (deadlock-free on any backend)
        if self.rank % 2:
            ops = [o for pair in zip(ops[1::2], ops[0::2]) for o in pair]
        for w in dist.batch_isend_irecv(ops):
            w.wait()  # NCCL: the current stream waits; gloo: the host waits


class LocalRing:
    """Shared state of ``world`` ranks running as threads of one process.

    Two FIFO inboxes per rank, each written only by one neighbour (the ordered P2P
    channels of simulator.py:201-234): ``ready[j]`` holds the receive buffers rank j+1
    offers for rank j's next send, ``data[j]`` the completion events of the sends into
    rank j's buffers."""

    def __init__(self, world: int, timeout: float = STALL_TIMEOUT_S):
        if world < 1:
            raise ValueError("world must be >= 1")
        self.world = world
        self.timeout = timeout
        self.ready = [queue.Queue() for _ in range(world)]
        self.data = [queue.Queue() for _ in range(world)]
        self.aborted = threading.Event()
        self._shared = {}
        self._barrier = threading.Barrier(world)

    def comm(self, rank: int) -> "LocalComm":
        return LocalComm(self, rank)

    def abort(self):
        self.aborted.set()
        self._barrier.abort()

    def get(self, q: queue.Queue, rank: int):
        waited = 0.0
        while True:
            if self.aborted.is_set():
                raise RuntimeError(f"ring aborted (rank {rank})")
            try:
                return q.get(timeout=0.25)
            except queue.Empty:
                waited += 0.25
                if waited >= self.timeout:
                    self.abort()
                    raise RuntimeError(f"ring channel stalled (rank {rank})")

    def all_gather(self, rank: int, key, value) -> list:
        """Every rank's ``value`` for ``key`` (host objects; blocks until all posted)."""
        slot = self._shared.setdefault(key, [None] * self.world)
        slot[rank] = value
        self._barrier.wait(timeout=self.timeout)
        out = list(slot)
        self._barrier.wait(timeout=self.timeout)
        if rank == 0:
            self._shared.pop(key, None)
        return out


def _record(ref: torch.Tensor):
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(ref.device))
    return ev


def _copy_async(dst: torch.Tensor, src: torch.Tensor):
    """Copy-engine copy on the current stream (peer copy over NVLink across devices)."""
    from . import _lib
    if dst.numel() != src.numel() or dst.dtype != src.dtype:
        raise ValueError("hop buffers differ in size or dtype")
    if not (dst.is_contiguous() and src.is_contiguous()):
        raise ValueError("hop buffers must be contiguous")
    nbytes = src.numel() * src.element_size()
    if nbytes == 0:
        return
    st = torch.cuda.current_stream(src.device).cuda_stream
    _lib.check(_lib.lib().sa_memcpy_async(dst.data_ptr(), src.data_ptr(), nbytes, st),
               "sa_memcpy_async")


class LocalComm(Comm):
    """One rank of a ``LocalRing`` (see there).  Per exchange:
    1. offer my receive buffers to the previous rank, with an event marking the point on
       my stream after which they may be overwritten;
    2. take the next rank's offer, make my stream wait for its event, copy my send
       buffers into its receive buffers (copy engine), record a completion event and
       post it to the next rank;
    3. take the previous rank's completion event and make my stream wait for it.
    Every event is recorded before it is handed over, so no wait can precede its record
    (the enqueued work stays acyclic)."""

    name = "local"
    peer_memory = True

    def __init__(self, ring: LocalRing, rank: int):
        self.ring = ring
        self.rank = rank
        self.world = ring.world
        self.next = (rank + 1) % ring.world
        self.prev = (rank - 1) % ring.world
        self._n = 0  # collective sequence number (every rank calls in the same order)

    def _key(self, what):
        self._n += 1
        return (what, self._n)

    def peer_views(self, t):
        return self.ring.all_gather(self.rank, self._key("views"), t)

    def sync_all(self, ref):
        ev = _record(ref) if ref.is_cuda else None
        evs = self.ring.all_gather(self.rank, self._key("sync"), ev)
        if ref.is_cuda:
            cur = torch.cuda.current_stream(ref.device)
            for j, e in enumerate(evs):
                if j != self.rank:
                    cur.wait_event(e)

    def exchange(self, send, recv):
        r = self.ring
        cuda = recv[0].is_cuda
        r.ready[self.prev].put((list(recv), _record(recv[0]) if cuda else None))
        dst, free = r.get(r.ready[self.rank], self.rank)
        if len(dst) != len(send):
            raise RuntimeError("ring peers disagree on the hop's tensors")
        if cuda:
            torch.cuda.current_stream(send[0].device).wait_event(free)
            for s, d in zip(send, dst):
                _copy_async(d, s)
            done = _record(send[0])
        else:
            for s, d in zip(send, dst):
                d.copy_(s)
            done = None
        r.data[self.next].put(done)
        ev = r.get(r.data[self.rank], self.rank)
        if cuda and ev is not None:
            torch.cuda.current_stream(recv[0].device).wait_event(ev)


def run_local_ring(world: int, fn, devices=None, timeout: float = STALL_TIMEOUT_S):
    """Run ``fn(rank, comm)`` for every rank as a thread of this process (LocalComm).

    ``devices``: the CUDA device of each rank (default: none -- CPU, or whatever ``fn``
    uses).  Each CUDA rank gets its own compute stream.  Returns the per-rank results;
    the first exception of any rank is re-raised after all threads joined
    (simulator.py:221-233)."""
    ring = LocalRing(world, timeout)
    results = [None] * world
    errors = []

    def worker(j):
        try:
            if devices is not None:
                dev = torch.device(devices[j])
                with torch.cuda.device(dev), torch.cuda.stream(torch.cuda.Stream(dev)):
                    results[j] = fn(j, ring.comm(j))
                    torch.cuda.current_stream(dev).synchronize()
            else:
                results[j] = fn(j, ring.comm(j))
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errors.append((j, e))
            ring.abort()

    threads = [threading.Thread(target=worker, args=(j,), daemon=True) for j in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        errors.sort(key=lambda x: isinstance(x[1], RuntimeError) and "aborted" in str(x[1]))
        raise errors[0][1]
    return results


def default_comm(group=None):
    """The comm of ``group`` under torch.distributed, or None (one rank)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        return NcclComm(group)
    return None


# ----------------------------------------------------------------------------- streams
_tls = threading.local()


def _side_streams(device: torch.device):
    """Two persistent side streams per (thread, device): K/V hops and dK/dV hops.  Created
    once (never from the shared pool on each call, which could alias other users'
    streams such as the host API's copy streams)."""
    cache = getattr(_tls, "streams", None)
    if cache is None:
        cache = _tls.streams = {}
    key = device.index
    if key not in cache:
        cache[key] = (torch.cuda.Stream(device=device), torch.cuda.Stream(device=device))
    return cache[key]


class _Streams:
    """Compute on the current stream, hops on side streams (CUDA); no-ops on CPU."""

    def __init__(self, ref: torch.Tensor):
        self.cuda = ref.is_cuda
        self.compute = self.kv = self.dkv = None
        if self.cuda:
            self.compute = torch.cuda.current_stream(ref.device)
            self.kv, self.dkv = _side_streams(ref.device)

    def on(self, stream):
        return torch.cuda.stream(stream) if self.cuda else contextlib.nullcontext()

    def event(self, stream, timing=False):
        if not self.cuda:
            return None
        e = torch.cuda.Event(enable_timing=timing)
        e.record(stream)
        return e

    def wait(self, stream, ev):
        if ev is not None and self.cuda:
            stream.wait_event(ev)


class _HopTimer:
    def __init__(self, st: _Streams, stats):
        self.on = stats is not None and st.cuda
        self.stats = stats
        self.st = st
        self.pending = []

    def start(self, stream):
        return self.st.event(stream, timing=True) if self.on else None

    def stop(self, stream, start, rnd, what, tensors):
        if self.on:
            nbytes = sum(t.numel() * t.element_size() for t in tensors)
            self.pending.append((HopRecord(rnd, what, nbytes), start,
                                 self.st.event(stream, timing=True)))

    def fill(self):
        if not self.on:
            return
        for rec, a, b in self.pending:
            b.synchronize()
            rec.ms = a.elapsed_time(b)
            self.stats.hops.append(rec)


def kv_parts(c: int, tile: int = 128) -> list:
    """Row ranges of the held stripe's keys, in launch order, for the backward's
    pipelined dK/dV hop: the upper half first (a quarter of the work under a causal mask),
    then the lower half.  Round i+1 launches its parts in the same order, so each part's
    accumulator rows have the previous parts' compute time to arrive: no hop is exposed.
    Two parts cost 1.0 % of the block at c = 32k (3 parts -- upper half, next quarter,
    lowest quarter -- cost 2.8 %, `scripts/parts_probe.py`).  Blocks of fewer than 2 key
    tiles run in one part."""
    nt = -(-c // tile)
    if nt < 2:
        return [(0, c)]
    mid = min(c, (nt // 2) * tile)
    return [(mid, c), (0, mid)]


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
        self.on = enabled and ref.is_cuda
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


def _rank_world(group, comm):
    if comm is not None:
        return comm.rank, comm.world
    if dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def ring_forward(q, k, v, *, group=None, layout: str = "striped", softmax_scale: float,
                 block_ops: BlockOps | None = None, stats: RingStats | None = None,
                 count_tiles: bool = False, workspace: Workspace | None = None,
                 comm: Comm | None = None):
    """Forward for this rank's stripe.  q [c,Hq,D], k/v [c,Hkv,D] (bf16 on GPU).

    ``comm``: the hop backend (default: NCCL P2P over ``group`` when torch.distributed
    runs with more than one rank).  Returns (out [c,Hq,D] bf16, lse [Hq,c] fp32) in
    local (permuted) order, like run_schedule's outputs (simulator.py:237-277)."""
    bops = block_ops or BlockOps()
    if comm is None:
        comm = default_comm(group)
    rank, world = _rank_world(group, comm)
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
    st = _Streams(q)
    hops = _HopTimer(st, stats)
    bufs = [(_alloc(ws, f"kbuf{b}", k.shape, k.dtype, k.device),
             _alloc(ws, f"vbuf{b}", v.shape, v.dtype, v.device)) for b in range(2)]
    cur = (k, v)
    for i in range(world):
        held = (rank - i) % world
        nxt = bufs[i % 2]
        kv_ready = None
        if i < world - 1:
            # nxt's previous reader (round i-1) has finished; cur is complete
            st.wait(st.kv, st.event(st.compute))
            with st.on(st.kv):
                h0 = hops.start(st.kv)
                comm.exchange(list(cur), list(nxt))
                hops.stop(st.kv, h0, i, "kv", cur)
            kv_ready = st.event(st.kv)
        kind = masks.block_mask(layout, rank, held, world)
        before = int(tiles.item()) if (tiles is not None and stats is not None) else 0
        timer.start()
        bops.fwd_block(q, cur[0], cur[1], o_acc, lse, out, softmax_scale, kind, i == 0,
                       i == world - 1, tiles)
        timer.stop()
        if stats is not None:
            after = int(tiles.item()) if tiles is not None else 0
            stats.rounds.append(StepRecord(i, held, int(kind), after - before))
        if i < world - 1:
            st.wait(st.compute, kv_ready)
            cur = nxt
    if stats is not None:
        timer.fill(stats.rounds)
        hops.fill()
    return out, lse


def ring_backward(dout, q, k, v, out, lse, *, group=None, layout: str = "striped",
                  softmax_scale: float, block_ops: BlockOps | None = None,
                  stats: RingStats | None = None, workspace: Workspace | None = None,
                  comm: Comm | None = None, deterministic: bool = False,
                  fused_dkv: bool = False):
    """Backward for this rank's stripe -> (dq, dk, dv) bf16 in local order.

    ``fused_dkv`` (peer-memory comms only): no dK/dV hops -- each round's kernel adds
    into the held stripe's home accumulator on its owner rank directly (see below).

    ``deterministic``: the dQ reduce-adds of every launch happen in a fixed order (a
    zeroed int32 semaphore per query tile, see sa_bwd_block_ex), so reruns are
    bit-identical (verify.py:216-227); dK / dV are deterministic either way.

    Per round the held block runs in key parts (``kv_parts``); each part's fp32 dK/dV
    rows hop to the next rank on the dK/dV stream as soon as the part retires, and the
    next round's K/V hop is issued right after the first part's (so with NCCL, whose
    P2P ops to one peer share an internal stream, it does not delay that hop).  The
    accumulators are home after N hops."""
    bops = block_ops or BlockOps()
    if comm is None:
        comm = default_comm(group)
    rank, world = _rank_world(group, comm)
    c, hq, d = q.shape
    hkv = k.shape[1]
    dev = q.device
    ws = workspace
    dsum = _alloc(ws, "dsum", (hq, c), torch.float32, dev)
    dq_acc = _alloc(ws, "dq_acc", (c, hq, d), torch.float32, dev)
    bops.bwd_preprocess(out, dout, dsum, dq_acc)
    det = {}
    if deterministic:
        det["dq_sem"] = _alloc(ws, "dq_sem", (hq * (-(-c // 64)),), torch.int32, dev, zero=True)
    timer = _StepTimer(q, stats is not None)
    if world == 1 and hasattr(bops, "bwd_block_final"):
        # one step: dK / dV come out of the kernel as bf16 (no fp32 accumulators / casts)
        kind = masks.block_mask(layout, 0, 0, 1)
        dk = _alloc(ws, "dk", k.shape, k.dtype, dev)
        dv = _alloc(ws, "dv", v.shape, v.dtype, dev)
        timer.start()
        bops.bwd_block_final(q, k, v, dout, lse, dsum, dq_acc, dk, dv, softmax_scale, kind,
                             **det)
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
        bops.bwd_block(q, k, v, dout, lse, dsum, dq_acc, dk_acc, dv_acc, softmax_scale, kind,
                       **det)
        timer.stop()
        if stats is not None:
            stats.rounds.append(StepRecord(0, 0, int(kind)))
    elif fused_dkv:
        # SURVEY 8(f)3, fused rotation: no dK/dV hop at all.  Every stripe's fp32 dK/dV
        # accumulator stays on its home rank; the block kernel of whichever rank holds the
        # stripe in a round reduce-adds its contribution straight into the home buffer
        # through peer memory (NVLink) from its epilogue, tile by tile as CTAs retire.
        if deterministic:
            raise ValueError("fused_dkv adds into the home buffers in arrival order; "
                             "use the travelling accumulators for deterministic=True")
        if not getattr(comm, "peer_memory", False):
            raise ValueError(f"fused_dkv needs a peer-memory comm (LocalComm / IpcComm), "
                             f"got {getattr(comm, 'name', comm)!r}")
        st = _Streams(q)
        hops = _HopTimer(st, stats)
        homes_k = comm.peer_views(dk_acc)
        homes_v = comm.peer_views(dv_acc)
        comm.sync_all(q)  # every home buffer is zeroed before anyone adds into it
        kv_bufs = [(_alloc(ws, f"bkbuf{b}", k.shape, k.dtype, dev),
                    _alloc(ws, f"bvbuf{b}", v.shape, v.dtype, dev)) for b in range(2)]
        cur = (k, v)
        for i in range(world):
            held = (rank - i) % world
            nxt = kv_bufs[i % 2]
            kv_ready = None
            if i < world - 1:
                st.wait(st.kv, st.event(st.compute))
                with st.on(st.kv):
                    h0 = hops.start(st.kv)
                    comm.exchange(list(cur), list(nxt))
                    hops.stop(st.kv, h0, i, "kv", cur)
                kv_ready = st.event(st.kv)
            kind = masks.block_mask(layout, rank, held, world)
            timer.start()
            bops.bwd_block(q, cur[0], cur[1], dout, lse, dsum, dq_acc, homes_k[held],
                           homes_v[held], softmax_scale, kind)
            timer.stop()
            if stats is not None:
                stats.rounds.append(StepRecord(i, held, int(kind)))
            if i < world - 1:
                st.wait(st.compute, kv_ready)
                cur = nxt
        comm.sync_all(q)  # every rank's contributions to my stripe are in
        if stats is not None:
            hops.fill()
    else:
        st = _Streams(q)
        hops = _HopTimer(st, stats)
        kv_bufs = [(_alloc(ws, f"bkbuf{b}", k.shape, k.dtype, dev),
                    _alloc(ws, f"bvbuf{b}", v.shape, v.dtype, dev)) for b in range(2)]
        dspare = (_alloc(ws, "dk_spare", dk_acc.shape, torch.float32, dev),
                  _alloc(ws, "dv_spare", dv_acc.shape, torch.float32, dev))
        cur = (k, v)
        dcur = (dk_acc, dv_acc)
        parts = kv_parts(c)
        arrived = [None] * len(parts)  # dK/dV-stream events: part p of dcur has arrived
        for i in range(world):
            held = (rank - i) % world
            nxt = kv_bufs[i % 2]
            round_start = st.event(st.compute)  # round i-1's kernels (nxt's reader) done
            kv_ready = None
            kind = masks.block_mask(layout, rank, held, world)
            timer.start()
            sent = [None] * len(parts)
            for pi, (r0, r1) in enumerate(parts):
                st.wait(st.compute, arrived[pi])  # this part's accumulator rows are here
                bops.bwd_block(q, cur[0], cur[1], dout, lse, dsum, dq_acc, dcur[0], dcur[1],
                               softmax_scale, kind, key_rows=(r0, r1), **det)
                st.wait(st.dkv, st.event(st.compute))
                with st.on(st.dkv):
                    h0 = hops.start(st.dkv)
                    part = [dcur[0][r0:r1], dcur[1][r0:r1]]
                    comm.exchange(part, [dspare[0][r0:r1], dspare[1][r0:r1]])
                    hops.stop(st.dkv, h0, i, "dkv", part)
                sent[pi] = st.event(st.dkv)
                if pi == 0 and i < world - 1:
                    # the next round's K/V, behind the first part's dK/dV hop
                    st.wait(st.kv, round_start)
                    with st.on(st.kv):
                        h0 = hops.start(st.kv)
                        comm.exchange(list(cur), list(nxt))
                        hops.stop(st.kv, h0, i, "kv", cur)
                    kv_ready = st.event(st.kv)
            timer.stop()
            if stats is not None:
                stats.rounds.append(StepRecord(i, held, int(kind)))
            arrived = sent
            dcur, dspare = dspare, dcur
            if i < world - 1:
                st.wait(st.compute, kv_ready)
                cur = nxt
        for ev in arrived:  # the accumulators are home after the N-th hop
            st.wait(st.compute, ev)
        dk_acc, dv_acc = dcur
        if stats is not None:
            hops.fill()
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
                         block_ops: BlockOps | None = None, count_tiles: bool = False,
                         timings: list | None = None):
    """All N ranks' stripes on ONE device, rounds in order (the reference's serial
    executor, simulator.py:189-198).  Same kernels and merge as the distributed path.
    ``timings`` (a list): receives (round, rank, start, end) CUDA events per block."""
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
            ev = _ev_pair(timings)
            bops.fwd_block(qs[j], ks[held], vs[held], accs[j], lses[j], outs[j], softmax_scale,
                           kind, i == 0, i == n - 1, tiles)
            _ev_close(timings, ev, i, j)
            after = int(tiles.item()) if tiles is not None else 0
            stats[j].rounds.append(StepRecord(i, held, int(kind), after - before))
    return outs, lses, stats


def _ev_pair(timings):
    if timings is None:
        return None
    s = torch.cuda.Event(enable_timing=True)
    s.record()
    return s


def _ev_close(timings, start, i, j):
    if timings is None:
        return
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    timings.append((i, j, start, e))


def virtual_ring_backward(douts, qs, ks, vs, outs, lses, *, layout: str = "striped",
                          softmax_scale: float, block_ops: BlockOps | None = None,
                          timings: list | None = None, cast: bool = True):
    """Backward over all N stripes on one device; dK/dV accumulators stay with their
    stripe (index ``held``), exactly what the travelling buffers compute.  ``cast=False``
    returns the fp32 accumulators (timing runs)."""
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
            ev = _ev_pair(timings)
            bops.bwd_block(qs[j], ks[held], vs[held], douts[j], lses[j], dsums[j], dqs[j],
                           dks[held], dvs[held], softmax_scale, kind)
            _ev_close(timings, ev, i, j)
    if not cast:
        return dqs, dks, dvs
    res = []
    for acc, like in ((dqs, qs), (dks, ks), (dvs, vs)):
        outl = []
        for a, x in zip(acc, like):
            o = torch.empty_like(x)
            bops.cast(a, o)
            outl.append(o)
        res.append(outl)
    return tuple(res)
