"""Copy-engine ring hop between processes: CUDA IPC memory + event handles (``IpcComm``).

One process per GPU (torchrun).  The hop of ring.LocalComm, across processes: each rank
offers its receive buffers to the previous rank as (IPC memory handle, offset, bytes)
plus an interprocess event marking when they may be overwritten; the previous rank
waits on that event, copies its send buffers straight into them with
``cudaMemcpyAsync`` (copy engines over NVLink -- no NCCL kernels taking SMs from the
attention grid, SURVEY.md section 2.5 option ii), records its own interprocess event and
tells the receiver, whose stream then waits on it.  The per-hop host hand-off goes
through the torch.distributed store; every event is recorded before its handle is
named to a peer, so no wait can precede its record.  Memory handles are opened once per
peer allocation (the ring's workspaces are persistent) and cached.

This is the reference's ordered per-device channel (simulator.py:201-234) with device
buffers: sends to rank j+1 and receives from rank j-1 are matched by a per-comm sequence
number that every rank advances in the same order.
"""

from __future__ import annotations

import ctypes
import itertools
import pickle
from datetime import timedelta

import torch
import torch.distributed as dist

from . import _lib
from .ring import STALL_TIMEOUT_S, Comm

_HANDLE = 64
_instances = itertools.count()


def _handle_bytes(buf) -> bytes:
    return bytes(bytearray(buf))


class _DevPtr:
    """A raw device pointer as a __cuda_array_interface__ object (zero-copy torch view)."""

    def __init__(self, ptr: int, shape, dtype: torch.dtype):
        typestr = {torch.float32: "<f4", torch.bfloat16: "<V2", torch.int32: "<i4"}[dtype]
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 2, "strides": None}


class IpcComm(Comm):
    name = "ipc"
    peer_memory = True

    def __init__(self, group=None, store=None, timeout: float = 20 * STALL_TIMEOUT_S):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        glob = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
        self.next_rank = (self.rank + 1) % self.world
        self.prev_rank = (self.rank - 1) % self.world
        self.next, self.prev = glob(self.next_rank), glob(self.prev_rank)
        # the default store's own timeout is left alone (NCCL init and torch.distributed
        # use it); every wait here carries its own.  Default 10 min: a rank's host can lag
        # its peers by whole rounds of GPU work (seconds each at 786k) when it synchronises.
        self.store = store if store is not None else dist.distributed_c10d._get_default_store()
        self.timeout = timeout
        self.prefix = f"sa_ipc/{next(_instances)}/"
        self.seq = 0
        self._lib = _lib.lib()
        self._free_ev, free_h = self._create_event()
        self._done_ev, done_h = self._create_event()
        self._sync_ev, sync_h = self._create_event()
        self.store.set(f"{self.prefix}ev/{self.rank}", pickle.dumps((free_h, done_h, sync_h)))
        self._n = 0  # collective sequence number (peer_views / sync_all)
        self._peer_ev = {}   # (rank, which) -> opened event
        self._opened = {}    # handle bytes -> opened base pointer
        self._mine = {}      # local base pointer -> (handle bytes)

    # ------------------------------------------------------------------ plumbing
    def _check(self, rc, what):
        _lib.check(rc, what)

    def _create_event(self):
        ev = ctypes.c_void_p()
        h = (ctypes.c_char * _HANDLE)()
        self._check(self._lib.sa_ipc_event_create(ctypes.byref(ev), h), "sa_ipc_event_create")
        return ev, _handle_bytes(h)

    def _fetch(self, key):
        """The value of `key` once a peer has set it (bounded wait: the reference's
        'ring channel stalled', simulator.py:40)."""
        try:
            self.store.wait([key], timedelta(seconds=self.timeout))
        except Exception as e:  # noqa: BLE001 - store timeout
            raise RuntimeError(f"ring channel stalled (rank {self.rank}, {key}): {e}") from e
        return self.store.get(key)

    def _get(self, key):
        v = self._fetch(key)
        self.store.delete_key(key)
        return v

    def _peer_event(self, rank, which):
        key = (rank, which)
        if key not in self._peer_ev:
            handles = pickle.loads(self._fetch(f"{self.prefix}ev/{rank}"))
            h = (ctypes.c_char * _HANDLE).from_buffer_copy(handles[which])
            ev = ctypes.c_void_p()
            self._check(self._lib.sa_ipc_event_open(h, ctypes.byref(ev)), "sa_ipc_event_open")
            self._peer_ev[key] = ev
        return self._peer_ev[key]

    def _describe(self, t: torch.Tensor):
        h = (ctypes.c_char * _HANDLE)()
        off = ctypes.c_int64()
        self._check(self._lib.sa_ipc_mem_handle(ctypes.c_void_p(t.data_ptr()), h,
                                                ctypes.byref(off)), "sa_ipc_mem_handle")
        return _handle_bytes(h), off.value, t.numel() * t.element_size()

    def _open(self, handle: bytes) -> int:
        if handle not in self._opened:
            h = (ctypes.c_char * _HANDLE).from_buffer_copy(handle)
            base = ctypes.c_void_p()
            self._check(self._lib.sa_ipc_mem_open(h, ctypes.byref(base)), "sa_ipc_mem_open")
            self._opened[handle] = base.value
        return self._opened[handle]

    # ------------------------------------------------------------------ the hop
    def exchange(self, send, recv):
        if not recv[0].is_cuda:
            raise ValueError("IpcComm moves CUDA tensors only")
        s = self.seq
        self.seq += 1
        stream = torch.cuda.current_stream(recv[0].device).cuda_stream
        # 1. offer my receive buffers to the previous rank
        self._check(self._lib.sa_event_record(self._free_ev, stream), "sa_event_record")
        self.store.set(f"{self.prefix}ready/{self.rank}/{s}",
                       pickle.dumps([self._describe(r) for r in recv]))
        # 2. write into the next rank's buffers once it allows it
        offer = pickle.loads(self._get(f"{self.prefix}ready/{self.next_rank}/{s}"))
        if len(offer) != len(send):
            raise RuntimeError("ring peers disagree on the hop's tensors")
        self._check(self._lib.sa_stream_wait_event(stream, self._peer_event(self.next_rank, 0)),
                    "sa_stream_wait_event")
        for t, (handle, off, nbytes) in zip(send, offer):
            if nbytes != t.numel() * t.element_size() or not t.is_contiguous():
                raise RuntimeError("hop buffer size mismatch")
            dst = self._open(handle) + off
            self._check(self._lib.sa_memcpy_async(ctypes.c_void_p(dst),
                                                  ctypes.c_void_p(t.data_ptr()), nbytes, stream),
                        "sa_memcpy_async")
        self._check(self._lib.sa_event_record(self._done_ev, stream), "sa_event_record")
        self.store.set(f"{self.prefix}done/{self.rank}/{s}", b"1")
        # 3. my buffers are filled once the previous rank's copies are
        self._get(f"{self.prefix}done/{self.prev_rank}/{s}")
        self._check(self._lib.sa_stream_wait_event(stream, self._peer_event(self.prev_rank, 1)),
                    "sa_stream_wait_event")

    # ------------------------------------------------------------------ collectives
    def _all_gather(self, tag, value: bytes) -> list:
        n = self._n
        self._n += 1
        self.store.set(f"{self.prefix}{tag}/{n}/{self.rank}", value)
        out = [self._fetch(f"{self.prefix}{tag}/{n}/{j}") for j in range(self.world)]
        # nobody deletes a key before every rank has read it: acknowledge, then clean up
        self.store.set(f"{self.prefix}{tag}_ack/{n}/{self.rank}", b"1")
        for j in range(self.world):
            self._fetch(f"{self.prefix}{tag}_ack/{n}/{j}")
        return out

    def peer_views(self, t):
        if t.dtype != torch.float32 or not t.is_contiguous():
            raise ValueError("peer_views: contiguous fp32 buffers only")
        mine = pickle.dumps(self._describe(t))
        views = []
        for j, blob in enumerate(self._all_gather("views", mine)):
            if j == self.rank:
                views.append(t)
                continue
            handle, off, nbytes = pickle.loads(blob)
            if nbytes != t.numel() * t.element_size():
                raise RuntimeError("peer buffers differ in size")
            ptr = self._open(handle) + off
            views.append(torch.as_tensor(_DevPtr(ptr, t.shape, t.dtype), device=t.device))
        return views

    def sync_all(self, ref):
        stream = torch.cuda.current_stream(ref.device).cuda_stream
        self._check(self._lib.sa_event_record(self._sync_ev, stream), "sa_event_record")
        n = self._n
        self._n += 1
        key = lambda j: f"{self.prefix}sync/{n}/{j}"
        self.store.set(key(self.rank), b"1")
        for j in range(self.world):
            if j != self.rank:
                self._fetch(key(j))
                self._check(self._lib.sa_stream_wait_event(stream, self._peer_event(j, 2)),
                            "sa_stream_wait_event")
        # the next record of any rank's sync event must follow every rank's wait on it
        self.store.set(f"{self.prefix}sync_ack/{n}/{self.rank}", b"1")
        for j in range(self.world):
            self._fetch(f"{self.prefix}sync_ack/{n}/{j}")

    def close(self):
        for base in self._opened.values():
            self._lib.sa_ipc_mem_close(ctypes.c_void_p(base))
        self._opened.clear()
        for ev in self._peer_ev.values():
            self._lib.sa_event_destroy(ev)
        self._peer_ev.clear()
