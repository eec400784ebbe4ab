"""The copy-engine IPC hop (ipc.IpcComm) between PROCESSES, on one GPU.

World sizes 2 and 4 as processes sharing cuda:0 (gloo only for the rendezvous / store):
the unchanged ring_forward / ring_backward with real kernels, side streams, double
buffers and the 2-part dK/dV hops, every hop a cudaMemcpyAsync into the next process's
IPC-mapped receive buffer ordered by interprocess events -- against the fp64 oracle.
No kernel waits on another process (the waits are stream-level event waits), so the
ranks need not run concurrently."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import ringref as R

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, layout, n, hq, hkv, d, out_q, fused=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, os.path.dirname(here))
        from paper_2311_09431_b200 import ring
        from paper_2311_09431_b200.ipc import IpcComm
        torch.cuda.set_device(0)
        rng = np.random.default_rng(17)
        q, k, v, do = (R.bf16_round(rng.standard_normal(s)) for s in
                       ((n, hq, d), (n, hkv, d), (n, hkv, d), (n, hq, d)))
        scheme = R.STRIPED if layout == "striped" else R.CONTIGUOUS
        rows = R.device_globals(scheme, n, world, rank)
        t = lambda a: torch.tensor(np.ascontiguousarray(a[rows]), dtype=torch.float32,
                                   device="cuda").bfloat16()
        comm = IpcComm()
        scale = 1 / math.sqrt(d)
        st = ring.RingStats(rank)
        with torch.cuda.stream(torch.cuda.Stream()):
            out, lse = ring.ring_forward(t(q), t(k), t(v), layout=layout, softmax_scale=scale,
                                         comm=comm, stats=st)
            dq, dk, dv = ring.ring_backward(t(do), t(q), t(k), t(v), out, lse, layout=layout,
                                            softmax_scale=scale, comm=comm, stats=st,
                                            fused_dkv=fused)
            torch.cuda.current_stream().synchronize()
        res = [x.float().cpu().numpy() for x in (out, lse, dq, dk, dv)]
        hops = [(h.what, h.nbytes) for h in st.hops]
        comm.close()
        out_q.put((rank, rows, res, hops))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,layout,fused", [(2, "striped", False), (4, "striped", False),
                                                (2, "ring", False), (4, "ring", False),
                                                (4, "striped", True)])
def test_ipc_ring_processes_on_one_gpu(world, layout, fused):
    """fused=True: no dK/dV hops; each process's kernels reduce-add into the other
    processes' IPC-mapped home accumulators (the fused rotation of SURVEY 8(f)3)."""
    n, hq, hkv, d = 2048, 4, 2, 128
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, layout, n, hq, hkv, d, out_q,
                                               fused))
             for r in range(world)]
    torch.cuda.empty_cache()  # the children open their own contexts on this GPU
    for p in procs:
        p.start()
    results = []
    waited = 0.0
    while len(results) < world:
        try:
            results.append(out_q.get(timeout=2.0))
        except Exception:  # queue.Empty: fail fast if a rank died instead of hanging
            waited += 2.0
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if dead or waited > 300:
                for p in procs:
                    p.kill()
                pytest.fail(f"IPC ranks failed (exit codes {dead}) or timed out")
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rng = np.random.default_rng(17)
    q, k, v, do = (R.bf16_round(rng.standard_normal(s)) for s in
                   ((n, hq, d), (n, hkv, d), (n, hkv, d), (n, hq, d)))
    scale = 1 / math.sqrt(d)
    o_ref, lse_ref = R.dense_forward(q, k, v, scale)
    dq_ref, dk_ref, dv_ref = R.dense_backward(q, k, v, do, scale)
    c = n // world
    for rank, rows, (o, lse, dq, dk, dv), hops in results:
        assert np.max(np.abs(o - o_ref[rows])) <= 2e-2
        assert np.max(np.abs(lse - lse_ref[:, rows])) <= 2e-3
        for got, want in ((dq, dq_ref), (dk, dk_ref), (dv, dv_ref)):
            assert np.max(np.abs(got - want[rows])) <= 2e-2
        # (N-1) K/V hops in the forward and N-1 in the backward, 3 dK/dV parts per round
        kv = [b for w, b in hops if w == "kv"]
        assert len(kv) == 2 * (world - 1) and all(b == 2 * c * hkv * d * 2 for b in kv)
        dkv = [b for w, b in hops if w == "dkv"]
        assert sum(dkv) == (0 if fused else world * 2 * c * hkv * d * 4)
