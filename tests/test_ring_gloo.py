"""Multi-process (gloo, CPU) tests of the ring driver's host logic.

world_size 2 and 4 processes run paper_2311_09431_b200.ring.ring_forward / ring_backward
unchanged, with the oracle block ops injected (tests/cpu_blockops.py).  Each rank's
outputs must equal the dense oracle restricted to that rank's stripe: this checks the
rotation schedule (held index (j - i) mod N, simulator.py:115-117), the mask chosen per
(rank, round), the LSE merge, and the dK/dV accumulators' N-hop trip home."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ringref as R


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, layout, result_q, c_rank=16):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, here)
        sys.path.insert(0, os.path.dirname(here))
        from cpu_blockops import OracleBlockOps
        from paper_2311_09431_b200 import ring, telemetry

        n, hq, hkv, d = c_rank * world, 4, 2, 8
        rng = np.random.default_rng(7)
        q, k, v, do = (rng.standard_normal(s) for s in ((n, hq, d), (n, hkv, d), (n, hkv, d),
                                                         (n, hq, d)))
        scheme = R.STRIPED if layout == "striped" else R.CONTIGUOUS
        rows = R.device_globals(scheme, n, world, rank)
        t = lambda a: torch.tensor(np.ascontiguousarray(a[rows]))
        ops = OracleBlockOps()
        stats = ring.RingStats(rank)
        out, lse = ring.ring_forward(t(q), t(k), t(v), layout=layout, softmax_scale=0.3,
                                     block_ops=ops, stats=stats)
        dq, dk, dv = ring.ring_backward(t(do), t(q), t(k), t(v), out, lse, layout=layout,
                                        softmax_scale=0.3, block_ops=ops)
        o_ref, lse_ref = R.dense_forward(q, k, v, 0.3)
        dq_ref, dk_ref, dv_ref = R.dense_backward(q, k, v, do, 0.3)
        errs = {
            "out": float(np.max(np.abs(out.numpy() - o_ref[rows]))),
            "lse": float(np.max(np.abs(lse.numpy() - lse_ref[:, rows]))),
            "dq": float(np.max(np.abs(dq.numpy() - dq_ref[rows]))),
            "dk": float(np.max(np.abs(dk.numpy() - dk_ref[rows]))),
            "dv": float(np.max(np.abs(dv.numpy() - dv_ref[rows]))),
        }
        held = [r.block_index for r in stats.rounds]
        kinds = [r.mask_kind for r in stats.rounds]
        # telemetry: every rank's stats on every rank, rows in the reference CSV schema
        everyone = telemetry.gather_stats(stats)
        run = telemetry.Run(layout, n // world, hq, everyone)
        csv_rows = telemetry.rows([run])
        imb = telemetry.step_imbalance(everyone)
        result_q.put((rank, errs, held, kinds, ops.calls, csv_rows, imb))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,c_rank", [(2, 16), (4, 16), (2, 512)])
@pytest.mark.parametrize("layout", ["striped", "ring"])
def test_ring_driver_over_gloo(world, c_rank, layout):
    """c_rank 512: the backward runs each block in 2 key parts whose dK/dV rows hop
    separately (ring.kv_parts)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, layout, q, c_rank))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rows0 = None
    for rank, errs, held, kinds, calls, csv_rows, imb in results:
        # every rank gathered the same table: world rounds x world devices, round-major
        assert len(csv_rows) == world * world
        assert [(r[1], r[2]) for r in csv_rows] == [(i, d) for i in range(world) for d in range(world)]
        assert all(r[3] == (r[2] - r[1]) % world for r in csv_rows)  # held = (j - i) mod N
        assert rows0 is None or csv_rows == rows0
        rows0 = csv_rows
        assert imb == [1.0] * world  # no CUDA timing on CPU
        for name, e in errs.items():
            assert e <= 1e-5, (rank, name, e)  # lse/out carried in fp32 by the driver
        assert held == [(rank - i) % world for i in range(world)]
        want = [R.block_kind(R.STRIPED if layout == "striped" else R.CONTIGUOUS, rank, h)
                for h in held]
        assert kinds == want
        fwd = [c for c in calls if c[0] == "fwd"]
        assert [c[2] for c in fwd] == [i == 0 for i in range(world)]
        assert [c[3] for c in fwd] == [i == world - 1 for i in range(world)]
