"""Threaded (one-process) ring ranks over ring.LocalComm, on CPU with the oracle block ops.

The same unchanged ring_forward / ring_backward as the gloo test, but the N ranks are
threads of this process exchanging through LocalComm's ordered inboxes -- the
reference's threaded executor (simulator.py:201-234).  Checks: outputs equal the dense
oracle on every rank, the rotation invariant, and that a rank that fails or stalls
aborts the ring with the reference's RuntimeError instead of hanging."""

import numpy as np
import pytest
import torch

from cpu_blockops import OracleBlockOps
from oracle import ringref as R


def _run(world, c_rank, layout, hkv=2, fused=False):
    from paper_2311_09431_b200 import ring
    n, hq, d = c_rank * world, 4, 8
    rng = np.random.default_rng(11)
    q, k, v, do = (rng.standard_normal(s) for s in ((n, hq, d), (n, hkv, d), (n, hkv, d),
                                                     (n, hq, d)))
    scheme = R.STRIPED if layout == "striped" else R.CONTIGUOUS

    def rank_fn(rank, comm):
        rows = R.device_globals(scheme, n, world, rank)
        t = lambda a: torch.tensor(np.ascontiguousarray(a[rows]))
        ops = OracleBlockOps()
        st = ring.RingStats(rank)
        out, lse = ring.ring_forward(t(q), t(k), t(v), layout=layout, softmax_scale=0.3,
                                     block_ops=ops, stats=st, comm=comm)
        dq, dk, dv = ring.ring_backward(t(do), t(q), t(k), t(v), out, lse, layout=layout,
                                        softmax_scale=0.3, block_ops=ops, comm=comm,
                                        fused_dkv=fused)
        return rows, st, out, lse, dq, dk, dv

    res = ring.run_local_ring(world, rank_fn)
    o_ref, lse_ref = R.dense_forward(q, k, v, 0.3)
    g_ref = R.dense_backward(q, k, v, do, 0.3)
    for rank, (rows, st, out, lse, dq, dk, dv) in enumerate(res):
        assert [r.block_index for r in st.rounds] == [(rank - i) % world for i in range(world)]
        assert np.max(np.abs(out.numpy() - o_ref[rows])) <= 1e-5
        assert np.max(np.abs(lse.numpy() - lse_ref[:, rows])) <= 1e-5
        for got, want in zip((dq, dk, dv), g_ref):
            assert np.max(np.abs(got.numpy() - want[rows])) <= 1e-5


@pytest.mark.parametrize("world,c_rank", [(2, 16), (3, 16), (4, 16), (2, 512)])
@pytest.mark.parametrize("layout", ["striped", "ring"])
def test_local_ring_threads_match_oracle(world, c_rank, layout):
    _run(world, c_rank, layout)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("layout", ["striped", "ring"])
def test_local_ring_fused_dkv_matches_oracle(world, layout):
    """no dK/dV hops -- each round adds into the held stripe's home buffer
    on its owner (peer memory), then a stream-level barrier before the casts."""
    _run(world, 16, layout, fused=True)


def test_fused_dkv_needs_peer_memory():
    from paper_2311_09431_b200 import ring

    class NoPeer(ring.Comm):
        rank, world = 0, 2

    q = torch.zeros(4, 1, 8)
    with pytest.raises(ValueError, match="peer-memory"):
        ring.ring_backward(q, q, q, q, q, torch.zeros(1, 4), softmax_scale=1.0,
                           block_ops=OracleBlockOps(), comm=NoPeer(), fused_dkv=True)


def test_local_ring_failure_aborts_instead_of_hanging():
    from paper_2311_09431_b200 import ring

    def rank_fn(rank, comm):
        if rank == 1:
            raise ValueError("rank 1 broke")
        x = torch.zeros(4)
        comm.exchange([x], [torch.empty(4)])

    with pytest.raises(ValueError, match="rank 1 broke"):
        ring.run_local_ring(3, rank_fn, timeout=5.0)


def test_local_ring_stall_times_out():
    from paper_2311_09431_b200 import ring

    def rank_fn(rank, comm):
        if rank == 0:  # never joins the hop: the others' channel stalls
            return None
        comm.exchange([torch.zeros(2)], [torch.empty(2)])

    with pytest.raises(RuntimeError, match="stalled|aborted"):
        ring.run_local_ring(2, rank_fn, timeout=1.0)
