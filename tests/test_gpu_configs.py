"""GPU parity at the BASELINE.json configs themselves (what bench.py measures).

* configs[0] exactly: S = 8192, 8 heads, d 64, N = 4 ranks, striped AND ring, forward and
  backward, run by the real ring driver (ring_forward / ring_backward with its side
  streams, double buffers and 2-part dK/dV hops) with the 4 ranks as threads sharing
  this GPU (ring.LocalComm: copy-engine hops) -- against the fp64 dense oracle
  (oracle/ringref.py: dense_forward pinned to the reference's simulate, dense_backward
  pinned by autograd / finite differences).
* configs[1] exactly: S = 32k, 32 heads, d 128 at N = 1 (the benched block kernels), plus
  its GQA variant (32 q / 8 kv); and the headline S = 256k, 32 heads at N = 1.  The dense
  fp64 oracle is O(S^2) in memory, so the reference here is the same math restated in
  fp32 torch on the GPU, chunked over query rows (TF32 off): every row of O, LSE, dQ, dK
  and dV of the checked heads is compared, not a sample.

Tolerances are the north star's: bf16 outputs max-abs <= 2e-2 and rel-L2 <= 1e-2 against
the reference on the same bf16-rounded inputs; fp32 LSE <= 2e-3.  One refinement: a bf16
output of magnitude >= 4 has a half-ulp of 1.6e-2 by itself (dK / dV of a GQA kv head sum
four q heads and reach that range), so the per-element bound is 2e-2 + 2^-7 |ref| (one
bf16 ulp relative on top of the absolute bound); rel-L2 stays 1e-2.
"""

import math

import numpy as np
import pytest
import torch

from oracle import ringref as R

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2, LSE_ABS = 2e-2, 1e-2, 2e-3


def _check(got, want, name):
    got = got.float()
    want = want.float()
    assert torch.isfinite(got).all(), name
    diff = (got - want).abs()
    err = diff.max().item()
    rel = ((got - want).norm() / want.norm().clamp_min(1e-30)).item()
    excess = (diff - (MAX_ABS + 2.0 ** -7 * want.abs())).max().item()
    assert excess <= 0, (name, err, excess)
    assert rel <= REL_L2, (name, rel)
    return err, rel


def _check_np(got, want, name):
    return _check(torch.as_tensor(np.asarray(got)), torch.as_tensor(np.asarray(want)), name)


# ------------------------------------------------------------------ configs[0], N = 4 ring
@pytest.mark.parametrize("layout,fused", [("striped", False), ("ring", False), ("striped", True)])
def test_config0_ring_fwd_bwd_threads_on_one_gpu(layout, fused):
    """fused=True: the fused rotation (no dK/dV hops; the kernels reduce-add into the
    held stripe's home accumulator on its owner rank through peer memory)."""
    from paper_2311_09431_b200 import ring
    n_dev, n, h, d = 4, 8192, 8, 64
    scale = 1.0 / math.sqrt(d)
    rng = np.random.default_rng(2024)
    q, k, v, do = (R.bf16_round(rng.standard_normal((n, h, d))) for _ in range(4))
    scheme = R.STRIPED if layout == "striped" else R.CONTIGUOUS

    def rank_fn(rank, comm):
        rows = R.device_globals(scheme, n, n_dev, rank)
        t = lambda a: torch.tensor(np.ascontiguousarray(a[rows]), dtype=torch.float32,
                                   device="cuda").bfloat16()
        st = ring.RingStats(rank)
        out, lse = ring.ring_forward(t(q), t(k), t(v), layout=layout, softmax_scale=scale,
                                     comm=comm, stats=st)
        dq, dk, dv = ring.ring_backward(t(do), t(q), t(k), t(v), out, lse, layout=layout,
                                        softmax_scale=scale, comm=comm, stats=st,
                                        fused_dkv=fused)
        torch.cuda.current_stream().synchronize()
        return (rows, [r.block_index for r in st.rounds[:n_dev]],
                *(x.float().cpu().numpy() for x in (out, lse, dq, dk, dv)))

    res = ring.run_local_ring(n_dev, rank_fn, devices=["cuda:0"] * n_dev, timeout=120.0)
    o_ref, lse_ref = R.dense_forward(q, k, v, scale)
    dq_ref, dk_ref, dv_ref = R.dense_backward(q, k, v, do, scale)
    got = {x: np.empty_like(o_ref if x != "lse" else lse_ref) for x in ("o", "lse", "dq")}
    got["dk"], got["dv"] = np.empty_like(dk_ref), np.empty_like(dv_ref)
    for rank, (rows, held, o, lse, dq, dk, dv) in enumerate(res):
        assert held == [(rank - i) % n_dev for i in range(n_dev)]  # simulator.py:115-117
        got["o"][rows], got["lse"][:, rows], got["dq"][rows] = o, lse, dq
        got["dk"][rows], got["dv"][rows] = dk, dv
    _check_np(got["o"], o_ref, "out")
    assert np.max(np.abs(got["lse"] - lse_ref)) <= LSE_ABS
    _check_np(got["dq"], dq_ref, "dq")
    _check_np(got["dk"], dk_ref, "dk")
    _check_np(got["dv"], dv_ref, "dv")


# ------------------------------------------------------------------ fp32 torch restatement
def reference_head(q, k, v, do, scale, chunk=2048):
    """fp32 causal attention fwd + bwd of ONE head (q/do [n, d], k/v [n, d], fp32 CUDA)
    chunked over query rows: the math of oracle.ringref.dense_forward / dense_backward
    (attention.py:121-143 forward).  Returns o, lse, dq, dk, dv."""
    n, d = q.shape
    o = torch.empty_like(q)
    lse = torch.empty(n, device=q.device)
    cols = torch.arange(n, device=q.device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        s = (q[a:b] @ k[:b].T) * scale
        s.masked_fill_(cols[None, :b] > torch.arange(a, b, device=q.device)[:, None], -math.inf)
        m = s.amax(dim=1, keepdim=True)
        p = torch.exp(s - m)
        z = p.sum(dim=1, keepdim=True)
        o[a:b] = (p @ v[:b]) / z
        lse[a:b] = (m + torch.log(z))[:, 0]
        del s, p
    dsum = (do * o).sum(dim=1)
    dq = torch.empty_like(q)
    dk = torch.zeros_like(k)
    dv = torch.zeros_like(v)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        s = (q[a:b] @ k[:b].T) * scale
        s.masked_fill_(cols[None, :b] > torch.arange(a, b, device=q.device)[:, None], -math.inf)
        p = torch.exp(s - lse[a:b, None])
        del s
        ds = p * (do[a:b] @ v[:b].T - dsum[a:b, None])
        dq[a:b] = (ds @ k[:b]) * scale
        dk[:b] += (ds.T @ q[a:b]) * scale
        dv[:b] += p.T @ do[a:b]
        del p, ds
    return o, lse, dq, dk, dv


def _run_block_and_check(n, hq, hkv, d, heads, seed):
    """N = 1 (one block, the benched path) at full size; every row of `heads` checked."""
    from paper_2311_09431_b200 import ring
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        gen = torch.Generator(device="cuda").manual_seed(seed)
        mk = lambda hh: torch.randn(n, hh, d, device="cuda", generator=gen).bfloat16()
        q, k, v, do = mk(hq), mk(hkv), mk(hkv), mk(hq)
        scale = 1.0 / math.sqrt(d)
        out, lse = ring.ring_forward(q, k, v, layout="striped", softmax_scale=scale)
        dq, dk, dv = ring.ring_backward(do, q, k, v, out, lse, layout="striped",
                                        softmax_scale=scale)
        torch.cuda.synchronize()
        group = hq // hkv
        dk_ref = {}
        dv_ref = {}
        for h in heads:
            g = h // group
            o_r, lse_r, dq_r, dk_r, dv_r = reference_head(q[:, h].float(), k[:, g].float(),
                                                           v[:, g].float(), do[:, h].float(),
                                                           scale)
            _check(out[:, h], o_r, f"out h{h}")
            assert (lse[h] - lse_r).abs().max().item() <= LSE_ABS, f"lse h{h}"
            _check(dq[:, h], dq_r, f"dq h{h}")
            dk_ref[g] = dk_ref.get(g, 0) + dk_r
            dv_ref[g] = dv_ref.get(g, 0) + dv_r
            del o_r, lse_r, dq_r, dk_r, dv_r
        # dK / dV of a kv head sum over its whole q-head group: check the groups whose
        # q heads were all restated
        for g in dk_ref:
            if all(h in heads for h in range(g * group, (g + 1) * group)):
                _check(dk[:, g], dk_ref[g], f"dk g{g}")
                _check(dv[:, g], dv_ref[g], f"dv g{g}")
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def test_config1_32k_32heads_fwd_bwd_all_rows():
    """configs[1] exactly: seq 32768, 32 heads, d 128 (the benched single-B200 block)."""
    _run_block_and_check(32768, 32, 32, 128, heads=[0, 7, 19, 31], seed=31)


def test_config1_gqa_32k_all_rows():
    """Same shape with the Llama-3-8B GQA ratio (configs[3]: 32 q / 8 kv heads)."""
    _run_block_and_check(32768, 32, 8, 128, heads=[0, 1, 2, 3, 28, 29, 30, 31], seed=32)


def test_headline_256k_32heads_fwd_bwd_all_rows():
    """The metric's shape (configs[2]: seq 256k, 32 heads, d 128) at N = 1."""
    _run_block_and_check(262144, 32, 32, 128, heads=[0, 31], seed=33)


@pytest.mark.parametrize("n,hq,hkv", [(262144, 4, 4), (524288, 8, 2)])
@pytest.mark.parametrize("layout", ["striped", "ring"])
def test_headline_256k_eight_rank_ring_equals_single_block(layout, n, hq, hkv):
    """configs[2]'s N = 8 schedule at full length (256k, c = 32768 per rank; 4 heads), and
    configs[3]'s (512k, c = 65536, GQA 4:1 on 8 of its q heads): all 64 (rank, round)
    blocks with their masks, LSE merges and travelling dK / dV accumulators (the serial
    executor) reproduce the N = 1 block -- which the tests here check row by row against
    the fp32 restatement -- after unpermuting (attention commutes with the stripe
    permutation, pkg/tests/test_layout.py:106-125)."""
    from paper_2311_09431_b200 import Layout, ring
    d, n_dev = 128, 8
    gen = torch.Generator(device="cuda").manual_seed(36)
    q, do = (torch.randn(n, hq, d, device="cuda", generator=gen).bfloat16() for _ in range(2))
    k, v = (torch.randn(n, hkv, d, device="cuda", generator=gen).bfloat16() for _ in range(2))
    scale = 1.0 / math.sqrt(d)
    out1, lse1 = ring.ring_forward(q, k, v, softmax_scale=scale)
    g1 = ring.ring_backward(do, q, k, v, out1, lse1, softmax_scale=scale)
    lay = Layout("striped" if layout == "striped" else "contiguous", n, n_dev)
    c = n // n_dev
    sh = lambda x: [s.contiguous() for s in lay.permute(x).split(c)]
    qs, ks, vs, dos = sh(q), sh(k), sh(v), sh(do)
    outs, lses, _ = ring.virtual_ring_forward(qs, ks, vs, layout=layout, softmax_scale=scale)
    gs = ring.virtual_ring_backward(dos, qs, ks, vs, outs, lses, layout=layout,
                                    softmax_scale=scale)
    torch.cuda.synchronize()
    _check(lay.gather(outs), out1.float(), "out")
    lse8 = lay.gather([x.t().contiguous() for x in lses]).t()
    assert (lse8 - lse1).abs().max().item() <= LSE_ABS
    for name, got, want in zip(("dq", "dk", "dv"), gs, g1):
        _check(lay.gather(got), want.float(), name)


def test_config3_512k_gqa_one_kv_group_all_rows():
    """configs[3] (Llama-3-8B GQA 32 q / 8 kv heads, seq 512k) at N = 1: every row of a
    whole kv group (q heads 0-3) incl. its summed dK / dV."""
    _run_block_and_check(524288, 32, 8, 128, heads=[0, 1, 2, 3], seed=34)


def test_config4_786k_long_sequence_all_rows():
    """configs[4]'s sequence length (786k) at N = 1 with 8 of its 64 heads (the kernels'
    per-head work does not depend on the head count): rows of heads 0 and 7."""
    _run_block_and_check(786432, 8, 8, 128, heads=[0, 7], seed=35)
