"""GPU: seeded random sweep of block shapes (ragged c around the 128 / 256 tile and pair
boundaries, GQA ratios, both head dims, every mask kind, carried state) through the forward
and backward kernels against the CPU oracle."""

import math
import os

import numpy as np
import pytest
import torch

from oracle import ringref as R

pytestmark = pytest.mark.gpu

O_MAX_ABS, O_REL_L2, LSE_ABS = 2e-2, 1e-2, 2e-3


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


def _cases(n=None, seed=2024):
    # SA_FUZZ_N widens the sweep for an extended run (profiles/r02_fuzz_extended.log)
    n = int(os.environ.get("SA_FUZZ_N", "40")) if n is None else n
    rng = np.random.default_rng(seed)
    cs = [127, 129, 255, 257, 383, 385, 511, 513, 640, 767, 769, 896]
    out = []
    for _ in range(n):
        c = int(rng.choice(cs))
        d = int(rng.choice([64, 128]))
        hkv = int(rng.integers(1, 3))
        hq = hkv * int(rng.choice([1, 2, 4]))
        kind = int(rng.choice([1, 2, 3]))
        steps = int(rng.integers(1, 3))  # 2: a carried (o_acc, lse) merge
        out.append((c, hq, hkv, d, kind, steps))
    return out


@pytest.fixture(scope="module")
def ops():
    from paper_2311_09431_b200 import ops as _ops
    return _ops


@pytest.mark.parametrize("c,hq,hkv,d,kind,steps", _cases())
def test_random_block_shapes(ops, c, hq, hkv, d, kind, steps):
    g = torch.Generator(device="cuda").manual_seed(c * 131 + hq * 7 + d + kind + steps)
    scale = 1.0 / math.sqrt(d)
    q = torch.randn(c, hq, d, device="cuda", generator=g).bfloat16()
    kvs = [(torch.randn(c, hkv, d, device="cuda", generator=g).bfloat16(),
            torch.randn(c, hkv, d, device="cuda", generator=g).bfloat16()) for _ in range(steps)]
    kinds = [kind] + [1] * (steps - 1)
    o_acc = torch.empty(c, hq, d, device="cuda")
    lse = torch.empty(hq, c, device="cuda")
    out = torch.empty(c, hq, d, device="cuda", dtype=torch.bfloat16)
    for i, ((k, v), kd) in enumerate(zip(kvs, kinds)):
        ops.fwd_block(q, k, v, o_acc, lse, out, scale, kd, i == 0, i == steps - 1)
    torch.cuda.synchronize()
    qn = q.float().cpu().numpy().astype(np.float64)
    st = R.Accum.fresh(c, hq, d)
    for (k, v), kd in zip(kvs, kinds):
        R.process_block(st, qn * scale, k.float().cpu().numpy().astype(np.float64),
                        v.float().cpu().numpy().astype(np.float64), kd, c, c)
    o_ref, lse_ref = R.finalize(st, allow_dead=True)
    o = out.float().cpu().numpy()
    ls = lse.cpu().numpy()
    dead = np.isneginf(lse_ref)
    np.testing.assert_array_equal(np.isneginf(ls), dead)
    assert np.max(np.abs(ls[~dead] - lse_ref[~dead])) <= LSE_ABS
    assert np.max(np.abs(o - o_ref)) <= O_MAX_ABS
    assert rel_l2(o, o_ref) <= O_REL_L2

    # backward of the first step's block against the fp64 restatement
    if steps == 1:
        do = torch.randn(c, hq, d, device="cuda", generator=g).bfloat16()
        k, v = kvs[0]
        dsum = torch.empty(hq, c, device="cuda")
        dq = torch.empty(c, hq, d, device="cuda")
        dk = torch.zeros(c, hkv, d, device="cuda")
        dv = torch.zeros(c, hkv, d, device="cuda")
        lse_t = torch.tensor(lse_ref, device="cuda", dtype=torch.float32).contiguous()
        out_t = torch.tensor(o_ref, device="cuda").bfloat16()
        ops.bwd_preprocess(out_t, do, dsum, dq)
        ops.bwd_block(q, k, v, do, lse_t, dsum, dq, dk, dv, scale, kind)
        torch.cuda.synchronize()
        don = do.float().cpu().numpy().astype(np.float64)
        outn = out_t.float().cpu().numpy().astype(np.float64)
        dsum_ref = np.einsum("shd,shd->hs", don, outn)
        want = R.block_backward(qn, k.float().cpu().numpy().astype(np.float64),
                                v.float().cpu().numpy().astype(np.float64), don,
                                lse_ref.astype(np.float32).astype(np.float64), dsum_ref, kind,
                                scale)
        for name, got, w in (("dq", dq, want[0]), ("dk", dk, want[1]), ("dv", dv, want[2])):
            gg = got.cpu().numpy()
            assert np.max(np.abs(gg - w)) <= O_MAX_ABS, (name, np.max(np.abs(gg - w)))
            assert rel_l2(gg, w) <= O_REL_L2, (name, rel_l2(gg, w))
