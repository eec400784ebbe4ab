"""GPU parity of the forward block kernel (K2+K3) against the CPU oracle.

Bar (north star): bf16 outputs within max-abs 2e-2 and rel-L2 1e-2 of the oracle run
in fp64 on the same bf16-rounded inputs; LSE (fp32 output) within 2e-3 abs."""

import math

import numpy as np
import pytest
import torch

from oracle import ringref as R
from conftest import load_golden

pytestmark = pytest.mark.gpu

O_MAX_ABS, O_REL_L2, LSE_ABS = 2e-2, 1e-2, 2e-3


@pytest.fixture(scope="module")
def ops():
    from paper_2311_09431_b200 import ops as _ops
    return _ops


def block_ref(q, k, v, kind, scale):
    """Oracle block op: process_block (simulator.py:144-186) on a fresh accumulator."""
    c = q.shape[0]
    st = R.Accum.fresh(c, q.shape[1], v.shape[2])
    R.process_block(st, q.astype(np.float64) * scale, k.astype(np.float64), v.astype(np.float64),
                    kind, c, c)
    return R.finalize(st, allow_dead=True)


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


def run_block(ops, q, k, v, kind, scale):
    c, hq, d = q.shape
    out = torch.empty(c, hq, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(hq, c, device="cuda", dtype=torch.float32)
    tiles = torch.zeros(1, device="cuda", dtype=torch.int64)
    ops.fwd_block(q, k, v, None, lse, out, scale, kind, True, True, tiles)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), lse.cpu().numpy(), int(tiles.item())


@pytest.mark.parametrize("kind", [2, 3, 1])
@pytest.mark.parametrize("c,hq,hkv,d", [(128, 1, 1, 128), (256, 2, 2, 128), (384, 2, 1, 64),
                                         (1000, 2, 2, 128), (100, 1, 1, 64), (2048, 4, 2, 128),
                                         (1, 1, 1, 128), (300, 3, 3, 64)])
def test_block_forward_matches_oracle(ops, kind, c, hq, hkv, d):
    g = torch.Generator(device="cuda").manual_seed(c * 7 + hq + d + kind)
    q = torch.randn(c, hq, d, device="cuda", generator=g).bfloat16()
    k = torch.randn(c, hkv, d, device="cuda", generator=g).bfloat16()
    v = torch.randn(c, hkv, d, device="cuda", generator=g).bfloat16()
    scale = 1.0 / math.sqrt(d)
    if kind == 3 and c == 1:
        pytest.skip("a 1-row strict block has no allowed pair at all")
    out, lse, tiles = run_block(ops, q, k, v, kind, scale)
    o_ref, lse_ref = block_ref(q.float().cpu().numpy(), k.float().cpu().numpy(),
                               v.float().cpu().numpy(), kind, scale)
    dead = np.isneginf(lse_ref)
    np.testing.assert_array_equal(np.isneginf(lse), dead)
    assert np.max(np.abs(lse[~dead] - lse_ref[~dead])) <= LSE_ABS
    assert np.max(np.abs(out - o_ref)) <= O_MAX_ABS
    assert rel_l2(out, o_ref) <= O_REL_L2
    if kind == 3:
        assert dead[:, 0].all() and not dead[:, 1:].any()  # strict: local row 0 is dead
        assert np.all(out[0] == 0)
    # tile accounting: the kernels compute exactly the reference's non-SKIP 128x128 tiles
    from paper_2311_09431_b200.masks import kernel_tile_census
    assert tiles == hq * kernel_tile_census(kind, c).n_computed


def test_block_state_matches_reference_process_round(ops):
    """Per-(rank, round) block outputs vs the reference's _process_round (golden)."""
    g = load_golden("block_striped_n4_c256_d128_j1.npz")
    n_dev, c, d, j, _ = g["meta"].tolist()
    qs = R.partition(g["q"][:, None, :], R.STRIPED, n_dev)
    ks = R.partition(g["k"][:, None, :], R.STRIPED, n_dev)
    vs = R.partition(g["v"][:, None, :], R.STRIPED, n_dev)
    to = lambda a: torch.tensor(np.ascontiguousarray(a), device="cuda").bfloat16()
    for i in range(n_dev):
        kk = (j - i) % n_dev
        st = R.Accum(g["acc"][i][:, None, :].copy(), g["m"][i][None].copy(), g["l"][i][None].copy())
        o_ref, lse_ref = R.finalize(st, allow_dead=True)
        out, lse, _ = run_block(ops, to(qs[j]), to(ks[kk]), to(vs[kk]), R.striped_kind(j, kk),
                                1.0 / math.sqrt(d))
        dead = np.isneginf(lse_ref)
        np.testing.assert_array_equal(np.isneginf(lse), dead)
        assert np.max(np.abs(lse[~dead] - lse_ref[~dead])) <= LSE_ABS
        assert np.max(np.abs(out - o_ref)) <= O_MAX_ABS


def test_merge_across_steps_in_kernel(ops):
    """Carry (o_acc, lse) through several launches: equals one dense pass over all keys."""
    c, h, d = 512, 2, 128
    gen = torch.Generator(device="cuda").manual_seed(3)
    q = torch.randn(c, h, d, device="cuda", generator=gen).bfloat16()
    ks = [torch.randn(c, h, d, device="cuda", generator=gen).bfloat16() for _ in range(3)]
    vs = [torch.randn(c, h, d, device="cuda", generator=gen).bfloat16() for _ in range(3)]
    kinds = [2, 1, 3]
    o_acc = torch.empty(c, h, d, device="cuda")
    lse = torch.empty(h, c, device="cuda")
    out = torch.empty(c, h, d, device="cuda", dtype=torch.bfloat16)
    for i in range(3):
        ops.fwd_block(q, ks[i], vs[i], o_acc, lse, out, 0.1, kinds[i], i == 0, i == 2)
    torch.cuda.synchronize()
    # oracle: fold the three blocks into one accumulator (attention.py:296-328)
    qn = q.float().cpu().numpy().astype(np.float64) * 0.1
    st = R.Accum.fresh(c, h, d)
    for i in range(3):
        R.process_block(st, qn, ks[i].float().cpu().numpy().astype(np.float64),
                        vs[i].float().cpu().numpy().astype(np.float64), kinds[i], 128, 128)
    o_ref, lse_ref = R.finalize(st)
    assert np.max(np.abs(out.float().cpu().numpy() - o_ref)) <= O_MAX_ABS
    assert np.max(np.abs(lse.cpu().numpy() - lse_ref)) <= LSE_ABS


def test_fully_masked_step_keeps_state(ops):
    c, h, d = 256, 1, 64
    q, k, v = (torch.randn(c, h, d, device="cuda").bfloat16() for _ in range(3))
    o_acc = torch.empty(c, h, d, device="cuda")
    lse = torch.empty(h, c, device="cuda")
    out = torch.empty(c, h, d, device="cuda", dtype=torch.bfloat16)
    ops.fwd_block(q, k, v, o_acc, lse, out, 0.125, 2, True, False)
    lse0 = lse.clone()
    ops.fwd_block(q, k, v, o_acc, lse, out, 0.125, 0, False, True)  # SKIP on the last step
    torch.cuda.synchronize()
    out1, lse1, _ = run_block(ops, q, k, v, 2, 0.125)
    assert torch.equal(lse, lse0)
    assert np.array_equal(out.float().cpu().numpy(), out1)


@pytest.mark.parametrize("d", [128, 64])
@pytest.mark.parametrize("kind", [2, 1])
def test_extreme_and_growing_scores(ops, d, kind):
    """The reference's extreme-score stability test (tests/test_attention.py:289-305) at
    kernel scale: scores spanning hundreds (deep exp underflow, no inf / NaN), and scores
    that grow along the keys so the running max rises by far more than the lazy-rescale
    threshold in every 128-key tile (the O rescale path runs every step)."""
    c, h = 1024, 2
    g = torch.Generator(device="cuda").manual_seed(11 + d + kind)
    # (a) wide scores: |q.k| up to a few hundred
    q = (torch.rand(c, h, d, device="cuda", generator=g) * 10 - 5).bfloat16()
    k = (torch.rand(c, h, d, device="cuda", generator=g) * 10 - 5).bfloat16()
    v = torch.randn(c, h, d, device="cuda", generator=g).bfloat16()
    # (b) growing scores: s(x, y) = 0.5 y for every query
    qg = torch.ones(c, h, d, device="cuda").bfloat16()
    ramp = (0.5 * torch.arange(c, device="cuda", dtype=torch.float32) / d)[:, None, None]
    kg = (ramp * torch.ones(c, h, d, device="cuda")).bfloat16()
    for qq, kk in ((q, k), (qg, kg)):
        out, lse, _ = run_block(ops, qq, kk, v, kind, 1.0)
        assert np.isfinite(out).all() and np.isfinite(lse).all()
        o_ref, lse_ref = block_ref(qq.float().cpu().numpy(), kk.float().cpu().numpy(),
                                   v.float().cpu().numpy(), kind, 1.0)
        assert np.max(np.abs(out - o_ref)) <= O_MAX_ABS
        assert rel_l2(out, o_ref) <= O_REL_L2
        # relative LSE bound: the scores themselves reach hundreds
        assert np.max(np.abs(lse - lse_ref) / np.maximum(1.0, np.abs(lse_ref))) <= LSE_ABS
