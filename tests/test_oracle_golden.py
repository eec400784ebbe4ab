"""Pin the CPU oracle (oracle/ringref.py) to golden vectors produced by the
reference itself (tests/golden/make_golden.py ran ringsim).  CPU only."""

import numpy as np
import pytest

from oracle import ringref as R
from conftest import golden_forward_cases, load_golden


def test_layout_maps_match_reference(tables):
    for case in tables["layout"]:
        for d, want in enumerate(case["globals"]):
            got = R.device_globals(case["scheme"], case["n_seq"], case["n_dev"], d)
            assert got.tolist() == want
            for x, g in enumerate(want):
                assert R.global_of(case["scheme"], case["n_seq"], case["n_dev"], d, x) == g


def test_block_masks_match_reference(tables):
    for case in tables["masks"]:
        assert R.striped_kind(case["j"], case["k"]) == case["striped"]
        assert R.ring_kind(case["j"], case["k"]) == case["ring"]


def test_allowed_blocks_and_counts_match_reference(tables):
    for case in tables["allowed"]:
        c = case["c"]
        assert R.allowed_block(case["kind"], 0, c, 0, c).astype(int).tolist() == case["mask"]
        assert R.count_allowed(case["kind"], 0, c, 0, c) == case["count"]


def test_tile_census_and_sub_counts_match_reference(tables):
    for case in tables["census"]:
        cen = R.tile_census(case["kind"], case["c"], case["c"], case["tq"], case["tk"])
        assert (cen.n_full, cen.n_partial, cen.n_skip) == (case["full"], case["partial"], case["skip"])
        if case["grid"] is not None:
            grid = R.classify_tiles(case["kind"], case["c"], case["c"], case["tq"], case["tk"])
            assert grid == case["grid"]
        if case["sub_counts"] is not None:
            tq, tk = case["tq"], case["tk"]
            for ti, row in enumerate(case["sub_counts"]):
                for tj, want in enumerate(row):
                    got = R.count_allowed(case["kind"], ti * tq, (ti + 1) * tq, tj * tk, (tj + 1) * tk)
                    assert got == want


def test_schedule_stats_and_speedup_match_reference(tables):
    for case in tables["schedule"]:
        for scheme, key in ((R.CONTIGUOUS, "ring"), (R.STRIPED, "striped")):
            stats = R.schedule_work_stats(scheme, case["n_dev"], case["c"], case["tq"], case["tk"])
            got = [[[r.round, r.block_index, r.tiles_total, r.tiles_skipped, r.tiles_partial,
                     r.tiles_full, r.interactions_computed, r.interactions_required]
                    for r in ws.rounds] for ws in stats]
            assert got == case[key]
        ring = R.schedule_work_stats(R.CONTIGUOUS, case["n_dev"], case["c"], case["tq"], case["tk"])
        strp = R.schedule_work_stats(R.STRIPED, case["n_dev"], case["c"], case["tq"], case["tk"])
        assert R.simulated_speedup(ring, strp) == pytest.approx(case["speedup"], rel=1e-15)


def test_kat_single_token(tables):
    o, lse = R.dense_forward(np.array([[3.0, -1.0]]), np.array([[0.5, 2.0]]),
                             np.array([[7.0, 8.0]]), softmax_scale=1.0)
    assert o[:, 0].tolist() == tables["kat_single"]
    assert lse[0, 0] == pytest.approx(3.0 * 0.5 - 2.0)


@pytest.mark.parametrize("name", golden_forward_cases())
def test_ring_forward_matches_reference(name):
    g = load_golden(name)
    n_dev, n_seq, heads, d, tile, _ = g["meta"].tolist()
    scheme = R.STRIPED if str(g["algo"]) == "striped" else R.CONTIGUOUS
    o, lse, stats = R.ring_forward(g["q"], g["k"], g["v"], n_dev, scheme, 1.0 / np.sqrt(d),
                                   tile_q=tile, tile_k=tile)
    assert np.max(np.abs(o - g["o"])) <= 1e-12
    assert np.max(np.abs(lse - g["lse"])) <= 1e-12
    got = [[[r.round, r.block_index, r.tiles_total, r.tiles_skipped, r.tiles_partial, r.tiles_full,
             r.interactions_computed, r.interactions_required] for r in ws.rounds] for ws in stats]
    assert got == g["stats"].tolist()
    # and the dense oracle agrees (N-independent ground truth)
    od, lsed = R.dense_forward(g["q"], g["k"], g["v"], 1.0 / np.sqrt(d))
    assert np.max(np.abs(od - g["o"])) <= 1e-12
    assert np.max(np.abs(lsed - g["lse"])) <= 1e-12


def test_per_step_block_state_matches_reference():
    g = load_golden("block_striped_n4_c256_d128_j1.npz")
    n_dev, c, d, j, _ = g["meta"].tolist()
    q, k, v = (g[x].astype(np.float64) for x in ("q", "k", "v"))
    qs = R.partition(q[:, None, :] / np.sqrt(d), R.STRIPED, n_dev)
    ks = R.partition(k[:, None, :], R.STRIPED, n_dev)
    vs = R.partition(v[:, None, :], R.STRIPED, n_dev)
    for i in range(n_dev):
        kk = (j - i) % n_dev
        st = R.Accum.fresh(c, 1, d)
        R.process_block(st, qs[j], ks[kk], vs[kk], R.striped_kind(j, kk), c, c)
        assert np.max(np.abs(st.acc[:, 0] - g["acc"][i])) <= 1e-12
        np.testing.assert_array_equal(np.isneginf(st.m[0]), np.isneginf(g["m"][i]))
        fin = np.isfinite(g["m"][i])
        assert np.max(np.abs(st.m[0][fin] - g["m"][i][fin])) <= 1e-12
        assert np.max(np.abs(st.l[0] - g["l"][i])) <= 1e-12
        if kk > j:  # strict step: local row 0 is dead (l == 0, m == -inf)
            assert g["l"][i][0] == 0 and np.isneginf(g["m"][i][0])


def test_merge_of_step_states_equals_full_ring():
    g = load_golden("block_striped_n4_c256_d128_j1.npz")
    n_dev, c, d, j, _ = g["meta"].tolist()
    o_acc, lse_acc = None, None
    for i in range(n_dev):
        st = R.Accum(g["acc"][i][:, None, :].copy(), g["m"][i][None].copy(), g["l"][i][None].copy())
        o, lse = R.finalize(st, allow_dead=True)
        o_acc, lse_acc = (o, lse) if o_acc is None else R.merge(o_acc, lse_acc, o, lse)
    q, k, v = (g[x].astype(np.float64) for x in ("q", "k", "v"))
    od, lsed = R.dense_forward(q, k, v, 1.0 / np.sqrt(d))
    rows = R.device_globals(R.STRIPED, c * n_dev, n_dev, j)
    assert np.max(np.abs(o_acc - od[rows])) <= 1e-12
    assert np.max(np.abs(lse_acc[0] - lsed[0, rows])) <= 1e-12


def test_partition_gather_roundtrip_with_companions():
    x = np.arange(8 * 3).reshape(8, 3)
    pos = np.arange(8)
    for scheme in (R.STRIPED, R.CONTIGUOUS):
        for n in (1, 2, 4, 8):
            sh = R.partition(x, scheme, n)
            assert np.array_equal(R.gather(sh, scheme), x)
            assert np.array_equal(R.gather(R.partition(pos, scheme, n), scheme), pos)
    assert R.partition(pos, R.STRIPED, 2)[1].tolist() == [1, 3, 5, 7]


def test_bf16_round_is_rne():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, -2.5e-3, 3.0e38], dtype=np.float32)
    import torch
    want = torch.tensor(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(R.bf16_round(x), want)
