"""Generate golden vectors by running the REFERENCE itself (ringsim).

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports ``ringsim`` from /root/reference/pkg/src (read-only), evaluates the
reference's own functions on seeded inputs and writes ``tests/golden/*.npz`` /
``*.json``.  The committed fixtures pin ``oracle/ringref.py`` (CPU tests) and
the CUDA path (GPU tests) to the reference's outputs.

Inputs are rounded to bfloat16 first (values exactly representable in bf16,
stored as float32) so the GPU consumes bit-identical inputs; the reference then
runs on their float64 upcast with ``precision="double", scale=True``.
LSE is read from the reference accumulator as ``m + ln l`` after
``simulator._run_serial``; finalize() does not mutate state.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from ringsim import attention as A  # noqa: E402
from ringsim import layout as L  # noqa: E402
from ringsim import simulator as S  # noqa: E402

from oracle.ringref import bf16_round  # noqa: E402

KIND = {A.MaskKind.FULLY_MASKED: 0, A.MaskKind.FULLY_UNMASKED: 1,
        A.MaskKind.CAUSAL_INCLUSIVE: 2, A.MaskKind.CAUSAL_EXCLUSIVE: 3}


def ref_forward_with_lse(algo, n_dev, q, k, v, tile):
    """One head through the reference: (O, LSE, stats) in token order."""
    n_seq, d = q.shape
    cfg = S.SimConfig(algo=algo, n_devices=n_dev, n_seq=n_seq, d_head=d, tile_q=tile, tile_k=tile,
                      precision="double", scale=True)
    run = S.simulate(cfg, inputs=(q, k, v))
    # LSE: rebuild the device states exactly as run_schedule does (simulator.py:261-272)
    layout = S.make_layout(cfg)
    batch = layout.partition(q * (1.0 / math.sqrt(d)), k, v)
    devs = [S.DeviceState(j, sh.q, j, sh.k, sh.v, A.SoftmaxAccumulator.fresh(cfg.block_size, d),
                          S.WorkStats(j)) for j, sh in enumerate(batch.shards)]
    outs = S._run_serial(cfg, devs)
    lse = layout.gather([dv.acc.m + np.log(dv.acc.l) for dv in devs])
    o2 = layout.gather(outs)
    assert np.array_equal(o2, run.output)
    return run.output, lse, run.stats


def stats_to_list(stats):
    return [[[r.round, r.block_index, r.tiles_total, r.tiles_skipped, r.tiles_partial, r.tiles_full,
              r.interactions_computed, r.interactions_required] for r in ws.rounds] for ws in stats]


def forward_case(name, algo, n_dev, n_seq, heads, d, tile, seed):
    rng = np.random.default_rng(seed)
    q, k, v = (bf16_round(rng.standard_normal((n_seq, heads, d))) for _ in range(3))
    o = np.empty((n_seq, heads, d))
    lse = np.empty((heads, n_seq))
    stats = None
    for h in range(heads):
        o[:, h], lse[h], st = ref_forward_with_lse(algo, n_dev, q[:, h].astype(np.float64),
                                                   k[:, h].astype(np.float64),
                                                   v[:, h].astype(np.float64), tile)
        stats = stats_to_list(st)
    np.savez_compressed(os.path.join(HERE, f"fwd_{name}.npz"), q=q, k=k, v=v, o=o, lse=lse,
                        stats=np.array(stats, dtype=np.int64),
                        meta=np.array([n_dev, n_seq, heads, d, tile, seed]),
                        algo=np.array(algo))


def block_case(name, n_dev, c, d, j, seed):
    """Per-(rank, step) block outputs of the reference's _process_round on a
    fresh accumulator, for every round of rank j (striped)."""
    rng = np.random.default_rng(seed)
    n_seq = c * n_dev
    q, k, v = (bf16_round(rng.standard_normal((n_seq, d))).astype(np.float64) for _ in range(3))
    cfg = S.SimConfig(algo="striped", n_devices=n_dev, n_seq=n_seq, d_head=d, tile_q=c, tile_k=c,
                      precision="double", scale=True)
    layout = S.make_layout(cfg)
    batch = layout.partition(q * (1.0 / math.sqrt(d)), k, v)
    accs, ms, ls = [], [], []
    for i in range(n_dev):
        kk = (j - i) % n_dev
        dev = S.DeviceState(j, batch.shards[j].q, kk, batch.shards[kk].k, batch.shards[kk].v,
                            A.SoftmaxAccumulator.fresh(c, d), S.WorkStats(j))
        S._process_round(cfg, dev, i)
        accs.append(dev.acc.acc)
        ms.append(dev.acc.m)
        ls.append(dev.acc.l)
    np.savez_compressed(os.path.join(HERE, f"block_{name}.npz"), q=q.astype(np.float32),
                        k=k.astype(np.float32), v=v.astype(np.float32), acc=np.array(accs),
                        m=np.array(ms), l=np.array(ls), meta=np.array([n_dev, c, d, j, seed]))


def tables():
    out = {}
    # layout maps (layout.py:62-79)
    out["layout"] = []
    for scheme in (L.Scheme.CONTIGUOUS, L.Scheme.STRIPED):
        for n_dev, n_seq in ((2, 4), (2, 16), (4, 16), (8, 64), (3, 12), (8, 8)):
            lay = L.Layout(scheme, n_seq, n_dev)
            out["layout"].append({"scheme": scheme.value, "n_dev": n_dev, "n_seq": n_seq,
                                  "globals": [lay.device_globals(d).tolist() for d in range(n_dev)]})
    # block masks (attention.py:155-183)
    out["masks"] = []
    for n_dev in (2, 3, 4, 8):
        for j in range(n_dev):
            for kk in range(n_dev):
                out["masks"].append({"n_dev": n_dev, "j": j, "k": kk,
                                     "striped": KIND[A.get_mask_striped(j, kk, 4).kind],
                                     "ring": KIND[A.get_mask_ring(j, kk, 4).kind]})
    # materialised masks and allowed counts
    out["allowed"] = []
    for kind in A.MaskKind:
        for c in (1, 2, 3, 5, 8):
            spec = A.MaskSpec(kind, c, c)
            out["allowed"].append({"kind": KIND[kind], "c": c,
                                   "mask": spec.materialize().astype(int).tolist(),
                                   "count": spec.count_allowed()})
    # tile census and sub-block counts (attention.py:97-118, 239-264)
    out["census"] = []
    for kind in A.MaskKind:
        for c, tq, tk in ((1536, 512, 512), (16, 4, 8), (32768, 128, 128), (256, 128, 128),
                          (384, 128, 128), (24, 6, 4), (12, 1, 1)):
            spec = A.MaskSpec(kind, c, c)
            cen = A.tile_census(spec, tq, tk)
            grid = A.classify_tiles(spec, tq, tk) if c <= 4096 else None
            sub = [[spec.count_allowed(ti * tq, (ti + 1) * tq, tj * tk, (tj + 1) * tk)
                    for tj in range(c // tk)] for ti in range(c // tq)] if c <= 1536 else None
            out["census"].append({"kind": KIND[kind], "c": c, "tq": tq, "tk": tk,
                                  "full": cen.n_full, "partial": cen.n_partial, "skip": cen.n_skip,
                                  "grid": None if grid is None else
                                  [[g.value for g in row] for row in grid],
                                  "sub_counts": sub})
    # closed-form schedule stats and speedups (simulator.py:280-341)
    out["schedule"] = []
    for n_dev, c, tq, tk in ((4, 8, 1, 1), (4, 16, 2, 2), (8, 32768, 128, 128), (2, 131072, 128, 128),
                             (4, 65536, 128, 128), (8, 65536, 128, 128), (8, 98304, 128, 128),
                             (4, 1024, 1, 1), (8, 32768, 2048, 4096)):
        ring = S.schedule_work_stats(S.Algo.RING, n_dev, c, tq, tk)
        strp = S.schedule_work_stats(S.Algo.STRIPED, n_dev, c, tq, tk)
        out["schedule"].append({"n_dev": n_dev, "c": c, "tq": tq, "tk": tk,
                                "ring": stats_to_list(ring), "striped": stats_to_list(strp),
                                "speedup": S.simulated_speedup(ring, strp)})
    # oracle known-answer tests (tests/test_attention.py:28-43 shapes)
    q = np.array([[3.0, -1.0]])
    kk = np.array([[0.5, 2.0]])
    v = np.array([[7.0, 8.0]])
    out["kat_single"] = A.oracle_causal_attention(q, kk, v).tolist()
    with open(os.path.join(HERE, "tables.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))


def main():
    tables()
    forward_case("striped_n4_s512_h2_d128", "striped", 4, 512, 2, 128, 32, 1)
    forward_case("ring_n4_s512_h2_d128", "ring", 4, 512, 2, 128, 32, 1)
    forward_case("striped_n2_s512_h2_d64", "striped", 2, 512, 2, 64, 64, 2)
    forward_case("striped_n3_s600_h1_d64", "striped", 3, 600, 1, 64, 40, 3)   # ragged c=200
    forward_case("striped_n4_s16_h1_d64", "striped", 4, 16, 1, 64, 2, 4)      # tiny c=4
    forward_case("ring_n8_s1024_h1_d128", "ring", 8, 1024, 1, 128, 128, 5)
    forward_case("striped_n8_s1024_h1_d128", "striped", 8, 1024, 1, 128, 128, 5)
    block_case("striped_n4_c256_d128_j1", 4, 256, 128, 1, 6)
    print("golden written to", HERE)


if __name__ == "__main__":
    main()
