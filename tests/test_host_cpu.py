"""CPU tests of the product's host logic and the C-ABI library surface (no GPU needed)."""

import ctypes

import numpy as np
import os
import re

import pytest
import torch

from oracle import ringref as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_host_masks_match_reference_tables(tables):
    from paper_2311_09431_b200 import masks
    for case in tables["masks"]:
        assert int(masks.get_mask_striped(case["j"], case["k"], case["n_dev"])) == case["striped"]
        assert int(masks.get_mask_ring(case["j"], case["k"], case["n_dev"])) == case["ring"]
    with pytest.raises(ValueError):
        masks.get_mask_striped(4, 0, 4)
    with pytest.raises(ValueError):
        masks.block_mask("zigzag", 0, 0)


def test_host_tile_classification_matches_reference(tables):
    from paper_2311_09431_b200 import masks
    for case in tables["census"]:
        if case["grid"] is None:
            continue
        tq, tk = case["tq"], case["tk"]
        for ti, row in enumerate(case["grid"]):
            for tj, cls in enumerate(row):
                got = masks.classify_bounds(case["kind"], ti * tq, (ti + 1) * tq, tj * tk,
                                            (tj + 1) * tk)
                assert got.value == cls


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
@pytest.mark.parametrize("c", [128, 256, 32768, 100, 300, 1])
def test_kernel_tile_census(kind, c):
    from paper_2311_09431_b200 import masks
    cen = masks.kernel_tile_census(kind, c)
    if c % 128 == 0:
        ref = R.tile_census(kind, c, c, 128, 128)
        assert (cen.n_full, cen.n_partial, cen.n_skip) == (ref.n_full, ref.n_partial, ref.n_skip)
    nt = -(-c // 128)
    assert cen.n_total == nt * nt
    assert masks.useful_pairs(kind, c) == R.count_allowed(kind, 0, c, 0, c)


def test_striped_rounds_are_balanced_at_kernel_tiles():
    """attention.py:239-264 at 128x128: inclusive and strict census identical for aligned
    blocks, so every striped round computes the same number of tiles on every rank."""
    from paper_2311_09431_b200 import masks
    for c in (128, 1024, 32768):
        a = masks.kernel_tile_census(masks.CAUSAL_INCLUSIVE, c)
        b = masks.kernel_tile_census(masks.CAUSAL_EXCLUSIVE, c)
        assert (a.n_full, a.n_partial, a.n_skip) == (b.n_full, b.n_partial, b.n_skip)


def test_layout_host_arithmetic(tables):
    from paper_2311_09431_b200 import Layout
    for case in tables["layout"]:
        lay = Layout(case["scheme"], case["n_seq"], case["n_dev"])
        for d, want in enumerate(case["globals"]):
            assert lay.device_globals(d).tolist() == want
            assert [lay.global_of(d, x) for x in range(lay.block_size)] == want
    with pytest.raises(ValueError):
        Layout("striped", 16, 3)
    with pytest.raises(ValueError):
        Layout("striped", 16, 4).global_of(4, 0)


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "striped_attn.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|int64_t)\s+(sa_\w+)\(", hdr, re.M)))


def test_c_abi_library_exports_every_declared_symbol():
    from paper_2311_09431_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2311_09431_b200 import build
        build.build()
    so = ctypes.CDLL(_lib.LIB_PATH)
    syms = _declared_symbols()
    assert len(syms) >= 9
    for s in syms:
        assert hasattr(so, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes binding out of sync with the header"
    lib = _lib.lib()
    assert lib.sa_abi_version() == 1


def test_c_abi_rejects_bad_arguments_without_launching():
    from paper_2311_09431_b200 import _lib
    lib = _lib.lib()
    # invalid arguments return > 0 before touching the device
    assert lib.sa_permute(None, None, 16, 3, 4, 1, 0, -1, None) > 0
    assert lib.sa_permute(1, 1, 16, 4, 6, 1, 0, -1, None) > 0          # row_bytes % 4
    assert lib.sa_fwd_block(16, 16, 16, None, 16, 16, 128, 2, 2, 96, 0.1, 2, 1, 1, None, None) > 0
    assert b"head dim" in lib.sa_last_error()
    assert lib.sa_fwd_block(16, 16, 16, None, 16, 16, 128, 3, 2, 128, 0.1, 2, 1, 1, None, None) > 0
    assert lib.sa_fwd_block(16, 16, 16, None, 16, 16, 128, 2, 2, 128, 0.1, 7, 1, 1, None, None) > 0
    assert lib.sa_bwd_block(16, 16, 16, 16, 16, 16, 16, 16, 16, 128, 2, 2, 128, -1.0, 2, None) > 0
    # misaligned operands / outputs (vector epilogue, TMA) are rejected before any launch
    assert lib.sa_fwd_block(18, 16, 16, None, 16, 16, 128, 2, 2, 128, 0.1, 2, 1, 1, None, None) > 0
    assert lib.sa_fwd_block(16, 16, 16, 20, 16, 16, 128, 2, 2, 128, 0.1, 2, 0, 1, None, None) > 0
    assert b"aligned" in lib.sa_last_error()
    assert lib.sa_fwd_block(16, 16, 16, None, 16, 24, 128, 2, 2, 128, 0.1, 2, 1, 1, None, None) > 0
    assert lib.sa_bwd_block(16, 16, 16, 16, 16, 16, 16, 20, 16, 128, 2, 2, 128, 0.1, 2, None) > 0
    assert b"aligned" in lib.sa_last_error()
    # sa_bwd_block_ex: exactly one dK/dV pair, whole range for bf16 outputs, aligned rows
    ex = lib.sa_bwd_block_ex
    assert ex(16, 16, 16, 16, 16, 16, 16, None, None, None, None, 256, 2, 2, 128, 0.1, 2, 0, -1,
              None, None) > 0
    assert b"dk_acc" in lib.sa_last_error()
    assert ex(16, 16, 16, 16, 16, 16, 16, 16, 16, 16, None, 256, 2, 2, 128, 0.1, 2, 0, -1,
              None, None) > 0
    assert ex(16, 16, 16, 16, 16, 16, 16, None, None, 16, 16, 256, 2, 2, 128, 0.1, 2, 128, -1,
              None, None) > 0
    assert b"whole key range" in lib.sa_last_error()
    assert ex(16, 16, 16, 16, 16, 16, 16, 16, 16, None, None, 256, 2, 2, 128, 0.1, 2, 64, -1,
              None, None) > 0
    assert b"128-aligned" in lib.sa_last_error()
    # copy / IPC helpers reject null arguments without touching the device
    assert lib.sa_memcpy_async(None, 16, 64, None) > 0
    assert lib.sa_ipc_mem_handle(None, None, None) > 0
    assert lib.sa_ipc_event_open(None, None) > 0
    assert lib.sa_event_record(None, None) > 0


def test_product_has_no_cpu_fallback():
    from paper_2311_09431_b200 import ops
    x = torch.zeros(128, 1, 64, dtype=torch.bfloat16)
    lse = torch.zeros(1, 128)
    with pytest.raises(ValueError, match="CUDA"):
        ops.fwd_block(x, x, x, None, lse, x, 0.1, 2, True, True)
    from paper_2311_09431_b200 import striped_attn_forward
    with pytest.raises(ValueError, match="CUDA"):
        striped_attn_forward(x, x, x)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2311_09431_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
                assert "oracle/" not in src.replace("oracle/ ", ""), f


def test_telemetry_csv_matches_reference_schema_and_oracle(tmp_path):
    """Rows of a (virtual, oracle-backed) ring run in the reference CSV schema
    (cli.py:38-49) equal the oracle's schedule_work_stats (simulator.py:280-315) at the
    kernel's 128 x 128 tiles; the kernel-counted tiles pass the census check."""
    import csv as _csv
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from cpu_blockops import OracleBlockOps
    from paper_2311_09431_b200 import ring, telemetry

    n_dev, c, hq, d = 4, 256, 2, 8
    rng = np.random.default_rng(3)
    for layout, scheme in (("striped", R.STRIPED), ("ring", R.CONTIGUOUS)):
        qs, ks, vs = ([torch.tensor(rng.standard_normal((c, hq, d))) for _ in range(n_dev)]
                      for _ in range(3))
        _, _, stats = ring.virtual_ring_forward(qs, ks, vs, layout=layout, softmax_scale=0.2,
                                                block_ops=OracleBlockOps(), count_tiles=True)
        run = telemetry.Run(layout, c, hq, stats)
        assert telemetry.check_tile_counts(run) == []
        path = tmp_path / f"{layout}.csv"
        telemetry.write_stats_csv(str(path), [run], extra=True)
        with open(path, encoding="utf-8") as fh:
            table = list(_csv.reader(fh))
        assert table[0] == telemetry.STATS_CSV_HEADER + telemetry.EXTRA_COLUMNS
        want = R.schedule_work_stats(scheme, n_dev, c, 128, 128)
        body = table[1:]
        assert len(body) == n_dev * n_dev
        for row in body:
            i, dev = int(row[1]), int(row[2])
            rs = want[dev].rounds[i]
            assert [int(x) for x in row[3:10]] == [rs.block_index, rs.tiles_total, rs.tiles_skipped,
                                                   rs.tiles_partial, rs.tiles_full,
                                                   rs.interactions_computed,
                                                   rs.interactions_required]
            assert int(row[11]) == hq * (rs.tiles_full + rs.tiles_partial)
        # a wrong count is reported
        stats[0].rounds[0].tiles_computed += 1
        assert len(telemetry.check_tile_counts(run)) == 1
