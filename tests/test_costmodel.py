"""CPU: the TMS cost model against values produced by the reference itself
(tests/golden/make_golden_tms.py -> tests/golden/tms.json)."""

import json
import os

import pytest

from paper_2311_09431_b200 import costmodel as C

with open(os.path.join(os.path.dirname(__file__), "golden", "tms.json")) as f:
    G = json.load(f)


def test_presets_match_reference():
    for name, vals in G["presets"].items():
        m = C.PRESETS[name]
        assert [m.n_vocab, m.d_model, m.d_ff, m.n_layer, m.n_head] == vals


def test_per_token_flops_match_reference():
    for name, v in G["per_token"].items():
        assert C.other_flops_per_token(C.PRESETS[name]) == pytest.approx(v["other"], rel=1e-15)
        assert C.attention_flops_per_token(C.PRESETS[name], 32768) == pytest.approx(v["attn_32k"],
                                                                                   rel=1e-15)


def test_reproduces_every_published_table_row():
    """Every row of the paper's table (as packaged by the reference): equal to the
    reference's unrounded value, and within the tables' 2-decimal rounding."""
    assert len(G["golden_rows"]) > 100
    for r in G["golden_rows"]:
        v = C.tms(C.PRESETS[r["model"]], r["n_seq"], r["mesh"][1], r["flop_weight"])
        assert v == pytest.approx(r["ref_tms"], rel=1e-12, abs=1e-12)
        assert abs(round(v, 2) - r["table_tms"]) <= C.TABLE_TOLERANCE + 1e-9, r


def test_extra_queries_and_table_match_reference():
    for r in G["extra"]:
        v = C.tms(C.PRESETS[r["model"]], r["n_seq"], r["sp"], r["flop_weight"])
        assert v == pytest.approx(r["ref_tms"], rel=1e-12)
    rows = C.tms_table(list(C.PRESETS.values()), [8192, 32768, 131072], [(1, 2), (2, 4), (1, 8)],
                       2.0)
    assert [(t.model, list(t.mesh), t.n_seq, t.tms) for t in rows] == \
        [(t["model"], t["mesh"], t["n_seq"], t["tms"]) for t in G["table"]]


def test_errors_mirror_reference():
    m = C.PRESETS["1b"]
    for bad in ((8192, 1, 2.0), (8192, 3, 2.0), (2, 4, 2.0), (8192, 2, 0.0)):
        with pytest.raises(ValueError):
            C.tms(m, *bad)
    with pytest.raises(ValueError):
        C.ModelPreset("x", 1, 0, 1, 1, 1)


def test_measured_tms_limits():
    """Measured form: equal attention times -> 1; no non-attention work -> the attention
    ratio; a 2x ring critical path with FLOP-proportional non-attention time matches the
    analytic model's structure."""
    m = C.PRESETS["7b"]
    assert C.measured_tms(m, 32768, 5.0, 5.0, 1000.0).tms == pytest.approx(1.0)
    r = C.measured_tms(m, 32768, 8.0, 4.0, 1e12)  # GEMMs ~free
    assert r.tms == pytest.approx(2.0, rel=1e-6)
    other = C.other_ms_per_layer(m, 32768, 1000.0)
    assert other == pytest.approx(C.other_flops_per_token(m) * 32768 * 3 / 1e15 * 1e3)
    with pytest.raises(ValueError):
        C.measured_tms(m, 32768, 0.0, 1.0, 1.0)
