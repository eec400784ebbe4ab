"""Training-step speedup of striped over ring attention (TMS), analytic and measured.

SURVEY.md section 8(f)4.  The reference's analytic model (``ringsim.costmodel``,
costmodel.py:65-128) counts per-token, per-layer matmul FLOPs of a decoder transformer:
everything outside attention (projections 8 d^2, a two-matrix MLP 4 d d_ff, the vocabulary
projection amortised over layers 2 d V / L, costmodel.py:65-73) plus the pairwise
attention work 4 n d (costmodel.py:76-79), weighted by ``flop_weight`` (attention run in a
costlier precision).  The critical path of a causal step keeps a fraction of the
unmasked attention work: (sp - 1/2) / sp on the ring schedule (costmodel.py:82-88), 1/2 on
the striped one (costmodel.py:91).  TMS is the ratio of the two weighted totals
(costmodel.py:115-127); the paper's tables (``data/tms_appendix.csv``) are reproduced
within the 2-decimal rounding they were printed with (``tests/test_costmodel.py``).

``measured_tms`` replaces the attention side by MEASURED B200 times: the ring and
striped per-step critical paths from ``bench.py`` (max over ranks, CUDA events), and
the non-attention side by its FLOPs at a measured dense-GEMM rate (MEASURED_PEAKS.json),
so the prediction reflects this implementation rather than an idealised FLOP count.
"""

from __future__ import annotations

from dataclasses import dataclass

TABLE_DECIMALS = 2
TABLE_TOLERANCE = 0.02  # the published tables print 2 decimals (costmodel.py:26)


@dataclass(frozen=True)
class ModelPreset:
    """Decoder hyper-parameters the FLOP model needs (costmodel.py:29-44)."""
    name: str
    n_vocab: int
    d_model: int
    d_ff: int
    n_layer: int
    n_head: int

    def __post_init__(self):
        for f in ("n_vocab", "d_model", "d_ff", "n_layer", "n_head"):
            if getattr(self, f) < 1:
                raise ValueError(f"{f} must be positive")

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_head


# costmodel.py:47-51 (Llama-style 1B / 3B / 7B)
PRESETS = {
    "1b": ModelPreset("1b", 32000, 2048, 5504, 22, 16),
    "3b": ModelPreset("3b", 32000, 3200, 8640, 26, 32),
    "7b": ModelPreset("7b", 32000, 4096, 11008, 32, 32),
}


def other_flops_per_token(m: ModelPreset) -> float:
    """Non-attention matmul FLOPs per token per layer (costmodel.py:65-73)."""
    d = float(m.d_model)
    return 8.0 * d * d + 4.0 * d * m.d_ff + 2.0 * d * m.n_vocab / m.n_layer


def attention_flops_per_token(m: ModelPreset, n_seq: int) -> float:
    """Unmasked pairwise FLOPs per token per layer: scores + value contraction
    (costmodel.py:76-79)."""
    return 4.0 * n_seq * m.d_model


def ring_critical_fraction(sp: int) -> float:
    """Share of the unmasked attention work on the ring schedule's critical path: round 0
    half-masked, every later round pinned by a full block (costmodel.py:82-88)."""
    if sp < 2:
        raise ValueError(f"sp must be at least 2, got {sp}")
    return (sp - 0.5) / sp


STRIPED_CRITICAL_FRACTION = 0.5  # costmodel.py:91


def _check(n_seq: int, sp: int, flop_weight: float):
    if sp < 2:
        raise ValueError(f"sp must be at least 2, got {sp}")
    if n_seq < sp or n_seq % sp:
        raise ValueError(f"sp={sp} must divide n_seq={n_seq}")
    if flop_weight <= 0:
        raise ValueError(f"flop_weight must be positive, got {flop_weight}")


def tms(m: ModelPreset, n_seq: int, sp: int, flop_weight: float = 2.0) -> float:
    """Analytic best-case striped-over-ring speedup of a training step, unrounded
    (costmodel.py:115-127: communication fully hidden, FLOP-proportional time)."""
    _check(n_seq, sp, flop_weight)
    other = other_flops_per_token(m)
    attn = flop_weight * attention_flops_per_token(m, n_seq)
    return (other + attn * ring_critical_fraction(sp)) / (other + attn * STRIPED_CRITICAL_FRACTION)


@dataclass(frozen=True)
class TableRow:
    model: str
    mesh: tuple  # (model-parallel label, sequence-parallel degree); mp is only a label
    n_seq: int
    tms: float   # rounded to TABLE_DECIMALS


def tms_table(models, seq_lens, meshes, flop_weight: float = 2.0) -> list:
    """One row per (model, mesh, n_seq), in that nesting order (costmodel.py:138-147)."""
    rows = []
    for m in models:
        for mp, sp in meshes:
            for n in seq_lens:
                rows.append(TableRow(m.name, (mp, sp), n, round(tms(m, n, sp, flop_weight),
                                                             TABLE_DECIMALS)))
    return rows


def other_ms_per_layer(m: ModelPreset, tokens: int, gemm_tflops: float,
                       passes: float = 3.0) -> float:
    """Non-attention time of one layer for ``tokens`` tokens at a dense-GEMM rate:
    FLOPs x passes (fwd + bwd = 3 x fwd) / rate."""
    return other_flops_per_token(m) * tokens * passes / (gemm_tflops * 1e12) * 1e3


@dataclass(frozen=True)
class MeasuredTms:
    tms: float
    other_ms: float
    attn_ring_ms: float
    attn_striped_ms: float


def measured_tms(m: ModelPreset, tokens_per_rank: int, attn_ring_ms: float,
                 attn_striped_ms: float, gemm_tflops: float) -> MeasuredTms:
    """Training-step speedup from measured per-layer attention critical paths (fwd+bwd,
    max over ranks) and the non-attention FLOPs at a measured GEMM rate; all heads of the
    layer are in the attention times."""
    if attn_ring_ms <= 0 or attn_striped_ms <= 0 or gemm_tflops <= 0:
        raise ValueError("times and rates must be positive")
    other = other_ms_per_layer(m, tokens_per_rank, gemm_tflops)
    return MeasuredTms((other + attn_ring_ms) / (other + attn_striped_ms), other, attn_ring_ms,
                       attn_striped_ms)
