"""Work / imbalance telemetry of the ring driver in the reference's CSV schema.

The reference writes one row per device per round with ``STATS_CSV_HEADER``
(cli.py:38-49, writer cli.py:125-146; rows ordered round-major, then device).  Here the
rows come from a real run: ``ring_forward(..., stats=RingStats(rank))`` records, per
round, the stripe held, the block mask kind, the tiles the kernel computed (its own
atomic counter) and the kernel's CUDA-event time.  The tile columns are the reference's
per-head census (attention.py:239-264) at the kernel's 128 x 128 tiles; the optional
extra columns carry what the simulator cannot know: heads, the kernel-counted tiles
(all heads) and the measured milliseconds.

``check_tile_counts`` is the work-accounting invariant of SURVEY.md section 8(f)2: the
tiles the kernels report equal heads x the census of the block's mask, every round.
``step_imbalance`` is the per-round max / mean of the ranks' kernel times (the
reference's critical path is the max, simulator.py:318-324).
"""

from __future__ import annotations

import csv
from dataclasses import dataclass
from typing import Iterable, Sequence

import torch.distributed as dist

from . import masks
from .ring import RingStats

STATS_CSV_HEADER = [
    "algo",
    "round",
    "device",
    "block_index",
    "tiles_total",
    "tiles_skipped",
    "tiles_partial",
    "tiles_full",
    "interactions_computed",
    "interactions_required",
]
EXTRA_COLUMNS = ["heads", "kernel_tiles_computed", "compute_ms"]


@dataclass(frozen=True)
class Run:
    """One ring run: layout ("striped" / "ring"), block size c, q heads, per-rank stats."""
    algo: str
    c: int
    heads: int
    stats: Sequence[RingStats]


def _row(run: Run, ws: RingStats, rec) -> list:
    cen = masks.kernel_tile_census(rec.mask_kind, run.c)
    t = masks.KERNEL_TILE
    return [run.algo, rec.round, ws.rank, rec.block_index, cen.n_total, cen.n_skip, cen.n_partial,
            cen.n_full, cen.n_computed * t * t, masks.useful_pairs(rec.mask_kind, run.c)]


def rows(runs: Iterable[Run], extra: bool = False) -> list[list]:
    out = []
    for run in runs:
        by_rank = sorted(run.stats, key=lambda s: s.rank)
        n_rounds = len(by_rank[0].rounds) if by_rank else 0
        for i in range(n_rounds):
            for ws in by_rank:
                rec = ws.rounds[i]
                r = _row(run, ws, rec)
                if extra:
                    r += [run.heads, rec.tiles_computed, f"{rec.compute_ms:.6f}"]
                out.append(r)
    return out


def write_stats_csv(path: str, runs: Iterable[Run], extra: bool = False) -> None:
    """The reference's stats CSV (header mandatory, UTF-8, newline-terminated rows);
    ``extra`` appends EXTRA_COLUMNS after the reference's ten."""
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(STATS_CSV_HEADER + (EXTRA_COLUMNS if extra else []))
        w.writerows(rows(runs, extra))


def check_tile_counts(run: Run) -> list[str]:
    """Rounds whose kernel tile count differs from heads x census (empty list = OK)."""
    bad = []
    for ws in run.stats:
        for rec in ws.rounds:
            want = run.heads * masks.kernel_tile_census(rec.mask_kind, run.c).n_computed
            if rec.tiles_computed != want:
                bad.append(f"rank {ws.rank} round {rec.round}: kernel {rec.tiles_computed} "
                           f"tiles, census {want}")
    return bad


def step_imbalance(stats: Sequence[RingStats]) -> list[float]:
    """Per round: max over ranks / mean over ranks of the measured kernel ms."""
    by_rank = sorted(stats, key=lambda s: s.rank)
    out = []
    for i in range(len(by_rank[0].rounds)):
        t = [ws.rounds[i].compute_ms for ws in by_rank]
        mean = sum(t) / len(t)
        out.append(max(t) / mean if mean > 0 else 1.0)
    return out


def gather_stats(stats: RingStats, group=None) -> list[RingStats]:
    """Every rank's RingStats on every rank (torch.distributed object all-gather)."""
    if not dist.is_initialized():
        return [stats]
    world = dist.get_world_size(group)
    out = [None] * world
    dist.all_gather_object(out, stats, group=group)
    return out
