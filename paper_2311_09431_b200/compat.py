"""ringsim-shaped entry points backed by the GPU path (drop-in for the reference API).

``run_schedule_gpu(config, batch)`` mirrors ``ringsim.simulator.run_schedule``
(simulator.py:237-277) and ``simulate_gpu(config, inputs)`` mirrors ``simulate``
(simulator.py:358-368): same argument objects (a ringsim ``SimConfig`` and
``PermutedBatch``, or anything with the same attributes), same preconditions and
``ValueError``s, same return shapes -- per-device outputs in local order plus per-device
``WorkStats`` -- so the reference's own property tests can target the GPU backend.

Differences, by design of the hot path: arithmetic is bf16 in / fp32 accumulate on the
GPU (the reference is fp64 / fp32 numpy), d_head must be 64 or 128, and the kernels
classify 128 x 128 tiles (the work counters below are still reported at the config's
tile_q x tile_k with the reference's own rule, attention.py:194-264).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import masks, ring


@dataclass(frozen=True)
class RoundStats:
    """simulator.py:92-103 (same fields), plus the kernel's own 128-tile count."""
    round: int
    block_index: int
    tiles_total: int
    tiles_skipped: int
    tiles_partial: int
    tiles_full: int
    interactions_computed: int
    interactions_required: int
    kernel_tiles_computed: int = 0


@dataclass
class WorkStats:
    device: int
    rounds: list = field(default_factory=list)


def _algo(config) -> str:
    a = getattr(config.algo, "value", config.algo)
    if a not in ("ring", "striped"):
        raise ValueError(f"unknown algo {a!r}")
    return a


def _census(kind: int, c: int, tq: int, tk: int):
    """tile_census (attention.py:239-264) via the interval rule, any tile size."""
    full = partial = skip = 0
    for ti in range(c // tq):
        for tj in range(c // tk):
            cls = masks.classify_bounds(kind, ti * tq, (ti + 1) * tq, tj * tk, (tj + 1) * tk)
            if cls is masks.TileClass.FULL:
                full += 1
            elif cls is masks.TileClass.PARTIAL:
                partial += 1
            else:
                skip += 1
    return full, partial, skip


def run_schedule_gpu(config, batch, device: str = "cuda"):
    """GPU counterpart of run_schedule: returns (outputs, stats) in local order."""
    algo = _algo(config)
    n, n_seq, d = config.n_devices, config.n_seq, config.d_head
    c = n_seq // n
    scheme = getattr(batch.layout.scheme, "value", batch.layout.scheme)
    if scheme != ("contiguous" if algo == "ring" else "striped"):
        raise ValueError(f"batch is partitioned {scheme}, but algo {algo} needs the other layout")
    if batch.layout.n_seq != n_seq or batch.layout.n_devices != n:
        raise ValueError("batch layout does not match the simulation config")
    if len(batch.shards) != n:
        raise ValueError(f"batch has {len(batch.shards)} shards, config wants {n}")
    for j, sh in enumerate(batch.shards):
        if np.shape(sh.q) != (c, d) or np.shape(sh.k) != (c, d) or np.shape(sh.v) != (c, d):
            raise ValueError(f"device {j} shard shape mismatch (want block {c} x d_head {d})")
    if d not in (64, 128):
        raise ValueError("the GPU kernels support d_head 64 or 128")
    to = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32,
                                   device=device).bfloat16()[:, None, :]
    qs = [to(sh.q) for sh in batch.shards]
    ks = [to(sh.k) for sh in batch.shards]
    vs = [to(sh.v) for sh in batch.shards]
    # the reference pre-scales q (simulator.py:365): the batch already carries it
    outs, _, kst = ring.virtual_ring_forward(qs, ks, vs, layout=algo, softmax_scale=1.0,
                                             count_tiles=True)
    dtype = np.float64 if getattr(config, "precision", "double") == "double" else np.float32
    outputs = [o[:, 0].float().cpu().numpy().astype(dtype) for o in outs]
    stats = []
    tq, tk = config.tile_q, config.tile_k
    for j in range(n):
        ws = WorkStats(j)
        for r in kst[j].rounds:
            full, partial, skip = _census(r.mask_kind, c, tq, tk)
            ws.rounds.append(RoundStats(r.round, r.block_index, full + partial + skip, skip,
                                        partial, full, (full + partial) * tq * tk,
                                        masks.useful_pairs(r.mask_kind, c), r.tiles_computed))
        stats.append(ws)
    return outputs, stats


def simulate_gpu(config, inputs):
    """GPU counterpart of simulate (simulator.py:358-368) for given (q, k, v) [n_seq, d]
    token-order arrays: scale, partition, run, gather.  Returns (output, outputs, stats)."""
    from .layout import Layout
    algo = _algo(config)
    q, k, v = (np.asarray(x, dtype=np.float64) for x in inputs)
    if getattr(config, "scale", False):
        q = q * (1.0 / math.sqrt(config.d_head))
    lay = Layout("contiguous" if algo == "ring" else "striped", config.n_seq, config.n_devices)

    @dataclass(frozen=True)
    class _Shard:
        q: np.ndarray
        k: np.ndarray
        v: np.ndarray

    @dataclass(frozen=True)
    class _Batch:
        layout: Layout
        shards: list

    shards = [_Shard(*(x[lay.device_globals(dv).numpy()] for x in (q, k, v)))
              for dv in range(config.n_devices)]
    outputs, stats = run_schedule_gpu(config, _Batch(lay, shards))
    out = np.empty((config.n_seq, config.d_head), dtype=outputs[0].dtype)
    for dv, o in enumerate(outputs):
        out[lay.device_globals(dv).numpy()] = o
    return out, outputs, stats
