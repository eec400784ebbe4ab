"""ringsim-shaped entry points backed by the GPU path (drop-in for the reference API).

``run_schedule_gpu(config, batch)`` mirrors ``ringsim.simulator.run_schedule``
(simulator.py:237-277) and ``simulate_gpu(config, inputs=None)`` mirrors ``simulate``
(simulator.py:358-368, returning a ``SimRun``): same argument objects (a ringsim ``SimConfig`` and
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


def _validate(config, scheme, n_seq_layout, n_dev_layout, n_shards, shard_shapes):
    """run_schedule's preconditions (simulator.py:237-260), same ValueErrors."""
    algo = _algo(config)
    n, n_seq, d = config.n_devices, config.n_seq, config.d_head
    c = n_seq // n
    if scheme != ("contiguous" if algo == "ring" else "striped"):
        raise ValueError(f"batch is partitioned {scheme}, but algo {algo} needs the other layout")
    if n_seq_layout != n_seq or n_dev_layout != n:
        raise ValueError("batch layout does not match the simulation config")
    if n_shards != n:
        raise ValueError(f"batch has {n_shards} shards, config wants {n}")
    for j, shp in enumerate(shard_shapes):
        if any(tuple(x) != (c, d) for x in shp):
            raise ValueError(f"device {j} shard shape mismatch (want block {c} x d_head {d})")
    if d not in (64, 128):
        raise ValueError("the GPU kernels support d_head 64 or 128")
    return algo, n, c


def _run_device_shards(config, algo, qs, ks, vs, n, c):
    """The N-round schedule on device shards [c, 1, d] bf16 -> (outs, WorkStats list)."""
    # the reference pre-scales q (simulator.py:365): the shards already carry it
    outs, _, kst = ring.virtual_ring_forward(qs, ks, vs, layout=algo, softmax_scale=1.0,
                                             count_tiles=True)
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
    return outs, stats


def _np_dtype(config):
    return np.float64 if getattr(config, "precision", "double") == "double" else np.float32


def run_schedule_gpu(config, batch, device: str = "cuda"):
    """GPU counterpart of run_schedule (simulator.py:237-277): a ringsim-shaped
    ``PermutedBatch`` (numpy shards) in, (outputs, stats) out, outputs in local order."""
    scheme = getattr(batch.layout.scheme, "value", batch.layout.scheme)
    algo, n, c = _validate(config, scheme, batch.layout.n_seq, batch.layout.n_devices,
                           len(batch.shards),
                           [(np.shape(sh.q), np.shape(sh.k), np.shape(sh.v))
                            for sh in batch.shards])
    to = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32,
                                   device=device).bfloat16()[:, None, :]
    qs = [to(sh.q) for sh in batch.shards]
    ks = [to(sh.k) for sh in batch.shards]
    vs = [to(sh.v) for sh in batch.shards]
    outs, stats = _run_device_shards(config, algo, qs, ks, vs, n, c)
    dtype = _np_dtype(config)
    return [o[:, 0].float().cpu().numpy().astype(dtype) for o in outs], stats


@dataclass
class SimRun:
    """simulator.py:344-355 (same fields): inputs, per-device results in local order,
    per-device WorkStats and the output reassembled in token order."""
    config: object
    q: np.ndarray
    k: np.ndarray
    v: np.ndarray
    layout: object
    outputs: list
    stats: list
    output: np.ndarray


def random_qkv(n_seq: int, d_head: int, seed: int, dtype=np.float64):
    """simulator.py:133-135: three standard-normal [n_seq, d_head] arrays, one seeded
    generator (the same draws as the reference)."""
    rng = np.random.default_rng(seed)
    return tuple(rng.standard_normal((n_seq, d_head), dtype=dtype) for _ in range(3))


def simulate_gpu(config, inputs=None, device: str = "cuda") -> SimRun:
    """GPU counterpart of simulate (simulator.py:358-368): generate (seeded
    ``random_qkv``, config.seed / config.dtype) or take (q, k, v) [n_seq, d_head], scale
    q when config.scale, partition with the K1 permute kernel, run the N rounds of the
    block kernels, gather with K1.  Returns a ``SimRun``."""
    from .layout import Layout
    algo = _algo(config)
    if inputs is None:
        dtype = getattr(config, "dtype", None) or _np_dtype(config)
        q, k, v = random_qkv(config.n_seq, config.d_head, getattr(config, "seed", 0), dtype)
    else:
        q, k, v = (np.asarray(x) for x in inputs)
    lay = Layout("contiguous" if algo == "ring" else "striped", config.n_seq, config.n_devices)
    q_in = q * q.dtype.type(1.0 / math.sqrt(config.d_head)) if getattr(config, "scale", False) \
        else q
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32,
                                    device=device).bfloat16()[:, None, :]
    batch = lay.partition(dev(q_in), dev(k), dev(v))  # K1 on the GPU
    _, n, c = _validate(config, lay.scheme.value, lay.n_seq, lay.n_devices, len(batch.shards),
                        [(tuple(sh.q.shape[::2]), tuple(sh.k.shape[::2]),
                          tuple(sh.v.shape[::2])) for sh in batch.shards])
    outs, stats = _run_device_shards(config, algo, [sh.q.contiguous() for sh in batch.shards],
                                     [sh.k.contiguous() for sh in batch.shards],
                                     [sh.v.contiguous() for sh in batch.shards], n, c)
    out_dtype = q.dtype if np.issubdtype(q.dtype, np.floating) else np.float64
    output = lay.gather(outs)[:, 0].float().cpu().numpy().astype(out_dtype)  # K1 inverse
    outputs = [o[:, 0].float().cpu().numpy().astype(out_dtype) for o in outs]
    return SimRun(config, q, k, v, lay, outputs, stats, output)
