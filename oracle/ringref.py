"""numpy restatement of the reference striped/ring attention path (TEST ORACLE).

See ``oracle/__init__.py``: test infrastructure only.  Multi-head tensors are
``[tokens, heads, d_head]`` (the product layout); the reference is single-head
``[tokens, d_head]`` (attention.py:10, attention.py:28-39) and is recovered with
``heads == 1``.  Grouped-query attention maps q-head ``h`` to kv-head
``h // (Hq // Hkv)`` (not in the reference).

Mask kinds use the reference's MaskKind order (attention.py:42-46) so the
integer codes are the ones the C ABI takes (include/striped_attn.h)::

    FULLY_MASKED = 0, FULLY_UNMASKED = 1, CAUSAL_INCLUSIVE = 2, CAUSAL_EXCLUSIVE = 3
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

FULLY_MASKED, FULLY_UNMASKED, CAUSAL_INCLUSIVE, CAUSAL_EXCLUSIVE = 0, 1, 2, 3
SKIP, PARTIAL, FULL = "skip", "partial", "full"  # TileClass, attention.py:49-52
CONTIGUOUS, STRIPED = "contiguous", "striped"    # Scheme, layout.py:20-22
RING, STRIPED_ALGO = "ring", "striped"           # Algo, simulator.py:43-45


# ----------------------------------------------------------------------------
# layout (layout.py)
# ----------------------------------------------------------------------------

def _check_layout(n_seq: int, n_dev: int) -> int:
    # layout.py:50-56 (Layout.__post_init__); N == 1 is allowed here because the
    # product supports single-GPU runs (no reference counterpart).
    if n_dev < 1:
        raise ValueError(f"need at least 1 device, got {n_dev}")
    if n_seq < n_dev or n_seq % n_dev:
        raise ValueError(f"{n_dev} devices must evenly divide sequence length {n_seq}")
    return n_seq // n_dev


def global_of(scheme: str, n_seq: int, n_dev: int, device: int, local: int) -> int:
    """layout.py:62-70: striped ``d + x*N``, contiguous ``d*c + x``."""
    c = _check_layout(n_seq, n_dev)
    if not (0 <= device < n_dev and 0 <= local < c):
        raise ValueError("device/local index out of range")
    return device * c + local if scheme == CONTIGUOUS else device + local * n_dev


def device_globals(scheme: str, n_seq: int, n_dev: int, device: int) -> np.ndarray:
    """layout.py:72-79: original positions owned by ``device`` in local order."""
    c = _check_layout(n_seq, n_dev)
    if not 0 <= device < n_dev:
        raise ValueError(f"device {device} out of range (N={n_dev})")
    x = np.arange(c, dtype=np.int64)
    return device * c + x if scheme == CONTIGUOUS else device + x * n_dev


def permutation(scheme: str, n_seq: int, n_dev: int) -> np.ndarray:
    """Concatenated device_globals: row p of the permuted sequence is token perm[p]."""
    return np.concatenate([device_globals(scheme, n_seq, n_dev, d) for d in range(n_dev)])


def partition(x, scheme: str, n_dev: int) -> list[np.ndarray]:
    """layout.py:81-101 for one tensor (Q, K, V or a companion array)."""
    x = np.asarray(x)
    return [x[device_globals(scheme, x.shape[0], n_dev, d)] for d in range(n_dev)]


def gather(shards, scheme: str) -> np.ndarray:
    """layout.py:103-117: exact inverse of ``partition``."""
    n_dev = len(shards)
    first = np.asarray(shards[0])
    n_seq = first.shape[0] * n_dev
    out = np.empty((n_seq,) + first.shape[1:], dtype=first.dtype)
    for d, sh in enumerate(shards):
        sh = np.asarray(sh)
        if sh.shape != first.shape:
            raise ValueError(f"shard {d} has shape {sh.shape}, expected {first.shape}")
        out[device_globals(scheme, n_seq, n_dev, d)] = sh
    return out


# ----------------------------------------------------------------------------
# masks and tiles (attention.py)
# ----------------------------------------------------------------------------

def striped_kind(j: int, k: int) -> int:
    """attention.py:172-183: key stripe k <= query stripe j -> inclusive, else strict."""
    return CAUSAL_INCLUSIVE if k <= j else CAUSAL_EXCLUSIVE


def ring_kind(j: int, k: int) -> int:
    """attention.py:155-169: k > j masked, k == j causal inclusive, k < j full."""
    if k > j:
        return FULLY_MASKED
    return CAUSAL_INCLUSIVE if k == j else FULLY_UNMASKED


def block_kind(scheme: str, j: int, k: int) -> int:
    """simulator.py:138-141 (_block_mask)."""
    return ring_kind(j, k) if scheme == CONTIGUOUS else striped_kind(j, k)


def allowed_block(kind: int, r0: int, r1: int, c0: int, c1: int) -> np.ndarray:
    """attention.py:83-92 (MaskSpec.allowed_block)."""
    if kind == FULLY_MASKED:
        return np.zeros((r1 - r0, c1 - c0), dtype=bool)
    if kind == FULLY_UNMASKED:
        return np.ones((r1 - r0, c1 - c0), dtype=bool)
    rows = np.arange(r0, r1)[:, None]
    cols = np.arange(c0, c1)[None, :]
    return cols <= rows if kind == CAUSAL_INCLUSIVE else cols < rows


def count_allowed(kind: int, r0: int, r1: int, c0: int, c1: int) -> int:
    """attention.py:97-118, restated as a per-row clamp sum in closed form."""
    if kind == FULLY_MASKED:
        return 0
    if kind == FULLY_UNMASKED:
        return (r1 - r0) * (c1 - c0)
    shift = 1 if kind == CAUSAL_INCLUSIVE else 0
    width = c1 - c0
    # row x allows clamp(x + shift - c0, 0, width) keys
    total = 0
    lo = max(r0, c0 - shift + 1)               # first row with >= 1 key
    sat = max(r0, c0 + width - shift)          # first saturated row
    hi = min(r1, sat)                          # rows [lo, hi) are on the slope
    if hi > lo:
        a, b = lo + shift - c0, hi - 1 + shift - c0
        total += (a + b) * (b - a + 1) // 2
    if r1 > sat:
        total += (r1 - sat) * width
    return total


def classify_bounds(kind: int, r0: int, r1: int, c0: int, c1: int) -> str:
    """attention.py:194-210 (_classify_bounds): interval test, no pair scan."""
    if kind == FULLY_MASKED:
        return SKIP
    if kind == FULLY_UNMASKED:
        return FULL
    if kind == CAUSAL_INCLUSIVE:
        if c1 - 1 <= r0:
            return FULL
        if c0 > r1 - 1:
            return SKIP
    else:
        if c1 <= r0:
            return FULL
        if c0 >= r1 - 1:
            return SKIP
    return PARTIAL


def classify_tiles(kind: int, rows: int, cols: int, tile_q: int, tile_k: int):
    """attention.py:213-225."""
    if rows % tile_q or cols % tile_k:
        raise ValueError("tile does not divide block")
    return [[classify_bounds(kind, ti * tile_q, (ti + 1) * tile_q, tj * tile_k, (tj + 1) * tile_k)
             for tj in range(cols // tile_k)] for ti in range(rows // tile_q)]


@dataclass(frozen=True)
class Census:
    n_full: int
    n_partial: int
    n_skip: int

    @property
    def n_total(self) -> int:
        return self.n_full + self.n_partial + self.n_skip


def tile_census(kind: int, rows: int, cols: int, tile_q: int, tile_k: int) -> Census:
    """attention.py:239-264, counted directly from classify_bounds per tile row."""
    if rows % tile_q or cols % tile_k:
        raise ValueError("tile does not divide block")
    gc = cols // tile_k
    full = skip = 0
    for ti in range(rows // tile_q):
        r0, r1 = ti * tile_q, (ti + 1) * tile_q
        if kind == FULLY_MASKED:
            skip += gc
            continue
        if kind == FULLY_UNMASKED:
            full += gc
            continue
        if kind == CAUSAL_INCLUSIVE:
            nf = (r0 + 1) // tile_k
            fs = (r1 - 1) // tile_k + 1
        else:
            nf = r0 // tile_k
            fs = (r1 - 2 + tile_k) // tile_k
        full += min(nf, gc)
        skip += gc - min(fs, gc)
    total = (rows // tile_q) * gc
    return Census(full, total - full - skip, skip)


# ----------------------------------------------------------------------------
# streaming softmax (attention.py:267-336)
# ----------------------------------------------------------------------------

@dataclass
class Accum:
    """SoftmaxAccumulator (attention.py:267-293) for every head of one block.

    acc [rows, H, Dv] unnormalised, m [H, rows] running max (-inf), l [H, rows]."""

    acc: np.ndarray
    m: np.ndarray
    l: np.ndarray

    @classmethod
    def fresh(cls, rows: int, heads: int, dv: int, dtype=np.float64) -> "Accum":
        return cls(np.zeros((rows, heads, dv), dtype), np.full((heads, rows), -np.inf, dtype),
                   np.zeros((heads, rows), dtype))


def _fold(acc, m, l, rows, scores, v_tile):
    """attention.py:321-328: carry = exp(m_old - m_new), p = exp(s - m_new)."""
    m_old = m[rows]
    m_new = np.maximum(m_old, scores.max(axis=1))
    carry = np.exp(m_old - m_new)
    p = np.exp(scores - m_new[:, None])
    acc[rows] = acc[rows] * carry[:, None] + p @ v_tile
    l[rows] = l[rows] * carry + p.sum(axis=1)
    m[rows] = m_new


def accumulate_tile(acc, m, l, q_tile, k_tile, v_tile, allowed=None):
    """attention.py:296-318 for one head: masked scores are -inf and rows with
    no allowed key are left untouched bit for bit."""
    scores = q_tile @ k_tile.T
    if allowed is not None and not allowed.all():
        scores[~allowed] = -np.inf
        live = allowed.any(axis=1)
        if not live.all():
            if live.any():
                _fold(acc, m, l, live, scores[live], v_tile)
            return
    _fold(acc, m, l, slice(None), scores, v_tile)


def process_block(state: Accum, q, k, v, kind: int, tile_q: int, tile_k: int, r_off=0):
    """simulator.py:144-186 (_process_round) for all heads: classify, row-major
    tile loop, accumulate.  q is already scaled (simulator.py:365).  Returns
    (n_full, n_partial, n_skip, computed, required) for ONE head."""
    c_q, hq, _ = q.shape
    c_k, hkv, _ = k.shape
    group = hq // hkv
    grid = classify_tiles(kind, c_q, c_k, tile_q, tile_k)
    nf = np_ = ns = comp = req = 0
    for ti, row in enumerate(grid):
        r0, r1 = ti * tile_q, (ti + 1) * tile_q
        for tj, cls in enumerate(row):
            if cls == SKIP:
                ns += 1
                continue
            c0, c1 = tj * tile_k, (tj + 1) * tile_k
            req += count_allowed(kind, r0, r1, c0, c1)
            comp += tile_q * tile_k
            allowed = None
            if cls == PARTIAL:
                np_ += 1
                allowed = allowed_block(kind, r0, r1, c0, c1)
            else:
                nf += 1
            for h in range(hq):
                accumulate_tile(state.acc[r0:r1, h], state.m[h, r0:r1], state.l[h, r0:r1],
                                q[r0:r1, h], k[c0:c1, h // group], v[c0:c1, h // group], allowed)
    return nf, np_, ns, comp, req


def finalize(state: Accum, allow_dead: bool = False):
    """attention.py:331-336 plus the LSE the reference leaves implicit (m + ln l).

    Returns (o [rows, H, Dv], lse [H, rows]).  A row with l == 0 is dead: the
    reference raises; with ``allow_dead`` (per-step block outputs) it gets o = 0
    and lse = -inf, the identity of the LSE merge."""
    dead = state.l == 0
    if dead.any() and not allow_dead:
        h, r = np.argwhere(dead)[0]
        raise ValueError(f"query row attended no keys (head {h}, row {r})")
    with np.errstate(divide="ignore", invalid="ignore"):
        lse = np.where(dead, -np.inf, state.m + np.log(np.where(dead, 1.0, state.l)))
        o = state.acc / np.where(dead, 1.0, state.l).T[:, :, None]
    return o, lse


def merge(o_a, lse_a, o_b, lse_b):
    """LSE merge of two partial softmax results (same rows): -inf safe.

    Equivalent to folding both key sets into one SoftmaxAccumulator
    (attention.py:321-328); not a reference function."""
    lse = np.logaddexp(lse_a, lse_b)
    with np.errstate(invalid="ignore"):
        wa = np.where(np.isneginf(lse_a), 0.0, np.exp(lse_a - lse))
        wb = np.where(np.isneginf(lse_b), 0.0, np.exp(lse_b - lse))
    return o_a * wa.T[:, :, None] + o_b * wb.T[:, :, None], lse


# ----------------------------------------------------------------------------
# ring schedule (simulator.py)
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class RoundStats:
    """simulator.py:92-103."""
    round: int
    block_index: int
    tiles_total: int
    tiles_skipped: int
    tiles_partial: int
    tiles_full: int
    interactions_computed: int
    interactions_required: int


@dataclass
class WorkStats:
    device: int
    rounds: list = field(default_factory=list)


def _as3(x):
    x = np.asarray(x)
    return x[:, None, :] if x.ndim == 2 else x


def ring_forward(q, k, v, n_dev: int, scheme: str, softmax_scale: float,
                 tile_q: int = 128, tile_k: int = 128, dtype=np.float64):
    """simulate() (simulator.py:358-368) with _run_serial (189-198), all heads.

    Inputs are global ``[S, H, D]`` in token order.  Returns
    (o [S,Hq,Dv], lse [Hq,S], stats) in token order."""
    q, k, v = (_as3(x).astype(dtype) for x in (q, k, v))
    n_seq = q.shape[0]
    c = _check_layout(n_seq, n_dev)
    tq, tk = min(tile_q, c), min(tile_k, c)
    qs = partition(q * dtype(softmax_scale), scheme, n_dev)
    ks = partition(k, scheme, n_dev)
    vs = partition(v, scheme, n_dev)
    states = [Accum.fresh(c, q.shape[1], v.shape[2], dtype) for _ in range(n_dev)]
    stats = [WorkStats(j) for j in range(n_dev)]
    held = list(range(n_dev))  # held_index starts at j (simulator.py:265)
    for i in range(n_dev):
        for j in range(n_dev):
            kk = held[j]
            kind = block_kind(scheme, j, kk)
            nf, np_, ns, comp, req = process_block(states[j], qs[j], ks[kk], vs[kk], kind, tq, tk)
            stats[j].rounds.append(RoundStats(i, kk, nf + np_ + ns, ns, np_, nf, comp, req))
        held = [held[(j - 1) % n_dev] for j in range(n_dev)]  # simulator.py:195-197
    outs = [finalize(s) for s in states]
    o = gather([o for o, _ in outs], scheme)
    lse = gather([l.T for _, l in outs], scheme).T
    return o, lse, stats


def schedule_work_stats(scheme: str, n_dev: int, c: int, tile_q: int, tile_k: int):
    """simulator.py:280-315 (closed form via tile_census)."""
    out = []
    for j in range(n_dev):
        ws = WorkStats(j)
        for i in range(n_dev):
            kk = (j - i) % n_dev
            kind = block_kind(scheme, j, kk)
            cen = tile_census(kind, c, c, tile_q, tile_k)
            ws.rounds.append(RoundStats(i, kk, cen.n_total, cen.n_skip, cen.n_partial, cen.n_full,
                                        (cen.n_full + cen.n_partial) * tile_q * tile_k,
                                        count_allowed(kind, 0, c, 0, c)))
        out.append(ws)
    return out


def round_critical_path(stats, i: int) -> int:
    """simulator.py:318-324."""
    return max(ws.rounds[i].interactions_computed for ws in stats)


def simulated_speedup(ring_stats, striped_stats) -> float:
    """simulator.py:327-341."""
    n = len(ring_stats)
    return (sum(round_critical_path(ring_stats, i) for i in range(n))
            / sum(round_critical_path(striped_stats, i) for i in range(n)))


# ----------------------------------------------------------------------------
# dense forward / backward (oracle_causal_attention, attention.py:121-143)
# ----------------------------------------------------------------------------

def dense_forward(q, k, v, softmax_scale: float, dtype=np.float64):
    """attention.py:121-143 for every head, plus LSE.  Returns (o, lse[H,S])."""
    q, k, v = (_as3(x).astype(dtype) for x in (q, k, v))
    n, hq, _ = q.shape
    group = hq // k.shape[1]
    tril = np.tril(np.ones((n, n), dtype=bool))
    o = np.empty((n, hq, v.shape[2]), dtype)
    lse = np.empty((hq, n), dtype)
    for h in range(hq):
        s = (q[:, h] * dtype(softmax_scale)) @ k[:, h // group].T
        s[~tril] = -np.inf
        m = s.max(axis=1, keepdims=True)
        p = np.exp(s - m)
        z = p.sum(axis=1, keepdims=True)
        o[:, h] = (p @ v[:, h // group]) / z
        lse[h] = (m + np.log(z))[:, 0]
    return o, lse


def dense_backward(q, k, v, do, softmax_scale: float, dtype=np.float64):
    """NOT REFERENCE (no backward exists in ringsim).  fp64 gradients
    of the causal forward above:  P = softmax(scale*QK^T + mask),
    dV = P^T dO,  dP = dO V^T,  dS = P o (dP - rowsum(dO o O)),
    dQ = scale * dS K,  dK = scale * dS^T Q  (summed over a GQA group)."""
    q, k, v, do = (_as3(x).astype(dtype) for x in (q, k, v, do))
    n, hq, _ = q.shape
    hkv = k.shape[1]
    group = hq // hkv
    tril = np.tril(np.ones((n, n), dtype=bool))
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    for h in range(hq):
        g = h // group
        s = (q[:, h] @ k[:, g].T) * dtype(softmax_scale)
        s[~tril] = -np.inf
        p = np.exp(s - s.max(axis=1, keepdims=True))
        p /= p.sum(axis=1, keepdims=True)
        o = p @ v[:, g]
        dsum = (do[:, h] * o).sum(axis=1, keepdims=True)
        dp = do[:, h] @ v[:, g].T
        ds = p * (dp - dsum)
        dv[:, g] += p.T @ do[:, h]
        dq[:, h] = dtype(softmax_scale) * (ds @ k[:, g])
        dk[:, g] += dtype(softmax_scale) * (ds.T @ q[:, h])
    return dq, dk, dv


def block_backward(q, k, v, do, lse, dsum, kind: int, softmax_scale: float, dtype=np.float64,
                   key_rows=None):
    """NOT REFERENCE.  One (rank, step) block of the ring backward: recompute
    P = exp(scale*QK^T - lse) under the block mask (same predicate as the
    forward, attention.py:172-183) with the GLOBAL lse, and return this block's
    (dq, dk, dv) contributions.  q/do/lse/dsum belong to the query stripe,
    k/v to the held key stripe.  ``key_rows=(r0, r1)`` keeps only the keys in
    [r0, r1) (the product's per-part backward launches)."""
    q, k, v, do = (_as3(x).astype(dtype) for x in (q, k, v, do))
    c_q, hq, _ = q.shape
    c_k, hkv, _ = k.shape
    group = hq // hkv
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    if kind == FULLY_MASKED:
        return dq, dk, dv
    allowed = allowed_block(kind, 0, c_q, 0, c_k)
    if key_rows is not None:
        keep = np.zeros(c_k, dtype=bool)
        keep[key_rows[0]:key_rows[1]] = True
        allowed = allowed & keep[None, :]
    for h in range(hq):
        g = h // group
        s = (q[:, h] @ k[:, g].T) * dtype(softmax_scale)
        with np.errstate(invalid="ignore"):
            p = np.where(allowed, np.exp(s - lse[h][:, None]), 0.0)
        dp = do[:, h] @ v[:, g].T
        ds = p * (dp - dsum[h][:, None])
        dv[:, g] += p.T @ do[:, h]
        dq[:, h] = dtype(softmax_scale) * (ds @ k[:, g])
        dk[:, g] += dtype(softmax_scale) * (ds.T @ q[:, h])
    return dq, dk, dv


def ring_backward(q, k, v, do, o, lse, n_dev: int, scheme: str, softmax_scale: float,
                  dtype=np.float64):
    """NOT REFERENCE.  The ring backward the product runs: dK/dV accumulators
    travel with their K/V block (same rotation as simulator.py:194-197) and
    arrive home after N hops.  Global token-order in and out."""
    q, k, v, do, o = (_as3(x).astype(dtype) for x in (q, k, v, do, o))
    dsum = np.einsum("shd,shd->hs", do, o)
    qs, ks, vs, dos = (partition(x, scheme, n_dev) for x in (q, k, v, do))
    lses = [x.T for x in partition(lse.T, scheme, n_dev)]
    dss = [x.T for x in partition(dsum.T, scheme, n_dev)]
    dq = [np.zeros_like(x) for x in qs]
    dk = [np.zeros_like(x) for x in ks]   # dk[b] travels with block b
    dv = [np.zeros_like(x) for x in vs]
    for i in range(n_dev):
        for j in range(n_dev):
            kk = (j - i) % n_dev
            a, b, cc = block_backward(qs[j], ks[kk], vs[kk], dos[j], lses[j], dss[j],
                                      block_kind(scheme, j, kk), softmax_scale, dtype)
            dq[j] += a
            dk[kk] += b
            dv[kk] += cc
    return gather(dq, scheme), gather(dk, scheme), gather(dv, scheme)


def bf16_round(x) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32 (for feeding the
    oracle the same values the GPU sees)."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(a.shape)


def useful_flops_fwd_bwd(n_seq: int, hq: int, d: int) -> float:
    """14*D FLOPs per useful causal (q,k) pair per q-head,
    pairs = Hq*S(S+1)/2  ->  7*D*Hq*S*(S+1)."""
    return 7.0 * d * hq * n_seq * (n_seq + 1)


def useful_flops_fwd(n_seq: int, hq: int, d: int) -> float:
    return 2.0 * d * hq * n_seq * (n_seq + 1)


def tiled_causal_backward(q, k, v, do, o, lse, softmax_scale: float, tile: int = 512,
                          dtype=np.float32):
    """NOT REFERENCE.  Flash-style tiled causal backward for one head ([S, D] arrays),
    O(S * tile) memory: the CPU counterpart of the GPU kernel used only as the
    ``bench.py`` CPU baseline (the reference has no backward).  lse is [S]."""
    q, k, v, do, o = (np.asarray(x, dtype=dtype) for x in (q, k, v, do, o))
    lse = np.asarray(lse, dtype=dtype)
    n = q.shape[0]
    dsum = (do * o).sum(axis=1)
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    sc = dtype(softmax_scale)
    for c0 in range(0, n, tile):
        c1 = min(n, c0 + tile)
        kt, vt = k[c0:c1], v[c0:c1]
        for r0 in range(c0 - c0 % tile, n, tile):
            r1 = min(n, r0 + tile)
            s = (q[r0:r1] @ kt.T) * sc
            p = np.exp(s - lse[r0:r1, None])
            if r0 < c1:  # diagonal tile: y <= x
                p[np.arange(c0, c1)[None, :] > np.arange(r0, r1)[:, None]] = 0
            dv[c0:c1] += p.T @ do[r0:r1]
            ds = p * (do[r0:r1] @ vt.T - dsum[r0:r1, None])
            dq[r0:r1] += sc * (ds @ kt)
            dk[c0:c1] += sc * (ds.T @ q[r0:r1])
    return dq, dk, dv


def tiled_causal_forward(q, k, v, softmax_scale: float, tile: int = 512, dtype=np.float32):
    """The reference's streaming-softmax forward (attention.py:296-328 via
    simulator.py:144-186) for one head, causal, row-major tiles.  Returns (o, lse)."""
    q, k, v = (np.asarray(x, dtype=dtype) for x in (q, k, v))
    st = Accum.fresh(q.shape[0], 1, v.shape[1], dtype)
    process_block(st, (q * dtype(softmax_scale))[:, None], k[:, None], v[:, None],
                  CAUSAL_INCLUSIVE, tile, tile)
    o, lse = finalize(st)
    return o[:, 0], lse[0]
