"""Host-side block-mask selection and tile accounting (mirror of ringsim.attention).

These are the integer decisions the host makes before launching a block kernel:
which MaskKind a (query stripe j, key stripe k) pair gets, and how many 128x128
tiles the kernel will compute / skip.  The kernels re-derive the per-tile class
in-kernel with the same interval rule.  Reference: attention.py:42-52 (enums),
155-183 (block masks), 194-264 (tile classification / census).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

# MaskKind codes, same order as attention.py:42-46 and include/striped_attn.h.
FULLY_MASKED, FULLY_UNMASKED, CAUSAL_INCLUSIVE, CAUSAL_EXCLUSIVE = 0, 1, 2, 3

KERNEL_TILE = 128  # the block kernels' query/key tile edge


class MaskKind(enum.IntEnum):
    FULLY_MASKED = FULLY_MASKED
    FULLY_UNMASKED = FULLY_UNMASKED
    CAUSAL_INCLUSIVE = CAUSAL_INCLUSIVE
    CAUSAL_EXCLUSIVE = CAUSAL_EXCLUSIVE


class TileClass(enum.Enum):
    SKIP = "skip"
    PARTIAL = "partial"
    FULL = "full"


def _check(j: int, k: int, n_devices: int | None):
    if j < 0 or k < 0:
        raise ValueError(f"block indices must be non-negative, got j={j}, k={k}")
    if n_devices is not None and (j >= n_devices or k >= n_devices):
        raise ValueError(f"block indices j={j}, k={k} out of range for {n_devices} devices")


def get_mask_striped(j: int, k: int, n_devices: int | None = None) -> MaskKind:
    """attention.py:172-183: query stripe j vs key stripe k.  Local row x of stripe j
    is token j + x*N, column y of stripe k is k + y*N; allowed iff k + yN <= j + xN,
    i.e. y <= x when k <= j (inclusive) and y < x when k > j (strict)."""
    _check(j, k, n_devices)
    return MaskKind.CAUSAL_INCLUSIVE if k <= j else MaskKind.CAUSAL_EXCLUSIVE


def get_mask_ring(j: int, k: int, n_devices: int | None = None) -> MaskKind:
    """attention.py:155-169: contiguous blocks are all-or-nothing off the diagonal."""
    _check(j, k, n_devices)
    if k > j:
        return MaskKind.FULLY_MASKED
    return MaskKind.CAUSAL_INCLUSIVE if k == j else MaskKind.FULLY_UNMASKED


def block_mask(layout: str, j: int, k: int, n_devices: int | None = None) -> MaskKind:
    """simulator.py:138-141 (_block_mask): layout 'striped' or 'ring'."""
    if layout == "striped":
        return get_mask_striped(j, k, n_devices)
    if layout in ("ring", "contiguous"):
        return get_mask_ring(j, k, n_devices)
    raise ValueError(f"layout must be 'striped' or 'ring', got {layout!r}")


def classify_bounds(kind: int, r0: int, r1: int, c0: int, c1: int) -> TileClass:
    """attention.py:194-210 -- the same rule the kernels evaluate per 128x128 tile."""
    if kind == FULLY_MASKED:
        return TileClass.SKIP
    if kind == FULLY_UNMASKED:
        return TileClass.FULL
    if kind == CAUSAL_INCLUSIVE:
        if c1 - 1 <= r0:
            return TileClass.FULL
        if c0 > r1 - 1:
            return TileClass.SKIP
    else:
        if c1 <= r0:
            return TileClass.FULL
        if c0 >= r1 - 1:
            return TileClass.SKIP
    return TileClass.PARTIAL


@dataclass(frozen=True)
class TileCensus:
    n_full: int
    n_partial: int
    n_skip: int

    @property
    def n_total(self) -> int:
        return self.n_full + self.n_partial + self.n_skip

    @property
    def n_computed(self) -> int:
        return self.n_full + self.n_partial


def kernel_tile_census(kind: int, c: int, tile: int = KERNEL_TILE) -> TileCensus:
    """Tiles one head of a c x c block computes in the kernels (ragged edges round up).

    Equals attention.py:239-264 (tile_census) whenever tile divides c."""
    nt = -(-c // tile)
    full = partial = skip = 0
    for ti in range(nt):
        r0, r1 = ti * tile, (ti + 1) * tile
        for tj in range(nt):
            cls = classify_bounds(kind, r0, r1, tj * tile, (tj + 1) * tile)
            if cls is TileClass.FULL and (tj + 1) * tile > c:
                cls = TileClass.PARTIAL  # ragged last key tile carries a bound mask
            if cls is TileClass.FULL:
                full += 1
            elif cls is TileClass.PARTIAL:
                partial += 1
            else:
                skip += 1
    return TileCensus(full, partial, skip)


def useful_pairs(kind: int, c: int) -> int:
    """Allowed (q, k) pairs of a c x c block: MaskSpec.count_allowed (attention.py:97-118)."""
    if kind == FULLY_MASKED:
        return 0
    if kind == FULLY_UNMASKED:
        return c * c
    return c * (c + 1) // 2 if kind == CAUSAL_INCLUSIVE else c * (c - 1) // 2
