"""Cost of running one ring round's backward in key parts (ring.kv_parts, so the dK/dV
hop of each part overlaps the later parts) against one launch, on one B200.

    python scripts/parts_probe.py [--c 32768 --h 32 --iters 10]
"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_09431_b200 import ops, ring  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--c", type=int, default=32768)
ap.add_argument("--h", type=int, default=32)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
dev = "cuda"
q, k, v, do = (torch.randn(a.c, a.h, 128, device=dev).bfloat16() for _ in range(4))
lse = torch.randn(a.h, a.c, device=dev).abs() + 10.0
dsum = torch.randn(a.h, a.c, device=dev)
dq = torch.zeros(a.c, a.h, 128, device=dev)
dk, dv = torch.zeros_like(dq), torch.zeros_like(dq)
s = 1 / math.sqrt(128)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.iters


for kind in (1, 3):
    one = timed(lambda: ops.bwd_block(q, k, v, do, lse, dsum, dq, dk, dv, s, kind))
    res = [f"kind {kind} c={a.c} h={a.h}: one launch {one:.3f} ms"]
    nt = -(-a.c // 128)
    r = lambda t: min(a.c, t * 128)
    splits = {"ring.kv_parts": ring.kv_parts(a.c),
              "3 parts (half, quarter, quarter)": [(r(nt // 2), a.c), (r(nt // 4), r(nt // 2)),
                                                   (0, r(nt // 4))]}
    for name, parts in splits.items():
        t = timed(lambda: [ops.bwd_block(q, k, v, do, lse, dsum, dq, dk, dv, s, kind,
                                         key_rows=rr) for rr in parts])
        res.append(f"{name} ({len(parts)}) {t:.3f} ms (+{(t / one - 1) * 100:.1f} %)")
    print(", ".join(res))
