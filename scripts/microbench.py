"""Quick CUDA-event timing of the block kernels at cfg2 shape (seq 32k, 32 heads, D 128)."""
import argparse
import math
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_09431_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--c", type=int, default=32768)
ap.add_argument("--h", type=int, default=32)
ap.add_argument("--hkv", type=int, default=0)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--bwd", action="store_true")
ap.add_argument("--kinds", default="2,1")
a = ap.parse_args()
hkv = a.hkv or a.h
dev = "cuda"
q = torch.randn(a.c, a.h, a.d, device=dev).bfloat16()
k = torch.randn(a.c, hkv, a.d, device=dev).bfloat16()
v = torch.randn(a.c, hkv, a.d, device=dev).bfloat16()
out = torch.empty_like(q)
lse = torch.empty(a.h, a.c, device=dev)
scale = 1 / math.sqrt(a.d)
for kind in [int(x) for x in a.kinds.split(",")]:
    pairs = {1: a.c * a.c, 2: a.c * (a.c + 1) // 2, 3: a.c * (a.c - 1) // 2}[kind]
    flops = 4.0 * a.d * a.h * pairs
    for _ in range(3):
        ops.fwd_block(q, k, v, None, lse, out, scale, kind, True, True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        ops.fwd_block(q, k, v, None, lse, out, scale, kind, True, True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    print(f"fwd kind={kind} c={a.c} h={a.h} d={a.d}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s")
    if a.bwd:
        do = torch.randn_like(q)
        dsum = torch.empty(a.h, a.c, device=dev)
        dq = torch.empty(a.c, a.h, a.d, device=dev)
        dk = torch.zeros(a.c, hkv, a.d, device=dev)
        dv = torch.zeros(a.c, hkv, a.d, device=dev)
        ops.bwd_preprocess(out, do, dsum, dq)
        for _ in range(3):
            ops.bwd_block(q, k, v, do, lse, dsum, dq, dk, dv, scale, kind)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.iters):
            ops.bwd_block(q, k, v, do, lse, dsum, dq, dk, dv, scale, kind)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        print(f"bwd kind={kind}: {ms:.3f} ms  {2.5 * flops / ms / 1e9:.1f} TFLOP/s")
