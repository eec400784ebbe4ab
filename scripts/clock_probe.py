"""Backward block timing with the SM clock sampled during the timed loop (is the kernel
power-capped, and does removing a traffic source raise the clock?).

    SA_LIB_PATH=... [SA_BWD_DEBUG=8] python scripts/clock_probe.py [--c 65536 --iters 20]
"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402
from paper_2311_09431_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--c", type=int, default=65536)
ap.add_argument("--h", type=int, default=32)
ap.add_argument("--hkv", type=int, default=0)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--fwd", action="store_true", help="time the forward block instead")
a = ap.parse_args()
dev = "cuda"
hkv = a.hkv or a.h
q, do = (torch.randn(a.c, a.h, 128, device=dev).bfloat16() for _ in range(2))
k, v = (torch.randn(a.c, hkv, 128, device=dev).bfloat16() for _ in range(2))
out = torch.empty_like(q)
lse = torch.empty(a.h, a.c, device=dev)
s = 1 / math.sqrt(128)
ops.fwd_block(q, k, v, None, lse, out, s, 2, True, True)
dsum = torch.empty(a.h, a.c, device=dev)
dq = torch.empty(a.c, a.h, 128, device=dev)
dk, dv = torch.empty_like(k), torch.empty_like(v)
ops.bwd_preprocess(out, do, dsum, dq)
for _ in range(3):
    ops.bwd_block_final(q, k, v, do, lse, dsum, dq, dk, dv, s, 2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
step = (lambda: ops.fwd_block(q, k, v, None, lse, out, s, 2, True, True)) if a.fwd else \
    (lambda: ops.bwd_block_final(q, k, v, do, lse, dsum, dq, dk, dv, s, 2))
for _ in range(2):
    step()
torch.cuda.synchronize()
with ClockSampler(0) as clk:
    e0.record()
    for _ in range(a.iters):
        step()
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
flops = (4 if a.fwd else 10) * 128 * a.h * a.c * (a.c + 1) / 2
dbg = os.environ.get("SA_FWD_DEBUG" if a.fwd else "SA_BWD_DEBUG", "0")
print(f"{'fwd' if a.fwd else 'bwd'} c={a.c} debug={dbg}: {ms:.3f} ms "
      f"{flops / ms / 1e9:.1f} TFLOP/s  clocks {clk.summary()}")
