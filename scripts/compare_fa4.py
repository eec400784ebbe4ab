"""COMPARATOR ONLY (not product, not the reference): time the image's vendored FlashAttention-4
CuTe-DSL kernels (vllm.vllm_flash_attn.cute, library code) on the same causal shape as
bench.py's configs[1] block, to calibrate how far our hand-written kernels are from a
state-of-the-art Blackwell implementation on this GPU and power cap.

    python scripts/compare_fa4.py [--seq 32768 --heads 32 --dim 128]
"""
import argparse
import math
import sys

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--dim", type=int, default=128)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()

from vllm.vllm_flash_attn.cute.interface import flash_attn_func  # noqa: E402

S, H, D = a.seq, a.heads, a.dim
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn(1, S, H, D, device="cuda", generator=g).bfloat16() for _ in range(4))
q.requires_grad_(True)
k.requires_grad_(True)
v.requires_grad_(True)
pairs = H * S * (S + 1) / 2
for _ in range(3):
    out = flash_attn_func(q, k, v, causal=True)
    out = out[0] if isinstance(out, tuple) else out
    out.backward(do)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
tf, tb = [], []
for _ in range(a.iters):
    e[0].record()
    out = flash_attn_func(q, k, v, causal=True)
    out = out[0] if isinstance(out, tuple) else out
    e[1].record()
    out.backward(do)
    e[2].record()
    torch.cuda.synchronize()
    tf.append(e[0].elapsed_time(e[1]))
    tb.append(e[1].elapsed_time(e[2]))
fm, bm = sorted(tf)[len(tf) // 2], sorted(tb)[len(tb) // 2]
print(f"FA4 (vendored, comparator) causal S={S} H={H} D={D}: fwd {fm:.3f} ms "
      f"{4 * D * pairs / fm / 1e9:.1f} TFLOP/s, bwd (incl. its pre/post kernels) {bm:.3f} ms "
      f"{10 * D * pairs / bm / 1e9:.1f} TFLOP/s")
sys.stdout.flush()
