"""One traced backward launch (perf build: SA_NVCC_EXTRA=-DSA_PERF_TRACE=1): prints the
clock64 timeline of CTA $SA_BWD_TRACE for its first 16 iterations (slots: see bwd.cu SA_TR).

    SA_LIB_PATH=abtest/lib_x.so SA_BWD_TRACE=0 python scripts/bwd_trace.py [--c 16384]
"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_09431_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--c", type=int, default=16384)
ap.add_argument("--h", type=int, default=32)
a = ap.parse_args()
q, k, v, do = (torch.randn(a.c, a.h, 128, device="cuda").bfloat16() for _ in range(4))
out = torch.empty_like(q)
lse = torch.empty(a.h, a.c, device="cuda")
s = 1 / math.sqrt(128)
ops.fwd_block(q, k, v, None, lse, out, s, 2, True, True)
dsum = torch.empty(a.h, a.c, device="cuda")
dq = torch.empty(a.c, a.h, 128, device="cuda")
dk, dv = torch.empty_like(q), torch.empty_like(q)
ops.bwd_preprocess(out, do, dsum, dq)
tr = os.environ.pop("SA_BWD_TRACE", None)
for _ in range(3):
    ops.bwd_block_final(q, k, v, do, lse, dsum, dq, dk, dv, s, 2)
torch.cuda.synchronize()
if tr is not None:
    os.environ["SA_BWD_TRACE"] = tr
ops.bwd_block_final(q, k, v, do, lse, dsum, dq, dk, dv, s, 2)
torch.cuda.synchronize()
