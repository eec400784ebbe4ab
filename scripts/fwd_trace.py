"""One traced forward launch of the CTA-pair kernel (perf build: SA_NVCC_EXTRA=-DSA_PERF_TRACE=1):
prints the clock64 timeline of pair 0's leader for its first 16 kv tiles (slots: fwd_pair.cu SA_TR).

    SA_LIB_PATH=abtest/lib_perf.so SA_FWD_PAIR_TRACE=1 python scripts/fwd_trace.py [--c 16384]
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
q, k, v = (torch.randn(a.c, a.h, 128, device="cuda").bfloat16() for _ in range(3))
out = torch.empty_like(q)
lse = torch.empty(a.h, a.c, device="cuda")
tr = os.environ.pop("SA_FWD_PAIR_TRACE", None)
for _ in range(3):
    ops.fwd_block(q, k, v, None, lse, out, 1 / math.sqrt(128), 2, True, True)
torch.cuda.synchronize()
if tr is not None:
    os.environ["SA_FWD_PAIR_TRACE"] = tr
ops.fwd_block(q, k, v, None, lse, out, 1 / math.sqrt(128), 2, True, True)
torch.cuda.synchronize()
