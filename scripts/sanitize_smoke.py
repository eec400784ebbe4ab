"""Small launches of every product kernel, for compute-sanitizer (one tool per run):

    compute-sanitizer --tool memcheck  python scripts/sanitize_smoke.py
    compute-sanitizer --tool racecheck python scripts/sanitize_smoke.py
    compute-sanitizer --tool synccheck python scripts/sanitize_smoke.py

Covers: K1 permute (both directions), the CTA-pair forward (D = 128) and the 1-CTA forward
(D = 64) with ragged blocks and all mask kinds, the LSE merge across steps, the backward
(accumulating, final bf16, key-range parts, deterministic dQ), the casts, and a 2-rank
threaded ring through ring_forward / ring_backward (copy-engine hops)."""

import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_09431_b200 import api, ops, ring  # noqa: E402
from paper_2311_09431_b200.layout import Layout  # noqa: E402


def main():
    torch.manual_seed(0)
    dev = "cuda"
    # K1
    x = torch.randn(1000, 2, 64, device=dev).bfloat16()
    lay = Layout("striped", 1000, 4)
    assert torch.equal(lay.unpermute(lay.permute(x)), x)
    for d, c, hq, hkv in ((128, 300, 2, 1), (64, 260, 2, 2), (128, 512, 4, 2)):
        mk = lambda h: torch.randn(c, h, d, device=dev).bfloat16()
        q, k, v, do = mk(hq), mk(hkv), mk(hkv), mk(hq)
        s = 1 / math.sqrt(d)
        for kind in (1, 2, 3):
            o_acc = torch.zeros(c, hq, d, device=dev)
            lse = torch.empty(hq, c, device=dev)
            out = torch.empty(c, hq, d, device=dev).bfloat16()
            ops.fwd_block(q, k, v, o_acc, lse, out, s, kind, True, False)
            ops.fwd_block(q, k, v, o_acc, lse, out, s, 2, False, True)
        out, lse = api.striped_attn_forward(q, k, v)
        api.striped_attn_backward(do, q, k, v, out, lse)
        api.striped_attn_backward(do, q, k, v, out, lse, deterministic=True)
        dsum = torch.empty(hq, c, device=dev)
        dq = torch.empty(c, hq, d, device=dev)
        dk = torch.zeros(c, hkv, d, device=dev)
        dv = torch.zeros(c, hkv, d, device=dev)
        ops.bwd_preprocess(out, do, dsum, dq)
        for r0, r1 in ring.kv_parts(c):
            ops.bwd_block(q, k, v, do, lse, dsum, dq, dk, dv, s, 3, key_rows=(r0, r1))
    torch.cuda.synchronize()

    # 2-rank threaded ring (side streams, copy-engine hops, 3-part dK/dV hops, fused)
    n, h, d = 1024, 2, 128
    qs = [torch.randn(n // 2, h, d, device=dev).bfloat16() for _ in range(4)]

    def rank_fn(rank, comm):
        qq, kk, vv, dd = (t.roll(rank, 0).contiguous() for t in qs)
        o, l = ring.ring_forward(qq, kk, vv, softmax_scale=d ** -0.5, comm=comm)
        ring.ring_backward(dd, qq, kk, vv, o, l, softmax_scale=d ** -0.5, comm=comm)
        ring.ring_backward(dd, qq, kk, vv, o, l, softmax_scale=d ** -0.5, comm=comm,
                           fused_dkv=True)
        torch.cuda.current_stream().synchronize()

    ring.run_local_ring(2, rank_fn, devices=[dev, dev], timeout=600.0)
    torch.cuda.synchronize()
    print("sanitize smoke done")


if __name__ == "__main__":
    main()
