"""Device-only fwd+bwd time of one head group vs all heads (where the e2e overhead goes)."""
import sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_09431_b200 import ring

c, d = 32768, 128
for h in (32, 16, 8, 4, 2, 1):
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, do = (torch.randn(c, h, d, device="cuda", generator=g).bfloat16() for _ in range(4))
    wsp = ring.Workspace()
    def step():
        o, l = ring.ring_forward(q, k, v, softmax_scale=d ** -0.5, workspace=wsp)
        ring.ring_backward(do, q, k, v, o, l, softmax_scale=d ** -0.5, workspace=wsp)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(3, 32 // h)
    e0.record()
    for _ in range(n):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"heads {h:2d}: {ms:7.3f} ms  x{32 // h} groups = {ms * 32 / h:7.2f} ms for 32 heads")
