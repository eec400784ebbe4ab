"""e2e probe: host API step time (CUDA events) and CPU time per call, per head-group count."""
import math, sys, os, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_09431_b200.host import attention_fwd_bwd_host, ramp_groups

c, hq, d = 32768, 32, 128
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda: torch.randn(c, hq, d, device="cuda", generator=g).bfloat16().cpu().pin_memory()
q, k, v, do = mk(), mk(), mk(), mk()
out, dq, dk, dv = (torch.empty(c, hq, d, dtype=torch.bfloat16).pin_memory() for _ in range(4))
lse = torch.empty(hq, c, dtype=torch.float32).pin_memory()
def parse(x):
    if x == 'ramp':
        return ramp_groups(hq, hq)
    if ',' in x:
        return [int(y) for y in x.split(',')]
    return int(x)


for groups in [parse(x) for x in sys.argv[1:]] or [4, 8, 16, 32]:
    def step():
        ev = attention_fwd_bwd_host(q, k, v, do, out, lse, dq, dk, dv, softmax_scale=d ** -0.5,
                                    head_groups=groups)
        torch.cuda.current_stream().wait_event(ev)
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 8
    st0 = torch.cuda.memory_stats()
    e0.record()
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    t_cpu = (time.perf_counter() - t0) / n
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    st1 = torch.cuda.memory_stats()
    keys = ["num_device_alloc", "num_device_free", "num_alloc_retries", "num_sync_all_streams"]
    print({kk: st1.get(kk, 0) - st0.get(kk, 0) for kk in keys})
    flops = 7.0 * d * hq * c * (c + 1)
    print(f"groups {str(groups):>26s}: {ms:7.2f} ms/step  {flops / ms / 1e9:6.0f} TFLOP/s   cpu {t_cpu * 1e3:6.2f} ms/call")
