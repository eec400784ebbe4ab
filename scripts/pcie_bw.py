import torch, time, ctypes, sys
sys.path.insert(0, '.')
from paper_2311_09431_b200 import _lib
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device='cuda')
s = torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps): fn()
    e1.record(s); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
with torch.cuda.stream(s):
    print("h2d contiguous GB/s", n / t(lambda: d.copy_(h, non_blocking=True)) / 1e6)
    print("d2h contiguous GB/s", n / t(lambda: h.copy_(d, non_blocking=True)) / 1e6)
    for width in (8192, 2048, 256):
        pitch = 8192
        rows = n // pitch
        def f():
            _lib.check(_lib.lib().sa_memcpy2d_async(d.data_ptr(), width, h.data_ptr(), pitch, width, rows, s.cuda_stream), "x")
        ms = t(f)
        print(f"h2d 2D width {width}: GB/s", rows * width / ms / 1e6)
    # both directions at once
    d2 = torch.empty(n, dtype=torch.uint8, device='cuda'); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    s2 = torch.cuda.Stream()
    torch.cuda.synchronize()
    e0 = time.time()
    for _ in range(3):
        with torch.cuda.stream(s): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    print("bidirectional GB/s each", 3 * n / (time.time() - e0) / 1e9)
import os
print("cpus", os.cpu_count(), "numa affinity", os.sched_getaffinity(0).__len__())
