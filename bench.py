"""Benchmark: causal attention fwd+bwd TFLOP/s, striped vs ring, on 1..8 B200.

    python bench.py [--gpus N --steps K --warmup W]            # our CUDA path
    python bench.py --impl reference [...]                     # CPU reference arm
    torchrun --nproc-per-node N bench.py --gpus N ...          # N > 1: one rank per GPU

A step = one forward + backward of the whole attention layer over synthetic bf16
inputs of the BASELINE shape (one pass of the hot path).  N = 1 runs configs[1]
(seq 32k, 32 heads, d 128: the single-B200 block kernel, no ring).  N > 1 runs the
striped ring with a fixed 32k-token stripe per rank (seq = 32768 * N, so the
headline 256k shape at N = 8) and also times the ring (contiguous) layout for the
striped/ring ratio.  Useful FLOPs = 7 * D * Hq * S * (S + 1) (masked
and skipped pairs are not counted).  Inputs (1 GiB per rank) exceed the 126 MB L2, so
no flush is needed between steps.

One JSON line is printed by rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "causal attn fwd+bwd TFLOP/s/GPU, striped vs ring, seq 256k-786k, 1/2/4/8 B200"
STRIPE = 32768


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=0)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--stripe", type=int, default=STRIPE, help="tokens per rank")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--head-groups", type=int, default=8,
                    help="e2e: head groups streamed by the host API (copy/compute overlap); "
                         "0 = host.ramp_groups (small first/last groups)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ring-compare", action="store_true")
    return ap.parse_args()


def useful_flops(n_seq, hq, d):
    return 7.0 * d * hq * n_seq * (n_seq + 1)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ----------------------------------------------------------------------------- CPU arm
def cpu_sample(budget_s: float = 8.0):
    """Oracle port (ringsim's streaming forward restated + the builder's tiled backward)
    on one head of the config, as many tokens as fit the time budget.  Returns
    (TFLOP/s, seconds, description, threads)."""
    import numpy as np
    from oracle import ringref as R

    d = 128
    rng = np.random.default_rng(0)
    n = 2048
    # grow the sample until one fwd+bwd takes ~budget/4 (cost ~ n^2)
    while True:
        q, k, v, do = (rng.standard_normal((n, d)).astype(np.float32) for _ in range(4))
        t0 = time.perf_counter()
        o, lse = R.tiled_causal_forward(q, k, v, d ** -0.5, tile=512)
        R.tiled_causal_backward(q, k, v, do, o, lse, d ** -0.5, tile=512)
        dt = time.perf_counter() - t0
        if dt > budget_s / 4 or n >= 32768:
            break
        n *= 2
    flops = useful_flops(n, 1, d)
    threads = os.cpu_count() or 1
    desc = (f"1 of 32 heads, seq {n}, d 128, fp32 numpy: ringsim's tiled streaming-softmax "
            f"forward (tile 512) + builder tiled backward; BLAS threads = {threads}")
    return flops / dt / 1e12, dt, desc, threads


def arm_config(args, world):
    """The workload both arms report (the reference arm runs a bounded sample of it)."""
    hq, d = args.heads, args.dim
    hkv = args.kv_heads or hq
    c = args.stripe
    n_seq = c * world
    workload = ("configs[1]: single-B200 causal fwd+bwd, seq 32768, 32 heads, d 128 "
                "(block kernels, no ring)") if world == 1 else \
        (f"striped ring fwd+bwd, seq {n_seq} ({c} tokens/rank), {hq} heads, d {d}")
    return {"workload": workload, "seq": n_seq, "stripe_tokens_per_rank": c, "heads_q": hq,
            "heads_kv": hkv, "d_head": d, "layout": "striped", "parallelism": f"sp{world}",
            "l2": "inputs 1 GiB/rank > 126 MB L2, no flush",
            "useful_flops_per_step": useful_flops(n_seq, hq, d)}


def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    vals = []
    desc = threads = None
    for i in range(args.warmup + args.steps):
        v, dt, desc, threads = cpu_sample(budget_s=6.0)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": arm_config(args, world),
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "port",
                             "sample": desc},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2311_09431_b200 import _lib, ring

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    hq, d = args.heads, args.dim
    hkv = args.kv_heads or hq
    c = args.stripe
    n_seq = c * world
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    q = torch.randn(c, hq, d, device=dev, generator=gen).bfloat16()
    k = torch.randn(c, hkv, d, device=dev, generator=gen).bfloat16()
    v = torch.randn(c, hkv, d, device=dev, generator=gen).bfloat16()
    dout = torch.randn(c, hq, d, device=dev, generator=gen).bfloat16()
    scale = 1.0 / math.sqrt(d)

    # per-kernel CUDA events on the launching (current) stream
    class TimedOps(ring.BlockOps):
        def __init__(self):
            super().__init__()
            self.events = []  # (name, start, end)
            self._open = None  # start event of a backward round run in key parts

        def _wrap(self, name, fn, *a):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn(*a)
            e.record()
            self.events.append((name, s, e))

        def fwd_block(self, *a):
            self._wrap("fwd_block", super().fwd_block, *a)

        def bwd_block(self, *a, **kw):
            rows = kw.get("key_rows")
            if rows is None:
                self._wrap("bwd_block", super().bwd_block, *a)
                return
            # a round in key parts (ring.kv_parts, the lowest rows last): one entry per round
            if self._open is None:
                self._open = torch.cuda.Event(enable_timing=True)
                self._open.record()
            super().bwd_block(*a, **kw)
            if rows[0] == 0:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                self.events.append(("bwd_block", self._open, e))
                self._open = None

        def bwd_block_final(self, *a):  # the N = 1 backward (bf16 dK / dV out of the kernel)
            self._wrap("bwd_block", super().bwd_block_final, *a)

        def bwd_preprocess(self, *a):
            self._wrap("bwd_preprocess", super().bwd_preprocess, *a)

        def cast(self, *a):
            self._wrap("cast", super().cast, *a)

    def step(layout, bops):
        out, lse = ring.ring_forward(q, k, v, layout=layout, softmax_scale=scale, block_ops=bops)
        dq, dk, dv = ring.ring_backward(dout, q, k, v, out, lse, layout=layout,
                                        softmax_scale=scale, block_ops=bops)
        return out, dq

    def timed(layout, steps, warmup):
        bops = TimedOps()
        for _ in range(warmup):
            step(layout, bops)
        torch.cuda.synchronize()
        bops.events.clear()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        n0 = _lib.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step(layout, bops)
        e1.record()
        torch.cuda.synchronize()
        launches = _lib.launch_count() - n0
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1) / steps
        per = {}
        for name, s, e in bops.events:
            per.setdefault(name, []).append(s.elapsed_time(e))
        return ms, per, launches

    with ClockSampler(local) as clk:
        ms, per, launches = timed("striped", args.steps, args.warmup)
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total = useful_flops(n_seq, hq, d)
    value = total / (ms_max / 1e3) / 1e12

    # per-round rank imbalance of the block kernels (max/mean over ranks, per round)
    def imbalance(per_dict):
        rows = []
        for name in ("fwd_block", "bwd_block"):
            xs = per_dict.get(name, [])
            if not xs:
                continue
            rounds = [statistics.mean(xs[i::world]) for i in range(world)] if world > 1 else \
                [statistics.mean(xs)]
            rows.append(torch.tensor(rounds, device=dev, dtype=torch.float64))
        if not rows:
            return None
        mine = torch.stack(rows)
        if world > 1:
            allr = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(allr, mine)
            stk = torch.stack(allr)  # [rank, kernel, round]
            ratio = stk.max(0).values / stk.mean(0)
            return {"max": float(ratio.max()), "mean": float(ratio.mean())}
        return {"max": 1.0, "mean": 1.0}

    imb = imbalance(per)

    ring_cmp = None
    if world > 1 and not args.no_ring_compare:
        ms_r, per_r, _ = timed("ring", args.steps, max(1, args.warmup))
        tr = torch.tensor([ms_r], device=dev)
        dist.all_reduce(tr, op=dist.ReduceOp.MAX)
        ring_cmp = {"ring_ms_per_step": float(tr.item()),
                    "ring_value": total / (float(tr.item()) / 1e3) / 1e12,
                    "striped_over_ring": float(tr.item()) / ms_max,
                    "ring_rank_imbalance": imbalance(per_r)}

    # roofline of the dominant kernel (bwd block), achieved = useful FLOPs per launch / time
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    peak_burst = peaks.get("bf16_tflops", 1590.0)
    peak_sus = peaks.get("bf16_tflops_sustained", 1400.0)

    # training-step speedup (TMS) predicted from these measured attention
    # critical paths (one layer, all heads) + the layer's non-attention FLOPs at the
    # measured sustained GEMM rate, next to the reference's analytic model
    if ring_cmp is not None:
        from paper_2311_09431_b200 import costmodel as CM
        preset = next((m for m in CM.PRESETS.values() if m.n_head == hq and m.head_dim == d),
                      None)
        if preset is not None:
            mt = CM.measured_tms(preset, c, ring_cmp["ring_ms_per_step"], ms_max, peak_sus)
            ring_cmp["tms"] = {"model": preset.name, "n_seq": n_seq, "sp": world,
                               "measured": mt.tms, "other_ms_per_layer": mt.other_ms,
                               "analytic_flop_weight_1": CM.tms(preset, n_seq, world, 1.0),
                               "analytic_flop_weight_2": CM.tms(preset, n_seq, world, 2.0)}
    bwd_ms = statistics.mean(per["bwd_block"])
    fwd_ms = statistics.mean(per["fwd_block"])
    # per launch one rank processes one block of c x c pairs of one ring round; average
    # useful pairs per round = total useful pairs / (N * N) per rank-launch
    pairs_per_launch = hq * n_seq * (n_seq + 1) / 2 / (world * world)
    bwd_achieved = 10.0 * d * pairs_per_launch / (bwd_ms / 1e3) / 1e12
    fwd_achieved = 4.0 * d * pairs_per_launch / (fwd_ms / 1e3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get("bwd_block_bytes_per_launch")
    except OSError:
        pass
    kern_ms = sum(sum(xs) for xs in per.values()) / args.steps
    roofline = {"bound": "tensor", "kernel": "bwd_kernel (K5)", "achieved": bwd_achieved,
                "peak": peak_sus, "unit": "TFLOP/s", "frac": bwd_achieved / peak_sus,
                "frac_of_burst": bwd_achieved / peak_burst, "traffic": traffic,
                "peak_note": "sustained bf16 of MEASURED_PEAKS.json (kernel timed inside a long step)",
                "share_of_step": statistics.mean(per["bwd_block"]) * len(per["bwd_block"]) /
                args.steps / ms,
                "fwd_kernel": {"achieved": fwd_achieved, "frac": fwd_achieved / peak_sus,
                               "ms": fwd_ms},
                "bwd_ms": bwd_ms}

    # End to end through the public host API (paper_2311_09431_b200.host): inputs start in
    # pinned host memory, results end in pinned host memory; the H2D / D2H copies are in the
    # timed region (overlapped with compute across head groups by the API itself).
    e2e = None
    if not args.no_e2e:
        from paper_2311_09431_b200.host import attention_fwd_bwd_host, ramp_groups
        hq_h, hk_h, hv_h, hdo_h = (x.cpu().pin_memory() for x in (q, k, v, dout))
        hout = torch.empty(c, hq, d, dtype=torch.bfloat16).pin_memory()
        hdq = torch.empty(c, hq, d, dtype=torch.bfloat16).pin_memory()
        hdk = torch.empty(c, hkv, d, dtype=torch.bfloat16).pin_memory()
        hdv = torch.empty(c, hkv, d, dtype=torch.bfloat16).pin_memory()
        hlse = torch.empty(hq, c, dtype=torch.float32).pin_memory()
        if args.head_groups > 0:
            groups = args.head_groups
            while groups > 1 and (hq % groups or hkv % groups):
                groups //= 2
        else:
            groups = ramp_groups(hq, hkv)

        def e2e_step():
            ev = attention_fwd_bwd_host(hq_h, hk_h, hv_h, hdo_h, hout, hlse, hdq, hdk, hdv,
                                        layout="striped", softmax_scale=scale,
                                        head_groups=groups)
            torch.cuda.current_stream().wait_event(ev)

        n_e2e = max(2, min(args.steps, 5))
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(n_e2e):
            e2e_step()
        s1.record()
        torch.cuda.synchronize()
        te = torch.tensor([s0.elapsed_time(s1) / n_e2e], device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        bi = sum(x.numel() * x.element_size() for x in (hq_h, hk_h, hv_h, hdo_h))
        bo = sum(x.numel() * x.element_size() for x in (hout, hdq, hdk, hdv, hlse))
        e2e = {"value": total / (float(te.item()) / 1e3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
               "ms_per_step": float(te.item()), "head_groups": groups,
               "api": "paper_2311_09431_b200.host.attention_fwd_bwd_host (pinned host in/out; "
                      "C ABI via ctypes)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v_cpu, dt, desc, threads = cpu_sample()
        cpu = {"value": v_cpu, "unit": "TFLOP/s", "cores": threads, "kind": "port",
               "sample": desc, "seconds": dt}

    exposed = max(0.0, ms - kern_ms)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded normal bf16 q/k/v/dO)",
            "config": arm_config(args, world),
            "per_gpu_value": value / world,
            "gpu_launches": launches,
            "kernel_ms_per_step": {kname: sum(xs) / args.steps for kname, xs in per.items()},
            "exposed_non_kernel_ms_per_step": exposed,
            "rank_imbalance": imb,
            "striped_vs_ring": ring_cmp,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
