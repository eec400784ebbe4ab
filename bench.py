"""Benchmark: causal attention fwd+bwd TFLOP/s per GPU, striped vs ring, on 1..8 B200.

    python bench.py [--gpus N --steps K --warmup W] [--config cfg3]   # our CUDA path
    python bench.py --impl reference [...]                            # CPU reference arm
    python bench.py --virtual-ring 8 --config cfg3                    # N ranks on ONE GPU

A step = one forward + backward of the whole attention layer over synthetic bf16
inputs of a BASELINE shape (one pass of the hot path).  ``--config`` picks the shape
(SURVEY.md section 8(d) names; BASELINE.json configs[i]):

    cfg2  seq  32768, 32 q / 32 kv heads, d 128   configs[1] (single-B200 block kernel)
    cfg3  seq 262144, 32 / 32,              d 128   configs[2] (the metric's headline shape)
    cfg4  seq 524288, 32 / 8 (GQA),         d 128   configs[3]
    cfg5  seq 786432, 64 / 64,              d 128   configs[4]

The total sequence is fixed and split over the N ranks (c = seq / N tokens per rank,
strong scaling).  Default: cfg3 -- at N = 1 the whole 256k sequence is one block on one
B200 (it fits: ~20 GiB of device tensors); the configs[1] 32k shape is also measured at
N = 1 and reported under "secondary".  At N > 1 the striped ring runs over NCCL (or the
copy-engine IPC hop, ``--comm ipc``) and the ring (contiguous) layout is timed too.

``value`` is useful causal TFLOP/s PER GPU (the metric's unit): useful FLOPs
7 * D * Hq * S * (S + 1) (masked / skipped pairs not counted) / step time / N;
``aggregate_tflops`` is the whole-job figure.  Inputs (>= 1 GiB per rank) exceed the
126 MB L2, so no flush is needed between steps.

``--gpus N`` without torchrun re-launches itself under torch.distributed.run with N
ranks; it fails (exit 2) if fewer than N GPUs are visible.  One JSON line is printed by
rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "causal attn fwd+bwd TFLOP/s/GPU, striped vs ring, seq 256k-786k, 1/2/4/8 B200"

CONFIGS = {
    "cfg2": {"seq": 32768, "hq": 32, "hkv": 32, "d": 128, "index": 1,
             "desc": "configs[1]: single-B200 stripe-masked causal flash attention fwd+bwd, "
                     "seq 32k, 32 heads, d_head 128, bf16"},
    "cfg3": {"seq": 262144, "hq": 32, "hkv": 32, "d": 128, "index": 2,
             "desc": "configs[2]: striped causal attention fwd+bwd, seq 256k, 32 heads, "
                     "d_head 128, bf16 (the paper's headline shape)"},
    "cfg4": {"seq": 524288, "hq": 32, "hkv": 8, "d": 128, "index": 3,
             "desc": "configs[3]: Llama-3-8B-shaped GQA layer (32 q / 8 kv heads, d_head 128), "
                     "seq 512k, bf16"},
    "cfg5": {"seq": 786432, "hq": 64, "hkv": 64, "d": 128, "index": 4,
             "desc": "configs[4]: seq 786k causal, 64 heads, d_head 128, bf16"},
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--seq", type=int, default=0, help="override the config's sequence length")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "ipc"],
                    help="N > 1: ring hop backend (NCCL P2P or CUDA-IPC copy engines)")
    ap.add_argument("--fused", action="store_true",
                    help="N > 1 with --comm ipc: fused rotation (no dK/dV hops; the kernels "
                         "reduce-add into the owner's buffer through peer memory)")
    ap.add_argument("--virtual-ring", type=int, default=0,
                    help="time N virtual ranks on ONE GPU, per (rank, round) block")
    ap.add_argument("--csv", default="", help="--virtual-ring: write the stats CSV here")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--head-groups", type=int, default=0,
                    help="e2e: head groups streamed by the host API (copy/compute overlap); "
                         "0 = host.ramp_groups (small first/last groups: the least exposed "
                         "copy; at 256k e2e 1103.6 vs 1094.6 TFLOP/s with 8 equal groups)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-ring-compare", action="store_true")
    return ap.parse_args(argv)


def shape(args):
    cfg = dict(CONFIGS[args.config])
    if args.seq:
        cfg["seq"] = args.seq
    return cfg


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


def host_info():
    """CPU model, logical CPU count and this process's affinity."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = os.cpu_count()
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "affinity_cpus": aff}


# ----------------------------------------------------------------------------- CPU arm
def cpu_sample(d: int, budget_s: float = 8.0):
    """Oracle port (ringsim's streaming forward restated + the builder's tiled backward)
    on one head of the config, as many tokens as fit the time budget.  Returns
    (TFLOP/s, seconds, description, threads)."""
    import numpy as np
    from oracle import ringref as R

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
    hi = host_info()
    threads = hi["affinity_cpus"] or 1
    desc = (f"1 head, seq {n}, d {d}, fp32 numpy: ringsim's tiled streaming-softmax forward "
            f"(tile 512, attention.py:296-328 restated) + builder tiled backward; OpenBLAS on "
            f"{threads} threads; CPU {hi['cpu_model']}")
    return flops / dt / 1e12, dt, desc, threads


def arm_config(args, world):
    """The workload both arms report (the reference arm runs a bounded sample of it)."""
    s = shape(args)
    c = s["seq"] // world
    return {"workload": s["desc"] + (f" -- one block of {c} tokens on 1 GPU (no ring)"
                                     if world == 1 else f" -- striped ring over {world} GPUs, "
                                     f"{c} tokens per rank"),
            "config": args.config, "seq": s["seq"], "tokens_per_rank": c, "heads_q": s["hq"],
            "heads_kv": s["hkv"], "d_head": s["d"], "layout": "striped",
            "parallelism": f"sp{world}", "comm": args.comm if world > 1 else None,
            "fused_dkv": bool(args.fused and world > 1),
            "l2": "inputs >= 1 GiB per rank > 126 MB L2, no flush",
            "useful_flops_per_step": useful_flops(s["seq"], s["hq"], s["d"])}


def run_reference(args, rank, world):
    if rank != 0:
        return
    s = shape(args)
    vals = []
    desc = threads = None
    for i in range(args.warmup + args.steps):
        v, dt, desc, threads = cpu_sample(s["d"], budget_s=6.0)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": arm_config(args, world),
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "port",
                             "sample": desc, **host_info()},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- launching
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SHARE_GPU = os.environ.get("SA_BENCH_SHARE_GPU") == "1"


def self_launch(args):
    """--gpus N > 1 outside torchrun: re-run under torch.distributed.run with N ranks."""
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus and not SHARE_GPU:
            print(json.dumps({"error": f"--gpus {args.gpus} but only {have} GPU(s) visible"}),
                  flush=True)
            sys.exit(2)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd, env=env))


# ----------------------------------------------------------------------------- GPU arm
def make_inputs(torch, dev, c, hq, hkv, d, seed):
    gen = torch.Generator(device=dev).manual_seed(seed)
    mk = lambda h: torch.randn(c, h, d, device=dev, generator=gen, dtype=torch.float32) \
        .to(torch.bfloat16)
    q, k, v, dout = mk(hq), mk(hkv), mk(hkv), mk(hq)
    return q, k, v, dout


def timed_ops_class(ring, torch):
    class TimedOps(ring.BlockOps):
        """Per-kernel CUDA events on the launching (current) stream."""

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

    return TimedOps


def measure(torch, dist, ring, _lib, q, k, v, dout, scale, layout, steps, warmup, world,
            comm=None, stats=False, fused=False):
    """Time `steps` fwd+bwd steps (after `warmup`); returns (ms/step on this rank,
    per-kernel ms lists, launches, RingStats of the last step or None)."""
    TimedOps = timed_ops_class(ring, torch)
    bops = TimedOps()
    ws = ring.Workspace()

    def step(st=None):
        out, lse = ring.ring_forward(q, k, v, layout=layout, softmax_scale=scale, block_ops=bops,
                                     workspace=ws, comm=comm, stats=st)
        ring.ring_backward(dout, q, k, v, out, lse, layout=layout, softmax_scale=scale,
                           block_ops=bops, workspace=ws, comm=comm, stats=st,
                           fused_dkv=fused and world > 1)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    bops.events.clear()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    launches = _lib.launch_count() - n0
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / steps
    per = {}
    for name, s, e in bops.events:
        per.setdefault(name, []).append(s.elapsed_time(e))
    rstats = None
    if stats and world > 1:  # one extra (untimed) step that records hop times
        rstats = ring.RingStats(dist.get_rank())
        bops.events.clear()
        step(rstats)
        torch.cuda.synchronize()
    return ms, per, launches, rstats


def measured_traffic(config, world):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu
    capture of the same configuration (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            rec = json.load(f).get("by_config", {}).get(f"{config}_n{world}")
    except (OSError, ValueError):
        return None
    return rec


def roofline_block(per, steps, ms, hq, d, n_seq, world, peaks, config):
    peak_burst = peaks.get("bf16_tflops", 1590.0)
    peak_sus = peaks.get("bf16_tflops_sustained", 1400.0)
    bwd_ms = statistics.mean(per["bwd_block"])
    fwd_ms = statistics.mean(per["fwd_block"])
    # per launch one rank processes one block of one ring round; average useful pairs per
    # launch = total useful pairs / (N * N) rank-launches
    pairs_per_launch = hq * n_seq * (n_seq + 1) / 2 / (world * world)
    bwd_achieved = 10.0 * d * pairs_per_launch / (bwd_ms / 1e3) / 1e12
    fwd_achieved = 4.0 * d * pairs_per_launch / (fwd_ms / 1e3) / 1e12
    tr = measured_traffic(config, world) or {}
    # B200_PROFILING.md: the burst figure for a kernel timed alone, the sustained one for a
    # kernel timed inside a long step -- a step of a second or more runs at the power cap
    long_step = ms >= 1000.0
    peak = peak_sus if long_step else peak_burst
    return {"bound": "tensor", "kernel": "bwd_kernel (K5)", "achieved": bwd_achieved,
            "peak": peak, "unit": "TFLOP/s", "frac": bwd_achieved / peak,
            "frac_of_burst": bwd_achieved / peak_burst,
            "frac_of_sustained": bwd_achieved / peak_sus,
            "traffic": tr.get("bwd_block_bytes_per_launch"),
            "traffic_algorithmic_min": tr.get("bwd_block_algorithmic_bytes"),
            "peak_note": ("MEASURED_PEAKS.json bf16_tflops_sustained: the step is "
                          f"{ms / 1e3:.2f} s long and runs power-capped" if long_step else
                          "MEASURED_PEAKS.json bf16_tflops (burst): the step is short"),
            "useful_flops_per_launch": 10.0 * d * pairs_per_launch,
            "share_of_step": bwd_ms * len(per["bwd_block"]) / steps / ms,
            "bwd_ms": bwd_ms,
            "fwd_kernel": {"achieved": fwd_achieved, "frac": fwd_achieved / peak,
                           "frac_of_burst": fwd_achieved / peak_burst,
                           "frac_of_sustained": fwd_achieved / peak_sus, "ms": fwd_ms,
                           "useful_flops_per_launch": 4.0 * d * pairs_per_launch}}


def run_e2e(torch, dist, args, q, k, v, dout, scale, total, world, dev, comm=None):
    """End to end through the public host API (paper_2311_09431_b200.host): inputs start in
    pinned host memory, results end in pinned host memory; the H2D / D2H copies are in the
    timed region (overlapped with compute across head groups by the API itself)."""
    from paper_2311_09431_b200.host import attention_fwd_bwd_host, ramp_groups
    c, hq, d = q.shape
    hkv = k.shape[1]

    def pinned_like(x):
        h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        h.copy_(x)
        return h

    hq_h, hk_h, hv_h, hdo_h = (pinned_like(x) for x in (q, k, v, dout))
    hout = torch.empty(c, hq, d, dtype=torch.bfloat16, pin_memory=True)
    hdq = torch.empty(c, hq, d, dtype=torch.bfloat16, pin_memory=True)
    hdk = torch.empty(c, hkv, d, dtype=torch.bfloat16, pin_memory=True)
    hdv = torch.empty(c, hkv, d, dtype=torch.bfloat16, pin_memory=True)
    hlse = torch.empty(hq, c, dtype=torch.float32, pin_memory=True)
    if args.head_groups > 0:
        groups = args.head_groups
        while groups > 1 and (hq % groups or hkv % groups):
            groups //= 2
    else:
        groups = ramp_groups(hq, hkv)

    def e2e_step():
        ev = attention_fwd_bwd_host(hq_h, hk_h, hv_h, hdo_h, hout, hlse, hdq, hdk, hdv,
                                    layout="striped", softmax_scale=scale, head_groups=groups,
                                    comm=comm)
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
    return {"value": total / (float(te.item()) / 1e3) / 1e12 / world, "unit": "TFLOP/s",
            "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
            "ms_per_step": float(te.item()), "steps": n_e2e,
            "head_groups": groups if isinstance(groups, int) else list(groups),
            "api": "paper_2311_09431_b200.host.attention_fwd_bwd_host (pinned host in/out; "
                   "C ABI via ctypes)"}


def secondary_cfg2(torch, ring, _lib, dev, steps, peaks):
    """configs[1] (seq 32k, 32 heads, d 128) at N = 1: the block-kernel measurement."""
    s = CONFIGS["cfg2"]
    q, k, v, dout = make_inputs(torch, dev, s["seq"], s["hq"], s["hkv"], s["d"], 4321)
    scale = 1.0 / math.sqrt(s["d"])
    ms, per, launches, _ = measure(torch, None, ring, _lib, q, k, v, dout, scale, "striped",
                                   max(steps, 10), 3, 1)
    total = useful_flops(s["seq"], s["hq"], s["d"])
    roof = roofline_block(per, max(steps, 10), ms, s["hq"], s["d"], s["seq"], 1, peaks, "cfg2")
    del q, k, v, dout
    return {"workload": s["desc"], "value": total / (ms / 1e3) / 1e12, "unit": "TFLOP/s",
            "ms_per_step": ms, "gpu_launches": launches,
            "kernel_ms_per_step": {kk: sum(xs) / max(steps, 10) for kk, xs in per.items()},
            "roofline": roof}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.virtual_ring:
        return run_virtual_ring(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if world != args.gpus:
        msg = f"--gpus {args.gpus} but WORLD_SIZE={world}"
        if rank == 0:
            print(json.dumps({"error": msg}), flush=True)
        sys.exit(2)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2311_09431_b200 import _lib, ring

    local = int(os.environ.get("LOCAL_RANK", "0"))
    if SHARE_GPU and world > 1:
        # TEST MODE (SA_BENCH_SHARE_GPU=1): every rank on GPU 0, gloo for the host-side
        # collectives, the copy-engine IPC hop (NCCL cannot put two ranks on one GPU).  It
        # exercises the N > 1 code path end to end; its timings are of ranks time-sharing
        # one GPU and mean nothing.
        if args.comm != "ipc":
            print(json.dumps({"error": "SA_BENCH_SHARE_GPU needs --comm ipc"}), flush=True)
            sys.exit(2)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        if SHARE_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        if args.comm == "ipc":
            from paper_2311_09431_b200 import ipc
            comm = ipc.IpcComm()
    s = shape(args)
    hq, hkv, d, n_seq = s["hq"], s["hkv"], s["d"], s["seq"]
    if n_seq % world:
        raise SystemExit(f"seq {n_seq} not divisible by {world} ranks")
    c = n_seq // world
    q, k, v, dout = make_inputs(torch, dev, c, hq, hkv, d, 1234 + rank)
    scale = 1.0 / math.sqrt(d)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass

    with ClockSampler(local) as clk:
        ms, per, launches, rstats = measure(torch, dist, ring, _lib, q, k, v, dout, scale,
                                            "striped", args.steps, args.warmup, world, comm,
                                            stats=True, fused=args.fused)
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total = useful_flops(n_seq, hq, d)
    value = total / (ms_max / 1e3) / 1e12 / world

    def imbalance(per_dict):
        """Per ring round, max / mean over ranks of the block kernel time."""
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
            return {"max": float(ratio.max()), "mean": float(ratio.mean()),
                    "per_round_fwd": [float(x) for x in ratio[0]],
                    "per_round_bwd": [float(x) for x in ratio[-1]]}
        return {"max": 1.0, "mean": 1.0}

    imb = imbalance(per)
    kern_ms = sum(sum(xs) for xs in per.values()) / args.steps
    exposed = max(0.0, ms - kern_ms)
    comm_info = None
    if rstats is not None and rstats.hops:
        kvh = [h for h in rstats.hops if h.what == "kv"]
        dkh = [h for h in rstats.hops if h.what == "dkv"]
        gbs = lambda hs: (sum(h.nbytes for h in hs) / (sum(h.ms for h in hs) / 1e3) / 1e9
                          if hs and sum(h.ms for h in hs) > 0 else None)
        comm_info = {"backend": args.comm, "kv_hop_bytes": kvh[0].nbytes if kvh else 0,
                     "kv_hop_ms_mean": statistics.mean(h.ms for h in kvh) if kvh else None,
                     "kv_hop_gbs": gbs(kvh), "dkv_hop_gbs": gbs(dkh),
                     "note": "hop times from CUDA events on the comm streams (issue to "
                             "completion, peer waits included): GB/s is a lower bound on "
                             "the NVLink rate"}

    ring_cmp = None
    if world > 1 and not args.no_ring_compare:
        ms_r, per_r, _, _ = measure(torch, dist, ring, _lib, q, k, v, dout, scale, "ring",
                                    args.steps, max(1, args.warmup), world, comm,
                                    fused=args.fused)
        tr = torch.tensor([ms_r], device=dev)
        dist.all_reduce(tr, op=dist.ReduceOp.MAX)
        ring_cmp = {"ring_ms_per_step": float(tr.item()),
                    "ring_value": total / (float(tr.item()) / 1e3) / 1e12 / world,
                    "striped_over_ring": float(tr.item()) / ms_max,
                    "ring_rank_imbalance": imbalance(per_r)}
        from paper_2311_09431_b200 import costmodel as CM
        preset = next((m for m in CM.PRESETS.values() if m.n_head == hq and m.head_dim == d),
                      None)
        if preset is not None:
            mt = CM.measured_tms(preset, c, ring_cmp["ring_ms_per_step"], ms_max,
                                 peaks.get("bf16_tflops_sustained", 1400.0))
            ring_cmp["tms"] = {"model": preset.name, "n_seq": n_seq, "sp": world,
                               "measured": mt.tms, "other_ms_per_layer": mt.other_ms,
                               "analytic_flop_weight_1": CM.tms(preset, n_seq, world, 1.0),
                               "analytic_flop_weight_2": CM.tms(preset, n_seq, world, 2.0)}

    roofline = roofline_block(per, args.steps, ms, hq, d, n_seq, world, peaks, args.config)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(torch, dist, args, q, k, v, dout, scale, total, world, dev, comm)
    del q, k, v, dout
    torch.cuda.empty_cache()
    secondary = None
    if world == 1 and not args.no_secondary and args.config != "cfg2":
        secondary = secondary_cfg2(torch, ring, _lib, dev, args.steps, peaks)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v_cpu, dt, desc, threads = cpu_sample(d)
        cpu = {"value": v_cpu, "unit": "TFLOP/s", "cores": threads, "kind": "port",
               "sample": desc, "seconds": dt, **host_info()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded normal bf16 q/k/v/dO)",
            "config": arm_config(args, world),
            "aggregate_tflops": value * world,
            "gpu_launches": launches,
            "kernel_ms_per_step": {kname: sum(xs) / args.steps for kname, xs in per.items()},
            "exposed_non_kernel_ms_per_step": exposed,
            "exposed_non_kernel_pct": 100.0 * exposed / ms if ms > 0 else 0.0,
            "rank_imbalance": imb,
            "comm": comm_info,
            "striped_vs_ring": ring_cmp,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "secondary": secondary,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- virtual ring
def run_virtual_ring(args):
    """N ranks' blocks on ONE GPU, one (rank, round) block launch at a time (the
    reference's serial executor), each timed with CUDA events, for the striped and the
    ring layout.  Reports the measured counterparts of round_critical_path /
    simulated_speedup (simulator.py:318-341): sum over rounds of the max over ranks of
    the block time, their ring / striped ratio, and the per-round max / mean imbalance,
    next to the reference's closed form at the kernel's 128 x 128 tiles."""
    import torch

    from oracle import ringref as R  # closed form only: schedule_work_stats
    from paper_2311_09431_b200 import ring, telemetry

    n = args.virtual_ring
    s = shape(args)
    hq, hkv, d, n_seq = s["hq"], s["hkv"], s["d"], s["seq"]
    c = n_seq // n
    dev = torch.device("cuda", 0)
    scale = 1.0 / math.sqrt(d)
    gen = torch.Generator(device=dev).manual_seed(99)
    mk = lambda h: [torch.randn(c, h, d, device=dev, generator=gen).bfloat16() for _ in range(n)]
    qs, ks, vs, dos = mk(hq), mk(hkv), mk(hkv), mk(hq)
    # warm-up (module load, first-launch setup): one untimed fwd + bwd of a whole block
    w_out, w_lse = ring.ring_forward(qs[0], ks[0], vs[0], softmax_scale=scale)
    ring.ring_backward(dos[0], qs[0], ks[0], vs[0], w_out, w_lse, softmax_scale=scale)
    torch.cuda.synchronize()
    del w_out, w_lse
    res = {}
    runs = []
    with ClockSampler(0) as clk:
        for layout in ("striped", "ring"):
            # layout only changes which mask each (rank, round) gets; the inputs are the
            # same random stripes (the timing does not depend on the values)
            tf, tb = [], []
            outs, lses, stats = ring.virtual_ring_forward(qs, ks, vs, layout=layout,
                                                          softmax_scale=scale, timings=tf)
            acc = ring.virtual_ring_backward(dos, qs, ks, vs, outs, lses, layout=layout,
                                             softmax_scale=scale, timings=tb, cast=False)
            torch.cuda.synchronize()
            del acc
            t = [[0.0] * n for _ in range(n)]  # t[i][j] fwd+bwd ms of rank j in round i
            for lst in (tf, tb):
                for i, j, a, b in lst:
                    t[i][j] += a.elapsed_time(b)
            for j in range(n):
                for rec in stats[j].rounds:
                    rec.compute_ms = t[rec.round][j]
            runs.append(telemetry.Run(layout, c, hq, stats))
            crit = sum(max(row) for row in t)
            imb = [max(row) / (sum(row) / n) for row in t]
            res[layout] = {"critical_path_ms": crit, "sum_ms": sum(sum(r) for r in t),
                           "per_round_max_ms": [max(r) for r in t],
                           "per_round_imbalance": imb, "t_ms": t}
            del outs, lses
            torch.cuda.empty_cache()
    scheme = {"striped": R.STRIPED, "ring": R.CONTIGUOUS}
    closed = {}
    for lay in scheme:
        ws = R.schedule_work_stats(scheme[lay], n, c, 128, 128)
        closed[lay] = sum(max(w.rounds[i].interactions_computed for w in ws) for i in range(n))
    if args.csv:
        telemetry.write_stats_csv(args.csv, runs, extra=True)
    line = {"mode": "virtual_ring", "config": args.config, "workload": s["desc"],
            "n_virtual_ranks": n, "tokens_per_rank": c,
            "measured_striped_speedup": res["ring"]["critical_path_ms"] /
            res["striped"]["critical_path_ms"],
            "closed_form_speedup_128_tiles": closed["ring"] / closed["striped"],
            "striped": {k_: v_ for k_, v_ in res["striped"].items() if k_ != "t_ms"},
            "ring": {k_: v_ for k_, v_ in res["ring"].items() if k_ != "t_ms"},
            "striped_round_imbalance_max": max(res["striped"]["per_round_imbalance"]),
            "t_ms": {lay: res[lay]["t_ms"] for lay in res},
            "useful_tflops_striped_per_gpu_equiv":
                useful_flops(n_seq, hq, d) / n / (res["striped"]["critical_path_ms"] / 1e3) / 1e12,
            "csv": args.csv or None, "clocks": clk.summary()}
    # training-step speedup (TMS) from these measured per-layer critical
    # paths + the layer's non-attention FLOPs at the measured sustained GEMM rate, beside
    # the reference's analytic model (costmodel.py:109-128)
    from paper_2311_09431_b200 import costmodel as CM
    preset = next((m for m in CM.PRESETS.values() if m.n_head == hq and m.head_dim == d), None)
    if preset is not None:
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                gemm = json.load(f).get("bf16_tflops_sustained", 1400.0)
        except OSError:
            gemm = 1400.0
        mt = CM.measured_tms(preset, c, res["ring"]["critical_path_ms"],
                             res["striped"]["critical_path_ms"], gemm)
        line["tms"] = {"model": preset.name, "measured": mt.tms, "other_ms_per_layer": mt.other_ms,
                       "analytic_flop_weight_1": CM.tms(preset, n_seq, n, 1.0),
                       "analytic_flop_weight_2": CM.tms(preset, n_seq, n, 2.0),
                       "note": "GQA kv heads are not modelled by the preset" if hkv != hq
                       else None}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
