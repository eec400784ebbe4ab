"""bench.py's N > 1 code path end to end on ONE GPU (SA_BENCH_SHARE_GPU=1 test mode):
`--gpus 2` self-launches torch.distributed.run, both ranks share GPU 0 and hop over the
copy-engine IPC comm (travelling dK/dV, and the fused rotation).  Checks the JSON line's
multi-GPU fields (striped-vs-ring, rank imbalance, hop bytes / GB/s, TMS); the timings
of ranks time-sharing one GPU mean nothing and are not asserted."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("extra", [[], ["--fused"]])
def test_bench_two_ranks_shared_gpu(extra):
    env = dict(os.environ, SA_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--comm", "ipc", "--config", "cfg2", "--seq", "8192", "--steps", "2",
                        "--warmup", "1", "--no-cpu", *extra],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    line = json.loads(lines[-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "sp2"
    assert line["config"]["tokens_per_rank"] == 4096
    assert line["config"]["fused_dkv"] == ("--fused" in extra)
    assert line["value"] > 0 and abs(line["aggregate_tflops"] - 2 * line["value"]) < 1e-6
    sr = line["striped_vs_ring"]
    assert sr is not None and sr["ring_ms_per_step"] > 0 and "tms" in sr
    assert line["rank_imbalance"]["max"] >= 1.0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    comm = line["comm"]
    assert comm["backend"] == "ipc" and comm["kv_hop_bytes"] == 2 * 4096 * 32 * 128 * 2
