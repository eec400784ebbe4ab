"""bench.py's contract on a machine without the GPUs it is asked for (CPU-only here):
--gpus N > visible GPUs fails loudly (exit 2, an "error" JSON line) instead of printing
an N = 1 line; the reference arm prints one JSON line with the contract's keys; the
config table covers BASELINE.json's GPU configs."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=300):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                          capture_output=True, text=True, timeout=timeout, cwd=ROOT)


def test_gpus_beyond_visible_fails_loudly():
    r = _run("--gpus", "2")
    assert r.returncode == 2
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "error" in line and "--gpus 2" in line["error"]


def test_world_size_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="2", RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode == 2


def test_reference_arm_line():
    r = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "cfg2")
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "config", "cpu_baseline", "e2e", "impl"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["seq"] == 32768 and line["config"]["heads_q"] == 32


def test_config_table_matches_baseline():
    sys.path.insert(0, ROOT)
    import bench
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        configs = json.load(f)["configs"]
    for name, cfg in bench.CONFIGS.items():
        text = configs[cfg["index"]]
        assert str(cfg["hq"]) in text and str(cfg["d"]) in text, (name, text)
    assert bench.CONFIGS["cfg3"]["seq"] == 262144 and bench.CONFIGS["cfg4"]["hkv"] == 8
    assert bench.CONFIGS["cfg5"]["seq"] == 786432 and bench.CONFIGS["cfg5"]["hq"] == 64
    # useful FLOPs: 7 D Hq S (S + 1)
    assert bench.useful_flops(262144, 32, 128) == 7.0 * 128 * 32 * 262144 * 262145
