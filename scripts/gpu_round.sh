#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list (+ optional full capture).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
cat gpurun_out/bench_ref.json
if [ "${NCU:-0}" = "1" ]; then
  CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
  timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
fi
if [ "${NCU_FULL:-0}" = "1" ]; then
  CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
  timeout 300 $CMD > gpurun_out/plain_full.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|fwd_pair_kernel|fwd_kernel" \
      -s 2 -c 2 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
