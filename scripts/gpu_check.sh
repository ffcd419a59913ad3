#!/bin/bash
# One GPU round-trip: smoke, GPU parity tests, bench, ncu launch list + one full capture.
# Usage (under gpurun): bash scripts/gpu_check.sh [tests|bench|ncu|all]
set -u
what=${1:-all}
mkdir -p gpurun_out
st=gpurun_out/status.txt
: > $st
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/smi.txt 2>&1
if [[ $what == all || $what == tests ]]; then
  timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> $st
  timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> $st
fi
if [[ $what == all || $what == bench ]]; then
  timeout 600 python bench.py --steps 50 --warmup 5 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?" >> $st
fi
if [[ $what == all || $what == ncu ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sgmv -c 224 --csv \
    --log-file gpurun_out/launches.csv python bench.py --profile --warmup 1 --sites 224 ${BENCH_ARGS:-} > gpurun_out/ncu_launch.log 2>&1
  echo "ncu_launch=$?" >> $st
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_fast -s 20 -c 2 \
    -o gpurun_out/prof -f python bench.py --profile --warmup 1 --sites 32 ${BENCH_ARGS:-} > gpurun_out/ncu_full.log 2>&1
  echo "ncu_full=$?" >> $st
fi
cat $st
