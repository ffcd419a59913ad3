#!/bin/bash
# round-2 GPU check: parity tests, then compute-sanitizer over every kernel family
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/san
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --kernel-name kns=sgmv --kernel-name kns=dense --kernel-name kns=build_segments --kernel-name kns=permute \
     --print-limit 50 python scripts/sanitize.py > gpurun_out/san/$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san/$tool.log
done
