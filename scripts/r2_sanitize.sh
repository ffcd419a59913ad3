#!/bin/bash
# compute-sanitizer over every kernel family (scripts/sanitize.py), logs under gpurun_out/san/
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/san
CS=/usr/local/cuda/bin/compute-sanitizer
F="--kernel-name kns=sgmv --kernel-name kns=dense --kernel-name kns=build_segments --kernel-name kns=permute"
for tool in synccheck; do
  SAN_MAX_CLUSTER=${SAN_MAX_CLUSTER:-16} timeout 1500 $CS --tool $tool $F --print-limit 200 python scripts/sanitize.py > gpurun_out/san/$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san/$tool.log
done
