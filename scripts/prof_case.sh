#!/bin/bash
# ncu --set full on one configuration: prof_case.sh <tag> <bench args...>
tag=$1; shift
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgmv_fast -s 20 -c 1 \
  -o gpurun_out/prof_$tag -f python bench.py --profile --warmup 1 --sites 32 "$@" > gpurun_out/ncu_$tag.log 2>&1
echo "$tag=$?"
