#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/sync
CS="/usr/local/cuda/bin/compute-sanitizer --kernel-name kns=sgmv --print-limit 4"
i=0
for args in "8 1 9 0 0 0 0" "8 1 9 2 0 0 0" "8 1 9 4 0 0 0" "8 1 9 16 0 0 0" "8 1 9 16 0 1 0" "8 3 9 16 0 0 0" "8 0 4 16 0 0 0" "16 1 9 0 0 0 0" "8 1 9 16 1 0 0" "8 1 9 16 8 0 0"; do
  i=$((i+1))
  echo "== one $args" > gpurun_out/sync/$i.log
  timeout 300 $CS --tool synccheck python scripts/sanitize.py one $args >> gpurun_out/sync/$i.log 2>&1
  timeout 300 $CS --tool memcheck python scripts/sanitize.py one $args >> gpurun_out/sync/$i.log 2>&1
done

