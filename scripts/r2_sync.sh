#!/bin/bash
# synccheck over every kernel family with clusters capped at 8 (profiles/round2/sanitizer.md)
cd $GRAFT_REPO_ROOT; o=${OUT:-gpurun_out/sync}; mkdir -p $o
F="--kernel-name kns=sgmv --kernel-name kns=dense --kernel-name kns=build_segments --kernel-name kns=permute"
SAN_MAX_CLUSTER=8 timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool synccheck $F --print-limit 100 python scripts/sanitize.py > $o/san_synccheck.log 2>&1
echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|cases done" $o/san_synccheck.log
