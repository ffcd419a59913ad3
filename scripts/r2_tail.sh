#!/bin/bash
# synccheck at portable cluster sizes + the dense projection schedules
cd $GRAFT_REPO_ROOT; o=gpurun_out/tail; mkdir -p $o
SAN_MAX_CLUSTER=8 timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --kernel-name kns=sgmv --kernel-name kns=dense --kernel-name kns=build_segments --kernel-name kns=permute --print-limit 100 python scripts/sanitize.py > $o/synccheck_c8.log 2>&1; echo "synccheck=$?"
grep -E "ERROR SUMMARY|sanitize cases" $o/synccheck_c8.log
timeout 300 python scripts/dense_lora_bench.py > $o/dense.json 2> $o/dense.err; cat $o/dense.json
