#!/bin/bash
cd $GRAFT_REPO_ROOT; o=gpurun_out/dense; mkdir -p $o
timeout 120 python scripts/dense_debug.py 2>&1 | grep -v "rel err" | tail -30
timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --kernel-name kns=dense --print-limit 10 python scripts/dense_debug.py > $o/dbg_race.log 2>&1; echo race=$?; grep -E "RACECHECK SUMMARY|Error|hazard" $o/dbg_race.log | head
timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --kernel-name kns=dense --print-limit 10 python scripts/dense_debug.py > $o/dbg_mem.log 2>&1; echo mem=$?; grep -E "ERROR SUMMARY|Invalid" $o/dbg_mem.log | head
