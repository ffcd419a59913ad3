#!/bin/bash
cd $GRAFT_REPO_ROOT; o=gpurun_out/val2; mkdir -p $o
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $o/pytest_gpu.log 2>&1; tail -2 $o/pytest_gpu.log; grep FAILED $o/pytest_gpu.log | head
CS=/usr/local/cuda/bin/compute-sanitizer
F="--kernel-name kns=sgmv --kernel-name kns=dense --kernel-name kns=build_segments --kernel-name kns=permute"
for tool in racecheck synccheck memcheck; do
  mc=16; [[ $tool == synccheck ]] && mc=8
  SAN_MAX_CLUSTER=$mc timeout 1200 $CS --tool $tool $F --print-limit 100 python scripts/sanitize.py > $o/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|cases done" $o/san_$tool.log
done
cp build/variants/instr/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
timeout 120 python scripts/trace_tc.py --gen 4 --segments 2048 > $o/trace_c4_prefill.txt 2>&1
timeout 120 python scripts/trace_tc.py --gen 4 > $o/trace_c4.txt 2>&1
cat $o/trace_c4_prefill.txt
