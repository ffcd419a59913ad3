#!/bin/bash
# round-2 evidence: sanitizers over every kernel family (C <= 8 for synccheck), ncu launch
# lists + full captures of the headline, c3 (MMA pair) and c4 (streaming kernel)
cd $GRAFT_REPO_ROOT; o=${OUT:-gpurun_out/ev}; mkdir -p $o
CS=/usr/local/cuda/bin/compute-sanitizer
F="--kernel-name kns=sgmv --kernel-name kns=dense --kernel-name kns=build_segments --kernel-name kns=permute"
for tool in memcheck racecheck synccheck; do
  mc=16; [[ $tool == synccheck ]] && mc=8
  SAN_MAX_CLUSTER=$mc timeout 1200 $CS --tool $tool $F --print-limit 100 python scripts/sanitize.py > $o/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|cases done" $o/san_$tool.log
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none -k regex:sgmv -c 224 --csv --log-file $o/launches_headline.csv python bench.py --profile --warmup 1 --sites 224 > /dev/null 2>&1; echo "list1 rc=$?"
timeout 600 ncu --metrics $M --clock-control none -k regex:sgmv -c 30 --csv --log-file $o/launches_c3.csv python bench.py --preset c3 --profile --warmup 2 --sites 8 > /dev/null 2>&1; echo "list2 rc=$?"
timeout 600 ncu --metrics $M --clock-control none -k regex:sgmv -c 30 --csv --log-file $o/launches_c4.csv python bench.py --preset c4 --profile --warmup 2 --sites 8 > /dev/null 2>&1; echo "list3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_fast -s 20 -c 1 -o $o/prof_headline -f python bench.py --profile --warmup 1 --sites 32 > /dev/null 2>&1; echo "full1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_mma -s 4 -c 2 -o $o/prof_c3 -f python bench.py --preset c3 --profile --warmup 2 --sites 8 > /dev/null 2>&1; echo "full2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_stream -s 2 -c 1 -o $o/prof_c4 -f python bench.py --preset c4 --profile --warmup 2 --sites 8 > /dev/null 2>&1; echo "full3 rc=$?"
