#!/bin/bash
# phase traces of the MMA pair (instrumented build) + ncu of its two kernels at c3 / c4
cd $GRAFT_REPO_ROOT; o=gpurun_out/mmat; mkdir -p $o
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread --clock-control none -k regex:sgmv -c 12 --csv \
  --log-file $o/launches_c3.csv python bench.py --preset c3 --profile --warmup 2 --sites 8 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:sgmv -c 12 --csv \
  --log-file $o/launches_c4g3.csv python bench.py --preset c4 --profile --warmup 2 --sites 8 --tc-gen 3 > /dev/null 2>&1
cp build/variants/instr/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
S8=8,8,8,8,8,8,8,8
timeout 120 python scripts/trace_tc.py --segments $S8 --hidden 5120 --rank 64 > $o/trace_c3.txt 2>&1
timeout 120 python scripts/trace_tc.py --gen 3 > $o/trace_c4_g3.txt 2>&1
timeout 120 python scripts/trace_tc.py --gen 3 --segments 2048 > $o/trace_c4_prefill_g3.txt 2>&1
timeout 120 python scripts/trace_tc.py --gen 3 --segments 128,$(python -c "print(','.join(['1']*31))") --mma-min-rows 2 > $o/trace_c4_128_g3.txt 2>&1
tail -n 30 $o/*.txt
