#!/bin/bash
# synccheck co-residency hypothesis + c4 phase traces (instrumented build)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/sync2
CS="/usr/local/cuda/bin/compute-sanitizer --kernel-name kns=sgmv --print-limit 4 --tool synccheck"
i=0
for args in "8 0 8 16 0 0 0" "8 0 16 16 0 0 0" "8 0 9 16 0 0 0" "8 0 32 8 0 0 0" "8 0 64 4 0 1 0"; do
  i=$((i+1)); echo "== one $args" > gpurun_out/sync2/$i.log
  timeout 300 $CS python scripts/sanitize.py one $args >> gpurun_out/sync2/$i.log 2>&1
done
cp build/variants/instr/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
for split in 0 1; do
  timeout 120 python scripts/trace_tc.py --split $split > gpurun_out/trace_c4_split$split.txt 2>&1
done
timeout 120 python scripts/trace_tc.py --segments 128,$(python -c "print(','.join(['1']*31))") > gpurun_out/trace_c4_128.txt 2>&1
