#!/bin/bash
cd $GRAFT_REPO_ROOT; o=gpurun_out/tr9; mkdir -p $o
cp build/variants/instr/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
timeout 120 python scripts/trace_tc.py --gen 4 --segments 2048 > $o/trace_prefill.txt 2>&1
timeout 120 python scripts/trace_tc.py --gen 4 > $o/trace_c4.txt 2>&1
cat $o/trace_prefill.txt $o/trace_c4.txt
