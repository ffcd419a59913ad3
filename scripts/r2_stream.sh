#!/bin/bash
# K9 streaming kernel: parity, c4 benches against tc3, trace
cd $GRAFT_REPO_ROOT; o=gpurun_out/stream4; mkdir -p $o
timeout 900 python -m pytest tests/test_sgmv_gpu.py -q -m gpu -k "mma_pair_long or long_segments_tensor_core or dropin" > $o/pytest.log 2>&1; tail -3 $o/pytest.log
B="python bench.py --no-extras --no-e2e --no-cpu-baseline --no-traffic --steps 20 --warmup 3"
j() { echo "== $*" >> $o/bench.txt; timeout 300 $B "$@" 2>>$o/bench.err | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(round(d['value'],2),'us', round(d['roofline']['frac'],3))" >> $o/bench.txt; }
j --preset c4 --tc-gen 4
j --preset c4 --tc-gen 4 --dtype bf16
j --preset c4-128 --tc-gen 4
j --preset c4 --tc-gen 0
j --preset c4 --tc-gen 4 --rank 64
j --preset c4 --tc-gen 0 --rank 64
j --preset c3
cat $o/bench.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_stream -s 4 -c 1 \
  -o $o/prof_stream -f python bench.py --preset c4 --tc-gen 4 --profile --warmup 2 --sites 8 > $o/ncu.log 2>&1; echo "ncu rc=$?"
cp build/variants/instr/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
timeout 120 python scripts/trace_tc.py --gen 4 > $o/trace_c4_g4.txt 2>&1
timeout 120 python scripts/trace_tc.py --gen 4 --segments 2048 > $o/trace_c4_prefill_g4.txt 2>&1
cat $o/trace_c4_g4.txt $o/trace_c4_prefill_g4.txt
