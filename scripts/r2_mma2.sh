#!/bin/bash
# MMA pair (TMA version): parity, benches, traces
cd $GRAFT_REPO_ROOT; o=gpurun_out/mma5; mkdir -p $o
timeout 900 python -m pytest tests/test_sgmv_gpu.py -q -m gpu -x -k "mma or rank64 or grouped_sites_rank64 or baseline_shapes" > $o/pytest.log 2>&1; tail -3 $o/pytest.log
B="python bench.py --no-extras --no-e2e --no-cpu-baseline --no-traffic --steps 20 --warmup 3"
j() { echo "== $*" >> $o/bench.txt; timeout 300 $B "$@" 2>>$o/bench.err | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(round(d['value'],2),'us', round(d['roofline']['frac'],3))" >> $o/bench.txt; }
j --preset c3
j --preset c3-skewed
j --preset c3 --popularity identical
j --preset c3 --dtype bf16
j --preset c4 --tc-gen 3
j --preset c4-128 --tc-gen 3
j --preset c4-128 --tc-gen 3 --mma-min-rows 2
j --preset c4
cat $o/bench.txt
cp build/variants/instr/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
timeout 120 python scripts/trace_tc.py --segments 8,8,8,8,8,8,8,8 --hidden 5120 --rank 64 > $o/trace_c3.txt 2>&1
timeout 120 python scripts/trace_tc.py --gen 3 --segments 2048 > $o/trace_c4_prefill_g3.txt 2>&1
cat $o/trace_c3.txt $o/trace_c4_prefill_g3.txt
