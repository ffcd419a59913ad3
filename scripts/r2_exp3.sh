#!/bin/bash
# c3 / c4 diagnosis: per-variant bench lines, phase traces (instrumented build), synccheck at C <= 8
cd $GRAFT_REPO_ROOT; o=gpurun_out/exp3; mkdir -p $o
B="python bench.py --no-extras --no-e2e --no-cpu-baseline --no-traffic --steps 20 --warmup 3"
j() { echo "== $*" >> $o/bench.txt; timeout 300 $B "$@" 2>>$o/bench.err | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(round(d['value'],2),'us', round(d['roofline']['frac'],3), d['config'].get('launch'))" >> $o/bench.txt; }
j --preset c3
j --preset c3 --tc-min-rows 8
j --preset c3 --tc-min-rows 8 --dtype bf16
j --preset c4
j --preset c4 --segments 2048 --sites 32
j --preset c4 --segments 2048 --sites 32 --tc-min-rows 128
j --preset c4 --segments $(python -c "print(','.join(['1']*31))") --sites 32
j --preset c4-128
j --preset c4 --segments 512,512,512,512 --sites 32
cat $o/bench.txt
SAN_MAX_CLUSTER=8 timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --kernel-name kns=sgmv --kernel-name kns=dense \
  --kernel-name kns=build_segments --kernel-name kns=permute --print-limit 100 python scripts/sanitize.py > $o/synccheck_c8.log 2>&1
echo "synccheck rc=$?" >> $o/synccheck_c8.log; tail -3 $o/synccheck_c8.log
timeout 600 python -m pytest tests/test_sgmv_gpu.py -q -m gpu -k "tp_nccl" > $o/tp.log 2>&1; tail -3 $o/tp.log
cp build/variants/instr/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
timeout 120 python scripts/trace_tc.py > $o/trace_c4.txt 2>&1
timeout 120 python scripts/trace_tc.py --segments 2048 > $o/trace_c4_prefill.txt 2>&1
