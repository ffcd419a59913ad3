#!/bin/bash
cd $GRAFT_REPO_ROOT; o=gpurun_out/val3; mkdir -p $o
timeout 900 python -m pytest tests/test_sgmv_gpu.py -q -m gpu -p no:cacheprovider -k "long or mma or stream or generations" > $o/pytest.log 2>&1; tail -2 $o/pytest.log; grep FAILED $o/pytest.log | head
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck memcheck; do
  timeout 900 $CS --tool $tool --kernel-name kns=sgmv_stream --print-limit 20 python scripts/sanitize.py stream > $o/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|cases done" $o/san_$tool.log
done
B="python bench.py --no-extras --no-e2e --no-cpu-baseline --no-traffic --steps 20 --warmup 3"
for c in "--preset c4" "--preset c4 --dtype bf16" "--preset c4 --rank 64" "--preset c4 --prefill 4096"; do
  echo "$c: $(timeout 300 $B $c 2>>$o/err.txt | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(round(d['value'],2),'us', round(d['roofline']['frac'],3))")"
done
cp build/variants/instr/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
timeout 120 python scripts/trace_tc.py --gen 4 --segments 2048 > $o/trace_c4_prefill.txt 2>&1
cat $o/trace_c4_prefill.txt
