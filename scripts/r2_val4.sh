#!/bin/bash
cd $GRAFT_REPO_ROOT; o=gpurun_out/val11; mkdir -p $o
timeout 900 python -m pytest tests/test_sgmv_gpu.py -q -m gpu -p no:cacheprovider -k "long or mma or generations or mixed or pdl" > $o/pytest.log 2>&1; tail -2 $o/pytest.log; grep FAILED $o/pytest.log | head
B="python bench.py --no-extras --no-e2e --no-cpu-baseline --no-traffic --steps 20 --warmup 3"
for c in "--preset c4" "--preset c3"; do
  echo "$c: $(timeout 300 $B $c 2>>$o/err.txt | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(round(d['value'],2),'us', round(d['roofline']['frac'],3))")"
done
cp build/variants/instr/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
timeout 120 python scripts/trace_tc.py --gen 4 --segments 2048 > $o/trace_c3.txt 2>&1
cat $o/trace_c3.txt
