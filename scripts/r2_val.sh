#!/bin/bash
# full GPU suite + the BASELINE config benches (default plans)
cd $GRAFT_REPO_ROOT; o=${OUT:-gpurun_out/val7}; mkdir -p $o
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $o/pytest_gpu.log 2>&1; tail -3 $o/pytest_gpu.log; grep FAILED $o/pytest_gpu.log | head
B="python bench.py --no-extras --no-e2e --no-cpu-baseline --no-traffic --steps 20 --warmup 3"
j() { echo "== $*" >> $o/bench.txt; timeout 300 $B "$@" 2>>$o/bench.err | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(round(d['value'],2),'us', round(d['roofline']['frac'],3))" >> $o/bench.txt; }
for pre in c1 c2 c3 c3-skewed c4-128 c4 c5; do j --preset $pre; done
j --preset c4 --tc-gen 5
j --preset c4-128 --tc-gen 5
cat $o/bench.txt
