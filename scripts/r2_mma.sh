#!/bin/bash
# MMA pair: parity tests, c3 / c4 benches (A/B against the earlier paths), sanitizer on the new kernels
cd $GRAFT_REPO_ROOT; o=gpurun_out/mma; mkdir -p $o
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
j --preset c3 --rank 16 --hidden 4096
j --preset c4
j --preset c4-128
j --preset c2
cat $o/bench.txt
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --kernel-name kns=sgmv_mma python scripts/sanitize.py mma > $o/memcheck.log 2>&1; tail -2 $o/memcheck.log
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --kernel-name kns=sgmv_mma python scripts/sanitize.py mma > $o/racecheck.log 2>&1; tail -2 $o/racecheck.log
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --kernel-name kns=sgmv_mma python scripts/sanitize.py mma > $o/synccheck.log 2>&1; tail -2 $o/synccheck.log
