#!/bin/bash
# one-launch K7 (LSG_OPT_MMA_FUSED): parity tests, then A/B against the pair on the MMA presets
cd $GRAFT_REPO_ROOT; o=gpurun_out/k7f; mkdir -p $o
[ -z "$NOTEST" ] && timeout 900 python -m pytest tests/test_sgmv_gpu.py -q -m gpu -p no:cacheprovider -k "mma" -x > $o/pytest.log 2>&1; tail -3 $o/pytest.log
B="python bench.py --no-extras --no-e2e --no-cpu-baseline --no-traffic --steps 20 --warmup 3"
for c in "--preset c3" "--preset c3 --popularity skewed" "--preset c3 --popularity identical" "--preset c3 --hidden 4096"; do
  for m in ${MODES:-1 2}; do
    r=$(timeout 300 $B $c --mma-fused $m 2>>$o/err.txt | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(round(d['value'],2),'us', round(d['roofline']['frac'],3))")
    echo "$c | fused=$m | $r"
  done
done
