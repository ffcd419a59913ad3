#!/bin/bash
# A/B of library build variants (build/variants/<name>) on given bench presets
# usage: bash scripts/r2_variants.sh "<variant names>" "<preset args; ...>"
cd $GRAFT_REPO_ROOT; o=${OUT:-gpurun_out/var}; mkdir -p $o
cp paper_2310_18547_b200/lib/libsgmv_b200.so /tmp/prod.so
B="python bench.py --no-extras --no-e2e --no-cpu-baseline --no-traffic --steps 20 --warmup 3"
IFS=';' read -ra CASES <<< "$2"
for v in $1; do
  cp build/variants/$v/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
  for c in "${CASES[@]}"; do
    r=$(timeout 300 $B $c 2>>$o/err.txt | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(round(d['value'],2),'us', round(d['roofline']['frac'],3))")
    echo "$v | $c | $r" >> $o/ab.txt
  done
done
cp /tmp/prod.so paper_2310_18547_b200/lib/libsgmv_b200.so
cat $o/ab.txt
