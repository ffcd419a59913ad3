#!/bin/bash
# A/B of build/variants/<name> libraries against the product library on bench.py argument sets.
# Usage (under gpurun): VARIANTS="a b" bash scripts/r2_ab_args.sh "<args1>" "<args2>" ...
cd $GRAFT_REPO_ROOT; o=gpurun_out/abargs; mkdir -p $o
cp paper_2310_18547_b200/lib/libsgmv_b200.so /tmp/prod.so
for v in prod $VARIANTS; do
  if [ $v = prod ]; then cp /tmp/prod.so paper_2310_18547_b200/lib/libsgmv_b200.so
  else cp build/variants/$v/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so; fi
  for a in "$@"; do
    r=$(timeout 300 python bench.py $a --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-extras --no-traffic 2>>$o/err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3))")
    echo "$v [$a] $r" | tee -a $o/res.txt
  done
done
cp /tmp/prod.so paper_2310_18547_b200/lib/libsgmv_b200.so
