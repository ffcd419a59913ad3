#!/bin/bash
# A/B of the product library against build/variants/<name> on chosen presets (value only).
# Usage (under gpurun): bash scripts/r2_ab.sh "<presets>" <variant>... ; tests with K="<pytest -k expression>"
cd $GRAFT_REPO_ROOT; o=gpurun_out/ab; mkdir -p $o
presets=$1; shift
cp paper_2310_18547_b200/lib/libsgmv_b200.so /tmp/prod.so
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -k "$K" > $o/pytest.log 2>&1; echo "pytest=$?" >> $o/status.txt
  tail -3 $o/pytest.log
fi
for rep in 1 2; do
for v in prod "$@"; do
  if [ $v = prod ]; then cp /tmp/prod.so paper_2310_18547_b200/lib/libsgmv_b200.so
  else cp build/variants/$v/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so; fi
  for p in $presets; do
    r=$(timeout 300 python bench.py --preset $p --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-extras --no-traffic 2>$o/err_${v}_$p.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3))")
    echo "rep$rep $v $p $r" | tee -a $o/ab.txt
  done
done
done
cp /tmp/prod.so paper_2310_18547_b200/lib/libsgmv_b200.so
