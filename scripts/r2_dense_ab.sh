#!/bin/bash
# Dense projection A/B: parity tests + scripts/dense_lora_bench.py for the product library and
# build/variants/<name> libraries.  Usage (under gpurun): bash scripts/r2_dense_ab.sh <variant>...
cd $GRAFT_REPO_ROOT; o=gpurun_out/dense_ab; mkdir -p $o
cp paper_2310_18547_b200/lib/libsgmv_b200.so /tmp/prod.so
for v in prod "$@"; do
  if [ $v = prod ]; then cp /tmp/prod.so paper_2310_18547_b200/lib/libsgmv_b200.so
  else cp build/variants/$v/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so; fi
  timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -k dense > $o/pytest_$v.log 2>&1
  echo "$v tests: $(tail -1 $o/pytest_$v.log)"
  timeout 300 python scripts/dense_lora_bench.py > $o/bench_$v.json 2>$o/bench_$v.err
  echo "$v bench: $(cat $o/bench_$v.json)"
done
cp /tmp/prod.so paper_2310_18547_b200/lib/libsgmv_b200.so
