#!/bin/bash
cd $GRAFT_REPO_ROOT; o=gpurun_out/dense; mkdir -p $o
cp paper_2310_18547_b200/lib/libsgmv_b200.so /tmp/prod.so
for v in $1; do
  cp build/variants/$v/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
  echo "$v $(timeout 300 python scripts/dense_lora_bench.py 2>>$o/var.err)"
done
cp /tmp/prod.so paper_2310_18547_b200/lib/libsgmv_b200.so
