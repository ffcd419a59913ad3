#!/bin/bash
cd $GRAFT_REPO_ROOT; o=gpurun_out/dense; mkdir -p $o
cp paper_2310_18547_b200/lib/libsgmv_b200.so /tmp/prod.so
cp build/variants/dn_trace/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
timeout 300 python scripts/dense_trace.py 2>&1 | tail -12
cp /tmp/prod.so paper_2310_18547_b200/lib/libsgmv_b200.so
