#!/bin/bash
cd $GRAFT_REPO_ROOT; o=gpurun_out/dense; mkdir -p $o
timeout 600 python -m pytest tests/test_sgmv_gpu.py -q -m gpu -p no:cacheprovider -k "dense" -x > $o/pytest.log 2>&1; tail -2 $o/pytest.log
timeout 300 python scripts/dense_lora_bench.py > $o/bench.json 2> $o/bench.err; cat $o/bench.json; tail -3 $o/bench.err
cp paper_2310_18547_b200/lib/libsgmv_b200.so /tmp/prod.so
cp build/variants/dn_trace/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
timeout 300 python scripts/dense_trace.py 2>&1 | tail -9
cp /tmp/prod.so paper_2310_18547_b200/lib/libsgmv_b200.so
