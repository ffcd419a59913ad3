#!/bin/bash
# dense_lora (tensor-core GEMM + folded LoRA expand): parity tests, the fused-vs-unfused timing,
# compute-sanitizer on the dense case.
cd $GRAFT_REPO_ROOT; o=gpurun_out/dense; mkdir -p $o
timeout 600 python -m pytest tests/test_sgmv_gpu.py -q -m gpu -p no:cacheprovider -k "dense" -x > $o/pytest.log 2>&1; tail -3 $o/pytest.log
timeout 300 python scripts/dense_lora_bench.py > $o/bench.json 2> $o/bench.err; cat $o/bench.json; tail -3 $o/bench.err
for tool in memcheck racecheck synccheck; do
  timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $tool --kernel-name kns=dense --print-limit 20 python scripts/sanitize.py dense > $o/san_$tool.log 2>&1
  echo "$tool=$?"; tail -2 $o/san_$tool.log
done
