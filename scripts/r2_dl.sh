#!/bin/bash
cd $GRAFT_REPO_ROOT; o=gpurun_out/dl; mkdir -p $o
timeout 600 python -m pytest tests/test_sgmv_gpu.py -q -m gpu -p no:cacheprovider -k "dense" > $o/pytest.log 2>&1; tail -2 $o/pytest.log
timeout 300 python scripts/dense_lora_bench.py > $o/dense.json 2>$o/dense.err; cat $o/dense.json
for tool in memcheck racecheck synccheck; do
  timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $tool --kernel-name kns=dense --kernel-name kns=sgmv --print-limit 20 python scripts/sanitize.py dense > $o/san_$tool.log 2>&1
  echo "$tool=$?"; tail -1 $o/san_$tool.log
done
