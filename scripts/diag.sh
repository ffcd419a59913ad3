#!/bin/bash
mkdir -p gpurun_out
timeout 60 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --popularity skewed > gpurun_out/d_skew.json 2> gpurun_out/d_skew.err; echo "skewed rc=$?"
timeout 60 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --popularity skewed --no-l2-staging > gpurun_out/d_skew2.json 2> gpurun_out/d_skew2.err; echo "skewed no-staging rc=$?"
timeout 120 python -m pytest tests/test_sgmv_gpu.py -x -q -k "verify" > gpurun_out/d_verify.log 2>&1; echo "verify rc=$?"
timeout 300 python -m pytest tests/test_sgmv_gpu.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
