timeout 600 python -m pytest tests/test_sgmv_gpu.py -x -q > gpurun_out/tc_pytest.log 2>&1; echo "pytest=$?"
tail -5 gpurun_out/tc_pytest.log
for args in "" "--preset c4" "--preset c4 --segments 2048" "--preset c4 --prefill 8192" "--preset c4 --rank 32" "--preset c4 --rank 64" "--popularity uniform"; do
  timeout 200 python bench.py $args --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/tmp/o.err
  python -c "import json,sys; d=json.load(open('/tmp/o.json')); print(repr(sys.argv[1]), round(d['value'],3), 'us frac', round(d['roofline']['frac'],3))" "$args" || tail -3 /tmp/o.err
done 2>&1 | tee gpurun_out/tc_bench.txt
timeout 120 python scripts/trace_tc.py > gpurun_out/trace_tc.txt 2>&1; cat gpurun_out/trace_tc.txt
timeout 120 python scripts/trace_tc.py --segments 2048 >> gpurun_out/trace_tc.txt 2>&1; tail -16 gpurun_out/trace_tc.txt
