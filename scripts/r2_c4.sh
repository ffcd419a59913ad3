#!/bin/bash
# c4 (long prefill) on the streamed tensor-core kernel: parity, bench, phase trace, ncu
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/c4
timeout 900 python -m pytest tests/test_sgmv_gpu.py -x -q -m gpu -k "long_segment or streamed or tc_ or pdl_chain or mixed" > gpurun_out/c4/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c4/pytest.log
for pre in c4 c4-128; do
  for leg in 0 1 2; do
    timeout 300 python - <<PY > gpurun_out/c4/bench_${pre}_legacy${leg}.json 2>&1
import sys, subprocess, json
sys.argv = ["bench.py", "--preset", "$pre", "--no-extras", "--no-e2e", "--no-cpu-baseline", "--steps", "20"]
import paper_2310_18547_b200 as lsg
lsg.set_option(lsg._lib.LSG_OPT_TC_LEGACY, $leg)
import bench; bench.main()
PY
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sgmv -c 60 --csv \
  --log-file gpurun_out/c4/launches_c4.csv python bench.py --preset c4 --profile --warmup 2 --sites 8 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_tc_ -s 4 -c 2 \
  -o gpurun_out/c4/prof_tc3 -f python bench.py --preset c4 --profile --warmup 2 --sites 8 > gpurun_out/c4/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 python -m pytest tests/test_sgmv_gpu.py -x -q -m gpu -k "tp_" > gpurun_out/c4/pytest_tp.log 2>&1; echo "rc=$?" >> gpurun_out/c4/pytest_tp.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c4/bench_full.json 2> gpurun_out/c4/bench_full.err
cp build/variants/instr/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
timeout 120 python scripts/trace_tc.py > gpurun_out/c4/trace_c4.txt 2>&1
timeout 120 python scripts/trace_tc.py --segments 128,$(python -c "print(','.join(['1']*31))") > gpurun_out/c4/trace_c4_128.txt 2>&1
# c3 (rank 64, shared adapters) phase traces for several tile / cluster plans (instrumented build)
for cfg in "0 0" "0 8" "0 16" "8 0" "8 16" "1 0" "1 16"; do
  set -- $cfg
  timeout 120 python scripts/trace_phases.py --popularity uniform --batch 64 --hidden 5120 --rank 64 --tile-rows $1 --cluster $2 \
    > gpurun_out/c4/trace_c3_mt$1_c$2.txt 2>&1
done
