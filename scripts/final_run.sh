#!/bin/bash
# Round-end evidence in one GPU call: smoke, GPU tests, headline bench line, every
# BASELINE config, the popularity x batch sweep, the ncu launch list, one full
# single-launch capture and one steady-state graph capture.  Outputs -> gpurun_out/.
mkdir -p gpurun_out
st=gpurun_out/final_status.txt; : > $st
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> $st
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> $st
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?" >> $st
bash scripts/run_configs.sh > gpurun_out/configs.txt 2>&1; echo "configs=$?" >> $st
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --sweep > /dev/null 2> gpurun_out/sweep.err; echo "sweep=$?" >> $st
timeout 300 python scripts/adapter_load_bench.py > gpurun_out/adapter_load.json 2>&1; echo "adapter=$?" >> $st
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sgmv -c 224 --csv \
  --log-file gpurun_out/launches.csv python bench.py --profile --warmup 1 --sites 224 > gpurun_out/ncu_launch.log 2>&1
echo "ncu_launch=$?" >> $st
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_fast -s 20 -c 1 \
  -o gpurun_out/prof -f python bench.py --profile --warmup 1 --sites 32 > gpurun_out/ncu_full.log 2>&1
echo "ncu_full=$?" >> $st
timeout 900 ncu --graph-profiling graph --nvtx --nvtx-include "lsg_graph/" --set full --import-source on \
  --clock-control none -c 1 -o gpurun_out/prof_graph -f python bench.py --profile-graph --sites 224 > gpurun_out/ncu_graph.log 2>&1
echo "ncu_graph=$?" >> $st
cat $st
