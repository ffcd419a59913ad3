#!/bin/bash
cd $GRAFT_REPO_ROOT; o=gpurun_out/dense; mkdir -p $o
timeout 600 python -m pytest tests/test_sgmv_gpu.py -q -m gpu -p no:cacheprovider -k "dense" > $o/pytest.log 2>&1; tail -1 $o/pytest.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv \
  -k regex:dense --log-file $o/launches.csv python scripts/dense_lora_bench.py --profile > /dev/null 2>&1
python scripts/launch_list_summary.py $o/launches.csv 2>/dev/null | head -20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense -s 3 -c 1 -o $o/prof_dense -f python scripts/dense_lora_bench.py --profile > $o/ncu_full.log 2>&1
echo ncu_full=$?
