#!/bin/bash
# Round-2 evidence pass: smoke, GPU parity tests, the default bench line (with its
# sweep / configs / traffic extras), compute-sanitizer over every kernel family,
# ncu launch list + full captures of the headline, c3 and c4 kernels.
# Usage (under gpurun): bash scripts/r2_full.sh [tests] [bench] [san] [ncu]
cd $GRAFT_REPO_ROOT
o=${OUT:-gpurun_out/r2}; mkdir -p $o $o/san
st=$o/status.txt; : > $st
what="${*:-tests bench san ncu}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $o/smi.txt 2>&1
nproc > $o/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $o/host.txt
if [[ $what == *tests* ]]; then
  timeout 300 python __graft_entry__.py smoke > $o/smoke.log 2>&1; echo "smoke=$?" >> $st
  timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider ${PYTEST_ARGS:-} > $o/pytest_gpu.log 2>&1; echo "pytest=$?" >> $st
fi
if [[ $what == *bench* ]]; then
  timeout 900 python bench.py --steps 50 --warmup 5 > $o/bench.json 2> $o/bench.err; echo "bench=$?" >> $st
  timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_ref.json 2> $o/bench_ref.err; echo "bench_ref=$?" >> $st
fi
if [[ $what == *san* ]]; then
  CS=/usr/local/cuda/bin/compute-sanitizer
  F="--kernel-name kns=sgmv --kernel-name kns=dense --kernel-name kns=build_segments --kernel-name kns=permute"
  for tool in memcheck racecheck synccheck; do
    SAN_MAX_CLUSTER=${SAN_MAX_CLUSTER:-16} timeout 1200 $CS --tool $tool $F --print-limit 100 python scripts/sanitize.py ${SAN_WHICH:-} > $o/san/$tool.log 2>&1
    echo "$tool=$?" >> $st
  done
fi
if [[ $what == *ncu* ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sgmv -c 224 --csv \
    --log-file $o/launches_headline.csv python bench.py --profile --warmup 1 --sites 224 > $o/ncu_launch.log 2>&1
  echo "ncu_launch=$?" >> $st
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_fast -s 20 -c 1 \
    -o $o/prof_headline -f python bench.py --profile --warmup 1 --sites 32 > $o/ncu_full.log 2>&1
  echo "ncu_full=$?" >> $st
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv -s 4 -c 1 \
    -o $o/prof_c3 -f python bench.py --preset c3 --profile --warmup 2 --sites 8 > $o/ncu_c3.log 2>&1
  echo "ncu_c3=$?" >> $st
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sgmv -c 60 --csv \
    --log-file $o/launches_c4.csv python bench.py --preset c4 --profile --warmup 2 --sites 8 > /dev/null 2>&1
  echo "ncu_c4_list=$?" >> $st
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_stream -s 4 -c 1 \
    -o $o/prof_c4 -f python bench.py --preset c4 --profile --warmup 2 --sites 8 > $o/ncu_c4.log 2>&1
  echo "ncu_c4=$?" >> $st
fi
cat $st
