# launch list + one full capture of the tensor-core kernel on the c4 preset
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/tc_launches.csv \
  python bench.py --preset c4 --profile --warmup 1 --sites 8 > /dev/null 2>&1; echo "list=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgmv_tc -s 4 -c 1 \
  -o gpurun_out/prof_tc -f python bench.py --preset c4 --profile --warmup 1 --sites 8 > gpurun_out/ncu_tc.log 2>&1; echo "full=$?"
