#!/bin/bash
mkdir -p gpurun_out
for args in "--popularity distinct" "--popularity distinct --pdl 0" "--popularity distinct --cluster 4" "--popularity identical" "--popularity identical --cluster 8" "--popularity uniform --cluster 8"; do
  timeout 120 python scripts/trace_phases.py $args
done
