#!/bin/bash
mkdir -p gpurun_out
for c in ${TRACE_CS:-2 4}; do
  timeout 120 python scripts/trace_phases.py --popularity distinct --pdl 1 --cluster $c
done
