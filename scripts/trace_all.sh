#!/bin/bash
mkdir -p gpurun_out
for pop in ${TRACE_POPS:-distinct identical}; do
  for pdl in 1 0; do
    timeout 120 python scripts/trace_phases.py --popularity $pop --pdl $pdl
  done
done
