#!/bin/bash
# Experiment flags (LSG_EXP bits: 1 no L2 hint, 2 single A piece, 4 B issued first) at the headline shape.
for e in 0 1 2 4 3 7; do
  for c in 2 3 4; do
    LSG_EXP=$e timeout 120 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --cluster $c \
      | python -c "import json,sys;d=json.loads(sys.stdin.read());print('exp=$e C=$c', round(d['value'],3), 'us nopdl', round(d['us_per_launch_no_pdl'],3))"
  done
done
