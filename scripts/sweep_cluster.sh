#!/bin/bash
# Sweep the split-K cluster size at the headline shape (and a few popularities).
mkdir -p gpurun_out
run() {
  timeout 120 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e "$@" \
    | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$*', round(d['value'],3), 'us', round(d['roofline']['frac'],3), 'nopdl', round(d['us_per_launch_no_pdl'],3), 'iso', round(d['isolated_launch_us_median'],2), d['config']['launch'])"
}
for c in ${CS:-0 2 3 4}; do run --popularity distinct --cluster $c; done
for c in 0 4 8 16; do run --popularity identical --cluster $c; done
for c in 0 8 16; do run --popularity uniform --cluster $c; done
run --popularity skewed
