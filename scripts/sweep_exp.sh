#!/bin/bash
run() {
  timeout 120 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e "$@" \
    | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$*', round(d['value'],3), 'us nopdl', round(d['us_per_launch_no_pdl'],3), 'iso', round(d['isolated_launch_us_median'],2), d['config']['launch'])"
}
for c in 2 3 4; do run --cluster $c; run --cluster $c --no-l2-staging; done
for pop in identical uniform skewed; do run --popularity $pop; done
