#!/bin/bash
run() {
  timeout 150 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e "$@" > /tmp/b.json 2> /tmp/b.err
  if [ -s /tmp/b.json ]; then
    python -c "import json,sys;d=json.loads(open('/tmp/b.json').read());print('$*', round(d['value'],3), 'us nopdl', round(d['us_per_launch_no_pdl'],3), 'iso', round(d['isolated_launch_us_median'],2), d['config']['launch'])"
  else
    echo "$* FAILED"; tail -5 /tmp/b.err
  fi
}
for c in ${CS:-2 3 4}; do run --cluster $c; done
run --cluster 2 --no-l2-staging
for pop in identical uniform skewed; do run --popularity $pop; done
