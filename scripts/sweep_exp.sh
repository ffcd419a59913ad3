#!/bin/bash
run() {
  timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e "$@" > /tmp/b.json 2> /tmp/b.err
  if [ -s /tmp/b.json ]; then
    python -c "import json,sys;d=json.loads(open('/tmp/b.json').read());print('$*', round(d['value'],3), 'us nopdl', round(d['us_per_launch_no_pdl'],3), 'frac', round(d['roofline']['frac'],3), d['config']['launch'])"
  else
    echo "$* FAILED"; tail -5 /tmp/b.err
  fi
}
run
for pop in identical uniform skewed; do run --popularity $pop; done
for b in 1 8 32; do run --batch $b; done
for p in c1 c3 c3-bgmv c5 c4; do run --preset $p; done
