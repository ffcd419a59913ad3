#!/bin/bash
cd $GRAFT_REPO_ROOT; o=gpurun_out/ind; mkdir -p $o
timeout 600 python -m pytest tests/test_sgmv_gpu.py -q -m gpu -p no:cacheprovider -k "independent or verify or kernel_variants or pdl" > $o/pytest.log 2>&1; tail -2 $o/pytest.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-traffic > $o/bench.json 2> $o/bench.err
python -c "
import json; d=json.loads(open('$o/bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'grouped', d.get('grouped_us_per_site'), 'indep', d.get('independent_kv_up_us_per_site'), 'nopdl', d.get('us_per_launch_no_pdl'))
print(d.get('decode_step'))"
