#!/bin/bash
# GPU parity of the dense projection + the decode-step bench (incl. the L2-prefetch variant)
cd $GRAFT_REPO_ROOT; o=gpurun_out/check; mkdir -p $o
timeout 900 python -m pytest tests/test_sgmv_gpu.py -q -m gpu -p no:cacheprovider -k "dense or prefetch" > $o/pytest.log 2>&1; tail -2 $o/pytest.log
timeout 300 python scripts/dense_lora_bench.py > $o/dense.json 2> $o/dense.err; cat $o/dense.json
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-traffic > $o/bench.json 2> $o/bench.err; tail -2 $o/bench.err
python -c "
import json; d=json.loads(open('$o/bench.json').read().strip().splitlines()[-1])
print(json.dumps(d.get('decode_step'), indent=1))"
