#!/bin/bash
# One bench value per argument string (product library): bash scripts/r2_args.sh "<args1>" "<args2>" ...
cd $GRAFT_REPO_ROOT; o=gpurun_out/args; mkdir -p $o
for rep in 1 2; do
for a in "$@"; do
  r=$(timeout 300 python bench.py $a --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-extras --no-traffic 2>>$o/err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), round(d['roofline']['frac'],3))")
  echo "rep$rep [$a] $r" | tee -a $o/res.txt
done
done
