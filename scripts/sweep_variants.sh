#!/bin/bash
# Headline bench across experimental library builds (scripts/build_variant.sh) and cluster sizes.
# Usage (under gpurun): bash scripts/sweep_variants.sh "main mb3 mb4" "0 2 4" [extra bench args]
mkdir -p gpurun_out
variants=${1:-main}; clusters=${2:-0}; shift 2
for v in $variants; do
  if [[ $v == main ]]; then unset LSG_LIB_OVERRIDE; else export LSG_LIB_OVERRIDE=build/variants/$v/libsgmv_b200.so; fi
  for c in $clusters; do
    timeout 200 python bench.py --cluster $c --steps 30 --warmup 3 --no-cpu-baseline --no-e2e "$@" > /tmp/o.json 2>/tmp/o.err
    python -c "import json,sys; d=json.load(open('/tmp/o.json')); print(sys.argv[1], 'C', sys.argv[2], round(d['value'],3), 'us frac', round(d['roofline']['frac'],3), 'nopdl', round(d['us_per_launch_no_pdl'],2), 'iso', round(d['isolated_launch_us_median'],2), d['config']['launch'])" "$v" "$c" || tail -3 /tmp/o.err
  done
done
