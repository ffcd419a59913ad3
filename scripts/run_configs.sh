#!/bin/bash
# Every BASELINE.json config through bench.py (one JSON line each) -> gpurun_out/configs.jsonl
mkdir -p gpurun_out
out=gpurun_out/configs.jsonl
: > $out
for p in c1 c2 c3 c3-bgmv c4 c5; do
  timeout 600 python bench.py --preset $p --steps 30 --warmup 3 ${CFG_ARGS:-} >> $out 2> gpurun_out/cfg_$p.err || echo "{\"preset\": \"$p\", \"failed\": true}" >> $out
done
for pop in uniform skewed identical; do
  timeout 600 python bench.py --popularity $pop --steps 30 --warmup 3 --no-cpu-baseline ${CFG_ARGS:-} >> $out 2> gpurun_out/cfg_$pop.err
done
timeout 600 python bench.py --dtype bf16 --steps 30 --warmup 3 --no-cpu-baseline >> $out 2> gpurun_out/cfg_bf16.err
python - <<'PY'
import json
for l in open("gpurun_out/configs.jsonl"):
    d = json.loads(l)
    if d.get("failed"):
        print(d); continue
    c = d["config"]
    print(f'{c.get("preset") or "-":8s} {c["workload"][:70]:70s} {d["value"]:8.2f} us  frac {d["roofline"]["frac"]:.3f}  '
          f'e2e {d["e2e"]["value"] if d.get("e2e") else None}  cpu {d.get("cpu_baseline", {}).get("value")}  launch {c["launch"]}')
PY
