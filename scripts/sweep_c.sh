# cluster-size sweep for decode batches: prints us/launch per (pop, batch, C)
for pop in distinct uniform identical; do
for b in 8 16 32 64 128; do
  line="$pop b=$b:"
  for c in 0 1 2 4 8 16; do
    timeout 100 python bench.py --popularity $pop --batch $b --cluster $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/dev/null
    v=$(python -c "import json; d=json.load(open('/tmp/o.json')); print(round(d['value'],2))" 2>/dev/null)
    line="$line C$c=$v"
  done
  echo "$line"
done; done
