#!/bin/bash
# c3 (rank 64 multi-row tiles) and c4 (cluster-free tensor-core pair): parity, A/B benches, ncu, traces
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/c34
timeout 1200 python -m pytest tests/test_sgmv_gpu.py -x -q -m gpu > gpurun_out/c34/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c34/pytest.log
run() {  # name, preset, extra python option lines
  timeout 300 python - "$@" <<'PY' >> gpurun_out/c34/ab.jsonl 2>> gpurun_out/c34/ab.err
import sys, json
name, preset, opts = sys.argv[1], sys.argv[2], sys.argv[3:]
sys.argv = ["bench.py", "--preset", preset, "--no-extras", "--no-e2e", "--no-cpu-baseline", "--steps", "20"]
import paper_2310_18547_b200 as lsg
for o in opts:
    k, v = o.split("=")
    lsg.set_option(int(k), int(v))
import io, contextlib, bench
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    bench.main()
d = json.loads(buf.getvalue().strip().splitlines()[-1])
print(json.dumps({"name": name, "preset": preset, "us": d["value"], "frac": d["roofline"]["frac"], "launch": d["config"]["launch"]}))
PY
}
for pre in c3 c3-skewed; do
  run "$pre auto" $pre
  run "$pre mt4 auto-c" $pre 3=4
  run "$pre mt8 c8" $pre 3=8 1=8
  run "$pre mt4 c8" $pre 3=4 1=8
  run "$pre mt4 c16" $pre 3=4 1=16
  run "$pre mt1" $pre 3=1
done
run "c3-bgmv" c3-bgmv
for pre in c4 c4-128; do
  run "$pre tc3" $pre
  run "$pre tc-fused" $pre 10=1
  run "$pre tc-stream" $pre 10=2
  run "$pre tc-split" $pre 6=1
done
run "c2 headline" c2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sgmv -c 60 --csv \
  --log-file gpurun_out/c34/launches_c4.csv python bench.py --preset c4 --profile --warmup 2 --sites 8 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sgmv -c 40 --csv \
  --log-file gpurun_out/c34/launches_c3.csv python bench.py --preset c3 --profile --warmup 2 --sites 8 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_fast -s 4 -c 1 \
  -o gpurun_out/c34/prof_c3 -f python bench.py --preset c3 --profile --warmup 2 --sites 8 > gpurun_out/c34/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_tc_ -s 4 -c 2 \
  -o gpurun_out/c34/prof_c4 -f python bench.py --preset c4 --profile --warmup 2 --sites 8 > gpurun_out/c34/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
cp build/variants/instr/libsgmv_b200.so paper_2310_18547_b200/lib/libsgmv_b200.so
timeout 120 python scripts/trace_tc.py > gpurun_out/c34/trace_c4.txt 2>&1
timeout 120 python scripts/trace_phases.py --popularity uniform --batch 64 --hidden 5120 --rank 64 > gpurun_out/c34/trace_c3.txt 2>&1
