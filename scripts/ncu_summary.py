"""Summarise an ncu report: duration, DRAM bytes, SM activity and the top stall sites."""
import csv
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return {h: (u, v) for h, u, v in zip(r[0], r[1], r[2])}


def main(rep, top=18):
    m = raw(rep)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_active.avg",
            "sm__cycles_active.max", "gpc__cycles_elapsed.max", "launch__grid_size", "launch__cluster_dim_x",
            "launch__registers_per_thread", "smsp__warps_active.avg.pct_of_peak_sustained_active",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
            "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
            "launch__shared_mem_per_block_dynamic"]
    for k in keys:
        if k in m:
            print(f"{k:60s} {m[k][1]} {m[k][0]}")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0
    data = [r for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]
    tot = sum(num(r[idx["Warp Stall Sampling (All Samples)"]]) for r in data)
    print("stall samples", tot)
    stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    agg = {k: sum(num(r[idx[k]]) for r in data) for k in stall_cols}
    print("by reason:", {k[6:]: v for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v})
    seen = set()
    for r in sorted(data, key=lambda r: -num(r[idx["Warp Stall Sampling (All Samples)"]])):
        if r[idx["Address"]] in seen:
            continue
        seen.add(r[idx["Address"]])
        s = num(r[idx["Warp Stall Sampling (All Samples)"]])
        if not s or len(seen) > top:
            break
        why = {k[6:]: r[idx[k]] for k in stall_cols if num(r[idx[k]])}
        print(f"{r[idx['Address']][-5:]} {s:5d} {r[idx['Source']][:64]:64s} {why}")


if __name__ == "__main__":
    main(sys.argv[1])
