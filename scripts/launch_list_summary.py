"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum,dram__bytes_read.sum,...):
per kernel, launches, mean duration, share of the listed time, DRAM bytes per launch."""
import csv
import sys
from collections import defaultdict


def main(path, label):
    rows = list(csv.reader(open(path)))
    hdr, per = None, defaultdict(lambda: defaultdict(list))
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            try:
                v = float(d["Metric Value"].replace(",", ""))
            except ValueError:
                continue
            per[d["Kernel Name"][:70]][d["Metric Name"]].append(v)
    print(f"ncu launch list ({label}): serialised, cold caches -- compare shares, not absolute times")
    tot = sum(sum(m["gpu__time_duration.sum"]) for m in per.values())
    for k, m in per.items():
        t = m["gpu__time_duration.sum"]
        rd = m.get("dram__bytes_read.sum", [0])
        print(f"{k:70s} launches {len(t):4d}  mean {sum(t) / len(t) / 1e3:7.2f} us  share {sum(t) / tot * 100:5.1f} %"
              f"  dram read/launch {sum(rd) / max(len(rd), 1) / 1e6:7.2f} MB")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
