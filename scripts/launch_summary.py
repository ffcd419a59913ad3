"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): launches, mean, share per kernel."""
import collections
import csv
import sys


def main(path, title=""):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    d = collections.defaultdict(list)
    for r in rows[i + 1:]:
        x = dict(zip(h, r))
        if x.get("Metric Name") == "gpu__time_duration.sum":
            scale = 1e-3 if x.get("Metric Unit") == "ns" else 1.0
            d[x["Kernel Name"][:100]].append(float(x["Metric Value"]) * scale)
    if title:
        print(title)
    print("(cold-cache, serialised launches: the SHARE of the step is what must match bench.py, not the absolute)")
    tot = sum(sum(v) for v in d.values())
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):5d} launches  mean {sum(v) / len(v):9.2f} us  share {sum(v) / tot:6.1%}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
