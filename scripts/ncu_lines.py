"""Aggregate ncu stall samples of one kernel by source line (via nvdisasm -g).
usage: ncu_lines.py <report> <obj.o> <mangled-kernel>"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, obj, name = sys.argv[1:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]
start = int(data[0][idx["Address"]], 16)
samp = defaultdict(int)
reasons = defaultdict(lambda: defaultdict(int))
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
seen = set()
for r in data:
    a = int(r[idx["Address"]], 16) - start
    if a in seen:
        continue
    seen.add(a)
    try:
        s = int(r[idx["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    samp[a] += s
    for k in stall_cols:
        try:
            reasons[a][k[6:]] += int(r[idx[k]])
        except ValueError:
            pass
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cubin)], capture_output=True, text=True).stdout
body = txt[txt.index(name + ":"):]
line_of = {}
cur = None
for l in body.splitlines():
    m = re.search(r'//## File ".*?([^/"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,5})\*/", l)
    if m:
        a = int(m.group(1), 16)
        if a in line_of:
            break
        line_of[a] = cur
by_line = defaultdict(int)
why = defaultdict(lambda: defaultdict(int))
for a, s in samp.items():
    ln = line_of.get(a, "?")
    by_line[ln] += s
    for k, v in reasons[a].items():
        why[ln][k] += v
tot = sum(by_line.values())
print("total samples", tot)
for ln, s in sorted(by_line.items(), key=lambda kv: -kv[1])[:25]:
    w = {k: v for k, v in sorted(why[ln].items(), key=lambda kv: -kv[1]) if v}
    print(f"{s:5d} {100*s/tot:5.1f}%  {ln:28s} {dict(list(w.items())[:4])}")
