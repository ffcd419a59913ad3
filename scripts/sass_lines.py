"""Map SASS offsets of a kernel (from an ncu report's absolute addresses) to source lines.
usage: sass_lines.py <obj.o> <mangled-kernel> <func_start_hex> <addr_hex>..."""
import re
import subprocess
import sys
import tempfile
import os

obj, name, start = sys.argv[1], sys.argv[2], int(sys.argv[3], 16)
addrs = [int(a, 16) - start for a in sys.argv[4:]]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cubin)], capture_output=True, text=True).stdout
body = txt[txt.index(name + ":"):]
body = body[: body.index("\n.L_x_", 100) if False else len(body)]
cur = None
for l in body.splitlines():
    m = re.search(r'//## File ".*?([^/"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,5})\*/", l)
    if m and int(m.group(1), 16) in addrs:
        print(hex(int(m.group(1), 16)), cur, l.strip()[:60])
        addrs.remove(int(m.group(1), 16))
    if not addrs:
        break
