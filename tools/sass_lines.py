#!/usr/bin/env python
"""Join an ncu SASS source page (per-instruction stall samples / executed
instructions) with nvdisasm line info to get per-CUDA-line totals.

    python tools/sass_lines.py gpurun_out/prof_C5.ncu-rep <kernel cubin> <mangled name> [top]
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, cubin, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
base = int(data[0][0], 16)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
lines = dis.splitlines()
start = next(i for i, ln in enumerate(lines) if ln.startswith("//---") and (".text." + fn + " ") in ln)
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith("//---")), len(lines))
line_of = {}
cur = None
for ln in lines[start:end]:
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if ln.strip().startswith("//##") and m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r'\s*/\*([0-9a-f]+)\*/', ln)
    if m and cur is not None:
        line_of[int(m.group(1), 16)] = cur
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = [hdr.index(h) for h in reasons]
st, ins = defaultdict(float), defaultdict(float)
why = defaultdict(lambda: defaultdict(float))
for r in data:
    off = int(r[0], 16) - base
    l = line_of.get(off, ("?", -1))
    st[l] += float(r[si] or 0)
    ins[l] += float(r[ie] or 0)
    for h, i in zip(reasons, ri):
        try:
            why[l][h] += float(r[i] or 0)
        except ValueError:
            pass
ts, ti = sum(st.values()), sum(ins.values())
srcs = {}


def text(f, n):
    if f not in srcs:
        try:
            srcs[f] = open(f).read().splitlines()
        except OSError:
            srcs[f] = []
    src = srcs[f]
    return src[n - 1].strip()[:80] if 0 < n <= len(src) else "?"


print(f"{'file:line':>18} {'stall%':>7} {'inst%':>7}  source")
for l in sorted(st, key=lambda k: -st[k])[:top]:
    s = text(*l)
    top2 = sorted(why[l].items(), key=lambda kv: -kv[1])[:2]
    tw = " ".join(f"{k[6:]}:{100 * v / max(st[l], 1):.0f}%" for k, v in top2)
    fl = f"{l[0].split('/')[-1]}:{l[1]}"
    print(f"{fl:>18} {100 * st[l] / ts:7.1f} {100 * ins[l] / ti:7.1f}  {tw:28s} {s}")
