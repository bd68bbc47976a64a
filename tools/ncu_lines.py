"""Per-source-line warp-stall samples of one kernel in an ncu report (needs -lineinfo + --import-source):
python tools/ncu_lines.py REPORT CUBIN_OBJ KERNEL_SUBSTRING SOURCE_FILE [top]"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kname, srcfile = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(dis) if kname in l and l.startswith(".text.")][0]
line, a2l = None, {}
for l in dis[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'line (\d+)', l)
    if m and os.path.basename(srcfile) in l:
        line = int(m.group(1))
    m2 = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m2 and line:
        a2l[int(m2.group(1), 16)] = line
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr, rows = r[1], r[2:]
samp = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
base = int(rows[0][0], 16)
agg, ins = collections.Counter(), collections.Counter()
for x in rows:
    a = int(x[0], 16) - base
    agg[a2l.get(a, -1)] += int(x[samp] or 0)
    ins[a2l.get(a, -1)] += int(x[ie] or 0)
S, I = sum(agg.values()), sum(ins.values())
src = open(srcfile).read().split("\n")
for ln, v in agg.most_common(top):
    print(f"{ln:5d} {100 * v / S:5.1f}% smp {100 * ins[ln] / I:5.1f}% ins  {src[ln - 1].strip()[:90] if ln > 0 else '?'}")
