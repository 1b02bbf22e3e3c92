"""Per-function share of ncu stall samples / executed instructions by CUDA
source line ranges (profiling helper). Inlined helpers (common.cuh) count
where they are written, so their samples are listed separately.
usage: python scripts/ncu_byfunc.py report.ncu-rep source.cu"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, src = sys.argv[1], sys.argv[2]
lines = open(src).read().split("\n")
starts = []
for i, l in enumerate(lines, 1):
    m = re.match(r"^(?:__device__|__global__)[^(]*?\b(\w+)\s*\(", l)
    if m:
        starts.append((i, m.group(1)))
starts.sort()


def func_of(ln):
    name = "(file scope)"
    for s, n in starts:
        if s <= ln:
            name = n
    return name


txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, cur_file = None, ""
agg = defaultdict(lambda: [0, 0])
for r in rows:
    if r and r[0] == "File Path" and len(r) > 1:
        cur_file = r[1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        si, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        continue
    if not hdr or not r or not r[0].strip().isdigit():
        continue
    ln = int(r[0])
    s = int(r[si]) if r[si].isdigit() else 0
    e = int(r[ie]) if r[ie].isdigit() else 0
    key = func_of(ln) if (cur_file == "" or cur_file.endswith("pms8g_search.cu")) else cur_file.split("/")[-1] + ":" + str(ln)
    agg[key][0] += s
    agg[key][1] += e
tot_s = sum(v[0] for v in agg.values()) or 1
tot_e = sum(v[1] for v in agg.values()) or 1
for k, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"{100 * s / tot_s:6.1f}% samples {100 * e / tot_e:6.1f}% inst  {k}")
