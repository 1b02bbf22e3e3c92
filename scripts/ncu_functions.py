"""Per-function share of ncu stall samples and executed instructions for one
kernel (profiling helper): SASS addresses from the ncu source page are mapped
to the noinline-function labels nvdisasm prints for the same build.
usage: python scripts/ncu_functions.py report.ncu-rep object.o kernel-mangled-substring"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
si, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = [(int(r[0], 16), int(r[si] or 0), int(r[ie] or 0)) for r in rows[2:] if r and r[0].startswith("0x")]
base = data[0][0]

with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", os.path.join(td, cub)], capture_output=True, text=True).stdout.split("\n")
start = end = None
for i, l in enumerate(sass):
    if l.startswith("\t.section") and ".text." in l:
        if start is not None and end is None:
            end = i
        if kname in l and start is None:
            start = i
sec = sass[start:end]
marks = [(0, "<kernel body>")]
pat = re.compile(r"(filter_push|filter_one_row|lazy_push|publish|maybe_donate_dfs|verify_all|prepare_tuple_swar|"
                 r"prepare_tuple|enum_loop_fast|enumerate_verify|starving|order_positions|ensure_row|dfs|begin_anchor)")
last_addr = 0
for l in sec:
    s = l.strip()
    m = re.match(r"/\*([0-9a-f]{4,})\*/", s)
    if m:
        last_addr = int(m.group(1), 16)
    elif s.endswith(":") and s.startswith("$") and "search_kernel" in s:
        fm = pat.search(s)
        if fm:
            marks.append((last_addr + 16, fm.group(1)))
marks.sort()
agg = defaultdict(lambda: [0, 0])
for a, smp, ins in data:
    off = a - base
    name = "<kernel body>"
    for mo, nm in marks:
        if mo <= off:
            name = nm
        else:
            break
    agg[name][0] += smp
    agg[name][1] += ins
ts = sum(v[0] for v in agg.values())
ti = sum(v[1] for v in agg.values())
print(f"total samples {ts}, warp instructions {ti / 1e9:.2f} G")
for k, (s_, i_) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:22s} samples {100.0 * s_ / ts:5.1f}%  instr {100.0 * i_ / ti:5.1f}%  ({i_ / 1e9:.2f} G)")
