"""Sum ncu instructions/samples per source region (profiling helper).
usage: python scripts/ncu_regions.py report.ncu-rep name:lo-hi ..."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
regions = []
for a in sys.argv[2:]:
    name, rng = a.split(":")
    lo, hi = rng.split("-")
    regions.append((name, int(lo), int(hi)))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, cur_file, data = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1]
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        data.append((cur_file, int(r[0]), r))
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
tot_s = sum(int(r[si] or 0) for f, l, r in data if r[si].isdigit())
tot_i = sum(int(r[ie] or 0) for f, l, r in data if r[ie].isdigit())
print(f"total samples {tot_s} instructions {tot_i/1e9:.2f}G")
for name, lo, hi in regions:
    s = sum(int(r[si]) for f, l, r in data if f.endswith("pms8g_search.cu") and lo <= l <= hi and r[si].isdigit())
    i = sum(int(r[ie]) for f, l, r in data if f.endswith("pms8g_search.cu") and lo <= l <= hi and r[ie].isdigit())
    print(f"{name:12s} samples {100*s/tot_s:5.1f}%  instr {i/1e9:7.2f}G ({100*i/tot_i:5.1f}%)")
other = sum(int(r[si]) for f, l, r in data if not f.endswith("pms8g_search.cu") and r[si].isdigit())
print(f"other files  samples {100*other/tot_s:5.1f}%")
