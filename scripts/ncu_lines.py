"""Aggregate ncu source-page samples per CUDA source line (profiling helper).
usage: python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
lines = []
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "File Path", "Function Name"):
        lines.append(r)
if not hdr:
    sys.exit("no source table")
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
tot = sum(int(r[si] or 0) for r in lines if r[si].isdigit())
lines.sort(key=lambda r: -int(r[si]) if r[si].isdigit() else 0)
print(f"total samples {tot}")
for r in lines[:top]:
    s = int(r[si]) if r[si].isdigit() else 0
    print(f"{s:8d} {100*s/max(1,tot):5.1f}%  inst={r[ie]:>12}  L{r[0]:>4}: {r[1][:110]}")
