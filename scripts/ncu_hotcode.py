"""Hot-code footprint of one ncu report per SASS function (profiling helper):
bytes of the instructions that cover 99% of the executed instructions, and
no_instruction stall samples, per noinline function of the kernel's text
section (offsets from the object's symbol table).
usage: python scripts/ncu_hotcode.py report.ncu-rep object.o kernel-mangled-substring"""
import csv
import io
import re
import subprocess
import sys

rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
elf = subprocess.run(["cuobjdump", "-elf", obj], capture_output=True, text=True).stdout
sym = elf[elf.index(".section .symtab"):]
funcs = []
for line in sym.split("\n"):
    f = line.split()
    if len(f) >= 7 and kname in f[-1] and f[-1].startswith("$"):
        m = re.search(r"43d2bc0f\d+([A-Za-z_]+?)(?:ILi|ERK|Ev|Eb|Ei|E)", f[-1].split("$")[2]) if f[-1].count("$") >= 2 else None
        nm = re.sub(r"^.*?(\d+)([a-z_]+)$", r"\2", f[-1].split("$")[2][-60:])
        nm = m.group(1) if m else nm
        funcs.append((int(f[1], 16), int(f[2], 16), nm))
funcs.sort()
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ie, ni, ad = hdr.index("Instructions Executed"), hdr.index("stall_no_inst"), hdr.index("Address")
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        data.append((int(r[ad], 16), int(r[ie] or 0), int(r[ni] or 0)))
    except ValueError:
        pass
data.sort()
base = data[0][0]
tot = sum(d[1] for d in data)
hot = set()
acc = 0
for d in sorted(data, key=lambda d: -d[1]):
    acc += d[1]
    hot.add(d[0])
    if acc >= 0.99 * tot:
        break


def fn(off):
    name = "kernel body"
    for s, sz, n in funcs:
        if s <= off < s + sz:
            name = n
    return name


agg = {}
for a, e, n in data:
    k = fn(a - base)
    x = agg.setdefault(k, [0, 0, 0, 0])
    x[0] += e
    x[1] += n
    x[2] += 16 * (a in hot)
    x[3] += 16
tn = sum(v[1] for v in agg.values()) or 1
print(f"hot code (99% of executed instructions): {len(hot) * 16 / 1024:.1f} KB of {len(data) * 16 / 1024:.0f} KB")
print(f"{'function':24s} {'dyn inst':>8s} {'no_inst':>8s} {'hot KB':>7s} {'size KB':>7s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][2]):
    if v[2] or v[1]:
        print(f"{k:24s} {100 * v[0] / tot:7.1f}% {100 * v[1] / tn:7.1f}% {v[2] / 1024:7.1f} {v[3] / 1024:7.1f}")
