"""Print the SASS of one noinline function of a kernel (profiling helper).
usage: python scripts/sass_fn.py object.o kernel-mangled function-substring [every]"""
import re
import subprocess
import sys

obj, kern, fname = sys.argv[1], sys.argv[2], sys.argv[3]
every = int(sys.argv[4]) if len(sys.argv) > 4 else 1
elf = subprocess.run(["cuobjdump", "-elf", obj], capture_output=True, text=True).stdout
sym = elf[elf.index(".section .symtab"):]
lo = hi = None
for line in sym.split("\n"):
    f = line.split()
    if len(f) >= 7 and f[-1].startswith("$") and kern in f[-1] and fname in f[-1].split("$")[2]:
        lo, hi = int(f[1], 16), int(f[1], 16) + int(f[2], 16)
        break
sass = subprocess.run(["cuobjdump", "-sass", "-fun", kern, obj], capture_output=True, text=True).stdout
n = 0
for l in sass.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m and lo <= int(m.group(1), 16) < hi:
        if n % every == 0:
            print(m.group(1), m.group(2).strip()[:100])
        n += 1
print("instructions:", n)
