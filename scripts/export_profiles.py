"""Export the judged summaries of the ncu reports in gpurun_out/ into profiles/
(details page, per-function shares, hot lines, headline metrics) and refresh
profiles/ncu_traffic.json, which bench.py reads for roofline.traffic.
usage: python scripts/export_profiles.py TAG REPORT.ncu-rep KEY "description" [TAG REPORT KEY "description" ...]
  TAG: file stem under profiles/ (e.g. r02_ncu_search_50_21); KEY: ncu_traffic.json key (e.g. 50_21)"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_1307_0571_b200", "csrc", "pms8g_search.cu")


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


def fnum(x):
    return float(x.replace(",", ""))


args = sys.argv[1:]
tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
for i in range(0, len(args), 4):
    tag, rep, key, desc = args[i:i + 4]
    out = os.path.join(ROOT, "profiles", tag)
    open(out + "_details.csv", "w").write(run(["ncu", "-i", rep, "--page", "details", "--csv"]))
    open(out + "_functions.txt", "w").write(run([sys.executable, os.path.join(ROOT, "scripts", "ncu_byfunc.py"), rep, SRC]))
    open(out + "_lines.txt", "w").write(run([sys.executable, os.path.join(ROOT, "scripts", "ncu_lines.py"), rep, "60"]))
    open(out + "_summary.txt", "w").write(run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep]))
    raw = list(csv.reader(io.StringIO(run(["ncu", "-i", rep, "--page", "raw", "--csv"]))))
    m = dict(zip(raw[0], raw[2]))
    u = dict(zip(raw[0], raw[1]))

    def byts(name):
        v, unit = fnum(m[name]), u[name].lower()
        return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}.get(unit, 1)

    def ms(name):
        v, unit = fnum(m[name]), u[name].lower()
        return v * {"ns": 1e-6, "us": 1e-3, "ms": 1, "s": 1e3, "usecond": 1e-3, "msecond": 1, "second": 1e3, "nsecond": 1e-6}.get(unit, 1)

    rd, wr = byts("dram__bytes_read.sum"), byts("dram__bytes_write.sum")
    traffic[key] = {
        "traffic_bytes": int(rd + wr), "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
        "smsp__issue_active": round(fnum(m["smsp__issue_active.avg.pct_of_peak_sustained_active"]) / 100, 4),
        "pipe_alu": round(fnum(m["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"]) / 100, 4),
        "pipe_xu": round(fnum(m.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "0")) / 100, 4),
        "kernel_ms": round(ms("gpu__time_duration.sum"), 2),
        "kernel": m.get("Kernel Name", ""),
        "source": f"profiles/{tag}_details.csv: {desc}",
    }
    print(tag, json.dumps(traffic[key]))
traffic["_note"] = ("per search_kernel launch, ncu --set full --clock-control none (one launch); traffic = dram__bytes_read.sum + "
                    "dram__bytes_write.sum; refreshed by scripts/export_profiles.py")
json.dump(traffic, open(tpath, "w"), indent=1)
