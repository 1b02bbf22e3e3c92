"""(50,21) CPU-vs-GPU on the same depth-1 branches of S1 l-mer 0 (a full S1
l-mer of the reference takes ≳35 h single-thread). The
reference (oracle/_ref/pms8ref `branch`: MotifSearch::push/pop on the
branching row, OpenMP over the branches, all host threads) and the GPU
(ParallelOptions(branches=...)) search the same branches; the motif sets must
match. Prints one JSON line.
usage: python scripts/branch_compare_50_21.py [0,1,2,3]"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1307_0571_b200 as P  # noqa: E402

idx = sys.argv[1] if len(sys.argv) > 1 else "0,1,2,3"
threads = os.cpu_count() or 1
t0 = time.perf_counter()
out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "pms8ref"), "branch", "50", "21", "1", "0", idx, "0",
                      str(threads)], capture_output=True, text=True, check=True).stdout
ref_wall = time.perf_counter() - t0
br, ref_motifs, ref_secs = [], set(), {}
for ln in out.splitlines():
    f = ln.split()
    if f and f[0] == "BRANCH":
        j, seq, off, sec = int(f[1]), int(f[2]), int(f[3]), float(f[4])
        br.append((0, seq, off))
        ref_secs[j] = sec
        ref_motifs.update(f[5:])
inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=50, d=21, seed=1, mutation=P.MutationMode.exactly_d))
opts = P.ParallelOptions(branches=br)
P.run_parallel(inst.problem, P.SolverConfig(), opts)  # warm-up (module load, context)
rep = P.RunReport()
t0 = time.perf_counter()
got = P.run_parallel(inst.problem, P.SolverConfig(), opts, rep)
gpu_wall = time.perf_counter() - t0
print(json.dumps({
    "workload": "(50,21) planted DNA n=20 m=600 exactly-d seed 1: depth-1 branches " + idx +
                " of S1 l-mer 0's branching row",
    "branches": [list(b) for b in br],
    "reference": {"wall_s": ref_wall, "per_branch_thread_s": ref_secs, "threads": threads,
                  "kind": "reference (oracle/_ref, OpenMP over branches)"},
    "gpu": {"wall_s": gpu_wall, "device_s": rep.device_seconds, "threshold": rep.device_threshold,
            "pushes": rep.counters.stacks_explored, "tuples": rep.counters.neighborhoods,
            "candidates": rep.counters.neighbors_visited, "verify_compares": rep.verify_compares},
    "speedup_wall": ref_wall / gpu_wall,
    "motifs_identical": sorted(ref_motifs) == got, "motifs": got}))
