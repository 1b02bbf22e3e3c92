"""Throughput of several instances per (l,d) (the paper averages 5 seeds,
PAPER.md:368): sequential solve() calls (device context cached between
calls) vs one solve_batch() call (instances concurrent, SMs split between
them). Prints one JSON line per config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_0571_b200 as P  # noqa: E402

for l, d in ((13, 4), (17, 6)):
    seeds = [1, 2, 3, 4, 5]
    probs = [P.generate_planted_instance(P.PlantedInstanceSpec(l=l, d=d, seed=s, mutation=P.MutationMode.exactly_d)
                                         ).problem for s in seeds]
    for _ in range(2):  # warm-up (module load, context cache)
        seq = [P.solve(p) for p in probs]
        bat = P.solve_batch(probs)
    ts, tb = [], []
    for _ in range(5):
        t0 = time.perf_counter()
        seq = [P.solve(p) for p in probs]
        ts.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        bat = P.solve_batch(probs)
        tb.append(time.perf_counter() - t0)
    ts, tb = sorted(ts)[2], sorted(tb)[2]
    s1 = len(seeds) * (600 - l + 1)
    print(json.dumps({"config": f"({l},{d}) seeds 1-5", "sequential_s": ts, "batch_s": tb,
                      "sequential_s1_lmers_per_s": s1 / ts, "batch_s1_lmers_per_s": s1 / tb,
                      "identical": seq == bat}), flush=True)
