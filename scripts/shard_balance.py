"""Load balance of the interleaved S1 l-mer sharding, measured on one GPU.

Each shard r of N (S1 offsets j with j % N == r) is exactly the work rank r
does in an N-GPU run; running the N shards back to back on one B200 and
taking mean/max of their device times gives the parallel efficiency the
interleaved split allows (collective and launch costs excluded; they are
measured separately by bench.py). usage:
    python scripts/shard_balance.py L D [N ...] > profiles/rXX_shard_balance_L_D.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_0571_b200 as P  # noqa: E402

l, d = int(sys.argv[1]), int(sys.argv[2])
ns = [int(x) for x in sys.argv[3:]] or [2, 4, 8]
inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=l, d=d, seed=1, mutation=P.MutationMode.exactly_d))
out = {"workload": f"({l},{d}) planted DNA n=20 m=600 exactly-d seed 1", "shards": {}}
full = None
for N in [1] + ns:
    times = []
    for r in range(N):
        ctx = P.Context(20, 600, l, d, P.Alphabet.dna(), P.SolverConfig(),
                        P.ParallelOptions(shard_rank=r, shard_count=N))
        ctx.load_codes(inst.codes.ctypes.data, False)
        ctx.run()  # warm
        ctx.run()
        times.append(ctx.kernel_ms()[0])
        ctx.close()
    if N == 1:
        full = times[0]
    mean, mx = sum(times) / N, max(times)
    out["shards"][str(N)] = {"search_ms": [round(x, 2) for x in times], "mean_ms": round(mean, 2),
                             "max_ms": round(mx, 2), "efficiency_mean_over_max": round(mean / mx, 4),
                             "efficiency_vs_1gpu": round(full / (N * mx), 4)}
    print(f"N={N} max {mx:.1f} ms mean {mean:.1f} ms eff(mean/max) {mean / mx:.3f} "
          f"eff(T1/(N*max)) {full / (N * mx):.3f}", file=sys.stderr, flush=True)
print(json.dumps(out))
