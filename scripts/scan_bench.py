"""Time the GPU brute-force scanner on (13,4) seed 1 (Sigma^13 = 67M words)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_0571_b200 as P  # noqa: E402

for l, d in ((11, 3), (13, 4), (14, 4)):
    inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=l, d=d, seed=1, mutation=P.MutationMode.exactly_d))
    for rep in range(2):
        r = P.RunReport()
        t0 = time.perf_counter()
        got = P.brute_force_solve(inst.problem, enumeration_guard=1 << 40, report=r)
        dt = time.perf_counter() - t0
    print(f"({l},{d}) brute force: {len(got)} motifs, wall {dt*1e3:.1f} ms, device {r.device_seconds*1e3:.1f} ms, "
          f"{4**l / r.device_seconds / 1e9:.2f} G words/s", flush=True)
