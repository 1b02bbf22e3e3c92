"""(50,21) depth-1 branch timings on the GPU: anchor 0's branches 0..N-1 of its
branching row (diagnostics: per-branch device time and counters)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_0571_b200 as P  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 4
inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=50, d=21, seed=1, mutation=P.MutationMode.exactly_d))
# anchor 0 branching row: row 7 (golden branches_50_21.json), offsets = branch index for this anchor
br = [(0, 7, j) for j in range(nb)]
rep = P.RunReport()
t0 = time.time()
got = P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(branches=br), rep)
dt = time.time() - t0
print(f"(50,21) anchor 0 branches 0..{nb-1}: {dt:.2f} s wall, device {rep.device_seconds:.2f} s, motifs {len(got)}, "
      f"t={rep.device_threshold} pushes={rep.counters.stacks_explored} tuples={rep.counters.neighborhoods} "
      f"cands={rep.counters.neighbors_visited} slots={rep.filter_slots} vcmp={rep.verify_compares} "
      f"nodes={rep.enum_nodes}", flush=True)
