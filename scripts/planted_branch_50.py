"""Time the (50,21) planted depth-1 branch on the GPU (diagnostics).
The anchor is the planted occurrence in sequence 0; the branch candidates
are the planted occurrences of every other sequence (only the one in the
anchor's branching row is a depth-1 branch, the others are skipped)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_0571_b200 as P  # noqa: E402

inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=50, d=21, seed=1, mutation=P.MutationMode.exactly_d))
pos = list(inst.positions)
motif = inst.motif
br = [(pos[0], s, pos[s]) for s in range(1, 20)]
rep = P.RunReport()
t0 = time.time()
got = P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(branches=br), rep)
print(f"planted branch (50,21): {time.time() - t0:.1f} s, {len(got)} motifs, planted motif found: {motif in got}",
      f"t={rep.device_threshold}", flush=True)
print(got[:10])
