"""Small searches that cover the t = 3..7 builds, the push queue, the early exit and the
level hand-off, for compute-sanitizer (memcheck / racecheck). usage: compute-sanitizer
--tool memcheck python scripts/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_0571_b200 as P  # noqa: E402


def planted(l, d, seed, n, m):
    return P.generate_planted_instance(
        P.PlantedInstanceSpec(n=n, m=m, l=l, d=d, seed=seed, mutation=P.MutationMode.exactly_d))


for (l, d, n, m, seed, ts) in [(34, 10, 8, 60, 3, (3, 5, 7)), (24, 8, 8, 50, 4, (4, 6, 7)), (13, 4, 20, 120, 1, (2, 3))]:
    inst = planted(l, d, seed, n, m)
    want = None
    for t in ts:
        got = P.solve(inst.problem, P.SolverConfig(threshold_override=t))
        assert inst.motif in got
        want = want or got
        assert got == want, (l, d, t)
    print(l, d, "ok", len(want))
