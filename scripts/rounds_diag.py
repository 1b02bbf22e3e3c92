import os, sys
sys.path.insert(0, "/root/repo")
import paper_1307_0571_b200 as P
for l, d in ((13, 4), (17, 6), (21, 8)):
    inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=l, d=d, seed=1, mutation=P.MutationMode.exactly_d))
    ctx = P.Context(20, 600, l, d, P.Alphabet.dna(), P.SolverConfig(), P.ParallelOptions())
    ctx.load_codes(inst.codes.ctypes.data, False)
    ctx.run(); ctx.run()
    c = ctx.counters()
    print((l, d), "search ms", ctx.kernel_ms()[0], "nodes", c[7], "rounds", c[395], "narrow", c[396],
          f"nodes/round {c[7]/max(1,c[395]):.2f} narrow frac {c[396]/max(1,c[395]):.2f}", flush=True)
