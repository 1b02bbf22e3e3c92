"""Quick GPU check: (13,4) seeds 1-5 vs golden; prints timings and counters."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_0571_b200 as P

gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "planted_13_4.json")))
for g in gold:
    inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=13, d=4, seed=g["seed"], mutation=P.MutationMode.exactly_d))
    rep = P.RunReport()
    t0 = time.time()
    got = P.solve(inst.problem, P.SolverConfig(), rep)
    t1 = time.time()
    got2 = P.solve(inst.problem, P.SolverConfig(), rep)
    t2 = time.time()
    print(g["seed"], got == g["motifs"], len(got), f"first {t1-t0:.3f}s second {t2-t1:.4f}s dev {rep.device_seconds*1e3:.2f}ms", rep.counters, rep.filter_slots, rep.verify_compares, rep.enum_nodes, flush=True)
    if got != g["motifs"]:
        print("GOT", got); print("EXP", g["motifs"])
for t in [1, 2, 3, 4]:
    inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=13, d=4, seed=1, mutation=P.MutationMode.exactly_d))
    rep = P.RunReport()
    got = P.solve(inst.problem, P.SolverConfig(threshold_override=t), rep)
    got = P.solve(inst.problem, P.SolverConfig(threshold_override=t), rep)
    print("t", t, got == gold[0]["motifs"], f"dev {rep.device_seconds*1e3:.2f}ms", rep.counters, flush=True)
for (l, d) in [(17, 6), (21, 8)]:
    for t in [3, 4]:
        inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=l, d=d, seed=1, mutation=P.MutationMode.exactly_d))
        rep = P.RunReport()
        t0 = time.time()
        got = P.solve(inst.problem, P.SolverConfig(threshold_override=t), rep)
        print(l, d, "t", t, got, f"wall {time.time()-t0:.3f}s dev {rep.device_seconds*1e3:.2f}ms", rep.counters, rep.filter_slots, rep.verify_compares, rep.enum_nodes, flush=True)
