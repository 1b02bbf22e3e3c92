"""Run one config on the GPU and print timing + device counters (diagnostics).
usage: python scripts/profile_run.py L D [t] [reps] [anchors-stride]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_0571_b200 as P  # noqa: E402

l, d = int(sys.argv[1]), int(sys.argv[2])
t = int(sys.argv[3]) if len(sys.argv) > 3 else 0
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
stride = int(sys.argv[5]) if len(sys.argv) > 5 else 1
inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=l, d=d, seed=1, mutation=P.MutationMode.exactly_d))
anchors = list(range(0, 600 - l + 1, stride)) if stride > 1 else None
shard = os.environ.get("SHARD")  # "r/N": interleaved shard r of N
sr, sn = (int(x) for x in shard.split("/")) if shard else (0, 1)
ctx = P.Context(20, 600, l, d, P.Alphabet.dna(), P.SolverConfig(threshold_override=t or None),
                P.ParallelOptions(anchors=anchors, shard_rank=sr, shard_count=sn,
                                  warps_per_block=int(os.environ.get("WARPS", "0"))))
ctx.load_codes(inst.codes.ctypes.data, False)
for r in range(reps):
    t0 = time.perf_counter()
    ctx.run()
    dt = time.perf_counter() - t0
rep = P.RunReport()
motifs = ctx.result(rep)
c = ctx.counters()
names = ["pushes", "viable", "slots", "tuples", "leaves", "emitted", "vcmp", "nodes", "clk_filter", "clk_pattern",
         "pair_rej", "tri_rej", "tasks", "donated", "replays"]
print(f"({l},{d}) t={rep.device_threshold} anchors={rep.subproblems} wall={dt*1e3:.2f}ms search={ctx.kernel_ms()[0]:.2f}ms "
      f"motifs={motifs}")
print("  " + " ".join(f"{n}={v}" for n, v in zip(names, c)))
hist = c[15:55]
if len(c) > 55:
    import torch
    props = torch.cuda.get_device_properties(0)
    ms = ctx.kernel_ms()[0]
    warps = 12 if (l <= 32 and rep.device_threshold <= 3) else 16  # search_default_warps
    tot = props.multi_processor_count * warps * ms * 1e-3 * 1.965e9
    for nm, lo in (("donated ranges", 56), ("donated nodes", 96)):
        print(f"  {nm} histogram: " + " ".join(f"{i}:{v}" for i, v in enumerate(c[lo:lo + 40]) if v))
    nlog = min(c[136], 14) if len(c) > 136 else 0
    for i in range(nlog):
        r = c[137 + 8 * i:145 + 8 * i]
        print(f"  long task kind={r[0]} anchor={r[1]} idx={r[2]} cycles={r[3]:.3e} tuples={r[4]} leaves={r[5]} "
              f"nodes={r[6]} prologue_cycles={r[7]}")
    print(f"  idle warp-cycles {c[55]:.3e} busy(filter+pattern) {c[8] + c[9]:.3e}"
          + (f" of {tot:.3e} available: idle {c[55] / tot:.1%}" if tot else ""))
if len(c) > 395:
    print(f"  cons_rej={c[395]}")
if len(c) > 397 + 48 - 1 and any(c[397:445]):
    for k in range(8):
        r = c[397 + 6 * k:403 + 6 * k]
        if r[0]:
            print(f"  level {k}: pushes={r[0]} stopped_early={r[1]} slots/push={r[2] / r[0]:.0f} "
                  f"cheap_survivors/push={r[3] / r[0]:.1f} kept/push={r[4] / r[0]:.1f} "
                  f"blocks_with_survivor/push={r[5] / r[0]:.1f} of {r[2] / r[0] / 32:.1f}")
if len(c) > 396 and c[396]:
    print(f"  enumeration rounds {c[396]} nodes/round {c[7] / c[396]:.2f} (fast loop, up to 16)")
print("  task cycles histogram (log2 bucket: count): " +
      " ".join(f"{i}:{v}" for i, v in enumerate(hist) if v))
