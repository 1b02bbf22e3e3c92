"""torchrun worker for tests/test_gpu_parity.py::test_shared_queue_ranks_*:
every rank maps GPU 0 (PMS8G_SINGLE_GPU test hook: ranks never wait on each
other inside a kernel), claims tasks from one shared pms8g_queue, and the
merged motif set and the per-rank static task counts are written by rank 0."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_0571_b200 as P  # noqa: E402
from paper_1307_0571_b200 import parallel as PP  # noqa: E402

C_STATIC = 394  # pms8g_device.cuh Ctr::C_STATIC


def main():
    l, d, seed, runs, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=l, d=d, seed=seed, mutation=P.MutationMode.exactly_d))
    q = PP.shared_queue(0)
    ctx = P.Context(20, 600, l, d, P.Alphabet.dna(), P.SolverConfig(), P.ParallelOptions(device=0, queue=q))
    ctx.load_codes(inst.codes.ctypes.data, False)
    res = []
    for _ in range(runs):
        ctx.run()
        ptr, cnt = ctx.keys()
        local = PP.device_keys_tensor(ptr, cnt).clone()
        merged = PP.merge_keys_device(PP.allgather_keys(local))
        motifs = PP.decode_keys(merged.cpu().numpy().view(np.uint64), l, "ACGT")
        statics = torch.tensor([ctx.counters()[C_STATIC]], dtype=torch.int64)
        dist.all_reduce(statics)
        mine = ctx.counters()[C_STATIC]
        res.append({"motifs": motifs, "statics": int(statics.item()), "mine": mine})
    # the public API path over the same queue (epochs continue)
    api = P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(device=0))
    if rank == 0:
        single = P.Context(20, 600, l, d, P.Alphabet.dna(), P.SolverConfig(), P.ParallelOptions(device=0))
        single.load_codes(inst.codes.ctypes.data, False)
        single.run()
        with open(out, "w") as f:
            json.dump({"runs": res, "api": api, "nstatic": single.counters()[C_STATIC]}, f)
        single.close()
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
