"""N>1 host path on CPU: world_size-2 gloo ranks shard the S1 l-mers exactly as
pms8g_options.shard_* does, each rank's motif keys (here from the C oracle,
standing in for the GPU) are unioned with parallel.allgather_keys, and the
union equals the single-process answer (union of per-subproblem
sets == whole-instance solve)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import _oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _keys(motifs):
    rows = []
    for mo in motifs:
        v = 0
        for ch in mo:
            v = (v << 2) | "ACGT".index(ch)
        rows.append([np.int64(np.uint64(v & ((1 << 64) - 1))), np.int64(v >> 64)])
    return torch.tensor(rows, dtype=torch.int64).reshape(-1, 2)


def _worker(rank, world, port, l, d, seed, anchors, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1307_0571_b200.parallel import allgather_keys, decode_keys, shard_offsets
        codes, _, _ = O.generate(l, d, seed, n=8, m=80)
        mine = [a for a in anchors if a in set(shard_offsets(80 - l + 1, rank, world))]
        motifs, _ = O.solve(codes, l, d, anchors=mine) if mine else ([], None)
        allk = allgather_keys(_keys(motifs))
        keys = np.unique(allk.numpy().view(np.uint64).reshape(-1, 2)[:, ::-1], axis=0)[:, ::-1]
        merged = decode_keys(np.ascontiguousarray(keys), l, "ACGT")
        if rank == 0:
            with open(out_path, "w") as f:
                f.write("\n".join(merged))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_union_equals_single_process(tmp_path, world):
    l, d, seed = 9, 2, 3
    anchors = list(range(0, 72))
    out = tmp_path / "merged.txt"
    mp.spawn(_worker, args=(world, _free_port(), l, d, seed, anchors, str(out)), nprocs=world, join=True)
    codes, _, _ = O.generate(l, d, seed, n=8, m=80)
    want, _ = O.solve(codes, l, d)
    got = [x for x in out.read_text().split("\n") if x]
    assert got == want
    assert len(want) > 0


def _gather_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1307_0571_b200.parallel import allgather_keys
        local = torch.arange(rank * 4, dtype=torch.int64).reshape(-1, 2)  # rank 0 sends nothing
        allk = allgather_keys(local)
        if rank == 0:
            np.save(out_path, allk.numpy())
    finally:
        dist.destroy_process_group()


def test_allgather_keys_variable_lengths(tmp_path):
    out = str(tmp_path / "g.npy")
    mp.spawn(_gather_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    assert got.shape == (2, 2)
    assert (got == np.arange(4).reshape(2, 2)).all()


def _queue_fallback_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1307_0571_b200.parallel import shared_queue
        q = shared_queue(0)  # no device here: every rank must agree on None (static split)
        with open(f"{out_path}.{rank}", "w") as f:
            f.write("none" if q is None else "queue")
    finally:
        dist.destroy_process_group()


def test_shared_queue_falls_back_together(tmp_path):
    # the collective that maps rank 0's claim counter into every GPU: when a
    # rank cannot map it, all ranks get None and use the static split
    out = str(tmp_path / "q")
    mp.spawn(_queue_fallback_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert [open(f"{out}.{r}").read() for r in range(2)] == ["none", "none"]
