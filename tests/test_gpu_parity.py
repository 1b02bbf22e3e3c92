"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (tests/golden/, produced by oracle/_ref) and the C oracle. Integer work:
every comparison is exact (bit-identical sorted motif lists)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import _oracle as O
import paper_1307_0571_b200 as P
from conftest import ROOT, golden

pytestmark = pytest.mark.gpu


def planted(l, d, seed, n=20, m=600):
    return P.generate_planted_instance(
        P.PlantedInstanceSpec(n=n, m=m, l=l, d=d, seed=seed, mutation=P.MutationMode.exactly_d))


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_planted_13_4_full_instance(seed):
    g = [x for x in golden("planted_13_4.json") if x["seed"] == seed][0]
    inst = planted(13, 4, seed)
    rep = P.RunReport()
    t = g["report"]["threshold"]
    # exact_tree: every row filtered at every push, as the reference does
    got = P.run_parallel(inst.problem, P.SolverConfig(threshold_override=t), P.ParallelOptions(exact_tree=True), rep)
    assert got == g["motifs"]
    assert P.solve(inst.problem, P.SolverConfig(threshold_override=t)) == g["motifs"]
    assert inst.motif in got
    # at the reference's threshold the GPU explores the identical tree
    assert rep.counters.stacks_explored == g["report"]["stacks_explored"]
    assert rep.counters.neighborhoods == g["report"]["neighborhoods"]
    assert rep.counters.neighbors_visited == g["report"]["neighbors_visited"]
    assert rep.counters.motifs_emitted == g["report"]["motifs_emitted"]
    assert rep.subproblems == 588


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_planted_17_6_full_instance(seed):
    g = [x for x in golden("planted_17_6.json") if x["seed"] == seed][0]
    inst = planted(17, 6, seed)
    got = P.solve(inst.problem)
    assert got == g["motifs"]
    assert inst.motif in got
    assert all(O.is_motif(inst.codes, 17, 6, mo) for mo in got)


def _anchor_parity(name, l, d):
    path = os.path.join(ROOT, "tests", "golden", name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    g = golden(name)
    inst = planted(l, d, g["seed"])
    for a in g["anchors"]:
        got = P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(anchors=[a["offset"]]))
        assert got == a["motifs"], a["offset"]


def test_anchor_sample_21_8():
    _anchor_parity("anchors_21_8.json", 21, 8)


def test_anchor_sample_23_9():
    _anchor_parity("anchors_23_9.json", 23, 9)
    # 24 more S1 l-mers (reference at threshold override 4: the set is t-invariant)
    _anchor_parity("anchors_23_9_more.json", 23, 9)


def test_full_instance_21_8_against_every_reference_anchor():
    # tests/golden/anchors_21_8_full.json: the reference's run_anchored motif
    # set of EVERY S1 l-mer of (21,8) seed 1 (make_golden.py heavy21full); the
    # whole-instance GPU answer must be their union (run_parallel,
    # src/parallel.cpp:88-90), and a spread of single S1 l-mers (including
    # the non-empty one) must match one by one
    g = golden("anchors_21_8_full.json")
    assert len(g["anchors"]) == 580
    inst = planted(21, 8, g["seed"])
    union = sorted({m for a in g["anchors"] for m in a["motifs"]})
    assert union and inst.motif in union
    assert P.solve(inst.problem) == union
    nonempty = [a for a in g["anchors"] if a["motifs"]]
    sample = nonempty + g["anchors"][::29]
    for a in sample:
        got = P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(anchors=[a["offset"]]))
        assert got == a["motifs"], a["offset"]
    # several S1 l-mers in one call: the union of theirs
    offs = [a["offset"] for a in sample]
    want = sorted({m for a in sample for m in a["motifs"]})
    assert P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(anchors=offs)) == want


@pytest.mark.parametrize("l,d,n,m,seed", [(34, 10, 6, 60, 1), (38, 11, 6, 60, 2), (45, 13, 5, 60, 6),
                                          (28, 9, 6, 50, 7), (24, 8, 6, 60, 5), (36, 11, 8, 60, 3),
                                          (26, 8, 9, 50, 4)])
def test_deep_switch_depths_against_oracle(l, d, n, m, seed):
    # the t >= 4 builds (consensus row rule, stack bound, 5/6/7-member tuples) on
    # one- and two-word l-mers, every t against the complete C oracle
    inst = planted(l, d, seed, n=n, m=m)
    want, _ = O.solve(inst.codes, l, d)
    assert inst.motif in want
    for t in range(3 if l > 32 else 2, min(n, 7) + 1):  # t=2 on l > 32: minutes of enumeration
        assert P.solve(inst.problem, P.SolverConfig(threshold_override=t)) == want, t


def test_small_random_and_edge_cases():
    for case in golden("small_random.json"):
        prob = P.Problem(case["sequences"], case["l"], case["d"])
        cfg = P.SolverConfig(threshold_override=case["t"] or None)
        assert P.solve(prob, cfg) == case["motifs"], case


def test_threshold_invariance():
    g = golden("planted_13_4.json")[0]
    inst = planted(13, 4, 1)
    for t in (1, 2, 3, 4, 5, 6, 20):
        assert P.solve(inst.problem, P.SolverConfig(threshold_override=t)) == g["motifs"], t


def test_prune_levels_and_row_order_do_not_change_output():
    codes, _, _ = O.generate(8, 2, 11, n=6, m=50)
    seqs = ["".join("ACGT"[c] for c in row) for row in codes]
    want = O.brute_force(codes, 8, 2)
    prob = P.Problem(seqs, 8, 2)
    for lvl in (P.PruneLevel.none, P.PruneLevel.pairs, P.PruneLevel.full):
        for sort_rows in (True, False):
            for t in (1, 2, 3):
                cfg = P.SolverConfig(prune_level=lvl, sort_rows=sort_rows, threshold_override=t)
                assert P.solve(prob, cfg) == want, (lvl, sort_rows, t)


def test_random_instances_vs_oracle():
    rng = np.random.default_rng(5)
    for _ in range(25):
        n = int(rng.integers(2, 9))
        l = int(rng.integers(5, 12))
        m = int(rng.integers(l, 60))
        d = int(rng.integers(0, 4))
        codes = rng.integers(0, 4, (n, m)).astype(np.uint8)
        seqs = ["".join("ACGT"[c] for c in row) for row in codes]
        want, _ = O.solve(codes, l, d)
        assert P.solve(P.Problem(seqs, l, d)) == want, (n, m, l, d)


def test_long_motifs_two_word_path():
    # l > 32 exercises the two-word bit planes (W=2); small n keeps it fast
    for l, d, seed in [(33, 3, 1), (40, 5, 2), (50, 8, 3), (64, 10, 4)]:
        inst = planted(l, d, seed, n=5, m=90)
        want, _ = O.solve(inst.codes, l, d)
        got = P.solve(inst.problem)
        assert got == want, (l, d)
        assert inst.motif in got


def test_reverify_and_caps():
    inst = planted(13, 4, 1)
    g = golden("planted_13_4.json")[0]
    assert P.solve(inst.problem, P.SolverConfig(reverify_against_originals=True)) == g["motifs"]
    with pytest.raises(P.SolverRuntimeError, match="motif cap of 3 exceeded"):
        P.solve(inst.problem, P.SolverConfig(max_motifs=3))
    assert P.solve(inst.problem, P.SolverConfig(max_motifs=100)) == g["motifs"]


def test_invalid_arguments():
    inst = planted(13, 4, 1)
    with pytest.raises(P.InvalidArgument, match=r"threshold must be in \[1, n\]"):
        P.solve(inst.problem, P.SolverConfig(threshold_override=21))
    with pytest.raises(P.InvalidArgument, match=r"threshold must be in \[1, n\]"):
        P.solve(inst.problem, P.SolverConfig(threshold_override=0))
    with pytest.raises(P.InvalidArgument, match="anchor offset"):
        P.run_parallel(inst.problem, None, P.ParallelOptions(anchors=[588]))


def test_shards_union_to_full_answer():
    g = [x for x in golden("planted_13_4.json") if x["seed"] == 3][0]
    inst = planted(13, 4, 3)
    union = set()
    for r in range(3):
        union |= set(P.run_parallel(inst.problem, None, P.ParallelOptions(shard_rank=r, shard_count=3)))
    assert sorted(union) == g["motifs"]


def test_device_merge_keys():
    import torch
    from paper_1307_0571_b200.parallel import merge_keys_device
    rng = np.random.default_rng(2)
    k = rng.integers(0, 1 << 40, (5000, 2)).astype(np.int64)
    k[:, 1] = rng.integers(0, 3, 5000)
    k = np.concatenate([k, k[:1000]])
    got = merge_keys_device(torch.as_tensor(k, device="cuda")).cpu().numpy()
    want = np.unique(k.view(np.uint64)[:, ::-1], axis=0)[:, ::-1].view(np.int64)
    assert (got == want).all()


def test_device_resident_context_matches():
    import torch
    g = golden("planted_13_4.json")[0]
    inst = planted(13, 4, 1)
    ctx = P.Context(20, 600, 13, 4)
    dev = torch.as_tensor(inst.codes, device="cuda").contiguous()
    torch.cuda.synchronize()
    ctx.load_codes(dev.data_ptr(), True)
    for _ in range(2):
        ctx.run()
        assert ctx.result() == g["motifs"]
    ctx.close()


def test_cli_solve_matches_reference_stdout(tmp_path):
    exe = os.path.join(ROOT, "paper_1307_0571_b200", "bin", "pms8g")
    f = tmp_path / "i.fa"
    subprocess.run([exe, "generate", "-l", "13", "-d", "4", "--seed", "1", "--mutation", "exact", "-o", str(f)],
                   check=True, capture_output=True)
    r = subprocess.run([exe, "solve", str(f)], capture_output=True, text=True)
    assert r.returncode == 0
    assert r.stdout.split() == golden("planted_13_4.json")[0]["motifs"]
    assert r.stderr.startswith("motifs=9 threshold=2 ")
    r = subprocess.run([exe, "solve", str(f), "--format", "json"], capture_output=True, text=True)
    assert json.loads(r.stdout)["motifs"] == golden("planted_13_4.json")[0]["motifs"]
    # no motif -> exit 1 (tools/pms8.cpp:183)
    g = tmp_path / "none.txt"
    g.write_text("AAAAAAAA\nCCCCCCCC\n")
    r = subprocess.run([exe, "solve", str(g), "-l", "8", "-d", "0"], capture_output=True, text=True)
    assert r.returncode == 1 and r.stdout == ""


def test_work_queue_wraparound_keeps_every_node(monkeypatch):
    # a 16-slot ring forces producers to wrap many times; the search tree must
    # still be the reference's exactly (no donated node lost or duplicated)
    g = golden("planted_13_4.json")[0]
    inst = planted(13, 4, 1)
    monkeypatch.setenv("PMS8G_QCAP", "16")
    rep = P.RunReport()
    got = P.run_parallel(inst.problem, P.SolverConfig(threshold_override=2),
                         P.ParallelOptions(warps_per_block=15, exact_tree=True), rep)
    assert got == g["motifs"]
    assert rep.counters.neighbors_visited == g["report"]["neighbors_visited"]
    assert rep.counters.motifs_emitted == g["report"]["motifs_emitted"]


def _branch_parity(name):
    path = os.path.join(ROOT, "tests", "golden", name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    for sample in golden(name):
        inst = planted(sample["l"], sample["d"], sample["seed"])
        for b in sample["branches"]:
            got = P.run_parallel(inst.problem, P.SolverConfig(),
                                 P.ParallelOptions(branches=[(sample["anchor"], b["seq"], b["offset"])]))
            assert got == b["motifs"], (sample["anchor"], b)


def test_branch_sample_50_21():
    # two-word (l=50) path at full size, t from the GPU rule: depth-1 branches
    # of S1 l-mer 0 and the planted depth-1 branch as the reference computed
    # them; the planted one is non-empty, so an all-empty output fails
    _branch_parity("branches_50_21.json")
    _branch_parity("branches_50_21_planted.json")
    sets = [b["motifs"] for name in ("branches_50_21.json", "branches_50_21_planted.json")
            for sample in golden(name) for b in sample["branches"]]
    assert any(sets)


def test_branch_planted_50_21():
    # the depth-1 branch (planted occurrence of sequence 0, planted occurrence
    # in its branching row) given as 19 candidate branches, size-independent
    # checks: the planted motif
    # is a common d-neighbour of a tuple of planted occurrences, all of which
    # survive every filter, so it must be emitted under this branch, and every
    # emitted motif must be a motif of the instance (CPU oracle check)
    # reference-pinned by branches_50_21_planted.json (test_branch_sample_50_21)
    inst = planted(50, 21, 1)
    pos = list(inst.positions)
    br = [(pos[0], s, pos[s]) for s in range(1, 20)]  # only the branching-row one is a branch
    got = P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(branches=br))
    assert inst.motif in got
    assert got == sorted(set(got))
    assert all(O.is_motif(inst.codes, 50, 21, mo) for mo in got)


def test_s1_sample_50_21():
    # whole S1 l-mers of (50,21) (the planted occurrence's offset in S1 plus
    # every 50th): the reference needs hours per S1 l-mer, so the checks are
    # size-independent — the planted motif is found, every motif passes the
    # CPU oracle's naive scan and the GPU scanner
    inst = planted(50, 21, 1)
    anchors = sorted({int(inst.positions[0])} | set(range(0, 551, 50)))
    got = P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(anchors=anchors))
    assert inst.motif in got
    assert all(O.is_motif(inst.codes, 50, 21, mo) for mo in got)
    assert all(ok for ok, _ in P.verify_motifs(inst.problem, got))


@pytest.mark.parametrize("l,d,seed", [(50, 21, 1), (50, 21, 2), (50, 21, 3), (23, 9, 1)])
def test_whole_heavy_instances(l, d, seed):
    # BASELINE's full sizes, whole instances (every S1 l-mer; (50,21) is the
    # bench step). The reference cannot finish these, so the checks are the
    # size-independent ones: the planted motif is in the output, the output is
    # sorted and duplicate-free, every motif passes the CPU oracle's naive scan
    # and the GPU scanner, and three interleaved shards union to the same set
    inst = planted(l, d, seed)
    got = P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions())
    assert inst.motif in got
    assert got == sorted(set(got))
    assert all(O.is_motif(inst.codes, l, d, mo) for mo in got)
    assert all(ok for ok, _ in P.verify_motifs(inst.problem, got))
    if l == 50:
        union = set()
        for r in range(3):
            union |= set(P.run_parallel(inst.problem, P.SolverConfig(),
                                        P.ParallelOptions(shard_rank=r, shard_count=3)))
        assert sorted(union) == got


def test_anchor_planted_21_8_and_23_9():
    _anchor_parity("anchors_21_8_planted.json", 21, 8)
    _anchor_parity("anchors_23_9_planted.json", 23, 9)
    g = golden("anchors_21_8_planted.json")
    assert any(a["motifs"] for a in g["anchors"])


@pytest.mark.parametrize("l,d,n,m,seed", [(7, 2, 40, 157, 1), (7, 2, 36, 150, 2), (9, 3, 36, 260, 1),
                                          (13, 4, 40, 120, 3)])
def test_more_than_32_sequences(l, d, n, m, seed):
    # n > 32 (the reference takes any n): the first 32 sequences are searched,
    # the GPU scanner keeps the motifs that occur in all n; the first three
    # instances have far more motifs in their first 32 sequences than overall
    inst = planted(l, d, seed, n=n, m=m)
    want, _ = O.solve(inst.codes, l, d)
    head, _ = O.solve(inst.codes[:32], l, d)
    assert inst.motif in want and (l > 9 or len(head) > len(want))
    rep = P.RunReport()
    assert P.solve(inst.problem, P.SolverConfig(), rep) == want
    assert P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(devices=[0, 0])) == want
    with pytest.raises(RuntimeError, match="motif cap"):
        P.solve(inst.problem, P.SolverConfig(max_motifs=len(want) - 1))
    assert P.solve(inst.problem, P.SolverConfig(max_motifs=len(want))) == want


def test_donated_tasks_replayed_without_level_handoff(monkeypatch):
    # PMS8G_DON_CAP=0: donated tasks carry no level, receivers rebuild it by
    # replaying the prefix pushes (the fallback for levels larger than a ring
    # slot); few S1 l-mers per call, so most of the work is donated
    monkeypatch.setenv("PMS8G_DON_CAP", "0")
    _anchor_parity("anchors_21_8_planted.json", 21, 8)
    inst = planted(36, 11, 3, n=8, m=60)
    want, _ = O.solve(inst.codes, 36, 11)
    for t in (4, 7):
        assert P.solve(inst.problem, P.SolverConfig(threshold_override=t)) == want, t
    _branch_parity("branches_50_21_planted.json")


def test_gpu_threshold_rule():
    assert [P.gpu_threshold(20, 600, l, d) for l, d in [(13, 4), (17, 6), (21, 8), (23, 9), (50, 21)]] == \
        [2, 3, 4, 4, 7]


@pytest.mark.parametrize("split", ["static", "queue"])
def test_sharded_ranks_on_one_gpu_match_golden(split):
    # torchrun with 2 ranks sharing GPU 0 (keys exchanged with gloo): the
    # per-rank shards (or the shared queue), allgather and device merge give
    # the full motif set
    import sys
    env = dict(os.environ, PMS8G_SINGLE_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--config", "13_4", "--steps", "1", "--no-cpu-baseline", "--split", split],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][0]
    out = json.loads(line)
    assert out["n_gpus"] == 2
    assert out["motifs"] == golden("planted_13_4.json")[0]["motifs"]


@pytest.mark.parametrize("world,l,d,seed", [(2, 13, 4, 2), (3, 17, 6, 1)])
def test_shared_queue_ranks_claim_every_task_once(tmp_path, world, l, d, seed):
    # ranks pull (S1 l-mer, branch) tasks from one epoch-tagged counter over
    # several consecutive runs: each run's static claims sum to the task count
    # of a single-device run (no task lost or repeated) and the merged motif
    # set equals the reference's
    import sys
    out = tmp_path / "q.json"
    env = dict(os.environ, PMS8G_SINGLE_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
                        "--master-addr", "127.0.0.1", "--master-port", "29541",
                        os.path.join(ROOT, "tests", "_queue_worker.py"), str(l), str(d), str(seed), "3", str(out)],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(out.read_text())
    want = [x for x in golden(f"planted_{l}_{d}.json") if x["seed"] == seed][0]["motifs"]
    assert res["nstatic"] > 0
    for run in res["runs"]:
        assert run["motifs"] == want
        assert run["statics"] == res["nstatic"]
    assert res["api"] == want


def test_jitter_hook_keeps_the_motif_set():
    # ParallelOptions' schedule-shaking hook (include/pms8/parallel.hpp:24-27):
    # every task sleeps a seeded random time first; the output must not change
    g = golden("planted_13_4.json")[0]
    inst = planted(13, 4, 1)
    for seed in (1, 2):
        got = P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(jitter_max_us=40, jitter_seed=seed))
        assert got == g["motifs"]


def test_worker_failure_names_the_subproblem(monkeypatch):
    # run_parallel aborts naming the failing offset (src/parallel.cpp:66-86);
    # a zero-capacity node overflow stack makes the first deep enumeration fail
    monkeypatch.setenv("PMS8G_NODE_CAP", "0")
    inst = planted(17, 6, 1)
    with pytest.raises(P.SolverRuntimeError, match=r"^subproblem at offset \d+ failed: enumeration stack overflow"):
        P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(anchors=list(range(0, 584, 8))))


def test_global_table_mode_matches(monkeypatch):
    # the l-mer table read from global memory (the mode instances beyond
    # shared memory use) gives the same motif sets; anchor lists bypass the
    # library's context cache, so the mode is chosen afresh
    monkeypatch.setenv("PMS8G_GLOBAL_TABLE", "1")
    g = golden("planted_17_6.json")[0]
    inst = planted(17, 6, 1)
    assert P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(anchors=list(range(584)))) == g["motifs"]
    g = golden("planted_13_4.json")[1]
    inst = planted(13, 4, 2)
    assert P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(anchors=list(range(588)))) == g["motifs"]
    _branch_parity("branches_50_21.json")


def test_large_instances_beyond_shared_memory():
    # n=20, m=2000: 39,020 two-word l-mers (624 KB) cannot be staged in shared
    # memory; the reference's motif sets (tests/golden/large.json)
    path = os.path.join(ROOT, "tests", "golden", "large.json")
    if not os.path.exists(path):
        pytest.skip("large.json not generated")
    for case in golden("large.json"):
        inst = planted(case["l"], case["d"], case["seed"], n=case["n"], m=case["m"])
        assert case["motif"] == inst.motif
        assert P.solve(inst.problem) == case["motifs"], (case["l"], case["d"])
