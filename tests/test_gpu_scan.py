"""GPU brute-force scanner (pms8g_verify_motifs / pms8g_brute_force — the
reference's `pms8 verify` and brute_force_solve, src/oracle.cpp:16-75) against
the C oracle and the reference's golden motif sets. Exact integer parity; the
exhaustive Sigma^l sweep is also an independent check of the PMS8 search path."""
import os
import subprocess

import numpy as np
import pytest

import _oracle as O
import paper_1307_0571_b200 as P
from conftest import ROOT, golden

pytestmark = pytest.mark.gpu
CLI = os.path.join(ROOT, "paper_1307_0571_b200", "bin", "pms8g")


def planted(l, d, seed, n=20, m=600, exact=True):
    return P.generate_planted_instance(P.PlantedInstanceSpec(
        n=n, m=m, l=l, d=d, seed=seed, mutation=P.MutationMode.exactly_d if exact else P.MutationMode.at_most_d))


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_brute_force_13_4_equals_reference_motif_set(seed):
    g = [x for x in golden("planted_13_4.json") if x["seed"] == seed][0]
    inst = planted(13, 4, seed)
    rep = P.RunReport()
    got = P.brute_force_solve(inst.problem, enumeration_guard=1 << 30, report=rep)
    assert got == g["motifs"]
    assert got == P.solve(inst.problem)
    assert rep.counters.neighbors_visited == 4 ** 13


def _random_problem(rng, sigma=4):
    n = int(rng.integers(2, 9))
    l = int(rng.integers(3, 9))
    m = int(rng.integers(l, 40))
    d = int(rng.integers(0, min(l, 4) + 1))
    codes = rng.integers(0, sigma, size=(n, m), dtype=np.uint8)
    return codes, l, d


@pytest.mark.parametrize("sigma", [4, 3, 2])
def test_brute_force_random_small_matches_oracle(sigma):
    rng = np.random.default_rng(100 + sigma)
    alpha = "ACGT"[:sigma]
    for _ in range(40):
        codes, l, d = _random_problem(rng, sigma)
        prob = P.Problem(["".join(alpha[c] for c in row) for row in codes], l, d, P.Alphabet.custom(alpha))
        want = O.brute_force(codes, l, d, sigma=sigma, cap=sigma ** l)
        want = ["".join(alpha["ACGT".index(ch)] for ch in w) for w in want]
        got = P.brute_force_solve(prob, enumeration_guard=sigma ** l)
        assert got == sorted(want), (codes.tolist(), l, d)


def test_brute_force_edges():
    # l == m, d == 0: the motif set is the common sequence, if any
    assert P.brute_force_solve(P.Problem(["ACGTAC", "ACGTAA"], 6, 0)) == []
    seqs = ["ACGTAC", "ACGTAC"]
    assert P.brute_force_solve(P.Problem(seqs, 6, 0)) == ["ACGTAC"]
    # d == l: every word of Sigma^l is a motif
    got = P.brute_force_solve(P.Problem(["ACGTACGT", "TTTTTTTT"], 5, 5))
    assert len(got) == 4 ** 5 and got == sorted(got)
    with pytest.raises(P.InvalidArgument, match="enumeration space 4\\^11 exceeds guard 1000000"):
        P.brute_force_solve(P.Problem(["ACGTACGTACGT"] * 2, 11, 2))


def test_verify_motifs_witnesses_match_naive_scan():
    inst = planted(17, 6, 1)
    codes = inst.codes
    rng = np.random.default_rng(7)
    cands = [inst.motif, "AGGGACACAAATCTACC", "ATGGACGGTTTTTAAGC"]
    # windows of the input (pass with d >= 0 in their own sequence) and mutants
    for _ in range(60):
        r, j = int(rng.integers(0, 20)), int(rng.integers(0, 584))
        w = list(inst.problem.sequences[r][j:j + 17])
        for p in rng.choice(17, size=int(rng.integers(0, 8)), replace=False):
            w[p] = "ACGT"[int(rng.integers(0, 4))]
        cands.append("".join(w))
    res = P.verify_motifs(inst.problem, cands)
    for mt, (ok, offs) in zip(cands, res):
        assert ok == O.is_motif(codes, 17, 6, mt)
        mc = O.codes_of([mt]).ravel()
        want = []
        for r in range(20):
            hd = np.array([(codes[r, j:j + 17] != mc).sum() for j in range(584)])
            hit = np.nonzero(hd <= 6)[0]
            if len(hit) == 0:
                break
            want.append(int(hit[0]))
        assert offs == want
        wo = []
        assert P.naive_is_motif(inst.problem, mt, wo) == ok and wo == want


def test_verify_two_word_motifs():
    inst = planted(50, 21, 1, n=8, m=200)
    res = P.verify_motifs(inst.problem, [inst.motif, "A" * 50])
    assert res[0][0] is True and len(res[0][1]) == 8
    assert res[1][0] == O.is_motif(inst.codes, 50, 21, "A" * 50)


def test_cli_verify(tmp_path):
    fa = tmp_path / "inst.fa"
    r = subprocess.run([CLI, "generate", "-l", "13", "-d", "4", "--seed", "1", "--mutation", "exact", "-o", str(fa)],
                       capture_output=True, text=True)
    assert r.returncode == 0
    planted_motif = r.stdout.strip()
    mf = tmp_path / "motifs.txt"
    mf.write_text(planted_motif + "\n" + "acgtacgtacgta\n")
    r = subprocess.run([CLI, "verify", str(fa), "-M", str(mf)], capture_output=True, text=True)
    lines = r.stdout.strip().split("\n")
    assert lines[0].startswith(planted_motif + "\tPASS\t")
    assert len(lines[0].split("\t")[2].split(",")) == 20
    passes = O.is_motif(_codes_from_fasta(fa), 13, 4, "ACGTACGTACGTA")
    assert lines[1].startswith("ACGTACGTACGTA\t" + ("PASS\t" if passes else "FAIL"))
    assert r.returncode == (0 if passes else 1)
    # a malformed motif: the earlier lines are still reported, then exit 2
    mf.write_text(planted_motif + "\nACGT\n")
    r = subprocess.run([CLI, "verify", str(fa), "-M", str(mf)], capture_output=True, text=True)
    assert r.returncode == 2 and r.stdout.startswith(planted_motif + "\tPASS")
    assert "has length 4, expected l=13" in r.stderr


def _codes_from_fasta(path):
    seqs, cur = [], []
    for line in open(path):
        line = line.strip()
        if not line or line.startswith(";"):
            continue
        if line.startswith(">"):
            if cur:
                seqs.append("".join(cur))
            cur = []
        else:
            cur.append(line)
    if cur:
        seqs.append("".join(cur))
    return O.codes_of(seqs)


# ---------------------------------------------------------------- batching
def test_solve_batch_matches_reference_per_instance():
    # the paper's protocol: several instances per (l,d), here
    # searched concurrently on one GPU, each with its share of the SMs
    for l, d, seeds in ((13, 4, [1, 2, 3, 4, 5]), (17, 6, [1, 2, 3])):
        gold = {g["seed"]: g["motifs"] for g in golden(f"planted_{l}_{d}.json")}
        probs = [planted(l, d, s).problem for s in seeds]
        reps = []
        got = P.solve_batch(probs, reports=reps)
        assert got == [gold[s] for s in seeds]
        assert len(reps) == len(seeds) and all(r.subproblems == 600 - l + 1 for r in reps)
    # more instances than concurrent lanes (waves) and a subset option
    probs = [planted(13, 4, s).problem for s in [1, 2, 3, 4, 5] * 2]
    got = P.solve_batch(probs, options=P.ParallelOptions(grid_blocks=37))
    gold = {g["seed"]: g["motifs"] for g in golden("planted_13_4.json")}
    assert got == [gold[s] for s in [1, 2, 3, 4, 5] * 2]
