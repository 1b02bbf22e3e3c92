"""Alphabets of 5..32 symbols on the GPU (the B-plane search,
paper_1307_0571_b200/csrc/pms8g_sigma.cu): motif sets
against the reference's own (tests/golden/protein.json, make_golden.py
protein) and the C oracle (pinned to the same golden in test_oracle.py)."""
import os
import subprocess

import numpy as np
import pytest

import _oracle as O
import paper_1307_0571_b200 as P
from conftest import ROOT, golden

pytestmark = pytest.mark.gpu


def _alphabet(name):
    return P.Alphabet.named(name)


@pytest.mark.parametrize("part", [0, 1])
def test_reference_motif_sets_larger_alphabets(part):
    cases = golden("protein.json")
    for case in cases[part::2]:
        prob = P.Problem(case["sequences"], case["l"], case["d"], _alphabet(case["alphabet"]))
        cfg = P.SolverConfig(threshold_override=case["t"] or None)
        assert P.solve(prob, cfg) == case["motifs"], (case["alphabet"], case["l"], case["d"])
        if case["planted"]:
            assert case["planted"] in case["motifs"]


@pytest.mark.parametrize("l,d,seed", [(11, 3, 1), (13, 4, 2), (15, 5, 3)])
def test_planted_protein_against_oracle(l, d, seed):
    n, m = 12, 120
    codes, motif, _ = O.generate(l, d, seed, n=n, m=m, sigma=20)
    sym = P.Alphabet.protein().symbols
    seqs = ["".join(sym[c] for c in row) for row in codes]
    want, _ = O.solve(codes, l, d, sigma=20, alphabet=sym)
    planted = "".join(sym[c] for c in motif)
    assert planted in want
    prob = P.Problem(seqs, l, d, P.Alphabet.protein())
    for t in (None, 2, 3, 4):
        assert P.solve(prob, P.SolverConfig(threshold_override=t)) == sorted(want), t
    rep = P.RunReport()
    assert P.run_parallel(prob, P.SolverConfig(reverify_against_originals=True), None, rep) == sorted(want)
    assert rep.motif_count == len(want)


def test_protein_subsets_caps_and_multi():
    case = [c for c in golden("protein.json") if c["alphabet"] == "protein" and c["l"] == 10 and c["t"] == 0][0]
    prob = P.Problem(case["sequences"], case["l"], case["d"], P.Alphabet.protein())
    w = len(case["sequences"][0]) - case["l"] + 1
    a = P.run_parallel(prob, P.SolverConfig(), P.ParallelOptions(anchors=list(range(0, w, 2))))
    b = P.run_parallel(prob, P.SolverConfig(), P.ParallelOptions(anchors=list(range(1, w, 2))))
    assert sorted(set(a) | set(b)) == case["motifs"]
    assert P.run_parallel(prob, P.SolverConfig(), P.ParallelOptions(devices=[0, 0])) == case["motifs"]
    big = [c for c in golden("protein.json") if len(c["motifs"]) > 100][0]
    prob = P.Problem(big["sequences"], big["l"], big["d"], _alphabet(big["alphabet"]))
    with pytest.raises(P.SolverRuntimeError, match="motif cap"):
        P.solve(prob, P.SolverConfig(max_motifs=10))


def test_cli_protein(tmp_path):
    exe = os.path.join(ROOT, "paper_1307_0571_b200", "bin", "pms8g")
    f = tmp_path / "p.fa"
    r = subprocess.run([exe, "generate", "-l", "10", "-d", "2", "-n", "10", "-m", "60", "--seed", "4",
                        "--alphabet", "protein", "--mutation", "exact", "-o", str(f)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    planted = r.stdout.strip()
    seqs = [x.strip() for x in f.read_text().split("\n") if x and not x.startswith((">", ";"))]
    codes = O.codes_of(seqs, P.Alphabet.protein().symbols)
    want, _ = O.solve(codes, 10, 2, sigma=20, alphabet=P.Alphabet.protein().symbols)
    r = subprocess.run([exe, "solve", str(f)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert r.stdout.split() == sorted(want) and planted in want
