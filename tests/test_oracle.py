"""Pins the C restatement (oracle/pms8_oracle.c) to the reference itself:
every expected value below was produced by the reference's own code
(oracle/_ref, see tests/golden/make_golden.py). CPU only."""
import hashlib

import pytest

import _oracle as O
from conftest import golden

KAT = golden("spec_kat.json")


def test_neighborhood_sizes_match_reference():
    for l, d, sigma, want in KAT["neighborhood_size"]:
        assert O.neighborhood_size(l, d, sigma) == want, (l, d)
    # SPEC.md:488 closed form
    assert O.neighborhood_size(13, 4) == "66379"


def test_threshold_model_matches_reference():
    for n, m, l, d, sigma, t in KAT["threshold"]:
        assert O.estimate_threshold(n, m, l, d, sigma) == t, (n, m, l, d)


def test_theorem1_and_consensus_kats():
    assert O.triple_ok("AA", "CC", "GG", 1, 1, 1) == KAT["triple_AA_CC_GG_111"] is False
    assert O.triple_ok("AAAA", "AAAT", "AATT", 1, 1, 1) == KAT["triple_AAAA_AAAT_AATT_111"] is True
    assert O.consensus_distance(["ACG", "ACT", "GCT"]) == KAT["consensus_ACG_ACT_GCT"] == 2
    assert O.consensus_distance(["AA", "CC", "GG", "TT"]) == KAT["consensus_AA_CC_GG_TT"] == 6
    for a, b, c, d1, d2, d3, ok in KAT["triples"]:
        assert O.triple_ok(a, b, c, d1, d2, d3) == bool(ok), (a, b, c, d1, d2, d3)


def test_common_neighborhood_matches_reference_in_order():
    assert len(O.common_neighborhood(["AC"], 1)) == KAT["cn_AC_d1"] == 7
    assert O.common_neighborhood(["AA", "TT"], 1) == KAT["cn_AA_TT_d1"] == ["AT", "TA"]
    for d, tup, want in KAT["neighborhoods"]:
        got = O.common_neighborhood(tup, d)
        assert got == want, (tup, d)
        # every prune level visits exactly the same leaves (neighborhood.hpp:14-20)
        assert O.common_neighborhood(tup, d, level=0) == want
        assert O.common_neighborhood(tup, d, level=1) == want


def test_generator_is_byte_identical_to_reference():
    for inst in golden("instances.json"):
        codes, motif, pos = O.generate(inst["l"], inst["d"], inst["seed"], inst["n"], inst["m"],
                                       inst["mode"] == "exact")
        seqs = ["".join("ACGT"[c] for c in row) for row in codes]
        assert "".join("ACGT"[c] for c in motif) == inst["motif"]
        assert list(pos) == inst["positions"]
        assert hashlib.sha256("\n".join(seqs).encode()).hexdigest() == inst["sha256"]


def test_small_random_instances_match_reference():
    for case in golden("small_random.json"):
        codes = O.codes_of(case["sequences"])
        if case["t"] > 8:
            continue
        got, _ = O.solve(codes, case["l"], case["d"], t=case["t"])
        assert got == case["motifs"], case
        if 4 ** case["l"] <= 1 << 14:
            assert O.brute_force(codes, case["l"], case["d"]) == case["motifs"]


def test_planted_13_4_seed1_matches_reference_with_counters():
    g = golden("planted_13_4.json")[0]
    codes, motif, _ = O.generate(13, 4, 1)
    got, ctr = O.solve(codes, 13, 4)
    assert got == g["motifs"]
    rep = g["report"]
    # same tree as the reference: pushes, tuples, leaves and emissions agree
    assert ctr[0] == rep["stacks_explored"]
    assert ctr[1] == rep["neighborhoods"]
    assert ctr[2] == rep["neighbors_visited"]
    assert ctr[3] == rep["motifs_emitted"]
    assert "".join("ACGT"[c] for c in motif) in got


@pytest.mark.parametrize("seed", [2, 3, 4, 5])
def test_planted_13_4_anchor_subsets(seed):
    g = [x for x in golden("planted_13_4.json") if x["seed"] == seed][0]
    codes, motif, pos = O.generate(13, 4, seed)
    got, _ = O.solve(codes, 13, 4, anchors=list(range(int(pos[0]) - 3, int(pos[0]) + 3)))
    planted = "".join("ACGT"[c] for c in motif)
    assert planted in got
    assert set(got) <= set(g["motifs"])


def test_threshold_invariance_on_small_instance():
    codes, _, _ = O.generate(9, 2, 7, n=6, m=60)
    base, _ = O.solve(codes, 9, 2, t=2)
    for t in (1, 3, 4, 6):
        assert O.solve(codes, 9, 2, t=t)[0] == base
    assert base == O.brute_force(codes, 9, 2)


def _protein_symbols(name):
    return "ACDEFGHIKLMNPQRSTVWY" if name == "protein" else name.split(":", 1)[1]


def test_oracle_matches_reference_on_larger_alphabets():
    # tests/golden/protein.json: the reference's run_parallel over alphabets of
    # 5..32 symbols (make_golden.py protein); the C restatement must agree
    for case in golden("protein.json"):
        sym = _protein_symbols(case["alphabet"])
        codes = O.codes_of(case["sequences"], sym)
        got, _ = O.solve(codes, case["l"], case["d"], case["t"], sigma=len(sym), alphabet=sym, cap=1 << 14)
        assert sorted(got) == case["motifs"], case["alphabet"]
