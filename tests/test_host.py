"""Host-side mirror of the reference interface (no GPU)."""
import pytest

import paper_1307_0571_b200 as P
from paper_1307_0571_b200.parallel import shard_offsets


def test_problem_validate_messages():
    with pytest.raises(P.InvalidArgument, match="no input sequences"):
        P.Problem([], 3, 1).validate()
    with pytest.raises(P.InvalidArgument, match="motif length must be >= 1"):
        P.Problem(["ACGT"], 0, 0).validate()
    with pytest.raises(P.InvalidArgument, match="exceeds sequence length"):
        P.Problem(["ACGT"], 5, 0).validate()
    with pytest.raises(P.InvalidArgument, match=r"mismatch budget must be in \[0, l\]"):
        P.Problem(["ACGT"], 3, 4).validate()
    with pytest.raises(P.InvalidArgument, match="has length 3, expected 4"):
        P.Problem(["ACGT", "ACG"], 2, 0).validate()
    # error naming 'U' at index 3
    with pytest.raises(P.InvalidArgument, match="sequence 0, position 3: symbol 'U'"):
        P.Problem(["ACGU"], 2, 0).validate()
    P.Problem(["ACGT", "TTTT"], 2, 1).validate()


def test_alphabet():
    a = P.Alphabet.dna()
    assert a.size() == 4 and a.name() == "dna"
    assert P.Alphabet.named("custom:acg").symbols == "ACG"
    with pytest.raises(P.InvalidArgument):
        P.Alphabet.named("klingon")
    with pytest.raises(P.InvalidArgument):
        P.Alphabet.custom("A")
    assert (a.encode(["ACGT", "TGCA"]) == [[0, 1, 2, 3], [3, 2, 1, 0]]).all()


def test_split_subproblems():
    # SPEC.md:417-418
    assert P.split_subproblems(P.Problem(["ACGTACGT"], 8, 0)) == [0]
    seqs = ["A" * 600] * 2
    assert len(P.split_subproblems(P.Problem(seqs, 13, 4))) == 588


def test_resolve_worker_count(monkeypatch):
    assert P.resolve_worker_count(3) == 3
    with pytest.raises(P.InvalidArgument):
        P.resolve_worker_count(0)
    monkeypatch.setenv("WORKER_COUNT", "5")
    assert P.resolve_worker_count() == 5


def test_shard_offsets_partition():
    for world in (1, 2, 3, 8):
        parts = [shard_offsets(588, r, world) for r in range(world)]
        flat = sorted(x for p in parts for x in p)
        assert flat == list(range(588))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        shard_offsets(10, 2, 2)


def test_canonical_motif_set():
    assert P.canonical_motif_set(["CA", "AC", "CA", "AA"]) == ["AA", "AC", "CA"]


def test_solve_batch_rejects_mixed_shapes():
    import paper_1307_0571_b200 as P
    a = P.Problem(["ACGTACGTAC", "ACGTACGTAA"], 5, 1)
    b = P.Problem(["ACGTACGTAC", "ACGTACGTAA"], 6, 1)
    import pytest
    with pytest.raises(P.InvalidArgument, match="same n, m, l, d"):
        P.solve_batch([a, b])
    assert P.solve_batch([]) == []
