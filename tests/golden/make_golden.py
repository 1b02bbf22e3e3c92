#!/usr/bin/env python3
"""Regenerate tests/golden/ from the reference itself (TEST INFRASTRUCTURE).

Runs oracle/_ref/pms8ref — the reference sources from /root/reference/proj/src
compiled unmodified by oracle/Makefile and driven through their public API by
oracle/ref_driver.cpp — and writes small JSON fixtures. Only runnable in the
build container (it needs /root/reference to build oracle/_ref); the fixtures
it writes are committed and travel to the GPU box.

    python tests/golden/make_golden.py quick        # seconds-to-minutes parts
    python tests/golden/make_golden.py protein      # alphabets of 5..32 symbols (seconds)
    python tests/golden/make_golden.py heavy17      # (17,6) seeds 1-5 full runs
    python tests/golden/make_golden.py heavy21      # (21,8) anchor sample
    python tests/golden/make_golden.py heavy21full  # (21,8) every S1 l-mer (~1.5 h on 8 threads)
    python tests/golden/make_golden.py heavy23      # (23,9) anchor sample
    python tests/golden/make_golden.py heavy23more  # (23,9) 24 more S1 l-mers (t=4 override)
    python tests/golden/make_golden.py heavy23quarter  # (23,9) every 4th S1 l-mer (t=4 override)
    python tests/golden/make_golden.py heavy50      # (50,21) depth-1 branch sample
    python tests/golden/make_golden.py heavyplanted # (21,8)/(23,9) planted S1 offsets
"""
import hashlib
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "..", "..", "oracle", "_ref", "pms8ref")
THREADS = os.cpu_count() or 8


def run(*args):
    out = subprocess.run([REF, *map(str, args)], capture_output=True, text=True, check=True)
    return out.stdout


def gen(l, d, seed, n=20, m=600, mode="exact"):
    lines = run("gen", l, d, seed, n, m, mode).strip().split("\n")
    motif = lines[0].split()[1]
    positions = [int(x) for x in lines[1].split()[1:]]
    seqs = lines[2:]
    return motif, positions, seqs


def parse_solve(text):
    motifs, report = [], None
    for line in text.strip().split("\n"):
        if line.startswith("REPORT "):
            report = json.loads(line[7:])
        elif line:
            motifs.append(line)
    return motifs, report


def dump(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w") as f:
        json.dump(obj, f, indent=1, sort_keys=True)
        f.write("\n")
    print("wrote", path)


def instances():
    out = []
    for (l, d) in [(13, 4), (17, 6), (21, 8), (23, 9), (50, 21)]:
        for seed in [1, 2, 3, 4, 5]:
            motif, pos, seqs = gen(l, d, seed)
            h = hashlib.sha256("\n".join(seqs).encode()).hexdigest()
            out.append({"l": l, "d": d, "seed": seed, "n": 20, "m": 600, "mode": "exact", "motif": motif,
                        "positions": pos, "sha256": h})
    # a few non-default generator settings (at-most-d, small n/m)
    for (l, d, seed, n, m, mode) in [(7, 1, 3, 5, 20, "exact"), (7, 1, 3, 5, 20, "atmost"), (5, 0, 1, 3, 10, "exact"),
                                     (15, 5, 9, 20, 600, "atmost")]:
        motif, pos, seqs = gen(l, d, seed, n, m, mode)
        out.append({"l": l, "d": d, "seed": seed, "n": n, "m": m, "mode": mode, "motif": motif, "positions": pos,
                    "sha256": hashlib.sha256("\n".join(seqs).encode()).hexdigest(), "sequences": seqs})
    dump("instances.json", out)


def solve_file(seqs, l, d, t=0, threads=1):
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
        f.write("\n".join(seqs) + "\n")
        path = f.name
    try:
        return parse_solve(run("file", path, l, d, threads, t))
    finally:
        os.unlink(path)


def small_random():
    """Tiny random instances (SPEC.md:335 grid: n<=5, m<=30, l<=7, d<=2) plus
    edge cases; motif sets from the reference's run_parallel."""
    rng = np.random.default_rng(20261020)
    cases = []
    for i in range(120):
        n = int(rng.integers(1, 6))
        l = int(rng.integers(2, 8))
        m = int(rng.integers(l, 31))
        d = int(rng.integers(0, 3))
        d = min(d, l)
        seqs = ["".join("ACGT"[x] for x in rng.integers(0, 4, m)) for _ in range(n)]
        cases.append((seqs, l, d, 0))
    # edge cases: m == l, d == 0, d == l, 2d >= l, n == 1, identical rows, t overrides
    cases.append((["ACGTACGT"], 8, 0, 0))
    cases.append((["ACGTA", "ACGTA", "TTTTT"], 5, 5, 0))
    cases.append((["AAAA", "AAAT"], 4, 0, 0))
    cases.append((["AAAAA", "TTTTT"], 4, 1, 0))
    cases.append((["ACGTTGCA", "ACGTTGCA", "ACGTTGCA"], 4, 2, 0))
    cases.append((["ACGTAC", "CAGTTC", "GGATCC", "TTACGA"], 3, 1, 0))
    cases.append((["ACGTACGTAC", "CAGTTCAGGT", "GGATCCATCG", "TTACGATTGA", "CCGATAGGCA"], 4, 1, 2))
    cases.append((["ACGTACGTAC", "CAGTTCAGGT", "GGATCCATCG", "TTACGATTGA", "CCGATAGGCA"], 4, 1, 5))
    cases.append((["ACGTACGTAC", "CAGTTCAGGT", "GGATCCATCG", "TTACGATTGA", "CCGATAGGCA"], 4, 1, 1))
    cases.append((["ACGTACGTACGTAC", "CAGTTCAGGTAAAC"], 6, 3, 0))
    # planted (7,1) n=5 m=20
    motif, pos, seqs = gen(7, 1, 3, 5, 20, "exact")
    cases.append((seqs, 7, 1, 0))
    out = []
    for seqs, l, d, t in cases:
        motifs, rep = solve_file(seqs, l, d, t)
        out.append({"sequences": seqs, "l": l, "d": d, "t": t, "motifs": motifs, "threshold": rep["threshold"]})
    dump("small_random.json", out)


def protein():
    """Alphabets of 5..32 symbols (the B-plane GPU path): planted protein
    instances from the reference generator and small random instances over
    custom alphabets, motif sets from the reference's run_parallel."""
    def solve_alpha(seqs, l, d, t, alphabet):
        with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
            f.write("\n".join(seqs) + "\n")
            path = f.name
        try:
            return parse_solve(run("file", path, l, d, 1, t, alphabet))
        finally:
            os.unlink(path)

    out = []
    for (l, d, n, m, seed, t) in [(8, 1, 10, 60, 1, 0), (10, 2, 10, 60, 2, 0), (12, 3, 8, 50, 3, 0),
                                  (13, 4, 6, 40, 4, 0), (9, 2, 12, 80, 5, 0), (10, 2, 10, 60, 2, 3),
                                  (12, 3, 8, 50, 3, 4), (11, 3, 6, 30, 6, 0)]:
        lines = run("gen", l, d, seed, n, m, "exact", "protein").strip().split("\n")
        motif, seqs = lines[0].split()[1], lines[2:]
        motifs, rep = solve_alpha(seqs, l, d, t, "protein")
        out.append({"alphabet": "protein", "l": l, "d": d, "t": t, "seed": seed, "planted": motif,
                    "sequences": seqs, "motifs": motifs, "threshold": rep["threshold"]})
    rng = np.random.default_rng(20261021)
    alphas = ["custom:ACGTN", "custom:ABCDEFGH", "protein", "custom:ABCDEFGHIJKLMNOPQRSTUVWXYZ012345",
              "custom:ZYXWVUTSRQ"]
    for i in range(60):
        a = alphas[i % len(alphas)]
        sym = "ACDEFGHIKLMNPQRSTVWY" if a == "protein" else a.split(":", 1)[1]
        n = int(rng.integers(2, 6))
        l = int(rng.integers(3, 8))
        m = int(rng.integers(l, 26))
        d = int(rng.integers(0, 3))
        seqs = ["".join(sym[x] for x in rng.integers(0, len(sym), m)) for _ in range(n)]
        motifs, rep = solve_alpha(seqs, l, d, 0, a)
        out.append({"alphabet": a, "l": l, "d": d, "t": 0, "seed": None, "planted": None, "sequences": seqs,
                    "motifs": motifs, "threshold": rep["threshold"]})
    dump("protein.json", out)


def planted_full(l, d, seeds, name):
    out = []
    for seed in seeds:
        motifs, rep = parse_solve(run("solve", l, d, seed, THREADS))
        out.append({"l": l, "d": d, "seed": seed, "motifs": motifs, "report": rep})
        print(l, d, seed, len(motifs), rep["wall_seconds"])
    dump(name, out)


def anchor_sample(l, d, seed, offsets, name, t=0, threads=THREADS):
    text = run("anchors", l, d, seed, threads, ",".join(map(str, offsets)), t)
    anchors = []
    timing = None
    for line in text.strip().split("\n"):
        f = line.split()
        if f[0] == "ANCHOR":
            anchors.append({"offset": int(f[1]), "seconds": float(f[2]), "stacks_explored": int(f[3]),
                            "neighborhoods": int(f[4]), "neighbors_visited": int(f[5]), "motifs_emitted": int(f[6]),
                            "motifs": f[7:]})
        elif f[0] == "TIMING":
            timing = json.loads(line[7:])
    dump(name, {"l": l, "d": d, "seed": seed, "anchors": anchors, "timing": timing})


def branch_sample(l, d, seed, anchor, idx, name):
    text = run("branch", l, d, seed, anchor, idx if isinstance(idx, str) else ",".join(map(str, idx)), 0, THREADS)
    branches = []
    brow = None
    for line in text.strip().split("\n"):
        f = line.split()
        if f[0] == "BRANCHROW":
            brow = {"row": int(f[1]), "size": int(f[2])}
        elif f[0] == "BRANCH":
            branches.append({"index": int(f[1]), "seq": int(f[2]), "offset": int(f[3]), "seconds": float(f[4]),
                             "motifs": f[5:]})
    return {"l": l, "d": d, "seed": seed, "anchor": anchor, "branch_row": brow, "branches": branches}


def branch2_planted(l, d, seed, anchor, t):
    # ref_driver branch2: the planted depth-1 branch as the union of its
    # depth-2 branches (reference push/pop/enumerate_and_collect)
    text = run("branch2", l, d, seed, t, THREADS)
    head = motifs = None
    for line in text.strip().split("\n"):
        f = line.split()
        if f[0] == "BRANCH1":
            head = dict(kv.split("=") for kv in f[1:])
        elif f[0] == "UNION":
            motifs, seconds = f[2:], float(f[1])
    assert int(head["anchor"]) == anchor
    return {"l": l, "d": d, "seed": seed, "anchor": anchor, "method": f"branch2 t={t} (depth-2 split)",
            "branches": [{"seq": int(head["u1_seq"]), "offset": int(head["u1_off"]), "seconds": seconds,
                          "depth2_branches": int(head["size"]), "motifs": motifs}]}


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "quick"
    if what == "quick":
        dump("spec_kat.json", json.loads(run("kat")))
        instances()
        small_random()
        planted_full(13, 4, [1, 2, 3, 4, 5], "planted_13_4.json")
    elif what == "protein":
        protein()
    elif what == "large":
        # beyond the shared-memory table: n=20, m=2000, l=50 (K = 39,020 two-word
        # l-mers, 624 KB), the reference's run_parallel on the whole instance
        out = []
        for (l, d, seed, n, m) in [(50, 12, 7, 20, 2000), (40, 10, 8, 20, 2000)]:
            motif, pos, seqs = gen(l, d, seed, n, m)
            motifs, rep = solve_file(seqs, l, d, 0, threads=int(os.environ.get("GOLDEN_THREADS", THREADS)))
            out.append({"l": l, "d": d, "seed": seed, "n": n, "m": m, "motif": motif, "motifs": motifs,
                        "threshold": rep["threshold"], "wall_seconds": rep["wall_seconds"],
                        "sha256": hashlib.sha256("\n".join(seqs).encode()).hexdigest()})
            print(l, d, len(motifs), rep["wall_seconds"])
        dump("large.json", out)
    elif what == "heavy17":
        planted_full(17, 6, [1, 2, 3, 4, 5], "planted_17_6.json")
    elif what == "heavy21":
        anchor_sample(21, 8, 1, list(range(0, 580, 37)), "anchors_21_8.json")
    elif what == "heavy21full":
        # every S1 l-mer of the (21,8) seed-1 instance, per anchor, at the
        # reference's threshold override t=4 (the motif set is t-invariant,
        # SPEC.md:369; t=4 halves the reference's time on this config)
        anchor_sample(21, 8, 1, list(range(0, 580)), "anchors_21_8_full.json", t=4,
                      threads=int(os.environ.get("GOLDEN_THREADS", THREADS)))
    elif what == "heavy23":
        anchor_sample(23, 9, 1, list(range(0, 578, 72)), "anchors_23_9.json")
    elif what == "heavy23more":
        # 24 more S1 l-mers of (23,9) spread over the instance, at the reference's
        # threshold override t=4 (t-invariant motif set; faster than its t=3)
        anchor_sample(23, 9, 1, list(range(13, 578, 24)), "anchors_23_9_more.json", t=4)
    elif what == "heavy23quarter":
        # every 4th S1 l-mer of (23,9) (144 of 578), t=4 override: ~40 min on 8 threads
        anchor_sample(23, 9, 1, list(range(2, 578, 4)), "anchors_23_9_quarter.json", t=4)
    elif what == "heavyplanted":
        # the S1 offset holding the planted occurrence in sequence 0, so the
        # heavy-config anchor parity includes a non-empty motif set
        p21 = gen(21, 8, 1)[1][0]
        p23 = gen(23, 9, 1)[1][0]
        anchor_sample(21, 8, 1, [p21, p21 + 1], "anchors_21_8_planted.json")
        anchor_sample(23, 9, 1, [p23], "anchors_23_9_planted.json")
    elif what == "heavy50":
        samples = [branch_sample(50, 21, 1, 0, [0, 1, 3], "x")]
        dump("branches_50_21.json", samples)
    elif what == "heavy50planted":
        # the planted S1 offset and the planted occurrence in its branching row
        # (one core needs hours for it at the reference's t = 5; at t = 6 and
        # split into its depth-2 branches over THREADS cores it takes minutes;
        # the motif set does not depend on t or on the split)
        p50 = gen(50, 21, 1)[1][0]
        dump("branches_50_21_planted.json", [branch2_planted(50, 21, 1, p50, 6)])
    else:
        raise SystemExit("unknown part " + what)


if __name__ == "__main__":
    main()
