"""The C ABI library: loads on a CPU-only host, exports every symbol that
include/pms8g.h declares, and its host-side pieces (generator, threshold
model, key decode, CLI generate) match the reference. No GPU compute here."""
import hashlib
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1307_0571_b200 as P
from paper_1307_0571_b200 import _capi
from conftest import ROOT, golden


def header_functions():
    text = open(os.path.join(ROOT, "include", "pms8g.h")).read()
    return sorted(set(re.findall(r"\b(pms8g_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _capi.lib()
    declared = header_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_capi.EXPORTS) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(r"\bT " + name + r"\b", out), name


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(7|8|9)\d", out)


def test_generator_matches_reference_instances():
    for inst in golden("instances.json"):
        spec = P.PlantedInstanceSpec(n=inst["n"], m=inst["m"], l=inst["l"], d=inst["d"], seed=inst["seed"],
                                     mutation=P.MutationMode.exactly_d if inst["mode"] == "exact"
                                     else P.MutationMode.at_most_d)
        got = P.generate_planted_instance(spec)
        assert got.motif == inst["motif"]
        assert got.positions == inst["positions"]
        assert hashlib.sha256("\n".join(got.problem.sequences).encode()).hexdigest() == inst["sha256"]


def test_threshold_model_matches_reference():
    for n, m, l, d, sigma, t in golden("spec_kat.json")["threshold"]:
        assert P.estimate_threshold(n, m, l, d, sigma) == t


def test_decode_keys_roundtrip():
    from paper_1307_0571_b200.parallel import decode_keys
    rng = np.random.default_rng(1)
    for l in (1, 13, 31, 32, 33, 50, 64):
        motifs = ["".join("ACGT"[c] for c in rng.integers(0, 4, l)) for _ in range(20)]
        keys = np.zeros((20, 2), np.uint64)
        for i, mo in enumerate(motifs):
            v = 0
            for ch in mo:
                v = (v << 2) | "ACGT".index(ch)
            keys[i, 0] = v & ((1 << 64) - 1)
            keys[i, 1] = v >> 64
        assert decode_keys(keys, l, "ACGT") == motifs
        # integer order of keys == lexicographic order of motifs
        order = sorted(range(20), key=lambda i: (int(keys[i, 1]), int(keys[i, 0])))
        assert [motifs[i] for i in order] == sorted(motifs)


def test_cli_generate_matches_reference_fasta(tmp_path):
    exe = os.path.join(ROOT, "paper_1307_0571_b200", "bin", "pms8g")
    out = tmp_path / "i.fa"
    r = subprocess.run([exe, "generate", "-l", "13", "-d", "4", "--seed", "1", "--mutation", "exact", "-o", str(out)],
                       capture_output=True, text=True)
    assert r.returncode == 0
    assert r.stdout.strip() == "AGGGACACAAATC"
    text = out.read_text().splitlines()
    assert text[0] == "; format=pms8-planted-instance-v1"
    assert "; motif=AGGGACACAAATC" in text
    seqs, cur = [], ""
    for line in text:
        if line.startswith(">"):
            if cur:
                seqs.append(cur)
            cur = ""
        elif not line.startswith(";"):
            assert len(line) <= 70
            cur += line
    seqs.append(cur)
    inst = [x for x in golden("instances.json") if (x["l"], x["d"], x["seed"]) == (13, 4, 1)][0]
    assert hashlib.sha256("\n".join(seqs).encode()).hexdigest() == inst["sha256"]


def test_cli_usage_errors_exit_2(tmp_path):
    exe = os.path.join(ROOT, "paper_1307_0571_b200", "bin", "pms8g")
    assert subprocess.run([exe], capture_output=True).returncode == 2
    assert subprocess.run([exe, "solve"], capture_output=True).returncode == 2
    f = tmp_path / "x.txt"
    f.write_text("ACGT\nACGT\n")
    r = subprocess.run([exe, "solve", str(f)], capture_output=True, text=True)
    assert r.returncode == 2 and "-l and -d are required" in r.stderr
    r = subprocess.run([exe, "solve", str(f), "-l", "9", "-d", "1"], capture_output=True, text=True)
    assert r.returncode == 2 and "exceeds sequence length" in r.stderr


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=13, d=4, seed=1, mutation=P.MutationMode.exactly_d))
    with pytest.raises(P.DeviceError, match="no CPU fallback"):
        P.solve(inst.problem)


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_scanner_has_no_cpu_fallback():
    inst = P.generate_planted_instance(P.PlantedInstanceSpec(l=8, d=1, n=4, m=30, seed=1))
    with pytest.raises(P.DeviceError, match="no CPU fallback"):
        P.brute_force_solve(inst.problem)
    with pytest.raises(P.DeviceError, match="no CPU fallback"):
        P.verify_motifs(inst.problem, [inst.motif])
    # argument errors are reported before any device work (Problem::validate, check_guard)
    with pytest.raises(P.InvalidArgument, match="exceeds guard"):
        P.brute_force_solve(inst.problem, enumeration_guard=1000)
    with pytest.raises(P.InvalidArgument, match="expected l=8"):
        P.verify_motifs(inst.problem, ["ACGT"])


def test_gpu_switch_depth_rule():
    # host-side model (no device): the GPU-tuned switch depth of the five
    # BASELINE configs; the reference's own rule gives 2,3,3,3,5
    cfgs = [(13, 4), (17, 6), (21, 8), (23, 9), (50, 21)]
    assert [P.gpu_threshold(20, 600, l, d) for l, d in cfgs] == [2, 3, 4, 4, 7]
    assert [P.estimate_threshold(20, 600, l, d) for l, d in cfgs] == [2, 3, 3, 3, 5]
