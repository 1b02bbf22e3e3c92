"""Several GPUs behind one blocking C call (pms8g_solve_multi / pms8g_multi_*,
the reference's run_parallel with GPUs as the worker team,
src/parallel.cpp:35-118). On a one-GPU box the device list repeats GPU 0:
the contexts then share its HBM counter and the motif sets travel by peer
copy; devices=[0] exercises the NCCL allgather path with one rank. The motif
set must equal the reference's (tests/golden) in every mode."""
import ctypes
import json
import os
import subprocess

import numpy as np
import pytest

import paper_1307_0571_b200 as P
from paper_1307_0571_b200 import _capi
from conftest import ROOT, golden

pytestmark = pytest.mark.gpu


def planted(l, d, seed):
    return P.generate_planted_instance(P.PlantedInstanceSpec(l=l, d=d, seed=seed, mutation=P.MutationMode.exactly_d))


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_solve_multi_13_4_matches_reference(devices):
    for g in golden("planted_13_4.json")[:3]:
        inst = planted(13, 4, g["seed"])
        rep = P.RunReport()
        got = P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(devices=devices), rep)
        assert got == g["motifs"], (devices, g["seed"])
        assert rep.gpus == len(devices)


@pytest.mark.parametrize("seed", [1, 2])
def test_solve_multi_17_6_shared_counter(seed):
    g = [x for x in golden("planted_17_6.json") if x["seed"] == seed][0]
    inst = planted(17, 6, seed)
    for _ in range(2):  # the cached handle's epochs stay in step across calls
        assert P.run_parallel(inst.problem, P.SolverConfig(), P.ParallelOptions(devices=[0, 0])) == g["motifs"]


def _multi(devices, inst, l, d, env=None):
    L = _capi.lib()
    o = _capi.Options()
    L.pms8g_default_options(ctypes.byref(o))
    h = ctypes.c_void_p()
    err = ctypes.create_string_buffer(512)
    devs = np.asarray(devices, np.int32)
    rc = L.pms8g_multi_create(20, 600, l, d, b"ACGT", ctypes.byref(o), devs.ctypes.data, len(devs), ctypes.byref(h),
                              err, 512)
    assert rc == 0, err.value
    try:
        exch = L.pms8g_multi_exchange(h).decode()
        codes = np.ascontiguousarray(inst.codes)
        res = _capi.Result()
        rc = L.pms8g_multi_run(h, codes.ctypes.data, ctypes.byref(res), err, 512)
        assert rc == 0, err.value
        raw = ctypes.string_at(res.motifs, res.count * res.l).decode() if res.count else ""
        got = [raw[i * l:(i + 1) * l] for i in range(res.count)]
        L.pms8g_result_free(ctypes.byref(res))
        return got, exch
    finally:
        L.pms8g_multi_destroy(h)


def test_multi_static_split_and_exchange_modes(monkeypatch):
    g = golden("planted_13_4.json")[1]
    inst = planted(13, 4, g["seed"])
    got, exch = _multi([0, 0], inst, 13, 4)
    assert got == g["motifs"] and exch == "peer-copy"
    monkeypatch.setenv("PMS8G_MULTI_STATIC", "1")  # offset % N == rank instead of the shared counter
    got, _ = _multi([0, 0, 0], inst, 13, 4)
    assert got == g["motifs"]
    monkeypatch.delenv("PMS8G_MULTI_STATIC")
    got, exch = _multi([0], inst, 13, 4)
    assert got == g["motifs"]
    assert exch in ("nccl-allgather", "peer-copy")


def test_cli_devices_flag(tmp_path):
    exe = os.path.join(ROOT, "paper_1307_0571_b200", "bin", "pms8g")
    f = tmp_path / "i.fa"
    subprocess.run([exe, "generate", "-l", "13", "-d", "4", "--seed", "1", "--mutation", "exact", "-o", str(f)],
                   check=True, capture_output=True)
    r = subprocess.run([exe, "solve", str(f), "--devices", "0,0", "--format", "json"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    doc = json.loads(r.stdout)
    assert doc["motifs"] == golden("planted_13_4.json")[0]["motifs"]
    assert doc["report"]["workers"] == 2
    # the reference's report schema (tools/pms8.cpp:31-60), keys sorted as nlohmann prints them
    rep = doc["report"]
    assert list(rep) == sorted(["n", "m", "l", "d", "alphabet", "threshold", "workers", "subproblems", "motif_count",
                                "wall_seconds", "sample_seconds", "pattern_seconds", "memory", "counters", "command"])
    assert list(rep["memory"]) == sorted(["pair_matrix_words", "row_matrix_words", "row_bookkeeping_words",
                                          "packed_words", "lookup_table_words", "tracked_total_words",
                                          "tracked_total_bytes"])
    assert rep["memory"]["tracked_total_bytes"] == 8 * rep["memory"]["tracked_total_words"]
    assert rep["threshold"] == 2  # the reference's estimate_threshold for (13,4), not the device's depth
    r = subprocess.run([exe, "solve", str(f)], capture_output=True, text=True)
    assert r.stderr.startswith("motifs=9 threshold=2 workers=1 ")
