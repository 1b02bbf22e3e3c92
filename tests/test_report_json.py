"""`pms8 solve --format json` parity (CPU): pms8g_report_json's bytes against
nlohmann::json's dump(2) of the same values — the library and call the
reference CLI uses (tools/pms8.cpp:31-60,171-176). The helper
tests/helpers/json_ref.cpp is compiled here against the nlohmann header
shipped in this image; the test is skipped if that header is absent."""
import ctypes
import os
import shutil
import subprocess

import pytest

import paper_1307_0571_b200 as P
from paper_1307_0571_b200 import _capi

HERE = os.path.dirname(os.path.abspath(__file__))
NLOHMANN = None
for cand in ["/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty",
             "/usr/include", "/usr/local/include"]:
    if os.path.exists(os.path.join(cand, "nlohmann", "json.hpp")):
        NLOHMANN = cand
        break


@pytest.fixture(scope="module")
def json_ref(tmp_path_factory):
    if NLOHMANN is None or shutil.which("g++") is None:
        pytest.skip("nlohmann/json.hpp or g++ not available")
    exe = str(tmp_path_factory.mktemp("jr") / "json_ref")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", NLOHMANN, "-o", exe,
                    os.path.join(HERE, "helpers", "json_ref.cpp")], check=True)
    return exe


CASES = [
    # (alphabet, command, report fields, motifs)
    ("dna", "pms8g solve inst.fa --format json",
     dict(n=20, m=600, l=13, d=4, threshold=2, gpus=1, subproblems=588, motif_count=3, wall_seconds=0.0123456,
          sample_seconds=0.004, pattern_seconds=0.0083456, pair_matrix_words=3457440, row_matrix_words=0,
          row_bookkeeping_words=912345, packed_words=17640, lookup_table_words=0, stacks_explored=60564,
          neighborhoods=59976, neighbors_visited=19110000, motifs_emitted=15),
     ["AGGGACACAAATC", "AGGGACACAAATG", "TGGGACACAAATC"]),
    ("custom:TGCA", 'weird "quoted" \\ cmd\ttab',
     dict(n=3, m=10, l=4, d=1, threshold=1, gpus=1, subproblems=7, motif_count=0, wall_seconds=1.5e-05,
          sample_seconds=123456789.25, pattern_seconds=0.0, pair_matrix_words=1, row_matrix_words=2,
          row_bookkeeping_words=3, packed_words=4, lookup_table_words=0, stacks_explored=0, neighborhoods=0,
          neighbors_visited=0, motifs_emitted=0),
     []),
    ("dna", "x",
     dict(n=20, m=600, l=50, d=21, threshold=5, gpus=8, subproblems=551, motif_count=1, wall_seconds=171.23,
          sample_seconds=2e20, pattern_seconds=0.1 + 0.2, pair_matrix_words=10 ** 12, row_matrix_words=7,
          row_bookkeeping_words=0, packed_words=0, lookup_table_words=0, stacks_explored=2 ** 40,
          neighborhoods=1, neighbors_visited=2, motifs_emitted=3),
     ["A" * 50]),
]


def ours(alphabet, command, f, motifs):
    res = _capi.Result()
    flat = "".join(motifs).encode()
    buf = ctypes.create_string_buffer(flat + b"\0")
    res.count = len(motifs)
    res.l = f["l"]
    res.motifs = ctypes.cast(buf, ctypes.c_char_p)
    for k, v in f.items():
        setattr(res.report, k, v)
    L = _capi.lib()
    n = L.pms8g_report_json(ctypes.byref(res), alphabet.encode(), command.encode(), None, 0)
    out = ctypes.create_string_buffer(n + 1)
    assert L.pms8g_report_json(ctypes.byref(res), alphabet.encode(), command.encode(), out, n + 1) == n
    return out.value.decode()


@pytest.mark.parametrize("case", range(len(CASES)))
def test_report_json_bytes_match_nlohmann(json_ref, case):
    alphabet, command, f, motifs = CASES[case]
    order = ["n", "m", "l", "d", "threshold", "gpus", "subproblems", "motif_count", "wall_seconds", "sample_seconds",
             "pattern_seconds", "pair_matrix_words", "row_matrix_words", "row_bookkeeping_words", "packed_words",
             "lookup_table_words", "stacks_explored", "neighborhoods", "neighbors_visited", "motifs_emitted"]
    stdin = alphabet + "\n" + command + "\n" + " ".join(repr(float(f[k])) if k.endswith("seconds") else str(f[k])
                                                        for k in order)
    stdin += f" {len(motifs)} " + " ".join(motifs) + "\n"
    want = subprocess.run([json_ref], input=stdin, capture_output=True, text=True, check=True).stdout
    assert ours(alphabet, command, f, motifs) + "\n" == want
