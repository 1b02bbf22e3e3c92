"""The reference-side binding on a B200: oracle/_ref/pms8ref_gpu is the
reference's generator (its own objects) calling run_parallel_gpu
(integration/parallel_gpu.cpp) -> libpms8g.so. Its motif sets must be the
reference's own (tests/golden)."""
import os
import subprocess

import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu
EXE = os.path.join(ROOT, "oracle", "_ref", "pms8ref_gpu")


@pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/pms8ref_gpu not built")
@pytest.mark.parametrize("seed", [1, 2])
def test_reference_caller_through_binding(seed):
    g = [x for x in golden("planted_13_4.json") if x["seed"] == seed][0]
    r = subprocess.run([EXE, "13", "4", str(seed)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().split("\n")
    assert lines[:-1] == g["motifs"]
    rep = lines[-1].split()
    assert rep[0] == "REPORT" and int(rep[1]) == g["report"]["threshold"] and int(rep[3]) == len(g["motifs"])
    # two "workers" = two device contexts (GPU 0 listed twice on a one-GPU box is not possible
    # through workers: devices 0..workers-1), so only check the one-GPU route here
