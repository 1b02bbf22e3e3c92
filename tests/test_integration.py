"""The reference-side binding (integration/parallel_gpu.cpp, shown in
INTEGRATION.md) compiles against the reference's own headers, and the
reference-side caller linked with it (oracle/_ref/pms8ref_gpu) fails loudly
without a GPU (no CPU fallback). CPU tests; the GPU run of the same binary is
in test_gpu_integration.py."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

REF_INC = "/root/reference/proj/include"
EXE = os.path.join(ROOT, "oracle", "_ref", "pms8ref_gpu")


@pytest.mark.skipif(not os.path.isdir(REF_INC) or shutil.which("g++") is None,
                    reason="reference headers only in the build container")
def test_binding_compiles_against_reference_headers():
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-I", REF_INC,
                        "-I", os.path.join(ROOT, "oracle", "boost_standin"), "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "integration", "parallel_gpu.cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/pms8ref_gpu not built")
def test_reference_caller_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = subprocess.run([EXE, "13", "4", "1"], capture_output=True, text=True)
    assert r.returncode == 2
    assert "no CUDA device" in r.stderr
