"""The C++ drop-in boundary: tests/cpp/test_facade.cpp is written against the
reference's API (the reference tests' idioms and known answers), compiled
against include/matchamg/*.hpp and linked only with libmatchamg.so +
libmamg_cuda.so (built by __graft_entry__.build())."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_facade")


def test_facade_binary_is_built():
    assert os.path.exists(BIN), "run __graft_entry__.build()"


def test_facade_fails_loudly_without_gpu():
    import shutil
    if shutil.which("nvidia-smi"):
        r = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True)
        if r.returncode == 0 and "GPU" in r.stdout:
            pytest.skip("a GPU is present")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    assert p.returncode != 0 and "no usable CUDA device" in (p.stdout + p.stderr)


@pytest.mark.gpu
def test_facade_reference_idioms_on_b200():
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failed" in p.stdout
