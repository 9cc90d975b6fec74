"""The C++ drop-in (include/lsort/lsort.hpp) compiles against the C-ABI
(CPU) and sorts / raises like the reference interface on the GPU."""
import os
import subprocess

import pytest

from lsort_testutil import ROOT

PKG = os.path.join(ROOT, "paper_2307_08637_b200")


def _build(tmp):
    exe = os.path.join(tmp, "dropin")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin.cpp"), "-L", PKG, "-llsort_cuda",
                    f"-Wl,-rpath,{PKG}", "-o", exe], check=True)
    return exe


def test_dropin_header_compiles(tmp_path):
    assert os.path.exists(_build(str(tmp_path)))


@pytest.mark.gpu
def test_dropin_runs_on_gpu(tmp_path):
    exe = _build(str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin ok" in r.stdout
