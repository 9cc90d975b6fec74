"""The C++ drop-in (include/lsort/lsort.hpp) compiles against the C-ABI
(CPU) and sorts / raises like the reference interface on the GPU; the
multi-GPU entry points are driven from C++ as well."""
import os
import subprocess

import pytest

from lsort_testutil import ROOT

PKG = os.path.join(ROOT, "paper_2307_08637_b200")


def _build(tmp, name="dropin"):
    exe = os.path.join(tmp, name)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-L", PKG, "-llsort_cuda",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{PKG}", "-o", exe], check=True)
    return exe


def test_dropin_header_compiles(tmp_path):
    assert os.path.exists(_build(str(tmp_path)))
    assert os.path.exists(_build(str(tmp_path), "dist_world1"))


@pytest.mark.gpu
def test_dropin_runs_on_gpu(tmp_path):
    exe = _build(str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin ok" in r.stdout


@pytest.mark.gpu
def test_dist_entry_points_from_cpp(tmp_path):
    """C++ host, no torch: lsort::dist_sorter (NCCL communicator owned by the
    library, world 1), lsort_cuda_sort_multi, and 4 emulated ranks."""
    exe = _build(str(tmp_path), "dist_world1")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dist ok" in r.stdout
