"""Build liblsort_cuda.so in-tree (nvcc for sm_100a, g++/OpenMP for the host generators).

    python -m paper_2307_08637_b200.build      # or __graft_entry__.build()

Incremental: objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(CSRC, "build")
LIB = os.path.join(PKG, "liblsort_cuda.so")
CLI = os.path.join(PKG, "lsort_cli")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fopenmp",
           "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")] + \
    os.environ.get("LSORT_NVCC_EXTRA", "").split()  # e.g. -DLSORT_DEBUG_DIRECT (device-side bounds checks)
CU_SOURCES = ["partition.cu", "models.cu", "basecase.cu", "cluster.cu", "util.cu", "engine.cu", "dist.cu", "classic.cu"]
CPP_SOURCES = ["gen.cpp", "keyio.cpp"]


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(ROOT, "include", "lsort_cuda.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def build(verbose: bool = False, ptxas_info: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = _headers()
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if _stale(o, [s] + hdrs):
            extra = ["-Xptxas", "-v"] if ptxas_info else []
            jobs.append([NVCC] + ARCH + NVFLAGS + extra + ["-c", s, "-o", o])
    for src in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if _stale(o, [s] + hdrs):
            jobs.append(["g++", "-O2", "-std=c++17", "-fPIC", "-fopenmp", "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o])
    logs = []
    if jobs:
        with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            for out in ex.map(_run, jobs):
                logs.append(out)
    if jobs or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        _run([NVCC] + ARCH + ["-shared", "-o", tmp] + objs +
             ["-Xcompiler", "-fopenmp", "-lcudart", "-lgomp", "-ldl"])
        os.replace(tmp, LIB)
    # the command-line harness (SPEC.md bench-cli), linked against the library
    cli_src = os.path.join(CSRC, "cli.cpp")
    if _stale(CLI, [cli_src, LIB] + hdrs):
        tmp = CLI + ".tmp"
        _run(["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
              cli_src, "-o", tmp, "-L", os.path.dirname(LIB), "-llsort_cuda", "-L", "/usr/local/cuda/lib64",
              "-lcudart", "-Wl,-rpath,$ORIGIN"])
        os.replace(tmp, CLI)
    text = "\n".join(logs)
    if verbose and text:
        print(text)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, ptxas_info="-v" in sys.argv))
