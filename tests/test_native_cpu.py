"""CPU-side checks of the product library (no GPU needed):
the C-ABI library loads and exports every symbol include/lsort_cuda.h
declares, defaults mirror SortConfig, context creation
fails cleanly without a GPU, and the product's host generators are
bit-identical to the oracle's restatement."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2307_08637_b200 as L
from paper_2307_08637_b200 import _native as N
from oracle import oracle as O
from lsort_testutil import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "lsort_cuda.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lsort_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = N.lib()
    syms = header_symbols()
    assert len(syms) >= 19
    for s in syms:
        assert hasattr(lib, s), f"missing export {s}"
    assert set(syms) == set(N.EXPORTS)


def test_header_constants_match_python_binding():
    """Every LSORT_FLAG_* / return code / memory and key kind of the header has the
    same value in the ctypes binding (a flag added on one side only is silent)."""
    text = open(os.path.join(ROOT, "include", "lsort_cuda.h")).read()
    defs = {m.group(1): int(m.group(2).rstrip("u"), 0)
            for m in re.finditer(r"#define\s+LSORT_(FLAG_[A-Z_]+)\s+(\d+u?)", text)}
    assert {"FLAG_PHASE_TIMING", "FLAG_STRICT_POLICY", "FLAG_CLUSTER", "FLAG_TEST_DIRECT_OVERFLOW",
            "FLAG_TEST_NO_PADDED_MEM"} <= set(defs)
    for name, v in defs.items():
        assert getattr(N, name) == v, name
    assert len(set(defs.values())) == len(defs)


def test_cfg_defaults_match_reference_sortconfig():
    c = N.lsort_cfg()
    N.lib().lsort_cfg_default(C.byref(c))
    d = L.SortConfig()
    for f in ("rmi_bucket_count", "tree_bucket_count", "min_rmi_input", "radix_base_case",
              "insertion_base_case", "first_sample_cap", "rmi_sample_cap", "base_case_capacity",
              "bucket_target"):
        assert getattr(c, f) == getattr(d, f), f
    assert c.max_duplicate_fraction == 0.10 and c.sample_fraction == 0.01
    # SPEC.md:369-372 defaults
    assert (c.rmi_bucket_count, c.tree_bucket_count, c.min_rmi_input) == (1024, 256, 100000)
    assert (c.radix_base_case, c.insertion_base_case, c.first_sample_cap) == (4096, 16, 8192)
    assert c.rmi_sample_cap == 1 << 20


def test_header_struct_layouts_match_ctypes(tmp_path):
    """Compile the public header with gcc and compare sizeof/offsetof to ctypes."""
    import subprocess
    structs = {"lsort_cfg": N.lsort_cfg, "lsort_rmi_header": N.lsort_rmi_header,
               "lsort_rmi_entry": N.lsort_rmi_entry, "lsort_tree": N.lsort_tree,
               "lsort_model_info": N.lsort_model_info, "lsort_stats": N.lsort_stats}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "lsort_cuda.h"', "int main(void){"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                 check=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(out[name]) == C.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(out[f"{name}.{f}"]) == getattr(cls, f).offset, f"{name}.{f}"


def test_context_without_gpu_fails_cleanly():
    h = C.c_void_p()
    rc = N.lib().lsort_cuda_ctx_create(C.byref(h), 0, None, 0)
    if rc == N.LSORT_OK:  # a visible GPU (whatever its device node is called)
        N.lib().lsort_cuda_ctx_destroy(h)
        pytest.skip("GPU present")
    assert not h.value


@pytest.mark.parametrize("dist,seed", [("uniform", 42), ("normal", 7), ("lognormal05", 7),
                                       ("exponential2", 7), ("mixgauss", 11), ("lognormal2", 19),
                                       ("rootdups", 3), ("twodups", 3), ("zipf", 3)])
def test_product_generators_match_oracle(dist, seed):
    n = 200_000
    a = L.generate(dist, n, seed)
    b = O.generate(dist, n, seed)
    assert a.dtype == b.dtype
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    if dist in L.FLOAT_DISTS:  # chunked generation == whole
        part = L.generate(dist, n, seed, first=12345, count=1000)
        assert np.array_equal(part.view(np.uint64), b[12345:13345].view(np.uint64))
