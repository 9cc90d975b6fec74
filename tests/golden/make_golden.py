"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs only in the build container, where /root/reference exists: it loads
oracle/_ref/libref.so (the reference's own keys/rng/models/verify compiled from
the unmodified sources under /root/reference/proj/src, see oracle/Makefile)
and records its outputs. The committed fixtures then travel to the GPU box,
where the reference is absent.

    python tests/golden/make_golden.py

Fixture contents (all outputs come from the reference build, never from the
C restatement under test):
  ref_models.npz  -- RMI cases: sorted sample, B, packed params P, probe keys,
                     predict() and PartitionModel::bucket_index() per probe;
                     SplitterTree cases: sample, budget, eq mode, splitters,
                     equality flags, bucket_count, classify() per probe;
                     codec, rng streams, duplicate_fraction, verify examples.
  generators.json -- fingerprints (multiset_hash, order hash) of the
                     synthetic config generators (these generators have no
                     reference code; the fingerprints pin the restatement's
                     own definition against drift, labelled as such).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def p(a):
    return a.ctypes.data_as(C.c_void_p)


def probes(sample: np.ndarray, rng: np.random.Generator, extra: int = 256) -> np.ndarray:
    lo, hi = int(sample[0]), int(sample[-1])
    parts = [sample[:: max(1, sample.size // 512)], sample[:8], sample[-8:],
             np.array([0, 1, 2**63 - 1, 2**63, 2**63 + 1, 2**64 - 2, 2**64 - 1], np.uint64)]
    if hi > lo:
        parts.append(rng.integers(lo, hi, extra, dtype=np.uint64, endpoint=True))
    parts.append(rng.integers(0, 2**64 - 1, 64, dtype=np.uint64, endpoint=True))
    if lo > 0:
        parts.append(np.array([lo - 1], np.uint64))
    if hi < 2**64 - 1:
        parts.append(np.array([hi + 1], np.uint64))
    return np.ascontiguousarray(np.concatenate([np.asarray(x, np.uint64) for x in parts]))


def rmi_cases(rng):
    cases = []
    # SPEC.md:119-121 examples
    cases.append(("spec_0_999_b4", np.arange(1000, dtype=np.uint64), 4))
    cases.append(("spec_0_1_b1", np.array([0, 1], np.uint64), 1))
    nrm = np.sort(O.encode(O.generate("normal", 10_000, 1)))
    cases.append(("spec_normal1e4_b64", nrm, 64))
    for dist, seed in [("uniform", 42), ("normal", 7), ("lognormal05", 7), ("exponential2", 7),
                       ("mixgauss", 11), ("lognormal2", 19)]:
        x = np.sort(O.encode(O.generate(dist, 8192, seed)))
        cases.append((f"{dist}_8192_b1024", x, 1024))
        cases.append((f"{dist}_8192_b64", x, 64))
    tw = np.sort(O.generate("twodups", 4096, 3))
    cases.append(("twodups_4096_b1024", tw, 1024))
    cases.append(("all_equal_b16", np.full(100, 7, np.uint64), 16))
    cases.append(("two_values_b8", np.array([5] * 50 + [9] * 50, np.uint64), 8))
    cases.append(("u64_wide_b256", np.sort(rng.integers(0, 2**64 - 1, 5000, dtype=np.uint64,
                                                        endpoint=True)), 256))
    return cases


def tree_cases(rng):
    cases = [("spec_0_255_k4", np.arange(256, dtype=np.uint64), 4, 1),
             ("spec_all7_k4", np.full(64, 7, np.uint64), 4, 1)]
    rd = np.sort(O.generate("rootdups", 8192 * 16, 3)[:8192])
    cases.append(("rootdups_k256", rd, 256, 1))
    zp = np.sort(O.generate("zipf", 8192, 3))
    cases.append(("zipf_k256", zp, 256, 1))
    cases.append(("zipf_k256_noeq", zp, 256, 0))
    u = np.sort(O.encode(O.generate("uniform", 8192, 42)))
    cases.append(("uniform_k256", u, 256, 1))
    cases.append(("uniform_k1024", u, 1024, 1))
    small = np.sort(rng.integers(0, 40, 1000, dtype=np.uint64))
    cases.append(("small_dups_k16", small, 16, 1))
    cases.append(("single_k2", np.array([3], np.uint64), 2, 1))
    return cases


def main():
    R = O.ref()
    if R is None:
        raise SystemExit("oracle/_ref/libref.so missing: run `make -C oracle` where /root/reference exists")
    rng = np.random.default_rng(20230717)
    arrays: dict[str, np.ndarray] = {}
    names = []
    for name, s, B in rmi_cases(rng):
        s = np.ascontiguousarray(s, np.uint64)
        P = np.zeros(4 + 4 * B, np.float64)
        assert R.ref_rmi_train(p(s), s.size, B, p(P)) == 0
        pr = probes(s, rng)
        pred = np.zeros(pr.size, np.float64)
        bucket = np.zeros(pr.size, np.uint32)
        R.ref_rmi_eval(p(s), s.size, B, B, 0.0, 1.0, p(pr), pr.size, p(pred), p(bucket))
        b1000 = np.zeros(pr.size, np.uint32)
        R.ref_rmi_eval(p(s), s.size, B, 1000, 0.0, 1.0, p(pr), pr.size, None, p(b1000))
        bsub = np.zeros(pr.size, np.uint32)  # forwarded model rescaled to a CDF sub-range
        R.ref_rmi_eval(p(s), s.size, B, 256, 0.25, 0.75, p(pr), pr.size, None, p(bsub))
        arrays.update({f"rmi/{name}/sample": s, f"rmi/{name}/B": np.array([B]),
                       f"rmi/{name}/P": P, f"rmi/{name}/probe": pr, f"rmi/{name}/pred": pred,
                       f"rmi/{name}/bucket": bucket, f"rmi/{name}/bucket1000": b1000,
                       f"rmi/{name}/bucket_sub": bsub})
        names.append(("rmi", name))
    for name, s, k, eq in tree_cases(rng):
        s = np.ascontiguousarray(s, np.uint64)
        pr = probes(s, rng)
        bucket = np.zeros(pr.size, np.uint32)
        spl = np.zeros(k, np.uint64)
        heavy = np.zeros(k, np.uint8)
        ns = C.c_uint32(0)
        bc = C.c_uint32(0)
        assert R.ref_tree_eval(p(s), s.size, k, eq, p(pr), pr.size, p(bucket), p(spl), p(heavy),
                               C.byref(ns), C.byref(bc)) == 0
        arrays.update({f"tree/{name}/sample": s, f"tree/{name}/k": np.array([k]),
                       f"tree/{name}/eq": np.array([eq]), f"tree/{name}/probe": pr,
                       f"tree/{name}/bucket": bucket,
                       f"tree/{name}/splitters": spl[: ns.value].copy(),
                       f"tree/{name}/heavy": heavy[: ns.value].copy(),
                       f"tree/{name}/bucket_count": np.array([bc.value])})
        names.append(("tree", name))
    # codec (keys.hpp:24-46)
    specials = np.array([0.0, -0.0, 1.0, -1.0, 3.5, -3.5, 5e-324, -5e-324, 2.2250738585072014e-308,
                         1.7976931348623157e308, -1.7976931348623157e308, np.inf, -np.inf, 0.5,
                         -0.5, 1e-300, -1e300], np.float64)
    x = np.ascontiguousarray(np.concatenate([specials, rng.standard_normal(200) * 1e3,
                                             rng.standard_normal(50) * 1e-200]))
    enc = np.array([R.ref_encode_double(float(v)) for v in x], np.uint64)
    dec = np.array([R.ref_decode_double(int(k)) for k in enc], np.float64)
    arrays.update({"codec/x": x, "codec/enc": enc, "codec/dec": dec})
    xn = np.ascontiguousarray(np.array([1.0, 2.0, np.nan, 4.0, np.nan], np.float64))
    outn = np.zeros(5, np.uint64)
    arrays["codec/nan_first"] = np.array([R.ref_encode_doubles(p(xn), p(outn), 5)])
    # rng streams (rng.hpp:13-53)
    for seed in (0, 1, 3, 7, 11, 19, 42, 2**64 - 1):
        for kind, nm in enumerate(["u64", "unit", "unit_open", "below", "normal", "exp"]):
            cnt = 64
            od = np.zeros(cnt, np.float64)
            ou = np.zeros(cnt, np.uint64)
            R.ref_rng_stream(seed, kind, 1000003, 2.0, cnt, p(od), p(ou))
            arrays[f"rng/{seed}/{nm}"] = ou if kind in (0, 3) else od
    # duplicate_fraction (models.cpp:187-193)
    dups = {"a": [1, 2, 3, 4], "b": [5, 5, 5, 5], "c": [], "d": [1, 1, 2, 3, 3, 3, 9]}
    for k, v in dups.items():
        a = np.ascontiguousarray(np.array(v, np.uint64))
        arrays[f"dup/{k}/in"] = a
        arrays[f"dup/{k}/out"] = np.array([R.ref_duplicate_fraction(p(a), a.size)])
    # verify (verify.hpp:17-29)
    vcases = {"a": [1, 2, 2, 3], "b": [2, 1], "c": [], "d": [1, 5, 3, 2], "e": [7]}
    for k, v in vcases.items():
        a = np.ascontiguousarray(np.array(v, np.uint64))
        fv = np.zeros(1, np.uint64)
        ok = R.ref_verify_sorted(p(a), a.size, p(fv))
        arrays[f"verify/{k}/in"] = a
        arrays[f"verify/{k}/out"] = np.array([ok, int(fv[0]), R.ref_multiset_hash(p(a), a.size)],
                                             np.uint64)
    np.savez_compressed(os.path.join(OUT, "ref_models.npz"), **arrays)

    # generator fingerprints (restatement-defined; pins drift only)
    gens = {}
    for dist, seed in [("uniform", 42), ("normal", 7), ("lognormal05", 7), ("exponential2", 7),
                       ("mixgauss", 11), ("lognormal2", 19), ("rootdups", 3), ("twodups", 3),
                       ("zipf", 3)]:
        n = 100_000
        v = O.generate(dist, n, seed)
        k = O.encode(v) if v.dtype == np.float64 else v
        order = int(np.bitwise_xor.reduce(k * np.arange(1, n + 1, dtype=np.uint64)))
        gens[dist] = {"n": n, "seed": seed, "multiset_hash": O.multiset_hash(k),
                      "order_hash": order, "first": [int(t) for t in k[:4]]}
    # SPEC.md:475-476 known sequences
    gens["spec_rootdups16_unshuffled"] = [i % 4 for i in range(16)]
    gens["spec_twodups8_unshuffled"] = [(i * i + 4) % 8 for i in range(8)]
    with open(os.path.join(OUT, "generators.json"), "w") as f:
        json.dump(gens, f, indent=1)
    print(f"wrote {len(names)} model cases, {len(arrays)} arrays")


if __name__ == "__main__":
    main()
