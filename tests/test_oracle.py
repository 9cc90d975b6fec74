"""CPU tests: pin the C oracle restatement to the reference.

(1) against the committed golden vectors produced by the reference build
    (tests/golden/make_golden.py -> oracle/_ref/libref.so), and
(2) live against oracle/_ref when it is present (build container),
(3) the SPEC known-answer examples,
(4) the oracle sort driver against numpy.sort on every config generator and
    the SPEC adversarial inputs.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from lsort_testutil import ROOT, golden_cases


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def G(golden):
    return golden


def route_defined(P, B, keys):
    """True where the reference's route() cast `size_t(t)` (models.hpp:63) is
    defined, i.e. not (t >= 2^64). Same IEEE ops as models.hpp:21,57,61."""
    with np.errstate(all="ignore"):
        xn = (np.asarray(keys, np.uint64).astype(np.float64) - P[2]) * P[3]
        t = (P[0] * xn + P[1]) * float(B)
        return ~(t >= 2.0 ** 64)


# ---------------------------------------------------------------- golden
def test_codec_golden(G):
    x, enc, dec = G["codec/x"], G["codec/enc"], G["codec/dec"]
    assert np.array_equal(O.encode(x), enc)
    assert np.array_equal(bits(O.decode(enc)), bits(dec))
    assert np.array_equal(bits(dec), bits(x))  # bitwise round trip incl. -0.0
    with pytest.raises(ValueError, match="index 2"):
        O.encode([1.0, 2.0, np.nan, 4.0, np.nan])
    assert int(G["codec/nan_first"][0]) == 2


def test_rng_golden(G):
    L = O.lib()
    for key in G.files:
        if not key.startswith("rng/"):
            continue
        _, seed, kind = key.split("/")
        seed = int(seed)
        ref = G[key]
        n = ref.size
        if kind == "u64":
            got = np.array([L.lso_rng_u64(seed, i) for i in range(n)], np.uint64)
        elif kind == "unit":
            got = np.array([L.lso_rng_unit(seed, i) for i in range(n)])
        elif kind == "unit_open":
            got = np.array([L.lso_rng_unit_open(seed, i) for i in range(n)])
        elif kind == "below":
            got = np.array([L.lso_rng_below(seed, i, 1000003) for i in range(n)], np.uint64)
        elif kind == "normal":  # two draws per value (rng.hpp:41-45)
            got = np.array([L.lso_rng_normal(seed, 2 * i) for i in range(n)])
        else:
            got = np.array([L.lso_rng_exponential(seed, i, 2.0) for i in range(n)])
        assert np.array_equal(np.asarray(got).view(np.uint64), np.asarray(ref).view(np.uint64)), key


@pytest.mark.parametrize("case", ["spec_0_999_b4", "spec_0_1_b1", "spec_normal1e4_b64",
                                  "uniform_8192_b1024", "normal_8192_b1024", "mixgauss_8192_b1024",
                                  "lognormal2_8192_b64", "twodups_4096_b1024", "all_equal_b16",
                                  "two_values_b8", "u64_wide_b256", "exponential2_8192_b1024",
                                  "lognormal05_8192_b64"])
def test_rmi_golden(G, case):
    s, B = G[f"rmi/{case}/sample"], int(G[f"rmi/{case}/B"][0])
    P = O.rmi_train(s, B)
    assert np.array_equal(bits(P), bits(G[f"rmi/{case}/P"])), "trained params differ"
    pr = G[f"rmi/{case}/probe"]
    ok = route_defined(P, B, pr)
    assert np.array_equal(bits(O.rmi_predict(P, B, pr))[ok], bits(G[f"rmi/{case}/pred"])[ok])
    assert np.array_equal(O.learned_bucket(P, B, B, pr)[ok], G[f"rmi/{case}/bucket"][ok])
    assert np.array_equal(O.learned_bucket(P, B, 1000, pr)[ok], G[f"rmi/{case}/bucket1000"][ok])
    assert np.array_equal(O.learned_bucket(P, B, 256, pr, 0.25, 0.75)[ok],
                          G[f"rmi/{case}/bucket_sub"][ok])
    # where the reference's size_t cast is undefined (t >= 2^64, models.hpp:63),
    # the restatement clamps to the last submodel (monotone)
    if not ok.all():
        assert np.all(O.rmi_predict(P, B, pr)[~ok] >= O.rmi_predict(P, B, [s[-1]])[0])


def test_rmi_all_golden_cases(G):
    for case in golden_cases(G, "rmi"):
        s, B = G[f"rmi/{case}/sample"], int(G[f"rmi/{case}/B"][0])
        assert np.array_equal(bits(O.rmi_train(s, B)), bits(G[f"rmi/{case}/P"])), case


def test_tree_golden(G):
    for case in golden_cases(G, "tree"):
        s = G[f"tree/{case}/sample"]
        k, eq = int(G[f"tree/{case}/k"][0]), int(G[f"tree/{case}/eq"][0])
        t = O.tree_build(s, k, bool(eq))
        m = t.nsplitters
        assert np.array_equal(np.array(t.splitters[:m], np.uint64), G[f"tree/{case}/splitters"]), case
        heavy = np.array([t.eq_offset[i + 1] - t.eq_offset[i] > 1 for i in range(m)], np.uint8)
        assert np.array_equal(heavy, G[f"tree/{case}/heavy"]), case
        assert t.bucket_count == int(G[f"tree/{case}/bucket_count"][0]), case
        assert np.array_equal(O.tree_classify(t, G[f"tree/{case}/probe"]), G[f"tree/{case}/bucket"]), case


def test_dup_and_verify_golden(G):
    for k in "abcd":
        assert O.duplicate_fraction(G[f"dup/{k}/in"]) == float(G[f"dup/{k}/out"][0])
    for k in "abcde":
        ok, fv = O.verify_sorted(G[f"verify/{k}/in"])
        exp = G[f"verify/{k}/out"]
        assert (int(ok), fv, O.multiset_hash(G[f"verify/{k}/in"])) == (int(exp[0]), int(exp[1]), int(exp[2]))


def test_generator_fingerprints():
    with open(os.path.join(ROOT, "tests", "golden", "generators.json")) as f:
        gens = json.load(f)
    for dist, g in gens.items():
        if dist.startswith("spec_"):
            continue
        v = O.generate(dist, g["n"], g["seed"])
        k = O.encode(v) if v.dtype == np.float64 else v
        assert O.multiset_hash(k) == g["multiset_hash"], dist
        order = int(np.bitwise_xor.reduce(k * np.arange(1, g["n"] + 1, dtype=np.uint64)))
        assert order == g["order_hash"], dist
    assert gens["spec_rootdups16_unshuffled"] == [0, 1, 2, 3] * 4
    assert gens["spec_twodups8_unshuffled"] == [4, 5, 0, 5, 4, 5, 0, 5]


# ------------------------------------------------------- live vs _ref
needs_ref = pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built (no /root/reference)")


@needs_ref
@pytest.mark.parametrize("dist,seed", [("uniform", 42), ("normal", 7), ("mixgauss", 11),
                                       ("lognormal2", 19), ("exponential2", 7), ("zipf", 3)])
def test_rmi_live_vs_reference(dist, seed):
    import ctypes as C
    R = O.ref()
    v = O.generate(dist, 20000, seed)
    s = np.sort(O.encode(v) if v.dtype == np.float64 else v)
    for B in (1, 3, 100, 1024):
        P = O.rmi_train(s, B)
        Pr = np.zeros_like(P)
        R.ref_rmi_train(O._p(s), s.size, B, O._p(Pr))
        assert np.array_equal(bits(P), bits(Pr)), (dist, B)
        pr = np.ascontiguousarray(s[::37])
        b = np.zeros(pr.size, np.uint32)
        R.ref_rmi_eval(O._p(s), s.size, B, 1024, 0.0, 1.0, O._p(pr), pr.size, None, O._p(b))
        assert np.array_equal(O.learned_bucket(P, B, 1024, pr), b)


# ------------------------------------------------ SPEC known answers
def test_spec_examples():
    assert O.encode([0.0])[0] == 0x8000000000000000
    e = O.encode([-1.0, -0.0, 0.0, 1.0])
    assert e[0] < e[1] < e[2] < e[3]                                       # :51, :69
    P = O.rmi_train(np.arange(1000, dtype=np.uint64), 4)
    assert 0.45 <= O.rmi_predict(P, 4, [500])[0] <= 0.55                   # :119
    P1 = O.rmi_train(np.array([0, 1], np.uint64), 1)
    p0, p1 = O.rmi_predict(P1, 1, [0, 1])
    assert 0 <= p0 <= p1 <= 1                                              # :120
    n = np.sort(O.encode(O.generate("normal", 10_000, 1)))
    Pn = O.rmi_train(n, 64)
    emp = np.arange(n.size) / n.size
    assert np.mean(np.abs(O.rmi_predict(Pn, 64, n) - emp)) <= 0.05         # :121
    assert O.rmi_predict(P, 4, [0])[0] == 0.0                              # :137 (below all)
    assert O.learned_bucket(P, 4, 1000, [2**64 - 1])[0] == 999             # :138/:146
    t = O.tree_build(np.arange(256, dtype=np.uint64), 4, True)
    assert list(t.splitters[: t.nsplitters]) == [63, 127, 191]             # :155
    t7 = O.tree_build(np.full(10, 7, np.uint64), 4, True)
    assert t7.bucket_count == 3 and list(O.tree_classify(t7, [6, 7, 8])) == [0, 1, 2]  # :156
    assert O.duplicate_fraction([1, 2, 3, 4]) == 0.0                       # :164
    assert O.duplicate_fraction([5, 5, 5, 5]) == 0.75                      # :165
    assert O.verify_sorted([2, 1]) == (False, 1)                           # :427


def test_monotone_property():
    """zero violations over random key pairs, every distribution."""
    rng = np.random.default_rng(5)
    for dist, seed in [("uniform", 42), ("normal", 7), ("mixgauss", 11), ("lognormal2", 19)]:
        s = np.sort(O.encode(O.generate(dist, 5000, seed)))
        P = O.rmi_train(s, 256)
        a = rng.integers(0, 2**64 - 1, 20000, dtype=np.uint64, endpoint=True)
        b = np.concatenate([s[:: 2], a[: 10000]])
        keys = np.sort(np.concatenate([a, b]))
        pr = O.rmi_predict(P, 256, keys)
        assert np.all(np.diff(pr) >= 0), dist
        assert pr.min() >= 0 and pr.max() <= 1


# ------------------------------------------------------- sort driver
@pytest.mark.parametrize("dist,seed", [("uniform", 42), ("normal", 7), ("lognormal05", 7),
                                       ("exponential2", 7), ("mixgauss", 11), ("lognormal2", 19),
                                       ("rootdups", 3), ("twodups", 3), ("zipf", 3)])
@pytest.mark.parametrize("n", [1000, 100_000, 300_000])
def test_oracle_sort_generators(dist, seed, n):
    v = O.generate(dist, n, seed)
    if v.dtype == np.float64:
        got = O.sort_doubles(v)
        assert np.array_equal(bits(got), bits(O.decode(np.sort(O.encode(v)))))
    else:
        assert np.array_equal(O.sort_keys(v), np.sort(v))


def test_oracle_sort_adversarial():
    n = 200_000
    rng = np.random.default_rng(1)
    cases = {
        "sorted": np.arange(n, dtype=np.uint64),
        "reversed": np.arange(n, dtype=np.uint64)[::-1].copy(),
        "all_equal": np.full(n, 42, np.uint64),
        "organ_pipe": np.concatenate([np.arange(n // 2), np.arange(n // 2)[::-1]]).astype(np.uint64),
        "near_constant": np.where(rng.random(n) < 1e-4, 7, 5).astype(np.uint64),
        "empty": np.zeros(0, np.uint64), "one": np.array([9], np.uint64),
        "wide": rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True),
    }
    for name, a in cases.items():
        assert np.array_equal(O.sort_keys(a), np.sort(a)), name


def test_oracle_policy_alg5():
    """SPEC.md:375-383 / acceptance 4: Uniform 1e6 -> learned; RootDups 1e6 and any 1e4 -> tree."""
    c = O.cfg()
    u = O.encode(O.generate("uniform", 1_000_000, 42))
    assert O.build_partition_model(u, 0, 0, c, 1024, 256)[0] == 0
    rd = O.generate("rootdups", 1_000_000, 3)
    assert O.build_partition_model(rd, 0, 0, c, 1024, 256)[0] == 1
    assert O.build_partition_model(u[:10_000], 0, 0, c, 1024, 256)[0] == 1


def test_oracle_nan():
    x = O.generate("normal", 1000, 7)
    x[[17, 500]] = np.nan
    with pytest.raises(ValueError, match="index 17"):
        O.sort_doubles(x)
