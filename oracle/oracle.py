"""CPU ORACLE bindings (test infrastructure only).

ctypes access to oracle/liblsort_oracle.so (the C restatement of the
reference hot path, see lsort_oracle.h) and, when present, oracle/_ref/libref.so
(the reference's own model layer compiled from /root/reference). Only tests/,
__graft_entry__.smoke() and bench.py's CPU baseline legs import this module;
the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblsort_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libref.so")

GEN = {
    "uniform": 0, "normal": 1, "lognormal05": 2, "exponential2": 3, "mixgauss": 4,
    "rootdups": 5, "twodups": 6, "zipf": 7, "lognormal2": 8,
}
FLOAT_GENS = {"uniform", "normal", "lognormal05", "exponential2", "mixgauss", "lognormal2"}

MAX_TREE = 1024


class Tree(C.Structure):
    _fields_ = [
        ("levels", C.c_uint32), ("leaf_origin", C.c_uint32),
        ("nsplitters", C.c_uint32), ("bucket_count", C.c_uint32),
        ("tree", C.c_uint64 * MAX_TREE), ("splitters", C.c_uint64 * MAX_TREE),
        ("eq_offset", C.c_uint32 * (MAX_TREE + 1)),
    ]


class Cfg(C.Structure):
    _fields_ = [
        ("rmi_bucket_count", C.c_uint32), ("tree_bucket_count", C.c_uint32),
        ("min_rmi_input", C.c_uint64), ("max_duplicate_fraction", C.c_double),
        ("radix_base_case", C.c_uint32), ("insertion_base_case", C.c_uint32),
        ("first_sample_cap", C.c_uint32), ("rmi_sample_cap", C.c_uint32),
        ("sample_fraction", C.c_double), ("seed", C.c_uint64), ("workers", C.c_uint32),
    ]


def build(quiet: bool = True) -> None:
    """make -C oracle (C restatement always; _ref only where /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        u64, f64, sz, vp = C.c_uint64, C.c_double, C.c_size_t, C.c_void_p
        L.lso_encode_double.restype = u64; L.lso_encode_double.argtypes = [f64]
        L.lso_decode_double.restype = f64; L.lso_decode_double.argtypes = [u64]
        L.lso_encode_doubles.restype = C.c_int64; L.lso_encode_doubles.argtypes = [vp, vp, sz]
        L.lso_decode_doubles.restype = None; L.lso_decode_doubles.argtypes = [vp, vp, sz]
        L.lso_splitmix64.restype = u64; L.lso_splitmix64.argtypes = [u64]
        L.lso_rng_u64.restype = u64; L.lso_rng_u64.argtypes = [u64, u64]
        L.lso_rng_unit.restype = f64; L.lso_rng_unit.argtypes = [u64, u64]
        L.lso_rng_unit_open.restype = f64; L.lso_rng_unit_open.argtypes = [u64, u64]
        L.lso_rng_below.restype = u64; L.lso_rng_below.argtypes = [u64, u64, u64]
        L.lso_rng_normal.restype = f64; L.lso_rng_normal.argtypes = [u64, u64]
        L.lso_rng_exponential.restype = f64; L.lso_rng_exponential.argtypes = [u64, u64, f64]
        L.lso_rmi_train.restype = C.c_int; L.lso_rmi_train.argtypes = [vp, sz, C.c_uint32, vp]
        L.lso_rmi_train_given_root.restype = C.c_int
        L.lso_rmi_train_given_root.argtypes = [vp, sz, C.c_uint32, vp]
        L.lso_rmi_predict.restype = f64; L.lso_rmi_predict.argtypes = [vp, C.c_uint32, u64]
        L.lso_learned_bucket.restype = C.c_uint32
        L.lso_learned_bucket.argtypes = [vp, C.c_uint32, C.c_uint32, f64, f64, u64]
        L.lso_tree_build.restype = C.c_int
        L.lso_tree_build.argtypes = [vp, sz, C.c_uint32, C.c_int, C.POINTER(Tree)]
        L.lso_tree_classify.restype = C.c_uint32
        L.lso_tree_classify.argtypes = [C.POINTER(Tree), u64]
        L.lso_duplicate_fraction.restype = f64; L.lso_duplicate_fraction.argtypes = [vp, sz]
        L.lso_verify_sorted.restype = C.c_int
        L.lso_verify_sorted.argtypes = [vp, sz, C.POINTER(u64)]
        L.lso_multiset_hash.restype = u64; L.lso_multiset_hash.argtypes = [vp, sz]
        L.lso_generate.restype = C.c_int
        L.lso_generate.argtypes = [C.c_int, u64, u64, u64, u64, vp, C.c_int]
        L.lso_cfg_default.restype = None; L.lso_cfg_default.argtypes = [C.POINTER(Cfg)]
        L.lso_seg_seed.restype = u64; L.lso_seg_seed.argtypes = [u64, u64, C.c_uint32]
        L.lso_first_sample_size.restype = u64
        L.lso_first_sample_size.argtypes = [C.POINTER(Cfg), u64]
        L.lso_rmi_sample_size.restype = u64
        L.lso_rmi_sample_size.argtypes = [C.POINTER(Cfg), u64]
        L.lso_build_partition_model.restype = C.c_int
        L.lso_build_partition_model.argtypes = [
            vp, u64, u64, C.c_uint32, C.POINTER(Cfg), C.c_uint32, C.c_uint32,
            C.POINTER(C.c_int), vp, C.POINTER(Tree), C.POINTER(f64)]
        L.lso_sort_keys.restype = C.c_int; L.lso_sort_keys.argtypes = [vp, u64, C.POINTER(Cfg)]
        L.lso_sort_doubles.restype = C.c_int
        L.lso_sort_doubles.argtypes = [vp, u64, C.POINTER(Cfg), C.POINTER(C.c_int64)]
        L.lso_radix_base_case_sort.restype = None
        L.lso_radix_base_case_sort.argtypes = [vp, u64, C.c_uint32]
        L.lso_learned_pivots.restype = sz
        L.lso_learned_pivots.argtypes = [vp, sz, vp, C.c_uint32, C.c_uint32, vp]
        L.lso_rank_le.restype = u64; L.lso_rank_le.argtypes = [vp, sz, u64]
        L.lso_pivot_quality.restype = f64; L.lso_pivot_quality.argtypes = [vp, sz, vp, sz, C.c_uint32]
        L.lso_eta.restype = f64; L.lso_eta.argtypes = [vp, sz, u64]
        L.lso_learned_bucket_many.restype = None
        L.lso_learned_bucket_many.argtypes = [vp, C.c_uint32, C.c_uint32, f64, f64, vp, sz, vp]
        L.lso_tree_classify_many.restype = None
        L.lso_tree_classify_many.argtypes = [C.POINTER(Tree), vp, sz, vp]
        L.lso_model_counting_sort.restype = None
        L.lso_model_counting_sort.argtypes = [vp, sz, vp, C.c_uint32, f64, f64, vp]
        L.lso_learned_sort_classic.restype = C.c_int
        L.lso_learned_sort_classic.argtypes = [vp, u64, C.POINTER(Cfg), vp]
        L.lso_std_sort_u64.restype = None; L.lso_std_sort_u64.argtypes = [vp, u64]
        L.lso_parallel_sort_u64.restype = None; L.lso_parallel_sort_u64.argtypes = [vp, u64, C.c_int]
        L.lso_max_threads.restype = C.c_int; L.lso_max_threads.argtypes = []
        _lib = L
    return _lib


def ref():
    """The reference's own model layer (oracle/_ref/libref.so) or None."""
    global _ref
    if _ref is None and os.path.exists(REF_PATH):
        R = C.CDLL(REF_PATH)
        u64, f64, sz, vp = C.c_uint64, C.c_double, C.c_size_t, C.c_void_p
        R.ref_encode_double.restype = u64; R.ref_encode_double.argtypes = [f64]
        R.ref_decode_double.restype = f64; R.ref_decode_double.argtypes = [u64]
        R.ref_encode_doubles.restype = C.c_int64; R.ref_encode_doubles.argtypes = [vp, vp, sz]
        R.ref_splitmix64.restype = u64; R.ref_splitmix64.argtypes = [u64]
        R.ref_rng_stream.restype = None
        R.ref_rng_stream.argtypes = [u64, C.c_int, u64, f64, sz, vp, vp]
        R.ref_rmi_train.restype = C.c_int; R.ref_rmi_train.argtypes = [vp, sz, C.c_uint32, vp]
        R.ref_rmi_eval.restype = C.c_int
        R.ref_rmi_eval.argtypes = [vp, sz, C.c_uint32, C.c_uint32, f64, f64, vp, sz, vp, vp]
        R.ref_tree_eval.restype = C.c_int
        R.ref_tree_eval.argtypes = [vp, sz, C.c_uint32, C.c_int, vp, sz, vp, vp, vp, vp, vp]
        R.ref_duplicate_fraction.restype = f64; R.ref_duplicate_fraction.argtypes = [vp, sz]
        R.ref_verify_sorted.restype = C.c_int; R.ref_verify_sorted.argtypes = [vp, sz, vp]
        R.ref_multiset_hash.restype = u64; R.ref_multiset_hash.argtypes = [vp, sz]
        _ref = R
    return _ref


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


# ---------------------------------------------------------------- wrappers
def encode(x) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    out = np.empty(x.shape, np.uint64)
    bad = lib().lso_encode_doubles(_p(x), _p(out), x.size)
    if bad >= 0:
        raise ValueError(f"NaN at index {bad}")
    return out


def decode(k) -> np.ndarray:
    k = _u64(k)
    out = np.empty(k.shape, np.float64)
    lib().lso_decode_doubles(_p(k), _p(out), k.size)
    return out


def model_counting_sort(keys, P, B: int, cdf_lo: float = 0.0, cdf_hi: float = 1.0) -> np.ndarray:
    """stable counting placement by predicted position."""
    k = _u64(keys).reshape(-1)
    out = np.empty_like(k)
    lib().lso_model_counting_sort(_p(k), k.size, _p(np.ascontiguousarray(P, np.float64)), B, cdf_lo, cdf_hi,
                                  _p(out))
    return out


def learned_sort_classic(keys, c: Cfg | None = None):
    """SPEC.md:402-410 on a copy: (sorted keys, non-empty sub-buckets, insertion swaps)."""
    a = _u64(keys).reshape(-1).copy()
    st = np.zeros(2, np.uint64)
    lib().lso_learned_sort_classic(_p(a), a.size, C.byref(c or cfg()), _p(st))
    return a, int(st[0]), int(st[1])


def std_sort(keys) -> np.ndarray:
    """std::sort on one thread (CPU baseline), in place on uint64 keys."""
    assert keys.dtype == np.uint64 and keys.flags["C_CONTIGUOUS"]
    lib().lso_std_sort_u64(_p(keys), keys.size)
    return keys


def parallel_sort(keys, threads: int = 0) -> np.ndarray:
    """__gnu_parallel::sort on `threads` OpenMP threads (CPU baseline), in place."""
    assert keys.dtype == np.uint64 and keys.flags["C_CONTIGUOUS"]
    lib().lso_parallel_sort_u64(_p(keys), keys.size, threads)
    return keys


def rmi_train(sorted_sample, B: int) -> np.ndarray:
    s = _u64(sorted_sample)
    P = np.zeros(4 + 4 * B, np.float64)
    if lib().lso_rmi_train(_p(s), s.size, B, _p(P)) != 0:
        raise ValueError("Rmi::train: invalid argument")
    return P


def rmi_train_given_root(sorted_sample, B: int, root_slope: float, root_intercept: float) -> np.ndarray:
    """Reference slicing + fits + enforce_monotonic under a given root model."""
    s = _u64(sorted_sample)
    P = np.zeros(4 + 4 * B, np.float64)
    P[0], P[1] = root_slope, root_intercept
    if lib().lso_rmi_train_given_root(_p(s), s.size, B, _p(P)) != 0:
        raise ValueError("Rmi::train: invalid argument")
    return P


def rmi_predict(P: np.ndarray, B: int, keys) -> np.ndarray:
    L = lib()
    return np.array([L.lso_rmi_predict(_p(P), B, int(k)) for k in _u64(keys)], np.float64)


def learned_bucket(P, B, bucket_count, keys, cdf_lo=0.0, cdf_hi=1.0) -> np.ndarray:
    k = _u64(keys).reshape(-1)
    P = np.ascontiguousarray(P, np.float64)
    out = np.empty(k.size, np.uint32)
    lib().lso_learned_bucket_many(_p(P), B, bucket_count, cdf_lo, cdf_hi, _p(k), k.size, _p(out))
    return out


def tree_build(sorted_sample, budget: int, equality_mode: bool = True) -> Tree:
    s = _u64(sorted_sample)
    t = Tree()
    if lib().lso_tree_build(_p(s), s.size, budget, int(equality_mode), C.byref(t)) != 0:
        raise ValueError("SplitterTree::build: invalid argument")
    return t


def tree_classify(t: Tree, keys) -> np.ndarray:
    k = _u64(keys).reshape(-1)
    out = np.empty(k.size, np.uint32)
    lib().lso_tree_classify_many(C.byref(t), _p(k), k.size, _p(out))
    return out


def duplicate_fraction(sorted_sample) -> float:
    s = _u64(sorted_sample)
    return lib().lso_duplicate_fraction(_p(s), s.size)


def learned_pivots(keys, P, B: int, b: int) -> np.ndarray:
    """Alg. 4: largest key per learned cell i < b-1, empty cells dropped."""
    a = _u64(keys)
    out = np.zeros(max(b - 1, 1), np.uint64)
    m = lib().lso_learned_pivots(_p(a), a.size, _p(np.ascontiguousarray(P, np.float64)), B, b, _p(out))
    return out[:m].copy()


def pivot_quality(sorted_keys, pivots, b: int) -> float:
    """sum_i |P(A <= p_i) - (i+1)/b|; ValueError unless len(pivots) + 1 == b."""
    s, p = _u64(sorted_keys), _u64(pivots)
    if p.size + 1 != b:
        raise ValueError("pivot count + 1 != b")
    return float(lib().lso_pivot_quality(_p(s), s.size, _p(p), p.size, b))


def eta(sorted_keys, pivot: int) -> float:
    """max(P(A <= p), 1 - P(A <= p)) - 1/2 (§3.1)."""
    s = _u64(sorted_keys)
    return float(lib().lso_eta(_p(s), s.size, int(pivot)))


def verify_sorted(a):
    a = _u64(a)
    fv = C.c_uint64(0)
    ok = lib().lso_verify_sorted(_p(a), a.size, C.byref(fv))
    return bool(ok), int(fv.value)


def multiset_hash(a) -> int:
    a = _u64(a)
    return int(lib().lso_multiset_hash(_p(a), a.size))


def generate(dist: str, n: int, seed: int, first: int = 0, count: int | None = None,
             threads: int = 0) -> np.ndarray:
    count = n - first if count is None else count
    out = np.empty(count, np.float64 if dist in FLOAT_GENS else np.uint64)
    if lib().lso_generate(GEN[dist], n, seed, first, count, _p(out), threads) != 0:
        raise ValueError("generate: bad arguments")
    return out


def cfg(**kw) -> Cfg:
    c = Cfg()
    lib().lso_cfg_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def sort_keys(a, c: Cfg | None = None) -> np.ndarray:
    a = _u64(a).copy()
    c = c or cfg()
    lib().lso_sort_keys(_p(a), a.size, C.byref(c))
    return a


def sort_doubles(a, c: Cfg | None = None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64)).copy()
    c = c or cfg()
    bad = C.c_int64(-1)
    rc = lib().lso_sort_doubles(_p(a), a.size, C.byref(c), C.byref(bad))
    if rc == 2:
        raise ValueError(f"NaN at index {bad.value}")
    return a


def build_partition_model(a, seg_begin: int, depth: int, c: Cfg, rmi_buckets: int,
                          tree_buckets: int):
    """Alg. 5 on segment a (encoded keys). Returns (kind, P or None, Tree or None, dup)."""
    a = _u64(a)
    kind = C.c_int(-1)
    P = np.zeros(4 + 4 * rmi_buckets, np.float64)
    t = Tree()
    dup = C.c_double(0)
    lib().lso_build_partition_model(_p(a), a.size, seg_begin, depth, C.byref(c), rmi_buckets,
                                    tree_buckets, C.byref(kind), _p(P), C.byref(t), C.byref(dup))
    return kind.value, (P if kind.value == 0 else None), (t if kind.value == 1 else None), dup.value
