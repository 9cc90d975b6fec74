"""B200-native parallel LearnedSort (AIPS2o, arXiv 2307.08637).

Python host mirror of the reference's sort interface: ``sort(a, cfg)`` over a
contiguous range of float64 / uint64 keys, in place, with
``SortConfig``. Every call goes through the C-ABI of
``liblsort_cuda.so`` (include/lsort_cuda.h): hand-written sm_100a kernels and a
C++ orchestrator. Device arrays are torch CUDA tensors (float64, int64 or
uint64); host arrays (numpy) are copied in and out inside the call. There is
no CPU fallback: the native library must be built (``build()``).

Error behaviour mirrors the reference: invalid arguments raise ValueError
(std::invalid_argument, models.cpp:40-43,135-138); a NaN in float64 input
raises ``NanError`` carrying the first NaN index (encode_doubles,
keys.hpp:34-42) and leaves the array unmodified.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import threading
from typing import Any

import numpy as np

from . import _native as N

__all__ = ["SortConfig", "Context", "NanError", "LsortError", "sort", "generate", "read_keys", "write_keys", "DISTS",
           "build", "default_context"]

DISTS = {"uniform": 0, "normal": 1, "lognormal05": 2, "exponential2": 3, "mixgauss": 4,
         "rootdups": 5, "twodups": 6, "zipf": 7, "lognormal2": 8}
FLOAT_DISTS = {"uniform", "normal", "lognormal05", "exponential2", "mixgauss", "lognormal2"}


def build(verbose: bool = False) -> str:
    from .build import build as _b
    return _b(verbose=verbose)


class LsortError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"lsort error {code}: {msg}")
        self.code = code


class NanError(ValueError):
    """NaN in float64 input (keys.hpp:34-42: rejected at ingestion with its index)."""

    def __init__(self, index: int):
        super().__init__(f"NaN at index {index}" if index >= 0 else "NaN in another rank's shard")
        self.index = index


@dataclasses.dataclass
class SortConfig:
    """SortConfig plus GPU extensions."""
    rmi_bucket_count: int = 1024
    tree_bucket_count: int = 256
    min_rmi_input: int = 100_000
    max_duplicate_fraction: float = 0.10
    radix_base_case: int = 4096
    insertion_base_case: int = 16
    first_sample_cap: int = 2 * 256 * 16
    rmi_sample_cap: int = 1 << 20
    sample_fraction: float = 0.01
    seed: int = 0x5EED
    workers: int = 0
    base_case_capacity: int = 16384
    bucket_target: int = 4096
    flags: int = 0

    def to_c(self) -> N.lsort_cfg:
        c = N.lsort_cfg()
        for f in dataclasses.fields(self):
            setattr(c, f.name, getattr(self, f.name))
        return c


def _check(ctx: "Context", rc: int):
    if rc == N.LSORT_OK:
        return
    msg = N.lib().lsort_cuda_last_error(ctx._h).decode() if ctx._h else ""
    if rc == N.LSORT_EINVAL:
        raise ValueError(msg or "invalid argument")
    raise LsortError(rc, msg)


def _torch():
    import torch
    return torch


def _key_kind_of(arr) -> int:
    dt = str(arr.dtype)
    if "float64" in dt:
        return N.KEY_F64
    if "int64" in dt or "uint64" in dt:
        return N.KEY_U64
    raise ValueError(f"keys must be float64, int64 or uint64 (got {arr.dtype})")


class Context:
    """One lsort_ctx (workspace + stream) on one device. Not thread-safe."""

    def __init__(self, device: int = 0, stream: Any = None, workspace_hint: int = 0):
        L = N.lib()
        h = C.c_void_p()
        rc = L.lsort_cuda_ctx_create(C.byref(h), device, stream, workspace_hint)
        if rc != N.LSORT_OK:
            raise LsortError(rc, f"cannot create context on device {device}")
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            N.lib().lsort_cuda_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- streams -----------------------------------------------------------
    def _sync_stream(self):
        """Order the native call after the work torch has queued: run on torch's
        current stream; when that is the legacy default stream (handle 0, which
        the C-ABI reads as 'the context's own stream'), wait for it first --
        a NCCL collective or an async copy feeding the keys would otherwise race
        the sort."""
        torch = _torch()
        cur = torch.cuda.current_stream(self.device)
        s = cur.cuda_stream
        if not s:
            cur.synchronize()
        N.lib().lsort_cuda_set_stream(self._h, C.c_void_p(s) if s else None)

    # -- the drop-in sort ----------------------------------------------------
    def sort(self, keys, cfg: SortConfig | None = None, encoded_f64: bool = False) -> dict:
        """In-place ascending sort. `keys`: torch CUDA tensor (device) or a
        contiguous numpy array (host; copied in/out inside the call)."""
        L = N.lib()
        cfg_c = (cfg or SortConfig()).to_c()
        stats = N.lsort_stats()
        nan = C.c_uint64(0)
        if isinstance(keys, np.ndarray):
            if not keys.flags["C_CONTIGUOUS"]:
                raise ValueError("host keys must be contiguous")
            kind, mem, ptr, n = _key_kind_of(keys), N.MEM_HOST, keys.ctypes.data, keys.size
            N.lib().lsort_cuda_set_stream(self._h, None)
        else:
            if not keys.is_cuda or not keys.is_contiguous():
                raise ValueError("device keys must be a contiguous CUDA tensor")
            self._sync_stream()
            kind, mem, ptr, n = _key_kind_of(keys), N.MEM_DEVICE, keys.data_ptr(), keys.numel()
        if encoded_f64:  # u64 keys in encoded form; sorted result decoded to float64 in place
            kind = N.KEY_ENC_F64
        rc = L.lsort_cuda_sort(self._h, C.c_void_p(ptr), n, kind, mem, C.byref(cfg_c), C.byref(stats),
                               C.byref(nan))
        if rc == N.LSORT_ENAN:
            raise NanError(int(nan.value))
        _check(self, rc)
        return stats.as_dict()

    def sort_classic(self, keys, cfg: SortConfig | None = None) -> dict:
        """learned_sort_classic: one RMI trained once, two
        partition rounds with that model, model-based counting sort + fix-up
        (lsort_cuda_sort_classic). Same arguments / errors as sort()."""
        cfg_c = (cfg or SortConfig()).to_c()
        stats = N.lsort_stats()
        nan = C.c_uint64(0)
        if isinstance(keys, np.ndarray):
            if not keys.flags["C_CONTIGUOUS"]:
                raise ValueError("host keys must be contiguous")
            kind, mem, ptr, n = _key_kind_of(keys), N.MEM_HOST, keys.ctypes.data, keys.size
            N.lib().lsort_cuda_set_stream(self._h, None)
        else:
            if not keys.is_cuda or not keys.is_contiguous():
                raise ValueError("device keys must be a contiguous CUDA tensor")
            self._sync_stream()
            kind, mem, ptr, n = _key_kind_of(keys), N.MEM_DEVICE, keys.data_ptr(), keys.numel()
        rc = N.lib().lsort_cuda_sort_classic(self._h, C.c_void_p(ptr), n, kind, mem, C.byref(cfg_c), C.byref(stats),
                                             C.byref(nan))
        if rc == N.LSORT_ENAN:
            raise NanError(int(nan.value))
        _check(self, rc)
        return stats.as_dict()

    def model_counting_sort(self, P: np.ndarray, submodels: int, d_keys, cdf_lo: float = 0.0, cdf_hi: float = 1.0):
        """model_counting_sort of one device segment (<= 8192
        uint64 keys): returns a new tensor placed by predicted position, stable."""
        torch = _torch()
        self._sync_stream()
        h, e = unpack_rmi(P, submodels)
        out = torch.empty_like(d_keys)
        rc = N.lib().lsort_cuda_model_counting_sort(self._h, C.byref(h), e.ctypes.data_as(C.c_void_p), cdf_lo, cdf_hi,
                                                    C.c_void_p(d_keys.data_ptr()), d_keys.numel(),
                                                    C.c_void_p(out.data_ptr()))
        _check(self, rc)
        return out

    def sort_batch(self, arrays, cfg: SortConfig | None = None) -> dict:
        """Sort several arrays (one key kind) in one call. Host (numpy) arrays:
        copies in / out pipelined against the sorts (lsort_cuda_sort_batch);
        CUDA tensors: up to three sorts run concurrently (lsort_cuda_sort_many). Raises
        NanError(index, array=i) for the first array holding a NaN (left
        untouched; the others are sorted)."""
        if not arrays:
            return {}
        kinds = {_key_kind_of(a) for a in arrays}
        if len(kinds) != 1:
            raise ValueError("sort_batch: all arrays must have the same key kind")
        device = not isinstance(arrays[0], np.ndarray)
        for a in arrays:
            if device:
                if isinstance(a, np.ndarray) or not a.is_cuda or not a.is_contiguous():
                    raise ValueError("sort_batch: device arrays must be contiguous CUDA tensors")
            elif not isinstance(a, np.ndarray) or not a.flags["C_CONTIGUOUS"]:
                raise ValueError("sort_batch: host arrays must be contiguous numpy arrays")
        m = len(arrays)
        if device:
            self._sync_stream()
            ptrs = (C.c_void_p * m)(*[a.data_ptr() for a in arrays])
            ns = (C.c_uint64 * m)(*[a.numel() for a in arrays])
            nans = (C.c_uint64 * m)()
            cfg_c = (cfg or SortConfig()).to_c()
            stats = N.lsort_stats()
            rc = N.lib().lsort_cuda_sort_many(self._h, ptrs, ns, m, kinds.pop(), C.byref(cfg_c), C.byref(stats),
                                              nans)
            if rc == N.LSORT_ENAN:
                i = next(i for i in range(m) if nans[i] != (1 << 64) - 1)
                err = NanError(int(nans[i]))
                err.array = i
                raise err
            _check(self, rc)
            return stats.as_dict()
        ptrs = (C.c_void_p * m)(*[a.ctypes.data for a in arrays])
        ns = (C.c_uint64 * m)(*[a.size for a in arrays])
        nans = (C.c_uint64 * m)()
        cfg_c = (cfg or SortConfig()).to_c()
        stats = N.lsort_stats()
        N.lib().lsort_cuda_set_stream(self._h, None)
        rc = N.lib().lsort_cuda_sort_batch(self._h, ptrs, ns, m, kinds.pop(), C.byref(cfg_c), C.byref(stats), nans)
        if rc == N.LSORT_ENAN:
            i = next(i for i in range(m) if nans[i] != (1 << 64) - 1)
            err = NanError(int(nans[i]))
            err.array = i
            raise err
        _check(self, rc)
        return stats.as_dict()

    def sort_forward(self, d_keys, P: np.ndarray, submodels: int, b_lo: int, b_hi: int, d_sorted_sample=None,
                     cfg: SortConfig | None = None, encoded_f64: bool = False) -> dict:
        """lsort_cuda_sort_forward: sort device keys of buckets [b_lo, b_hi) of the
        learned model P (packed) with its root level forwarded (no training)."""
        self._sync_stream()
        h, e = unpack_rmi(P, submodels)
        cfg_c = (cfg or SortConfig()).to_c()
        stats = N.lsort_stats()
        nan = C.c_uint64(0)
        kind = N.KEY_ENC_F64 if encoded_f64 else _key_kind_of(d_keys)
        sp = C.c_void_p(d_sorted_sample.data_ptr()) if d_sorted_sample is not None else None
        sn = d_sorted_sample.numel() if d_sorted_sample is not None else 0
        rc = N.lib().lsort_cuda_sort_forward(self._h, C.c_void_p(d_keys.data_ptr()), d_keys.numel(), kind,
                                             C.byref(cfg_c), C.byref(h), e.ctypes.data_as(C.c_void_p), b_lo, b_hi,
                                             sp, sn, C.byref(stats), C.byref(nan))
        if rc == N.LSORT_ENAN:
            raise NanError(int(nan.value))
        _check(self, rc)
        return stats.as_dict()

    def sort_buckets(self, d_keys, P: np.ndarray, submodels: int, b_lo: int, b_hi: int, sizes, d_sorted_sample=None,
                     cfg: SortConfig | None = None, encoded_f64: bool = False) -> dict:
        """lsort_cuda_sort_buckets: keys already grouped by the model's buckets
        [b_lo, b_hi) (sizes per bucket, in order); small buckets sorted in place,
        the rest recursed from level 1. encoded_f64: decode in the final stores."""
        self._sync_stream()
        h, e = unpack_rmi(P, submodels)
        sz = np.ascontiguousarray(np.asarray(sizes, dtype=np.uint64))
        stats = N.lsort_stats()
        c = (cfg or SortConfig()).to_c()
        kind = N.KEY_ENC_F64 if encoded_f64 else N.KEY_U64
        sp = C.c_void_p(d_sorted_sample.data_ptr()) if d_sorted_sample is not None else None
        sn = d_sorted_sample.numel() if d_sorted_sample is not None else 0
        rc = N.lib().lsort_cuda_sort_buckets(self._h, C.c_void_p(d_keys.data_ptr()), d_keys.numel(), kind, C.byref(c),
                                             C.byref(h), e.ctypes.data_as(C.c_void_p), b_lo, b_hi,
                                             sz.ctypes.data_as(C.c_void_p), sp, sn, C.byref(stats))
        _check(self, rc)
        return stats.as_dict()

    # -- unit entry points (parity tests) --------------------------------------
    def rmi_train(self, d_sorted_sample, submodels: int):
        """Rmi::train + enforce_monotonic on a sorted device sample -> packed P."""
        self._sync_stream()
        h = N.lsort_rmi_header()
        e = np.zeros((submodels, 4), np.float64)
        rc = N.lib().lsort_cuda_rmi_train(self._h, C.c_void_p(d_sorted_sample.data_ptr()),
                                          d_sorted_sample.numel(), submodels, C.byref(h),
                                          e.ctypes.data_as(C.c_void_p))
        _check(self, rc)
        return pack_rmi(h, e)

    def classify_rmi(self, P: np.ndarray, submodels: int, bucket_count: int, d_keys, cdf_lo=0.0,
                     cdf_hi=1.0, ids=True):
        torch = _torch()
        self._sync_stream()
        h, e = unpack_rmi(P, submodels)
        n = d_keys.numel()
        d_ids = torch.empty(n, dtype=torch.int32, device=d_keys.device) if ids else None
        d_hist = torch.empty(bucket_count, dtype=torch.int64, device=d_keys.device)
        rc = N.lib().lsort_cuda_classify_rmi(
            self._h, C.byref(h), e.ctypes.data_as(C.c_void_p), bucket_count, cdf_lo, cdf_hi,
            C.c_void_p(d_keys.data_ptr()), n, _key_kind_of(d_keys),
            C.c_void_p(d_ids.data_ptr()) if ids else None, C.c_void_p(d_hist.data_ptr()))
        _check(self, rc)
        return d_ids, d_hist

    def tree_build(self, d_sorted_sample, budget: int, equality_mode: bool = True) -> N.lsort_tree:
        self._sync_stream()
        t = N.lsort_tree()
        rc = N.lib().lsort_cuda_tree_build(self._h, C.c_void_p(d_sorted_sample.data_ptr()),
                                           d_sorted_sample.numel(), budget, int(equality_mode),
                                           C.byref(t))
        _check(self, rc)
        return t

    def classify_tree(self, t: N.lsort_tree, d_keys, ids=True):
        torch = _torch()
        self._sync_stream()
        n = d_keys.numel()
        d_ids = torch.empty(n, dtype=torch.int32, device=d_keys.device) if ids else None
        d_hist = torch.empty(t.bucket_count, dtype=torch.int64, device=d_keys.device)
        rc = N.lib().lsort_cuda_classify_tree(self._h, C.byref(t), C.c_void_p(d_keys.data_ptr()), n,
                                              _key_kind_of(d_keys),
                                              C.c_void_p(d_ids.data_ptr()) if ids else None,
                                              C.c_void_p(d_hist.data_ptr()))
        _check(self, rc)
        return d_ids, d_hist

    def build_model(self, d_keys, cfg: SortConfig | None = None):
        """Alg. 5 on the whole array: returns dict(kind, nbuckets, s1, s2, dup, P|tree)."""
        self._sync_stream()
        cfg_c = (cfg or SortConfig()).to_c()
        info = N.lsort_model_info()
        h = N.lsort_rmi_header()
        e = np.zeros((N.MAX_RMI, 4), np.float64)
        t = N.lsort_tree()
        rc = N.lib().lsort_cuda_build_model(self._h, C.c_void_p(d_keys.data_ptr()), d_keys.numel(),
                                            _key_kind_of(d_keys), C.byref(cfg_c), C.byref(info),
                                            C.byref(h), e.ctypes.data_as(C.c_void_p), C.byref(t))
        _check(self, rc)
        out = {"kind": info.kind, "nbuckets": info.nbuckets, "s1": info.first_sample,
               "s2": info.rmi_sample, "dup": info.duplicate_fraction}
        if info.kind == 0:
            out["P"] = pack_rmi(h, e[: h.submodels])
            out["B"] = h.submodels
        else:
            out["tree"] = t
        return out

    # -- pivot analysis (Alg. 4 / Table 1) -----------
    def learned_pivots(self, P: np.ndarray, submodels: int, b: int, d_keys, cells: bool = False):
        """Alg. 4: largest key of each learned cell i < b-1 (empty cells dropped),
        ascending; in the keys' representation (float64 for float keys).
        cells=True also returns each pivot's cell index."""
        self._sync_stream()
        h, e = unpack_rmi(P, submodels)
        out = np.zeros(max(b - 1, 1), np.uint64)
        cel = np.zeros(max(b - 1, 1), np.uint32)
        cnt = C.c_uint32(0)
        rc = N.lib().lsort_cuda_learned_pivots(self._h, C.byref(h), e.ctypes.data_as(C.c_void_p), b,
                                               C.c_void_p(d_keys.data_ptr()), d_keys.numel(),
                                               _key_kind_of(d_keys), out.ctypes.data_as(C.c_void_p),
                                               cel.ctypes.data_as(C.c_void_p), C.byref(cnt))
        _check(self, rc)
        out = out[:cnt.value].copy()
        if _key_kind_of(d_keys) == N.KEY_F64:
            out = out.view(np.float64)
        return (out, cel[:cnt.value].copy()) if cells else out

    def pivot_quality(self, d_sorted, pivots, b: int):
        """(distance, ranks): sum_i |P(A <= p_i) - (i+1)/b| over device-resident
        sorted keys; LsortError (EINVAL) unless len(pivots) + 1 == b."""
        self._sync_stream()
        p = np.ascontiguousarray(np.asarray(pivots)).view(np.uint64)
        d = C.c_double(0.0)
        ranks = np.zeros(max(p.size, 1), np.uint64)
        rc = N.lib().lsort_cuda_pivot_quality(self._h, C.c_void_p(d_sorted.data_ptr()), d_sorted.numel(),
                                              _key_kind_of(d_sorted), p.ctypes.data_as(C.c_void_p), p.size, b,
                                              C.byref(d), ranks.ctypes.data_as(C.c_void_p))
        _check(self, rc)
        return d.value, ranks[:p.size]

    def eta(self, d_sorted, pivot) -> float:
        """max(P(A <= p), 1 - P(A <= p)) - 1/2 (§3.1)."""
        self._sync_stream()
        pv = int(np.asarray(pivot).reshape(1).view(np.uint64)[0])
        out = C.c_double(0.0)
        rc = N.lib().lsort_cuda_eta(self._h, C.c_void_p(d_sorted.data_ptr()), d_sorted.numel(),
                                    _key_kind_of(d_sorted), pv, C.byref(out))
        _check(self, rc)
        return out.value

    def block_sort(self, d_keys):
        self._sync_stream()
        _check(self, N.lib().lsort_cuda_block_sort(self._h, C.c_void_p(d_keys.data_ptr()), d_keys.numel()))

    def verify(self, d_keys):
        """(sorted, first_violation, multiset_hash) -- verify.hpp:17-29 on device."""
        self._sync_stream()
        fv, hs = C.c_uint64(0), C.c_uint64(0)
        rc = N.lib().lsort_cuda_verify(self._h, C.c_void_p(d_keys.data_ptr()), d_keys.numel(),
                                       _key_kind_of(d_keys), C.byref(fv), C.byref(hs))
        _check(self, rc)
        return fv.value == 0, int(fv.value), int(hs.value)


def pack_rmi(h: N.lsort_rmi_header, e: np.ndarray) -> np.ndarray:
    """Packed P layout shared with the oracle: 4 header doubles then B x 4."""
    P = np.empty(4 + e.size, np.float64)
    P[:4] = [h.root_slope, h.root_intercept, h.key_base, h.key_scale]
    P[4:] = e.reshape(-1)
    return P


def unpack_rmi(P: np.ndarray, B: int):
    h = N.lsort_rmi_header(P[0], P[1], P[2], P[3], B, 0)
    e = np.ascontiguousarray(P[4: 4 + 4 * B].reshape(B, 4))
    return h, e


_tls = threading.local()


def default_context(device: int | None = None) -> Context:
    if device is None:
        device = _torch().cuda.current_device() if _torch().cuda.is_available() else 0
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def sort(keys, cfg: SortConfig | None = None) -> dict:
    """lsort::sort -- in-place ascending sort of float64 / uint64 keys."""
    dev = keys.device.index if hasattr(keys, "device") and getattr(keys, "is_cuda", False) else None
    return default_context(dev).sort(keys, cfg)


def generate(dist: str, n: int, seed: int, first: int = 0, count: int | None = None,
             threads: int = 0) -> np.ndarray:
    """Synthetic config inputs (host, glibc libm, reference Rng stream)."""
    count = n - first if count is None else count
    out = np.empty(count, np.float64 if dist in FLOAT_DISTS else np.uint64)
    rc = N.lib().lsort_gen_keys(DISTS[dist], n, seed, first, count, out.ctypes.data_as(C.c_void_p),
                                threads)
    if rc != N.LSORT_OK:
        raise ValueError("generate: bad arguments")
    return out


# --------------------------------------------------------------- key files
def write_keys(path: str, keys) -> None:
    """data.write_keys: 8-byte LE count + count 8-byte LE keys."""
    a = np.ascontiguousarray(keys)
    if a.dtype.itemsize != 8:
        raise ValueError("write_keys: 8-byte keys expected")
    err = C.create_string_buffer(512)
    rc = N.lib().lsort_write_keys(str(path).encode(), C.c_void_p(a.ctypes.data), a.size, err, 512)
    if rc != N.LSORT_OK:
        raise OSError(err.value.decode())


def read_keys(path: str) -> np.ndarray:
    """data.read_keys -> uint64 array; a truncated or
    oversized file raises OSError naming the expected and actual byte ranges."""
    err = C.create_string_buffer(512)
    n = C.c_uint64(0)
    rc = N.lib().lsort_read_keys(str(path).encode(), None, 0, C.byref(n), err, 512)
    if rc != N.LSORT_OK:
        raise OSError(err.value.decode())
    out = np.empty(n.value, np.uint64)
    rc = N.lib().lsort_read_keys(str(path).encode(), C.c_void_p(out.ctypes.data), out.size, C.byref(n), err, 512)
    if rc != N.LSORT_OK:
        raise OSError(err.value.decode())
    return out
