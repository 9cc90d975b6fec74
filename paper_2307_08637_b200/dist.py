"""Multi-GPU distributed LearnedSort: RMI splitters + one all-to-all.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch). Each rank
holds a shard; after ``DistSorter.sort`` rank r holds the r-th key range of
the global sorted order (variable length), so the concatenation over ranks is
the sorted input.

Steps per sort (collectives are torch.distributed; all device work is the C-ABI):
  1. every rank draws its share of the global RMI sample (device gather,
     reference Rng stream per rank, rng.hpp:35-37);
  2. all_gather of the samples; every rank sorts the identical global sample
     and trains the identical monotone RMI (deterministic kernels,
     models.cpp:39-131) -- no broadcast of parameters is needed;
  3. local histogram under the global model, all_reduce -> global histogram;
  4. rank boundaries = bucket-id cut points balancing the global counts
     (monotone F => ranks receive disjoint, ordered key ranges);
  5. destination-major partition of the local shard (the level-0 scatter with a
     bucket -> rank map), all_to_all of the counts, all_to_all_single of keys;
  6. local LearnedSort of the received (encoded) keys, decoded in place for
     float64.

``ops`` abstracts the device steps: the default (``NativeOps``) calls
liblsort_cuda.so; tests inject a CPU implementation to exercise this host
logic with gloo on CPU. The product path never uses a CPU fallback.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def splitmix64(x: int) -> int:
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def rank_bounds(hist: np.ndarray, world: int) -> np.ndarray:
    """Bucket cut points: rank r receives buckets [b[r], b[r+1]). Greedy
    equal-count split of the global histogram (identical on every rank)."""
    hist = np.asarray(hist, dtype=np.int64)
    B = hist.size
    total = int(hist.sum())
    pref = np.cumsum(hist)
    bounds = [0]
    for r in range(1, world):
        target = math.ceil(r * total / world)
        b = int(np.searchsorted(pref, target, side="left")) + 1  # first bucket after the cut
        b = min(max(b, bounds[-1]), B)
        bounds.append(b)
    bounds.append(B)
    return np.asarray(bounds, dtype=np.uint32)


def sample_shares(n_local: list[int], s_total: int) -> list[int]:
    """Per-rank sample sizes proportional to shard sizes (sum == s_total)."""
    N = sum(n_local)
    if N == 0:
        return [0] * len(n_local)
    shares = [s_total * n // N for n in n_local]
    rem = s_total - sum(shares)
    for i in range(rem):
        shares[i % len(shares)] += 1
    return [min(s, n) if n else 0 for s, n in zip(shares, n_local)]


def bucket_exchange_plan(hists: np.ndarray, bounds: np.ndarray, rank: int):
    """Host plan of the bucket-major exchange. hists: (world, B) per-source
    bucket counts (the all-gathered local histograms); bounds: rank bucket
    ranges. Returns (send counts per destination, receive counts per source,
    runs (src_off, dst_off, len) that turn the source-major receive buffer --
    source s's keys of buckets [lo, hi), bucket-major -- into bucket-major
    order with the sources in rank order inside each bucket, per-bucket sizes)."""
    hists = np.asarray(hists, dtype=np.int64)
    world = hists.shape[0]
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    send = [int(hists[rank, bounds[r]:bounds[r + 1]].sum()) for r in range(world)]
    mine = hists[:, lo:hi]
    recv = [int(mine[s].sum()) for s in range(world)]
    sizes = mine.sum(axis=0)
    bstart = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    before = np.zeros(hi - lo, np.int64)  # keys of the same bucket from lower ranks
    runs = []
    src_base = 0
    for s in range(world):  # vectorised over the buckets
        h = mine[s]
        src_off = src_base + np.concatenate([[0], np.cumsum(h)[:-1]]).astype(np.int64)
        nz = h > 0
        runs.append(np.stack([src_off[nz], (bstart + before)[nz], h[nz]], axis=1))
        before += h
        src_base += int(h.sum())
    runs = np.concatenate(runs, axis=0) if runs else np.zeros((0, 3), np.int64)
    return send, recv, runs.astype(np.uint64).reshape(-1, 3), sizes.astype(np.uint64)


class NativeOps:
    """Device steps through the C-ABI (liblsort_cuda.so)."""

    fused_decode = True  # local_sort(to_f64=True) decodes in its final stores

    def __init__(self, ctx):
        self.ctx = ctx

    def sample(self, keys, s: int, seed: int):
        import ctypes as C
        import torch
        from . import _native as N
        from . import _key_kind_of
        out = torch.empty(max(s, 1), dtype=torch.int64, device=keys.device)
        self.ctx._sync_stream()
        if s:
            rc = N.lib().lsort_cuda_dist_sample(self.ctx._h, C.c_void_p(keys.data_ptr()), keys.numel(),
                                                _key_kind_of(keys), seed, s, C.c_void_p(out.data_ptr()))
            self._check(rc)
        return out[:s]

    def train(self, sample, buckets: int):
        import ctypes as C
        from . import _native as N
        from . import pack_rmi
        h = N.lsort_rmi_header()
        e = np.zeros((buckets, 4), np.float64)
        self.ctx._sync_stream()
        rc = N.lib().lsort_cuda_dist_train(self.ctx._h, C.c_void_p(sample.data_ptr()), sample.numel(), buckets,
                                           C.byref(h), e.ctypes.data_as(C.c_void_p))
        self._check(rc)
        return pack_rmi(h, e)

    def histogram(self, keys, P, buckets: int):
        # lsort_cuda_dist_histogram: the level-0 classify kernel; it also keeps
        # the bucket ids, which lsort_cuda_dist_partition then reuses
        import ctypes as C
        import torch
        from . import _native as N
        from . import _key_kind_of, unpack_rmi
        h, e = unpack_rmi(P, buckets)
        hist = torch.zeros(buckets, dtype=torch.int64, device=keys.device)
        self.ctx._sync_stream()
        rc = N.lib().lsort_cuda_dist_histogram(self.ctx._h, C.c_void_p(keys.data_ptr()), keys.numel(),
                                               _key_kind_of(keys), C.byref(h), e.ctypes.data_as(C.c_void_p),
                                               C.c_void_p(hist.data_ptr()))
        self._check(rc)
        return hist

    def partition(self, keys, P, buckets: int, bounds: np.ndarray):
        import ctypes as C
        import torch
        from . import _native as N
        from . import _key_kind_of, unpack_rmi
        h, e = unpack_rmi(P, buckets)
        world = bounds.size - 1
        out = torch.empty(max(keys.numel(), 1), dtype=torch.int64, device=keys.device)
        counts = np.zeros(world, np.uint64)
        b = np.ascontiguousarray(bounds, dtype=np.uint32)
        self.ctx._sync_stream()
        rc = N.lib().lsort_cuda_dist_partition(self.ctx._h, C.c_void_p(keys.data_ptr()), keys.numel(),
                                               _key_kind_of(keys), C.byref(h), e.ctypes.data_as(C.c_void_p),
                                               b.ctypes.data_as(C.c_void_p), world, C.c_void_p(out.data_ptr()),
                                               counts.ctypes.data_as(C.c_void_p))
        self._check(rc)
        return out[: keys.numel()], [int(c) for c in counts]

    def local_sort(self, keys_u64, cfg, to_f64: bool = False, forward=None):
        # to_f64: the decode is fused into the local sort's final stores.
        # forward = (P, buckets, b_lo, b_hi, sorted global sample): the local root
        # level reuses the global model restricted to this rank's buckets
        if forward is not None:
            P, buckets, b_lo, b_hi, sample = forward
            if b_hi > b_lo:
                return self.ctx.sort_forward(keys_u64, P, buckets, b_lo, b_hi, sample, cfg, encoded_f64=to_f64)
        return self.ctx.sort(keys_u64, cfg, encoded_f64=to_f64)

    bucket_major = True  # partition_buckets / copy_runs / sort_buckets below

    def partition_buckets(self, keys, P, buckets: int):
        """Level-0 scatter by bucket (identity bucket -> "rank" map): bucket-major
        output (reuses the histogram's ids; cursors scanned on the device, so no
        counts come back -- the caller has the histograms)."""
        import ctypes as C
        import torch
        from . import _native as N
        from . import _key_kind_of, unpack_rmi
        h, e = unpack_rmi(P, buckets)
        out = torch.empty(max(keys.numel(), 1), dtype=torch.int64, device=keys.device)
        b = np.arange(buckets + 1, dtype=np.uint32)
        self.ctx._sync_stream()
        rc = N.lib().lsort_cuda_dist_partition(self.ctx._h, C.c_void_p(keys.data_ptr()), keys.numel(),
                                               _key_kind_of(keys), C.byref(h), e.ctypes.data_as(C.c_void_p),
                                               b.ctypes.data_as(C.c_void_p), buckets, C.c_void_p(out.data_ptr()),
                                               None)
        self._check(rc)
        return out[: keys.numel()], None

    def copy_runs(self, src, dst, runs):
        self.ctx.copy_runs(src, dst, runs)

    def sort_buckets(self, keys_u64, P, buckets, b_lo, b_hi, sizes, sample, cfg, to_f64=False):
        return self.ctx.sort_buckets(keys_u64, P, buckets, b_lo, b_hi, sizes, sample, cfg, encoded_f64=to_f64)

    def decode(self, keys_u64):
        import ctypes as C
        from . import _native as N
        self.ctx._sync_stream()
        self._check(N.lib().lsort_cuda_decode_inplace(self.ctx._h, C.c_void_p(keys_u64.data_ptr()),
                                                      keys_u64.numel()))
        return keys_u64.view(__import__("torch").float64)

    def _check(self, rc):
        from . import _check
        _check(self.ctx, rc)


@dataclass
class DistStats:
    n_in: int = 0
    n_out: int = 0
    sample: int = 0
    send_counts: tuple = ()
    bounds: tuple = ()
    local: dict | None = None


class DistSorter:
    """Globally sort per-rank shards. ``keys``: contiguous tensor (float64 or
    int64/uint64 bits) on this rank's device (or CPU with CPU ops)."""

    def __init__(self, ctx=None, cfg=None, group=None, ops=None, buckets: int = 1024):
        from . import SortConfig
        self.cfg = cfg or SortConfig()
        self.group = group
        self.ops = ops or NativeOps(ctx)
        self.buckets = buckets

    def sort(self, keys):
        import torch
        import torch.distributed as dist
        g = self.group
        rank, world = dist.get_rank(g), dist.get_world_size(g)
        import os
        import time
        trace = bool(os.environ.get("LSORT_DIST_TRACE")) and keys.is_cuda
        sync_at = set(filter(None, os.environ.get("LSORT_DIST_SYNC", "").split(",")))
        marks = []

        def mark(name):
            if trace or name in sync_at:
                torch.cuda.synchronize()
            elif "cur:" + name in sync_at:
                torch.cuda.current_stream().synchronize()
            if trace:
                marks.append((name, time.perf_counter()))

        mark("start")
        dev = keys.device
        is_f64 = keys.dtype == torch.float64
        n_local = keys.numel()
        # ---- 1. sample shares
        sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([n_local], dtype=torch.int64, device=dev), group=g)
        n_all = [int(t.item()) for t in sizes]
        N = sum(n_all)
        s_total = max(2, min(int(math.ceil(self.cfg.sample_fraction * N)), self.cfg.rmi_sample_cap))
        shares = sample_shares(n_all, s_total)
        seed = splitmix64(self.cfg.seed ^ splitmix64(0x6A09E667F3BCC908 + rank))
        mine = self.ops.sample(keys, shares[rank], seed)
        # ---- 2. all_gather samples (pad to the max share), identical global sample
        smax = max(shares)
        pad = torch.zeros(max(smax, 1), dtype=torch.int64, device=dev)
        pad[: mine.numel()] = mine
        gathered = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(gathered, pad, group=g)
        sample = torch.cat([gathered[r][: shares[r]] for r in range(world)]).contiguous()
        mark("sample+gather")
        P = self.ops.train(sample, self.buckets)
        mark("train")
        # ---- 3. global histogram
        hist = self.ops.histogram(keys, P, self.buckets).to(torch.int64)
        mark("histogram")
        if getattr(self.ops, "bucket_major", False):
            return self._sort_bucket_major(keys, P, hist, sample, s_total, n_local, is_f64, mark, marks, trace)
        dist.all_reduce(hist, group=g)
        # ---- 4. rank boundaries
        bounds = rank_bounds(hist.cpu().numpy(), world)
        # ---- 5. partition + exchange
        mark("allreduce+bounds")
        part, send = self.ops.partition(keys, P, self.buckets, bounds)
        mark("partition")
        send_t = torch.tensor(send, dtype=torch.int64, device=dev)
        recv_t = torch.empty(world, dtype=torch.int64, device=dev)
        dist.all_to_all_single(recv_t, send_t, group=g)
        recv = [int(x) for x in recv_t.cpu().tolist()]
        out = torch.empty(max(sum(recv), 1), dtype=torch.int64, device=dev)[: sum(recv)]
        dist.all_to_all_single(out, part, output_split_sizes=recv, input_split_sizes=send, group=g)
        mark("exchange")
        # ---- 6. local sort of encoded keys, decode
        from . import SortConfig
        lcfg = SortConfig(**{**self.cfg.__dict__})
        fused = is_f64 and getattr(self.ops, "fused_decode", False)
        if fused:  # native ops: forwarded root model + fused decode
            fwd = (P, self.buckets, int(bounds[rank]), int(bounds[rank + 1]), sample)
            local = self.ops.local_sort(out, lcfg, to_f64=True, forward=fwd)
        elif getattr(self.ops, "fused_decode", False):
            fwd = (P, self.buckets, int(bounds[rank]), int(bounds[rank + 1]), sample)
            local = self.ops.local_sort(out, lcfg, forward=fwd) if out.numel() else {}
        else:
            local = self.ops.local_sort(out, lcfg) if out.numel() else {}
        mark("local sort")
        if fused:
            result = out.view(torch.float64)
        else:
            result = self.ops.decode(out) if is_f64 else out
        mark("decode")
        if trace and rank == 0:
            print("[dist] " + " ".join(f"{marks[i][0]} {1e3 * (marks[i][1] - marks[i - 1][1]):.3f}"
                                     for i in range(1, len(marks))) + " ms", flush=True)
        stats = DistStats(n_in=n_local, n_out=int(out.numel()), sample=s_total, send_counts=tuple(send),
                          bounds=tuple(int(b) for b in bounds), local=local)
        return result, stats.__dict__

    def _sort_bucket_major(self, keys, P, hist, sample, s_total, n_local, is_f64, mark, marks, trace):
        """Steps 3-6 with a bucket-major exchange: every rank scatters its keys by
        bucket (not just by destination), the per-rank histograms are all-gathered
        (instead of all-reduced) so each rank knows where every (source, bucket)
        piece lands, the all-to-all's source-major receive buffer is regrouped by
        bucket with one run-gather copy (nothing to do at one rank), and the local
        sort starts at level 1 with the rank's buckets as its segments -- no second
        level-0 classify + scatter."""
        import torch
        import torch.distributed as dist
        g = self.group
        rank, world = dist.get_rank(g), dist.get_world_size(g)
        dev = keys.device
        hists = [torch.empty_like(hist) for _ in range(world)]
        dist.all_gather(hists, hist, group=g)
        H = torch.stack(hists).cpu().numpy()
        bounds = rank_bounds(H.sum(axis=0), world)
        mark("allreduce+bounds")
        part, _ = self.ops.partition_buckets(keys, P, self.buckets)
        mark("partition")
        send, recv, runs, sizes = bucket_exchange_plan(H, bounds, rank)
        if world == 1:  # nothing to exchange: the partition is already bucket-major
            out = part
        else:
            out = torch.empty(max(sum(recv), 1), dtype=torch.int64, device=dev)[: sum(recv)]
            dist.all_to_all_single(out, part, output_split_sizes=recv, input_split_sizes=send, group=g)
        if world > 1 and runs.shape[0] > 1:
            grouped = torch.empty_like(out)
            self.ops.copy_runs(out, grouped, runs)
            out = grouped
        mark("exchange")
        from . import SortConfig
        lcfg = SortConfig(**{**self.cfg.__dict__})
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        fused = is_f64 and getattr(self.ops, "fused_decode", False)
        local = (self.ops.sort_buckets(out, P, self.buckets, lo, hi, sizes, sample, lcfg, to_f64=fused)
                 if out.numel() else {})
        mark("local sort")
        if fused:
            result = out.view(torch.float64)
        else:
            result = self.ops.decode(out) if is_f64 else out
        mark("decode")
        if trace and rank == 0:
            print("[dist] " + " ".join(f"{marks[i][0]} {1e3 * (marks[i][1] - marks[i - 1][1]):.3f}"
                                     for i in range(1, len(marks))) + " ms", flush=True)
        stats = DistStats(n_in=n_local, n_out=int(out.numel()), sample=s_total, send_counts=tuple(send),
                          bounds=tuple(int(b) for b in bounds), local=local)
        return result, stats.__dict__
