"""Multi-GPU LearnedSort: the Python front end of the library's multi-GPU driver.

One process per GPU. Each rank holds a shard; after ``sort`` rank r holds the
r-th key range of the global sorted order (variable length), so the
concatenation over ranks is the sorted input.

``DistContext`` is one rank of the C++ driver (liblsort_cuda.so, csrc/dist.cu,
``lsort_cuda_sort_dist``): the library owns its NCCL communicator (rank 0's
unique id is broadcast over the caller's torch.distributed group) and runs
the whole sort -- global sample, global partition model (RMI, or a splitter
tree when the RMI cannot balance the ranks), all-gathered level-0 histograms,
rank cuts, the exchange fused into the level-0 scatter as NVLink stores into
the owners' receive buffers, and the local sort from level 1.

``DistSorter(ops=...)`` is a host-logic mirror of the same steps for tests:
torch.distributed collectives (gloo on CPU) around CPU stand-ins of the device
steps, sharing the driver's C++ rank plan (``lsort_dist_plan``). The product
path never uses it (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N


def splitmix64(x: int) -> int:
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def rank_seed(seed: int, rank: int) -> int:
    """The per-rank sampling stream of the driver (dist.cu step 2)."""
    return splitmix64(seed ^ splitmix64((0x6A09E667F3BCC908 + rank) & ((1 << 64) - 1)))


def sample_size(frac: float, cap: int, n: int) -> int:
    """SPEC.md:438 rmi sample size (engine sample_size_host)."""
    return max(2, int(math.ceil(min(frac * n, float(cap)))))


def sample_shares(n_local: list[int], s_total: int) -> list[int]:
    """Per-rank sample sizes proportional to shard sizes (sum == s_total), as dist.cu share_of."""
    Nt = sum(n_local)
    if Nt == 0:
        return [0] * len(n_local)
    shares = [s_total * n // Nt for n in n_local]
    tot = sum(shares)
    i = 0
    while tot < s_total:
        if n_local[i]:
            shares[i] += 1
            tot += 1
        i = (i + 1) % len(n_local)
    return [min(s, n) for s, n in zip(shares, n_local)]


def dist_plan(H: np.ndarray, eq: np.ndarray | None, rank: int) -> dict:
    """The driver's rank plan (C++ lsort_dist_plan, identical on every rank):
    cuts in global sorted positions (bucket boundaries, or anywhere inside an
    equality bucket), keys per rank, per-bucket owner / offset of this rank's
    keys in the owner's receive buffer, and this rank's received pieces
    (bucket, local offset, count)."""
    H = np.ascontiguousarray(np.asarray(H, dtype=np.uint64))
    world, nb = H.shape
    cuts = np.zeros(world + 1, np.uint64)
    recv = np.zeros(world, np.uint64)
    dest = np.zeros(nb, np.uint32)
    off = np.zeros(nb, np.uint64)
    pieces = np.zeros((nb, 3), np.uint64)
    npc = C.c_uint32(0)
    e = None if eq is None else np.ascontiguousarray(np.asarray(eq, dtype=np.uint8))
    rc = N.lib().lsort_dist_plan(world, nb, H.ctypes.data_as(C.c_void_p),
                                 None if e is None else e.ctypes.data_as(C.c_void_p), rank,
                                 cuts.ctypes.data_as(C.c_void_p), recv.ctypes.data_as(C.c_void_p),
                                 dest.ctypes.data_as(C.c_void_p), off.ctypes.data_as(C.c_void_p),
                                 pieces.ctypes.data_as(C.c_void_p), C.byref(npc))
    if rc != N.LSORT_OK:
        raise ValueError("lsort_dist_plan: bad arguments")
    return {"cuts": cuts.astype(np.int64), "recv": recv.astype(np.int64), "dest": dest,
            "dest_off": off.astype(np.int64), "pieces": pieces[: npc.value].astype(np.int64)}


def _group_info(group):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


class DistContext:
    """One rank of the multi-GPU driver (lsort_cuda_dist_create / lsort_cuda_sort_dist)."""

    def __init__(self, device: int | None = None, group=None):
        import torch
        self.rank, self.world = _group_info(group)
        self.device = torch.cuda.current_device() if device is None else device
        L = N.lib()
        nid = None
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():  # the library's own NCCL communicator
            obj = [None]
            if self.rank == 0:
                buf = C.create_string_buffer(128)
                rc = L.lsort_nccl_unique_id(buf)
                if rc != N.LSORT_OK:
                    raise RuntimeError("NCCL unavailable for the multi-GPU driver")
                obj = [bytes(buf.raw)]
            dist.broadcast_object_list(obj, src=0, group=group)
            nid = C.create_string_buffer(obj[0], 128)
        h = C.c_void_p()
        rc = L.lsort_cuda_dist_create(C.byref(h), self.device, self.world, self.rank, nid)
        if rc != N.LSORT_OK:
            raise RuntimeError(f"lsort_cuda_dist_create failed ({rc})")
        self._h = h
        self._out = None

    def close(self):
        if getattr(self, "_h", None):
            N.lib().lsort_cuda_dist_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _err(self) -> str:
        return N.lib().lsort_cuda_dist_last_error(self._h).decode()

    def sort(self, keys, cfg=None, out=None):
        """Globally sort this rank's shard (contiguous CUDA tensor: float64,
        int64 or uint64 bits). Returns (this rank's key range as a view of
        `out` -- or of a buffer this context keeps --, stats dict)."""
        import torch
        from . import NanError, SortConfig, _key_kind_of
        if not keys.is_cuda or not keys.is_contiguous():
            raise ValueError("keys must be a contiguous CUDA tensor")
        cur = torch.cuda.current_stream(self.device)
        if not cur.cuda_stream:
            cur.synchronize()
        N.lib().lsort_cuda_dist_set_stream(self._h, C.c_void_p(cur.cuda_stream) if cur.cuda_stream else None)
        cfg_c = (cfg or SortConfig()).to_c()
        kind = _key_kind_of(keys)
        n = keys.numel()
        for _ in range(2):
            if out is None:
                if self._out is None or self._out.dtype != keys.dtype or self._out.numel() < n + n // 4 + 65536:
                    self._out = torch.empty(n + n // 4 + 65536, dtype=keys.dtype, device=keys.device)
                dst = self._out
            else:
                dst = out
            st = N.lsort_stats()
            n_out = C.c_uint64(0)
            nan = C.c_uint64(0)
            rc = N.lib().lsort_cuda_sort_dist(self._h, C.c_void_p(keys.data_ptr()), n, kind,
                                              C.c_void_p(dst.data_ptr()), dst.numel(), C.byref(n_out),
                                              C.byref(cfg_c), C.byref(st), C.byref(nan))
            if rc == N.LSORT_ENOMEM and out is None:
                # some rank's buffer was short: every rank failed alike before any
                # key moved, so every rank grows (if it was short) and repeats
                if n_out.value > dst.numel():
                    self._out = torch.empty(n_out.value + n_out.value // 8 + 65536, dtype=keys.dtype,
                                            device=keys.device)
                continue
            break
        if rc == N.LSORT_ENAN:
            raise NanError(int(nan.value) if nan.value != (1 << 64) - 1 else -1)
        if rc != N.LSORT_OK:
            if rc == N.LSORT_EINVAL:
                raise ValueError(self._err())
            from . import LsortError
            raise LsortError(rc, self._err())
        d = st.as_dict()
        d["n_in"], d["n_out"] = n, int(n_out.value)
        return dst[: n_out.value], d


class DistSorter:
    """Globally sort per-rank shards. Native (ops=None): the C++ driver through
    DistContext. With ``ops`` (tests): the driver's steps mirrored in Python
    around CPU stand-ins of the device work (see tests/dist_cpu_ops.py)."""

    def __init__(self, ctx=None, cfg=None, group=None, ops=None):
        from . import SortConfig
        self.cfg = cfg or SortConfig()
        self.group = group
        self.ops = ops
        self._dc = None
        if ops is None:
            self._dc = DistContext(getattr(ctx, "device", None), group)

    def sort(self, keys):
        if self.ops is None:
            return self._dc.sort(keys, self.cfg)
        return self._mirror(keys)

    # --------------------------------------------------- host-logic mirror
    def _mirror(self, keys):
        """dist.cu steps 1-7 with torch.distributed collectives; `ops` does the
        per-rank device work on CPU. Keys move as in the fused scatter: every
        key of a moved bucket goes to (owner, dest_off[b] + its rank within
        this source's keys of b)."""
        import torch
        import torch.distributed as dist
        from . import NanError
        g, ops, cfg = self.group, self.ops, self.cfg
        rank, world = dist.get_rank(g), dist.get_world_size(g)
        is_f64 = keys.dtype == torch.float64
        k = ops.encode(keys)
        n = k.size
        # 1. shard sizes
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([n], dtype=torch.int64), group=g)
        n_all = [int(t.item()) for t in sizes]
        Nt = sum(n_all)
        if Nt == 0:
            return keys[:0], {"n_in": 0, "n_out": 0}
        # 2. sample shares, gather
        s_total = sample_size(cfg.sample_fraction, cfg.rmi_sample_cap, Nt)
        sh = sample_shares(n_all, s_total)
        mine = ops.sample(k, sh[rank], rank_seed(cfg.seed, rank))
        smax = max(max(sh), 1)
        pad = torch.zeros(smax, dtype=torch.int64)
        pad[: mine.size] = torch.from_numpy(mine.view(np.int64))
        gathered = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(gathered, pad, group=g)
        sample = np.sort(np.concatenate([gathered[r][: sh[r]].numpy().view(np.uint64) for r in range(world)]))
        # 3. global model (identical on every rank: the same sorted sample)
        model = ops.global_model(sample, Nt, cfg, world)
        # 4. local classify + histogram; all-gather with the NaN index
        ids = model.classify(k)
        nan = ops.nan_index(keys)
        msg = torch.from_numpy(np.concatenate([np.bincount(ids, minlength=model.nb).astype(np.int64), [nan]]))
        msgs = [torch.empty_like(msg) for _ in range(world)]
        dist.all_gather(msgs, msg, group=g)
        M = np.stack([m.numpy() for m in msgs])
        bad = [r for r in range(world) if M[r, -1] >= 0]
        if bad:
            raise NanError(int(M[bad[0], -1]) if bad[0] == rank else -1)
        H = M[:, :-1]
        # 5. plan (C++)
        pl = dist_plan(H, model.eq, rank)
        # 6. exchange: every moved key to (owner, dest_off[b] + rank within b)
        order = np.argsort(ids, kind="stable")
        sid = ids[order]
        first = np.searchsorted(sid, np.arange(model.nb))
        within = np.arange(n) - first[sid]
        dest = pl["dest"][sid].astype(np.int64)
        moved = dest != 0xFFFFFFFF
        pos = pl["dest_off"][sid] + within
        send_k, send_p, counts = [], [], []
        for r in range(world):
            sel = moved & (dest == r)
            send_k.append(k[order][sel])
            send_p.append(pos[sel])
            counts.append(int(sel.sum()))
        ct = torch.tensor(counts, dtype=torch.int64)
        rct = torch.empty(world, dtype=torch.int64)
        dist.all_to_all_single(rct, ct, group=g)
        rc = [int(x) for x in rct.tolist()]
        rk = torch.empty(sum(rc), dtype=torch.int64)
        rp = torch.empty(sum(rc), dtype=torch.int64)
        dist.all_to_all_single(rk, torch.from_numpy(np.concatenate(send_k).view(np.int64)),
                               output_split_sizes=rc, input_split_sizes=counts, group=g)
        dist.all_to_all_single(rp, torch.from_numpy(np.concatenate(send_p)),
                               output_split_sizes=rc, input_split_sizes=counts, group=g)
        nr = int(pl["recv"][rank])
        buf = np.zeros(nr, np.uint64)
        filled = np.zeros(nr, bool)
        rp_n = rp.numpy()
        assert rp_n.size == 0 or (rp_n.min() >= 0 and rp_n.max() < nr), "key outside the rank's range"
        buf[rp_n] = rk.numpy().view(np.uint64)
        filled[rp_n] = True
        # 7. local: equality pieces are fills, the rest sorted per bucket
        for b, at, cnt in pl["pieces"]:
            if model.eq[b]:
                buf[at:at + cnt] = model.eqval[b]
                filled[at:at + cnt] = True
            else:
                ops.local_sort(buf[at:at + cnt], model, int(b))
        assert filled.all(), "a received position was never written"
        out = ops.decode(buf) if is_f64 else torch.from_numpy(buf.view(np.int64))
        return out, {"n_in": n, "n_out": nr, "kind": model.kind, "cuts": pl["cuts"].tolist(),
                     "recv": pl["recv"].tolist()}


def sort_emulated(shards, cfg=None, out_caps=None, device: int | None = None):
    """TEST ENTRY (lsort_cuda_dist_emulate): len(shards) virtual ranks on one
    GPU run the driver's multi-rank data path (global model, rank cuts, the
    exchange fused into the scatter, local sorts) with emulated collectives.
    Returns ([per-rank output views], [per-rank stats]); raises NanError(index
    of the first rank holding a NaN) / LsortError like the driver."""
    import torch
    from . import LsortError, NanError, SortConfig, _key_kind_of
    W = len(shards)
    kinds = {_key_kind_of(s) for s in shards}
    if len(kinds) != 1:
        raise ValueError("shards must share one key kind")
    dev = shards[0].device.index if device is None else device
    total = sum(s.numel() for s in shards)
    caps = out_caps or [total + 1] * W
    outs = [torch.empty(max(c, 1), dtype=shards[0].dtype, device=shards[0].device) for c in caps]
    P = C.c_void_p * W
    U = C.c_uint64 * W
    st = (N.lsort_stats * W)()
    n_outs, nans = U(), U()
    err = C.create_string_buffer(512)
    torch.cuda.synchronize()
    rc = N.lib().lsort_cuda_dist_emulate(dev, W, P(*[s.data_ptr() for s in shards]), U(*[s.numel() for s in shards]),
                                         kinds.pop(), P(*[o.data_ptr() for o in outs]), U(*caps), n_outs,
                                         C.byref((cfg or SortConfig()).to_c()), st, nans, err, 512)
    if rc == N.LSORT_ENAN:
        r = next(i for i in range(W) if nans[i] != (1 << 64) - 1)
        e = NanError(int(nans[r]))
        e.rank = r
        raise e
    if rc != N.LSORT_OK:
        e = LsortError(rc, err.value.decode())
        e.n_outs = [int(v) for v in n_outs]
        raise e
    return [outs[r][: n_outs[r]] for r in range(W)], [st[r].as_dict() for r in range(W)]
