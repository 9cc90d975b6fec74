"""The distributed sort's native device steps (sample, global RMI train,
histogram, destination-major partition, local sort, decode) through the C-ABI,
with NCCL at world size 1 on one B200 (this run has one GPU; the multi-rank
host logic is covered by tests/test_dist_cpu.py with gloo)."""
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2307_08637_b200 as L  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def pg():
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("dist_name,seed", [("normal", 7), ("lognormal2", 19), ("rootdups", 3)])
def test_dist_sort_world1(pg, dist_name, seed):
    from paper_2307_08637_b200.dist import DistSorter
    x = O.generate(dist_name, 2_000_000, seed)
    t = torch.from_numpy(x if x.dtype == np.float64 else x.view(np.int64)).cuda()
    ctx = L.Context(0)
    out, st = DistSorter(ctx, L.SortConfig()).sort(t)
    got = out.cpu().numpy()
    if x.dtype == np.float64:
        exp = O.decode(np.sort(O.encode(x)))
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
    else:
        assert np.array_equal(got.view(np.uint64), np.sort(x))
    assert st["n_out"] == x.size and st["send_counts"] == (x.size,)


def test_dist_partition_destinations(pg):
    """lsort_cuda_dist_partition: destination-major output, counts per rank,
    every key routed by the bucket->rank map of the global model."""
    from paper_2307_08637_b200.dist import NativeOps, rank_bounds
    x = O.generate("uniform", 500_000, 42)
    t = torch.from_numpy(x).cuda()
    ops = NativeOps(L.Context(0))
    keys = O.encode(x)
    sample = torch.from_numpy(np.sort(keys[::50]).view(np.int64)).cuda()
    P = ops.train(sample.clone(), 512)
    hist = ops.histogram(t, P, 512).cpu().numpy()
    bounds = rank_bounds(hist, 4)
    part, counts = ops.partition(t, P, 512, bounds)
    assert sum(counts) == x.size
    ids = O.learned_bucket(P, 512, 512, keys)
    dest = np.searchsorted(bounds, ids, side="right") - 1
    assert counts == [int(c) for c in np.bincount(dest, minlength=4)]
    got = part.cpu().numpy().view(np.uint64)
    off = 0
    for r in range(4):
        seg = got[off:off + counts[r]]
        assert np.array_equal(np.sort(seg), np.sort(keys[dest == r]))
        off += counts[r]


@pytest.mark.parametrize("dist_name,seed,n", [("normal", 7, 2_000_000), ("lognormal2", 19, 1_000_000),
                                              ("uniform", 42, 3_000_000)])
def test_sort_buckets_from_level_one(dist_name, seed, n):
    """lsort_cuda_sort_buckets on a bucket-major level-0 partition (identity
    bucket map) of a sub-range [b_lo, b_hi) of the buckets: small buckets in
    place, the rest from level 1, decode fused -- equals the sorted keys."""
    from paper_2307_08637_b200.dist import NativeOps
    x = O.generate(dist_name, n, seed)
    keys = O.encode(x)
    ctx = L.Context(0)
    ops = NativeOps(ctx)
    t = torch.from_numpy(x).cuda()
    sample = torch.from_numpy(np.sort(keys[::100]).view(np.int64)).cuda()
    B = 512
    P = ops.train(sample.clone(), B)
    hist = ops.histogram(t, P, B).cpu().numpy()
    part, _ = ops.partition_buckets(t, P, B)  # cursors scanned on the device
    starts = np.concatenate([[0], np.cumsum(hist)])
    for b_lo, b_hi in [(0, B), (100, 300), (B - 7, B)]:
        seg = part[starts[b_lo]:starts[b_hi]].clone()
        st = ops.sort_buckets(seg, P, B, b_lo, b_hi, hist[b_lo:b_hi], sample, L.SortConfig(), to_f64=True)
        got = seg.view(torch.float64).cpu().numpy()
        ids = O.learned_bucket(P, B, B, keys)
        exp = O.decode(np.sort(keys[(ids >= b_lo) & (ids < b_hi)]))
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64)), (b_lo, b_hi)
        assert st["levels"] <= 2


def test_sort_buckets_edge_cases():
    """Empty buckets, only small buckets (no level 1), one huge bucket, u64 keys,
    zero keys; copy_runs with no runs and with overlapping-free reversals."""
    from paper_2307_08637_b200.dist import NativeOps
    ctx = L.Context(0)
    ops = NativeOps(ctx)
    rng = np.random.default_rng(9)
    keys = np.sort(rng.integers(0, 2**63, 600_000, dtype=np.uint64))
    sample = torch.from_numpy(keys[::60].copy().view(np.int64)).cuda()
    B = 256
    P = ops.train(sample.clone(), B)
    ids = O.learned_bucket(P, B, B, keys)
    for sizes_kind in ("real", "empties"):
        k = rng.permutation(keys)
        kid = O.learned_bucket(P, B, B, k)
        if sizes_kind == "empties":  # drop every other bucket's keys
            k = k[kid % 2 == 0]
            kid = kid[kid % 2 == 0]
        order = np.argsort(kid, kind="stable")
        part = torch.from_numpy(k[order].view(np.int64)).cuda()
        sizes = np.bincount(kid, minlength=B)
        ops.sort_buckets(part, P, B, 0, B, sizes, sample, L.SortConfig())
        assert np.array_equal(part.cpu().numpy().view(np.uint64), np.sort(k)), sizes_kind
    # one huge bucket of random keys (the model is not asked to be right)
    k = rng.integers(0, 2**64 - 1, 300_000, dtype=np.uint64, endpoint=True)
    t = torch.from_numpy(k.view(np.int64)).cuda()
    ops.sort_buckets(t, P, B, 3, 4, np.array([k.size]), None, L.SortConfig())
    assert np.array_equal(t.cpu().numpy().view(np.uint64), np.sort(k))
    # zero keys
    ops.sort_buckets(torch.empty(0, dtype=torch.int64, device="cuda"), P, B, 0, B, np.zeros(B, np.uint64), sample,
                     L.SortConfig())
    with pytest.raises(ValueError):  # sizes must add up to n
        ops.sort_buckets(t, P, B, 0, 2, np.array([1, 2]), None, L.SortConfig())
    # copy_runs: none, and pieces swapped
    src = torch.arange(10, dtype=torch.int64, device="cuda")
    dst = torch.zeros(10, dtype=torch.int64, device="cuda")
    ctx.copy_runs(src, dst, np.zeros((0, 3), np.uint64))
    assert int(dst.sum()) == 0
    ctx.copy_runs(src, dst, np.array([[0, 6, 4], [4, 0, 6]], np.uint64))
    assert dst.cpu().tolist() == [4, 5, 6, 7, 8, 9, 0, 1, 2, 3]
