"""Multi-rank host logic of the distributed sort (paper_2307_08637_b200/dist.py)
on CPU with gloo, world sizes 2 and 3: the concatenation of the per-rank
outputs in rank order must equal the sorted input (bit-exact), every rank's
range must be ordered w.r.t. its neighbours, and the split arithmetic must
be consistent."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_08637_b200.dist import rank_bounds, sample_shares, splitmix64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dist_name, n_per, out_dir, bucket_major=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from dist_cpu_ops import CpuOps, CpuOpsRankMajor
    from paper_2307_08637_b200 import SortConfig
    from paper_2307_08637_b200.dist import DistSorter
    total = n_per * world
    full = O.generate(dist_name, total, {"normal": 7, "lognormal2": 19, "uniform": 42, "zipf": 3}[dist_name])
    shard = full[rank * n_per:(rank + 1) * n_per].copy()
    if rank == world - 1:  # ragged shards
        shard = shard[: n_per // 2]
    t = torch.from_numpy(shard if shard.dtype == np.float64 else shard.view(np.int64))
    sorter = DistSorter(cfg=SortConfig(sample_fraction=0.05), ops=CpuOps() if bucket_major else CpuOpsRankMajor(),
                        buckets=256)
    out, st = sorter.sort(t)
    np.save(os.path.join(out_dir, f"out{rank}.npy"), out.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("bucket_major", [True, False], ids=["bucket_major", "rank_major"])
@pytest.mark.parametrize("world,dist_name", [(2, "normal"), (3, "lognormal2"), (2, "zipf")])
def test_distributed_sort_gloo(tmp_path, world, dist_name, bucket_major):
    n_per = 6000
    port = _free_port()
    mp.spawn(_worker, args=(world, port, dist_name, n_per, str(tmp_path), bucket_major), nprocs=world, join=True)
    from oracle import oracle as O
    seed = {"normal": 7, "lognormal2": 19, "uniform": 42, "zipf": 3}[dist_name]
    full = O.generate(dist_name, n_per * world, seed)
    parts = [full[r * n_per:(r + 1) * n_per] for r in range(world)]
    parts[-1] = parts[-1][: n_per // 2]
    data = np.concatenate(parts)
    outs = [np.load(tmp_path / f"out{r}.npy") for r in range(world)]
    got = np.concatenate(outs)
    if data.dtype == np.float64:
        exp = O.decode(np.sort(O.encode(data)))
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
    else:
        assert np.array_equal(got.view(np.uint64), np.sort(data))
    assert sum(o.size for o in outs) == data.size


def test_rank_bounds_and_shares():
    h = np.array([5, 0, 10, 3, 2, 0, 0, 30, 1, 1])
    for world in (1, 2, 3, 4, 8):
        b = rank_bounds(h, world)
        assert b[0] == 0 and b[-1] == h.size and np.all(np.diff(b.astype(np.int64)) >= 0)
        assert b.size == world + 1
    b = rank_bounds(np.ones(1024, np.int64), 4)
    assert list(b) == [0, 256, 512, 768, 1024]
    assert sum(sample_shares([100, 50, 0, 25], 70)) == 70
    assert sample_shares([100, 50, 0, 25], 70)[2] == 0
    assert splitmix64(0) == 0xE220A8397B1DCDAF


def test_bucket_exchange_plan():
    """Runs regroup the source-major receive buffer by bucket; sizes and counts add up."""
    from paper_2307_08637_b200.dist import bucket_exchange_plan
    rng = np.random.default_rng(3)
    for world in (1, 2, 3, 5):
        B = 64
        H = rng.integers(0, 7, (world, B))
        H[:, 5] = 0  # an empty bucket
        bounds = rank_bounds(H.sum(axis=0), world)
        sends = [bucket_exchange_plan(H, bounds, r)[0] for r in range(world)]
        for r in range(world):
            send, recv, runs, sizes = bucket_exchange_plan(H, bounds, r)
            assert recv == [sends[s][r] for s in range(world)]
            lo, hi = bounds[r], bounds[r + 1]
            assert np.array_equal(sizes, H[:, lo:hi].sum(axis=0))
            # simulate: source s sends its keys of my buckets bucket-major, tagged (bucket, s)
            buf = []
            for s_ in range(world):
                for b in range(lo, hi):
                    buf += [(b, s_)] * int(H[s_, b])
            dst = [None] * len(buf)
            for so, do, ln in runs.astype(np.int64):
                dst[do:do + ln] = buf[so:so + ln]
            assert dst == sorted(buf)  # bucket-major, sources in rank order inside a bucket
