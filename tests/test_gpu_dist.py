"""The multi-GPU driver (csrc/dist.cu) on one B200.

* lsort_cuda_dist_emulate: 2 / 4 / 8 virtual ranks on the one GPU run the
  driver's whole multi-rank data path -- global model, rank cuts, the exchange
  fused into the level-0 scatter (stores into the other ranks' receive
  buffers), local sorts -- with emulated collectives (host barriers; no kernel
  waits on another). The concatenation must equal numpy's sort bit for bit
  and rank loads must balance.
* DistContext: the NCCL communicator owned by the library (torch.distributed
  world 1 ships the unique id), IPC sharing, stream-ordered barrier.
* lsort_cuda_sort_buckets: keys already grouped by a model's buckets.
The multi-process host logic is covered by tests/test_dist_cpu.py (gloo)."""
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2307_08637_b200 as L  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2307_08637_b200.dist import sort_emulated  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dev(a):
    return torch.from_numpy(a if a.dtype == np.float64 else a.view(np.int64)).cuda()


def _expected(x):
    return O.decode(np.sort(O.encode(x))).view(np.uint64) if x.dtype == np.float64 else np.sort(x)


def _input(name, n):
    if name == "heavy":  # 40% one value: an equality bucket split across ranks
        rng = np.random.default_rng(5)
        a = rng.integers(0, 1 << 40, n, dtype=np.uint64)
        a[rng.random(n) < 0.4] = 123456789
        return a
    seeds = {"mixgauss": 11, "lognormal2": 19, "normal": 7, "rootdups": 3, "uniform": 42, "zipf": 3}
    return O.generate(name, n, seeds[name])


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name,n", [("mixgauss", 8_000_000), ("lognormal2", 6_000_000), ("normal", 4_000_000),
                                    ("heavy", 4_000_000), ("rootdups", 4_000_000)])
def test_dist_emulated_exact_and_balanced(world, name, n):
    x = _input(name, n)
    per = n // world
    shards = [_dev(x[r * per:(r + 1) * per if r < world - 1 else n]) for r in range(world)]
    outs, stats = sort_emulated(shards)
    got = np.concatenate([o.cpu().numpy().view(np.uint64) for o in outs])
    assert np.array_equal(got, _expected(x))
    loads = [o.numel() for o in outs]
    assert max(loads) <= 1.10 * n / world, loads
    if name == "mixgauss":
        assert stats[0]["level0_kind"] == 1, "the RMI cannot balance C3: the global model must be a tree"


def test_dist_emulated_ragged_empty_and_tiny():
    x = _input("lognormal2", 1_000_000)
    parts = [x[:600_000], x[600_000:600_000], x[600_000:600_010], x[600_010:]]  # an empty and a 10-key shard
    outs, _ = sort_emulated([_dev(p) for p in parts])
    got = np.concatenate([o.cpu().numpy().view(np.uint64) for o in outs])
    assert np.array_equal(got, _expected(x))
    for n in (0, 1, 5, 3000):  # tiny totals
        y = _input("uniform", 4 * n) if n else np.zeros(0)
        outs, _ = sort_emulated([_dev(y[r * n:(r + 1) * n]) for r in range(4)])
        got = np.concatenate([o.cpu().numpy().view(np.uint64) for o in outs])
        assert np.array_equal(got, _expected(y)), n


def test_dist_emulated_u64_extremes():
    rng = np.random.default_rng(3)
    a = np.concatenate([rng.integers(0, 2**64 - 1, 500_000, dtype=np.uint64, endpoint=True),
                        np.full(1000, 2**64 - 1, np.uint64), np.zeros(1000, np.uint64)])
    rng.shuffle(a)
    outs, _ = sort_emulated([_dev(p) for p in np.array_split(a, 3)])
    assert np.array_equal(np.concatenate([o.cpu().numpy().view(np.uint64) for o in outs]), np.sort(a))


def test_dist_emulated_nan_fails_every_rank():
    x = _input("normal", 400_000)
    parts = [p.copy() for p in np.array_split(x, 4)]
    parts[2][1234] = np.nan
    with pytest.raises(L.NanError) as e:
        sort_emulated([_dev(p) for p in parts])
    assert e.value.rank == 2 and e.value.index == 1234


def test_dist_emulated_small_output_buffer():
    x = _input("uniform", 400_000)
    shards = [_dev(p) for p in np.array_split(x, 2)]
    with pytest.raises(L.LsortError) as e:
        sort_emulated(shards, out_caps=[1000, 400_001])
    assert e.value.code == 3 and sum(e.value.n_outs) == x.size  # LSORT_ENOMEM, ranges reported


@pytest.fixture(scope="module")
def pg():
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("name,n", [("normal", 2_000_000), ("lognormal2", 3_000_000), ("rootdups", 2_000_000),
                                    ("heavy", 1_000_000)])
def test_dist_context_nccl_world1(pg, name, n):
    from paper_2307_08637_b200.dist import DistContext
    x = _input(name, n)
    dc = DistContext(0)
    for _ in range(2):  # the receive buffer registration is reused
        out, st = dc.sort(_dev(x))
        assert np.array_equal(out.cpu().numpy().view(np.uint64), _expected(x))
        assert st["n_out"] == n


@pytest.mark.parametrize("dist_name,seed,n", [("normal", 7, 2_000_000), ("lognormal2", 19, 1_000_000),
                                              ("uniform", 42, 3_000_000)])
def test_sort_buckets_from_level_one(dist_name, seed, n):
    """lsort_cuda_sort_buckets on keys grouped by a model's buckets (sub-range
    [b_lo, b_hi)): small buckets in place, the rest from level 1, decode fused."""
    x = O.generate(dist_name, n, seed)
    keys = O.encode(x)
    ctx = L.Context(0)
    sample = np.sort(keys[::100])
    B = 512
    P = ctx.rmi_train(_dev(sample), B)
    ids = O.learned_bucket(P, B, B, keys)
    order = np.argsort(ids, kind="stable")
    part = keys[order]
    hist = np.bincount(ids, minlength=B)
    starts = np.concatenate([[0], np.cumsum(hist)])
    ds = _dev(sample)
    for b_lo, b_hi in [(0, B), (100, 300), (B - 7, B)]:
        seg = _dev(part[starts[b_lo]:starts[b_hi]].copy())
        st = ctx.sort_buckets(seg, P, B, b_lo, b_hi, hist[b_lo:b_hi], ds, L.SortConfig(), encoded_f64=True)
        got = seg.view(torch.float64).cpu().numpy()
        exp = O.decode(np.sort(keys[(ids >= b_lo) & (ids < b_hi)]))
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64)), (b_lo, b_hi)
        assert st["levels"] <= 2


def test_sort_buckets_edge_cases():
    """Empty buckets, one huge bucket, zero keys, sizes that do not add up."""
    ctx = L.Context(0)
    rng = np.random.default_rng(9)
    keys = np.sort(rng.integers(0, 2**63, 600_000, dtype=np.uint64))
    B = 256
    P = ctx.rmi_train(_dev(keys[::60].copy()), B)
    sample = _dev(keys[::60].copy())
    for sizes_kind in ("real", "empties"):
        k = rng.permutation(keys)
        kid = O.learned_bucket(P, B, B, k)
        if sizes_kind == "empties":
            k = k[kid % 2 == 0]
            kid = kid[kid % 2 == 0]
        order = np.argsort(kid, kind="stable")
        part = _dev(k[order])
        ctx.sort_buckets(part, P, B, 0, B, np.bincount(kid, minlength=B), sample, L.SortConfig())
        assert np.array_equal(part.cpu().numpy().view(np.uint64), np.sort(k)), sizes_kind
    k = rng.integers(0, 2**64 - 1, 300_000, dtype=np.uint64, endpoint=True)
    t = _dev(k)
    ctx.sort_buckets(t, P, B, 3, 4, np.array([k.size]), None, L.SortConfig())
    assert np.array_equal(t.cpu().numpy().view(np.uint64), np.sort(k))
    ctx.sort_buckets(torch.empty(0, dtype=torch.int64, device="cuda"), P, B, 0, B, np.zeros(B, np.uint64), sample,
                     L.SortConfig())
    with pytest.raises(ValueError):
        ctx.sort_buckets(t, P, B, 0, 2, np.array([1, 2]), None, L.SortConfig())
