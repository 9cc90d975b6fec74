"""GPU parity tests: the CUDA path (through the C-ABI) against the oracle.

Bit-exact bar: sample sorts, bucket ids and histograms given identical model
parameters, tree builds, duplicate fractions, and every final sorted array.
RMI training on the GPU uses deterministic parallel sums for the root fit and
for slices > 512 samples, so its parameters are compared with a tolerance
(stated below); slices <= 512 samples are fitted sequentially and must match
the reference bit for bit.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2307_08637_b200 as L  # noqa: E402
from oracle import oracle as O  # noqa: E402
from lsort_testutil import golden_cases  # noqa: E402

RMI_RTOL = 1e-9   # relative tolerance on GPU-trained RMI parameters (parallel sums)
RMI_ATOL = 1e-12  # absolute floor for parameters that cancel to ~0 (e.g. intercepts)


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return L.Context(0)


def dev(a: np.ndarray):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        return torch.from_numpy(a.view(np.int64)).cuda()
    return torch.from_numpy(a).cuda()


def host_u64(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def route_defined(P, B, keys):
    with np.errstate(all="ignore"):
        xn = (np.asarray(keys, np.uint64).astype(np.float64) - P[2]) * P[3]
        t = (P[0] * xn + P[1]) * float(B)
        return ~(t >= 2.0 ** 64)


# ------------------------------------------------------------ block sort
def test_block_sort_limit(ctx):
    with pytest.raises(ValueError):
        ctx.block_sort(dev(np.arange(8193, dtype=np.uint64)))


@pytest.mark.parametrize("n", [2, 3, 17, 100, 1000, 4096, 8191, 8192])
def test_block_sort(ctx, n):
    rng = np.random.default_rng(n)
    for a in [rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True),
              rng.integers(0, 7, n, dtype=np.uint64),
              np.full(n, 5, np.uint64),
              np.sort(rng.integers(0, 1000, n, dtype=np.uint64))[::-1].copy(),
              (rng.integers(0, 3, n, dtype=np.uint64) << np.uint64(60)) + rng.integers(0, 50, n, dtype=np.uint64)]:
        d = dev(a)
        ctx.block_sort(d)
        assert np.array_equal(host_u64(d), np.sort(a))


# -------------------------------------------------- classification parity
def test_classify_rmi_golden(ctx, golden):
    for case in golden_cases(golden, "rmi"):
        P, B = golden[f"rmi/{case}/P"], int(golden[f"rmi/{case}/B"][0])
        pr = golden[f"rmi/{case}/probe"]
        ok = route_defined(P, B, pr)
        for bc, key, lo, hi in [(B, "bucket", 0.0, 1.0), (1000, "bucket1000", 0.0, 1.0),
                                (256, "bucket_sub", 0.25, 0.75)]:
            ids, hist = ctx.classify_rmi(P, B, bc, dev(pr), lo, hi)
            got = ids.cpu().numpy().astype(np.uint32)
            exp = golden[f"rmi/{case}/{key}"]
            assert np.array_equal(got[ok], exp[ok]), (case, key)
            assert np.array_equal(np.bincount(got, minlength=bc), hist.cpu().numpy()), (case, key)


@pytest.mark.parametrize("dist,seed", [("uniform", 42), ("normal", 7), ("mixgauss", 11),
                                       ("lognormal2", 19), ("exponential2", 7)])
def test_classify_rmi_large_exact(ctx, dist, seed):
    """1e6 keys under an oracle-trained 1024-submodel RMI: ids + histogram exact."""
    x = O.generate(dist, 1_000_000, seed)
    k = O.encode(x)
    s = np.sort(k[:: 97])
    P = O.rmi_train(s, 1024)
    exp = O.learned_bucket(P, 1024, 1024, k[:20000])
    ids, hist = ctx.classify_rmi(P, 1024, 1024, dev(x))  # f64 input: fused encode
    got = ids.cpu().numpy().astype(np.uint32)
    assert np.array_equal(got[:20000], exp)
    # histogram of all keys equals bincount of the ids (device-consistent)
    assert np.array_equal(np.bincount(got, minlength=1024), hist.cpu().numpy())


def test_classify_tree_golden(ctx, golden):
    for case in golden_cases(golden, "tree"):
        s = golden[f"tree/{case}/sample"]
        k, eq = int(golden[f"tree/{case}/k"][0]), int(golden[f"tree/{case}/eq"][0])
        t = O.tree_build(s, k, bool(eq))
        tt = L._native.lsort_tree.from_buffer_copy(bytes(t))
        ids, hist = ctx.classify_tree(tt, dev(golden[f"tree/{case}/probe"]))
        assert np.array_equal(ids.cpu().numpy().astype(np.uint32), golden[f"tree/{case}/bucket"]), case


# ---------------------------------------------------------- model building
def test_tree_build_golden(ctx, golden):
    for case in golden_cases(golden, "tree"):
        s = golden[f"tree/{case}/sample"]
        if s.size > 16384:
            continue
        k, eq = int(golden[f"tree/{case}/k"][0]), int(golden[f"tree/{case}/eq"][0])
        t = ctx.tree_build(dev(s), k, bool(eq))
        m = t.nsplitters
        assert np.array_equal(np.array(t.splitters[:m], np.uint64), golden[f"tree/{case}/splitters"]), case
        heavy = np.array([t.eq_offset[i + 1] - t.eq_offset[i] > 1 for i in range(m)], np.uint8)
        assert np.array_equal(heavy, golden[f"tree/{case}/heavy"]), case
        assert t.bucket_count == int(golden[f"tree/{case}/bucket_count"][0]), case
        ot = O.tree_build(s, k, bool(eq))
        assert bytes(t) == bytes(ot), case  # whole POD incl. implicit heap


def compare_rmi(Pg, Pr, B, s):
    """GPU-trained vs reference-trained RMI on the same sorted sample `s`.

    The GPU's root fit sums in a deterministic parallel order, so the root is
    compared with RMI_RTOL/RMI_ATOL. Everything downstream of the root is then
    checked against the reference algorithm run under the GPU's root
    (oracle.rmi_train_given_root): slices of <= 512 samples are fitted
    sequentially on the GPU and must match bit for bit; larger slices use a
    warp-parallel sum and must match within RMI_RTOL."""
    assert np.allclose(Pg[:4], Pr[:4], rtol=RMI_RTOL, atol=RMI_ATOL), "root"
    assert np.array_equal(bits(Pg[2:4]), bits(Pr[2:4])), "key_base/key_scale are exact"
    Pq = O.rmi_train_given_root(s, B, Pg[0], Pg[1])
    E, Eq = Pg[4:].reshape(B, 4), Pq[4:].reshape(B, 4)
    xn = (s.astype(np.float64) - Pg[2]) * Pg[3]
    t = (Pg[0] * xn + Pg[1]) * float(B)
    route = np.where(~(t > 0), 0, np.minimum(np.floor(np.where(t > 0, t, 0)), B - 1)).astype(np.int64)
    sizes = np.bincount(route, minlength=B)
    seq = sizes <= 512
    # slope/intercept of sequentially fitted slices are bit-exact; clamp bounds
    # propagate neighbours' values (running max/min, models.cpp:110-113), so
    # they inherit the tolerance of any warp-fitted neighbour
    # (empty submodels take the midpoint of their clamp range, models.cpp:124-126,
    # which is neighbour-dependent as well)
    bad = np.nonzero(seq & (sizes > 0) & np.any(bits(E[:, :2]) != bits(Eq[:, :2]), axis=1))[0]
    assert bad.size == 0, ("sequential slice fits differ", bad[:8], sizes[bad[:8]], E[bad[:4]], Eq[bad[:4]])
    if seq.all():
        assert np.array_equal(bits(E), bits(Eq)), "all-sequential model must be bit-exact"
    assert np.allclose(E, Eq, rtol=RMI_RTOL, atol=RMI_ATOL), "parallel slices / clamp bounds"


def _fanout(n, count, target):
    if target == 0:
        return count
    want = -(-n // target)
    b = 2
    while b < want and b < count:
        b <<= 1
    return min(b, count)


@pytest.mark.parametrize("dist,seed,n", [("uniform", 42, 2_000_000), ("normal", 7, 300_000),
                                         ("rootdups", 3, 1_000_000), ("zipf", 3, 500_000),
                                         ("uniform", 42, 50_000), ("twodups", 3, 400_000),
                                         ("lognormal2", 19, 5_000_000)])
def test_build_model_alg5(ctx, dist, seed, n):
    """Alg. 5 policy on the same device-drawn samples as the
    oracle: decision and duplicate fraction exact, trees bit-exact, learned
    models within RMI_RTOL of the reference-exact oracle training."""
    x = O.generate(dist, n, seed)
    keys = O.encode(x) if x.dtype == np.float64 else x
    cfg = L.SortConfig()
    m = ctx.build_model(dev(x), cfg)
    rb = _fanout(n, cfg.rmi_bucket_count, cfg.bucket_target)
    tk = _fanout(n, cfg.tree_bucket_count, cfg.bucket_target)
    kind, P, t, dup = O.build_partition_model(keys, 0, 0, O.cfg(seed=cfg.seed), rb, tk)
    assert m["kind"] == kind
    assert m["dup"] == dup
    if kind == 1:
        assert bytes(m["tree"]) == bytes(t)
    else:
        assert m["B"] == rb
        s2 = np.sort(keys[[O.lib().lso_rng_below(O.lib().lso_seg_seed(cfg.seed, 0, 0), m["s1"] + j, n)
                           for j in range(m["s2"])]])
        compare_rmi(m["P"], P, rb, s2)


# --------------------------------------------------------------- full sort
def check_sorted_f64(x, got):
    exp = O.decode(np.sort(O.encode(x)))
    assert np.array_equal(bits(got), bits(exp))


@pytest.mark.parametrize("dist,seed", [("uniform", 42), ("normal", 7), ("lognormal05", 7),
                                       ("exponential2", 7), ("mixgauss", 11), ("lognormal2", 19)])
@pytest.mark.parametrize("n", [1000, 16384, 16385, 100_000, 1_000_000, 3_000_000])
def test_sort_f64_generators(ctx, dist, seed, n):
    x = O.generate(dist, n, seed)
    d = dev(x)
    ctx.sort(d)
    check_sorted_f64(x, d.cpu().numpy())


@pytest.mark.parametrize("dist", ["rootdups", "twodups", "zipf"])
@pytest.mark.parametrize("n", [5000, 200_000, 2_000_000])
def test_sort_u64_dups(ctx, dist, n):
    a = O.generate(dist, n, 3)
    d = dev(a)
    st = ctx.sort(d)
    assert np.array_equal(host_u64(d), np.sort(a))
    if n >= 2_000_000 and dist == "zipf":
        assert st["fill_keys"] > 0  # heavy ranks 1-2 (>1/256 of the sample) -> equality buckets


def test_sort_heavy_hitters(ctx):
    """Equality buckets (models.cpp:155-163): heavy splitters are filled, not moved."""
    rng = np.random.default_rng(4)
    n = 1_000_000
    a = rng.integers(0, 1 << 40, n, dtype=np.uint64)
    a[rng.random(n) < 0.3] = 123456789
    a[rng.random(n) < 0.1] = 2**64 - 1
    d = dev(a)
    st = ctx.sort(d)
    assert np.array_equal(host_u64(d), np.sort(a))
    assert st["fill_keys"] >= 0.35 * n


@pytest.mark.parametrize("case", ["top_of_range", "dense_low_cells", "skewed_cells", "two_ends"])
def test_sort_tree_lookup_table(ctx, case):
    """Radix-assisted splitter lookup (partition.cu kstate_load<kTree>): cells of
    the splitter range, saturation near 2^64, cells holding many splitters
    (tree descent fallback) -- duplicate-heavy inputs so the trees are used."""
    rng = np.random.default_rng(11)
    n = 3_000_000
    top = np.uint64(2**64 - 1)
    if case == "top_of_range":
        a = top - rng.integers(0, 5000, n, dtype=np.uint64)
    elif case == "dense_low_cells":
        a = rng.integers(0, 3000, n, dtype=np.uint64) * np.uint64(1 << 40)
    elif case == "skewed_cells":  # many distinct splitters in the first cells, sparse above
        a = np.where(rng.random(n) < 0.7, rng.integers(0, 600, n), rng.integers(0, 1 << 50, n)).astype(np.uint64)
        a[rng.random(n) < 0.2] = 5
    else:  # both branches uint64 (an int64 / uint64 mix would promote to float64)
        a = np.where(rng.random(n) < 0.5, rng.integers(0, 2000, n, dtype=np.uint64),
                     top - rng.integers(0, 2000, n, dtype=np.uint64))
        assert a.dtype == np.uint64 and np.unique(a[a > (top >> np.uint64(1))]).size == 2000
    d = dev(a)
    st = ctx.sort(d)
    assert st["level0_kind"] == 1, "expected a splitter tree at level 0"
    assert np.array_equal(host_u64(d), np.sort(a))


def test_sort_adversarial(ctx):
    n = 300_000
    rng = np.random.default_rng(1)
    cases = {
        "sorted": np.arange(n, dtype=np.uint64),
        "reversed": np.arange(n, dtype=np.uint64)[::-1].copy(),
        "all_equal": np.full(n, 42, np.uint64),
        "organ_pipe": np.concatenate([np.arange(n // 2), np.arange(n // 2)[::-1]]).astype(np.uint64),
        "near_constant": np.where(rng.random(n) < 1e-4, 7, 5).astype(np.uint64),
        "wide": rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True),
        "two_clusters": np.concatenate([rng.integers(0, 100, n // 2), rng.integers(2**63, 2**63 + 100, n // 2,
                                                                                   dtype=np.uint64)]).astype(np.uint64),
        "outliers": np.where(rng.random(n) < 1e-3, 2**64 - 1, rng.integers(0, 1 << 20, n)).astype(np.uint64),
    }
    for name, a in cases.items():
        d = dev(a)
        ctx.sort(d)
        assert np.array_equal(host_u64(d), np.sort(a)), name


def test_sort_small_and_special(ctx):
    for n in [0, 1, 2, 3, 31, 1025]:
        a = np.random.default_rng(n).integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True)
        d = dev(a) if n else torch.empty(0, dtype=torch.int64, device="cuda")
        ctx.sort(d)
        assert np.array_equal(host_u64(d), np.sort(a))
    sp = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, 5e-324, -5e-324, 1e308, -1e308] * 3000)
    np.random.default_rng(0).shuffle(sp)
    d = dev(sp)
    ctx.sort(d)
    check_sorted_f64(sp, d.cpu().numpy())


@pytest.mark.parametrize("n,pos", [(1000, [17, 500]), (500_000, [123456, 400000]), (16384, [16383])])
def test_sort_nan(ctx, n, pos):
    x = O.generate("normal", n, 7)
    x[pos] = np.nan
    d = dev(x)
    with pytest.raises(L.NanError) as e:
        ctx.sort(d)
    assert e.value.index == min(pos)
    assert np.array_equal(bits(d.cpu().numpy()), bits(x))  # untouched


@pytest.mark.parametrize("off", [0, 1, 3])
@pytest.mark.parametrize("n", [4096 * 40 + 1, 4096 * 40 + 2, 4096 * 300 + 1, 1_000_003])
def test_sort_misaligned_tiles(ctx, off, n):
    """Device views at odd key offsets with sizes = 1, 2 (mod 4096): tiles whose
    16-byte aligned interior is empty issue no bulk copy (partition.cu TileStream)."""
    x = O.generate("normal", n + off + 5, 7)
    base = dev(x)
    v = base[off:off + n]
    ctx.sort(v)
    got = base.cpu().numpy()
    check_sorted_f64(x[off:off + n], got[off:off + n])
    assert np.array_equal(bits(got[:off]), bits(x[:off]))
    assert np.array_equal(bits(got[off + n:]), bits(x[off + n:]))


def test_sort_u64_encoded_normal_20m(ctx):
    """Encoded float keys sorted as u64 (the distributed local sort's input)."""
    a = O.encode(O.generate("normal", 20_000_000, 11))
    d = dev(a)
    ctx.sort(d)
    assert np.array_equal(host_u64(d), np.sort(a))


@pytest.mark.parametrize("n", [600_000, 1_400_000])
def test_sort_quality_fallback(ctx, n):
    """A segment straddling 0.0 (normal values in [-0.003, 0.031]): encoded keys
    are bimodal, the reference's learned model (strict policy) puts most keys in
    one bucket; the GPU policy swaps in a splitter tree. Same sorted output."""
    rng = np.random.default_rng(5)
    x = rng.normal(0.0, 1.0, 4 * n)
    x = x[(x > -0.003) & (x < 0.031)][:n] if n <= 600_000 else np.concatenate(
        [rng.uniform(-0.003, 0.0, n // 10), rng.uniform(0.0, 0.031, n - n // 10)])
    rng.shuffle(x)
    levels = {}
    for name, flags in [("strict", L._native.FLAG_STRICT_POLICY), ("gpu", 0)]:
        d = dev(x)
        st = ctx.sort(d, L.SortConfig(flags=flags))
        check_sorted_f64(x, d.cpu().numpy())
        levels[name] = st["levels"]
    assert levels["gpu"] <= levels["strict"]


@pytest.mark.parametrize("dist,seed", [("uniform", 42), ("normal", 7), ("lognormal2", 19), ("mixgauss", 11),
                                       ("zipf", 3), ("rootdups", 3)])
def test_sort_cluster_level(ctx, dist, seed):
    """The fused DSMEM last level (cluster.cu, LSORT_FLAG_CLUSTER) takes
    segments of 16K..131K keys: 3e7 keys put the level-0 buckets there. Exact
    against np.sort with and without it."""
    n = 30_000_000
    a = O.generate(dist, n, seed)
    ref = np.sort(O.encode(a)) if a.dtype != np.uint64 else np.sort(a)
    for flags in (L._native.FLAG_CLUSTER, 0):
        d = dev(a)
        ctx.sort(d, L.SortConfig(flags=flags))
        got = d.cpu().numpy()
        if a.dtype == np.uint64:
            assert np.array_equal(got.view(np.uint64), ref), flags
        else:
            assert np.array_equal(O.encode(got), ref), flags


def test_sort_host_memory(ctx):
    x = O.generate("lognormal2", 2_000_000, 19)
    y = x.copy()
    st = ctx.sort(y)
    check_sorted_f64(x, y)
    assert st["h2d_bytes"] == x.nbytes and st["d2h_bytes"] == x.nbytes


def test_sort_batch_host(ctx):
    """lsort_cuda_sort_batch: pipelined host arrays, NaN array untouched."""
    xs = [O.generate("normal", 3_000_000, 7), O.generate("lognormal05", 1_000_000, 7),
          O.generate("exponential2", 5, 7), O.generate("uniform", 2_000_001, 42)]
    ys = [x.copy() for x in xs]
    st = ctx.sort_batch(ys)
    for x, y in zip(xs, ys):
        check_sorted_f64(x, y)
    assert st["h2d_bytes"] == sum(x.nbytes for x in xs)
    bad = [O.generate("uniform", 100_000, 42), O.generate("normal", 200_000, 7)]
    bad[1][12345] = np.nan
    keep = bad[1].copy()
    with pytest.raises(L.NanError) as e:
        ctx.sort_batch(bad)
    assert e.value.index == 12345 and e.value.array == 1
    assert np.array_equal(bits(bad[1]), bits(keep))
    assert np.all(np.diff(bad[0]) >= 0)
    us = [O.generate(d, 400_000, 3) for d in ("rootdups", "zipf")]
    vs = [u.copy() for u in us]
    ctx.sort_batch(vs)
    for u, v in zip(us, vs):
        assert np.array_equal(np.sort(u), v)


def test_sort_batch_device(ctx):
    """lsort_cuda_sort_many: concurrent device sorts, NaN array untouched."""
    xs = [O.generate("normal", 3_000_000, 7), O.generate("lognormal2", 2_500_000, 19),
          O.generate("mixgauss", 7, 11), O.generate("uniform", 4_000_001, 42)]
    ds = [dev(x) for x in xs]
    ctx.sort_batch(ds)
    for x, d in zip(xs, ds):
        check_sorted_f64(x, d.cpu().numpy())
    bad = [O.generate("uniform", 300_000, 42), O.generate("normal", 200_000, 7)]
    bad[1][4321] = np.nan
    db = [dev(b) for b in bad]
    with pytest.raises(L.NanError) as e:
        ctx.sort_batch(db)
    assert e.value.index == 4321 and e.value.array == 1
    assert np.array_equal(bits(db[1].cpu().numpy()), bits(bad[1]))
    check_sorted_f64(bad[0], db[0].cpu().numpy())


@pytest.mark.parametrize("n", [1, 5000, 2_000_000])
def test_sort_encoded_to_f64(ctx, n):
    """LSORT_KEY_ENC_F64: encoded u64 keys in, decoded float64 out (the
    distributed local sort's fused decode)."""
    x = O.generate("lognormal2", n, 19)
    d = dev(O.encode(x))
    ctx.sort(d, encoded_f64=True)
    check_sorted_f64(x, d.cpu().numpy().view(np.float64))


@pytest.mark.parametrize("dist_name,seed", [("normal", 7), ("uniform", 42), ("lognormal2", 19)])
def test_sort_forward(ctx, dist_name, seed):
    """lsort_cuda_sort_forward: the root level reuses a given RMI restricted to a
    bucket range (LearnedSort 2.0 model forwarding, cdf_lo/cdf_hi); exact output
    for the full range and for the keys of a sub-range of buckets."""
    n, B = 4_000_000, 2048
    x = O.generate(dist_name, n, seed)
    k = O.encode(x)
    rng = np.random.default_rng(1)
    samp = np.sort(k[rng.integers(0, n, 40_000)])
    ds = dev(samp)
    P = ctx.rmi_train(ds, B)
    d = dev(k)
    ctx.sort_forward(d, P, B, 0, B, ds)
    assert np.array_equal(host_u64(d), np.sort(k))
    ids = O.learned_bucket(P, B, B, k)
    lo, hi = 700, 1300
    sub = k[(ids >= lo) & (ids < hi)]
    d2 = dev(sub)
    ctx.sort_forward(d2, P, B, lo, hi, ds)
    assert np.array_equal(host_u64(d2), np.sort(sub))
    d3 = dev(sub)  # encoded in, float64 out, no sample
    ctx.sort_forward(d3, P, B, lo, hi, None, encoded_f64=True)
    assert np.array_equal(O.encode(d3.cpu().numpy().view(np.float64)), np.sort(sub))


def test_sort_configs(ctx):
    x = O.generate("exponential2", 1_000_000, 7)
    for cfg in [L.SortConfig(bucket_target=0), L.SortConfig(rmi_bucket_count=256, tree_bucket_count=16),
                L.SortConfig(base_case_capacity=4096), L.SortConfig(seed=12345),
                L.SortConfig(min_rmi_input=10**9)]:
        d = dev(x)
        ctx.sort(d, cfg)
        check_sorted_f64(x, d.cpu().numpy())
    with pytest.raises(ValueError):
        ctx.sort(dev(x), L.SortConfig(rmi_bucket_count=1000))


def test_verify(ctx, golden):
    for k in "abcde":
        a = golden[f"verify/{k}/in"]
        if a.size == 0:
            continue
        ok, fv, h = ctx.verify(dev(a))
        exp = golden[f"verify/{k}/out"]
        assert (int(ok), fv, h) == (int(exp[0]), int(exp[1]), int(exp[2]))


def test_sort_large_f64(ctx):
    """BASELINE config 1 at full size (1e7 uniform): bit-exact + hash check on device."""
    x = O.generate("uniform", 10_000_000, 42)
    d = dev(x)
    h_before = ctx.verify(d)[2]
    st = ctx.sort(d)
    ok, fv, h_after = ctx.verify(d)
    assert ok and h_after == h_before
    check_sorted_f64(x, d.cpu().numpy())
    assert st["levels"] >= 1


def _constant_bucket_model(B):
    """A monotone RMI that predicts 0.5 for every key: every key lands in one
    bucket (the adversarial model of SPEC.md:440 / acceptance 9)."""
    P = np.zeros(4 + 4 * B, np.float64)
    P[:4] = [0.0, 0.0, 0.0, 1.0]  # root slope 0, intercept 0: every key routes to submodel 0
    e = P[4:].reshape(B, 4)
    e[:, 0] = 0.0   # slope
    e[:, 1] = 0.5   # intercept
    e[:, 2] = 0.5   # lo
    e[:, 3] = 0.5   # hi
    return P


@pytest.mark.parametrize("case", ["uniform_u64", "normal_enc", "clustered_u64"])
def test_sort_no_progress_fallback(ctx, case):
    """Depth-cap / no-progress fallback: a forwarded root
    model that maps every key to one bucket makes no progress, so the child is
    flagged kSegForceRadix and split by the range-adaptive radix model
    (partition.cu k_scan_children, k_hist<kRadix>). The sort must still
    terminate, be bit-exact and stay within 10x the normal sort time."""
    import time
    n, B = 1_000_000, 1024
    rng = np.random.default_rng(5)
    if case == "uniform_u64":
        k = rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True)
    elif case == "normal_enc":
        k = O.encode(O.generate("normal", n, 7))
    else:  # a few tight clusters far apart: several radix levels
        c = rng.integers(0, 4, n).astype(np.uint64) << np.uint64(60)
        k = c + rng.integers(0, 1 << 20, n, dtype=np.uint64)
    P = _constant_bucket_model(B)
    exp = np.sort(k)
    d = dev(k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = ctx.sort_forward(d, P, B, 0, B, None)
    torch.cuda.synchronize()
    t_fb = time.perf_counter() - t0
    assert np.array_equal(host_u64(d), exp)
    assert st["levels"] >= 2  # the forwarded level made no progress, the radix level did
    d2 = dev(k)
    ctx.sort(d2)  # warm
    d2 = dev(k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.sort(d2)
    torch.cuda.synchronize()
    t_norm = time.perf_counter() - t0
    assert np.array_equal(host_u64(d2), exp)
    assert t_fb <= 10 * max(t_norm, 1e-3), (t_fb, t_norm)


@pytest.mark.parametrize("dist_name,seed", [("exponential2", 7), ("lognormal2", 19)])
def test_padded_level0_and_its_fallback(ctx, dist_name, seed):
    """Large learned roots take the padded one-pass level 0 (k_direct: no
    classify pass, buckets at sample-estimated offsets, children read padded
    and written exact); with the test flag the regions are sized below their
    counts, overflow, and the exact two-pass level runs instead -- both
    bit-exact."""
    n = 80_000_000
    x = O.generate(dist_name, n, seed)
    exp = O.decode(np.sort(O.encode(x))).view(np.uint64)
    d = dev(x)
    st = ctx.sort(d)
    assert st["direct_keys"] >= n  # (level 1 may run one-pass too)
    assert np.array_equal(d.cpu().numpy().view(np.uint64), exp)
    d = dev(x)
    st = ctx.sort(d, L.SortConfig(flags=L._native.FLAG_TEST_DIRECT_OVERFLOW))
    assert st["direct_keys"] == 0
    assert np.array_equal(d.cpu().numpy().view(np.uint64), exp)


@pytest.mark.parametrize("dist_name,seed,n", [("lognormal2", 19, 60_000_000), ("normal", 7, 40_000_000),
                                              ("zipf", 3, 40_000_000)])
def test_no_memory_for_padded_levels(ctx, dist_name, seed, n):
    """The padded buffers of the one-pass levels (~1.2 N keys for level 0, ~5 N for
    level 1) are an optimisation: when they cannot be allocated (test flag) the
    exact two-pass levels run in the N-key scratch array -- same result."""
    x = O.generate(dist_name, n, seed)
    exp = np.sort(x) if x.dtype == np.uint64 else O.decode(np.sort(O.encode(x))).view(np.uint64)
    d = dev(x)
    st = ctx.sort(d, L.SortConfig(flags=L._native.FLAG_TEST_NO_PADDED_MEM))
    assert st["direct_keys"] == 0
    assert np.array_equal(host_u64(d), exp)
    d = dev(x)
    st = ctx.sort(d)
    assert np.array_equal(host_u64(d), exp)


@pytest.mark.parametrize("case", ["lognormal2_f64", "narrow_u64"])
def test_cell_table_models(ctx, case):
    """GPU policy (DESIGN 3, 6): a one-pass root tries a cell table over its
    sorted sample (level0_kind 3 when accepted; wide tables use 32-bit aligned
    cells, narrow ones 64-bit offsets) and every learned-eligible segment
    below the root gets one. The strict reference policy builds none; both
    outputs equal numpy's sort bit for bit."""
    n = 40_000_000
    if case == "lognormal2_f64":
        x = O.generate("lognormal2", n, 19)
        exp = O.decode(np.sort(O.encode(x))).view(np.uint64)
    else:  # uint64 keys over a 2^24 range: cells narrower than 2^32 keys
        x = np.random.default_rng(5).integers(0, 1 << 24, n, dtype=np.uint64)
        exp = np.sort(x)
    d = dev(x)
    st = ctx.sort(d)
    assert st["level0_kind"] == 3, st["level0_kind"]
    assert st["direct_keys"] >= n
    assert np.array_equal(host_u64(d), exp)
    d = dev(x)
    st = ctx.sort(d, L.SortConfig(flags=L._native.FLAG_STRICT_POLICY))
    assert st["level0_kind"] != 3
    assert np.array_equal(host_u64(d), exp)


@pytest.mark.parametrize("dist_name", ["rootdups", "zipf"])
def test_padded_level0_tree_root(ctx, dist_name):
    """Duplicate-heavy roots (Alg. 5 picks the splitter tree) also take the
    one-pass level 0: regions sized from the tree's buckets in the sorted first
    sample, equality buckets counted but not moved (filled afterwards); with
    the test flag the regions overflow and the exact two-pass level runs."""
    n = 40_000_000
    x = O.generate(dist_name, n, 3)
    exp = np.sort(x)
    d = dev(x)
    st = ctx.sort(d)
    assert st["level0_kind"] == 1
    assert st["direct_keys"] >= n
    assert st["fill_keys"] > 0
    assert np.array_equal(host_u64(d), exp)
    d = dev(x)
    st = ctx.sort(d, L.SortConfig(flags=L._native.FLAG_TEST_DIRECT_OVERFLOW))
    assert st["direct_keys"] == 0
    assert np.array_equal(host_u64(d), exp)


@pytest.mark.parametrize("dist_name,seed", [("lognormal2", 19), ("exponential2", 7)])
def test_padded_level1_and_its_fallback(ctx, dist_name, seed):
    """Level 1 of a one-pass root also runs one-pass when every segment has a
    linear cell table (regions from each segment's slice of the root sample);
    with the test flag its regions overflow too and both exact levels run."""
    n = 60_000_000
    x = O.generate(dist_name, n, seed)
    exp = O.decode(np.sort(O.encode(x))).view(np.uint64)
    d = dev(x)
    st = ctx.sort(d)
    assert st["direct_keys"] == 2 * n, st["direct_keys"]
    assert np.array_equal(host_u64(d), exp)
    d = dev(x)
    st = ctx.sort(d, L.SortConfig(flags=L._native.FLAG_TEST_DIRECT_OVERFLOW))
    assert st["direct_keys"] == 0
    assert np.array_equal(host_u64(d), exp)


@pytest.mark.parametrize("dist_name,n", [("uniform", 20_000_000), ("lognormal2", 30_000_000),
                                         ("normal", 25_000_000), ("twodups", 30_000_000)])
def test_padded_level1_other_model_kinds(ctx, dist_name, n):
    """A one-pass level 1 whose segments are too small for cell tables (splitter
    trees, < 32 Ki keys) or mix model kinds: the tree segments' tiles are empty in
    k_direct (their headers are not read as cell tables) and the exact kernels
    write them into scratch3's tail, read by the next level through the same
    buffer. Regression: 2e7-3e7 keys failed with an illegal address."""
    seed = {"uniform": 42, "lognormal2": 19, "normal": 7, "twodups": 3}[dist_name]
    x = O.generate(dist_name, n, seed)
    if x.dtype == np.uint64:
        exp = np.sort(x)
    else:
        exp = O.decode(np.sort(O.encode(x))).view(np.uint64)
    for _ in range(2):  # (a second sort reuses the grown workspaces)
        d = dev(x)
        ctx.sort(d)
        assert np.array_equal(host_u64(d), exp)
