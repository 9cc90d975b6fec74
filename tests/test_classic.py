"""LearnedSort 2.0 classic path.

CPU: the oracle's restatement (learned_sort_classic, model_counting_sort) on
SPEC examples. GPU (through the C-ABI): lsort_cuda_model_counting_sort equals
the oracle's stable placement bit for bit under the same RMI;
lsort_cuda_sort_classic equals numpy's sort on every BASELINE generator,
adversarial inputs, NaN and host memory, and its round-two occupancy is
~N/B^2 on uniform data (SPEC invariant)."""
import numpy as np
import pytest

from oracle import oracle as O

SEEDS = {"uniform": 42, "normal": 7, "lognormal05": 7, "exponential2": 7, "mixgauss": 11, "lognormal2": 19,
         "rootdups": 3, "twodups": 3, "zipf": 3}


def _trained(name, n, B, frac=0.05):
    x = O.generate(name, n, SEEDS[name])
    k = O.encode(x) if x.dtype == np.float64 else x
    rng = np.random.default_rng(4)
    s = np.sort(k[rng.integers(0, n, max(2, int(frac * n)))])
    return k, s, O.rmi_train(s, B)


def test_oracle_model_counting_sort_examples():
    # perfect distinct predictions -> exactly sorted
    k = np.array([40, 10, 30, 20], np.uint64)
    P = O.rmi_train(np.array([10, 20, 30, 40], np.uint64), 1)
    assert list(O.model_counting_sort(k, P, 1)) == [10, 20, 30, 40]
    # colliding predictions: every key present, ties keep the input order
    P2 = np.zeros(8)
    P2[3], P2[4 + 1], P2[4 + 2], P2[4 + 3] = 1.0, 0.5, 0.5, 0.5  # constant model
    out = O.model_counting_sort(np.array([9, 3, 7], np.uint64), P2, 1)
    assert list(out) == [9, 3, 7]


def test_oracle_model_counting_sort_displacement_bound():
    """Inversion distance of the output <= the model's max rank error per
    segment: no key lands farther from its sorted position than
    the largest |predicted - true| position error, +1 for the tie order."""
    k, s, P = _trained("uniform", 50_000, 64)
    seg = k[:1000]
    out = O.model_counting_sort(seg, P, 64)
    true = np.searchsorted(np.sort(seg), out)
    pred = O.learned_bucket(P, 64, seg.size, out)
    err = np.abs(pred.astype(np.int64) - np.searchsorted(np.sort(seg), out, side="left")).max()
    assert np.abs(true - np.arange(seg.size)).max() <= err + 1


@pytest.mark.parametrize("name", ["uniform", "lognormal2", "rootdups", "normal"])
def test_oracle_learned_sort_classic(name):
    k = O.encode(O.generate(name, 60_000, SEEDS[name])) if name in ("uniform", "lognormal2", "normal") else \
        O.generate(name, 60_000, SEEDS[name])
    out, nsub, swaps = O.learned_sort_classic(k, O.cfg(rmi_bucket_count=256))
    assert np.array_equal(out, np.sort(k))
    assert nsub > 0


def test_oracle_classic_sorted_input_unchanged():
    k = np.arange(0, 30_000, 3, dtype=np.uint64)
    out, _, swaps = O.learned_sort_classic(k, O.cfg(rmi_bucket_count=64))
    assert np.array_equal(out, k) and swaps == 0


# ------------------------------------------------------------------ GPU
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2307_08637_b200 as L
    return L.Context(0)


def _dev(a):
    return torch.from_numpy(a if a.dtype == np.float64 else a.view(np.int64)).cuda()


@pytest.mark.gpu
@pytest.mark.parametrize("name,B", [("uniform", 1024), ("lognormal2", 256), ("normal", 64), ("zipf", 1024)])
def test_model_counting_sort_matches_oracle(ctx, name, B):
    k, s, P = _trained(name, 200_000, B)
    rng = np.random.default_rng(1)
    for n in (1, 2, 17, 1000, 4096, 8192):
        seg = k[rng.integers(0, k.size, n)]
        for lo, hi in ((0.0, 1.0), (0.25, 0.5)):
            got = ctx.model_counting_sort(P, B, _dev(seg), lo, hi).cpu().numpy().view(np.uint64)
            assert np.array_equal(got, O.model_counting_sort(seg, P, B, lo, hi)), (n, lo, hi)


@pytest.mark.gpu
@pytest.mark.parametrize("name,n", [("uniform", 10_000_000), ("normal", 3_000_000), ("lognormal05", 2_000_000),
                                    ("exponential2", 2_000_000), ("mixgauss", 3_000_000), ("lognormal2", 5_000_000),
                                    ("rootdups", 2_000_000), ("twodups", 2_000_000), ("zipf", 2_000_000)])
def test_sort_classic_exact(ctx, name, n):
    x = O.generate(name, n, SEEDS[name])
    d = _dev(x)
    st = ctx.sort_classic(d)
    got = d.cpu().numpy()
    exp = O.decode(np.sort(O.encode(x))) if x.dtype == np.float64 else np.sort(x)
    assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
    assert st["levels"] >= 1


@pytest.mark.gpu
def test_sort_classic_round_two_occupancy(ctx):
    """SPEC.md invariant: average bucket occupancy after round two ~ N / B^2
    (within +-50%) on uniform data; round two happens for every bucket above
    the base-case capacity."""
    import paper_2307_08637_b200 as L
    n, B = 4_000_000, 64
    x = O.generate("uniform", n, 42)
    d = _dev(x)
    st = ctx.sort_classic(d, L.SortConfig(rmi_bucket_count=B, base_case_capacity=1024))
    assert np.array_equal(d.cpu().numpy(), np.sort(x))
    assert st["round2_buckets"] > 0
    occ = n / st["round2_buckets"]
    assert 0.5 * n / B**2 <= occ <= 1.5 * n / B**2, (occ, n / B**2)


@pytest.mark.gpu
def test_sort_classic_edges(ctx):
    import paper_2307_08637_b200 as L
    for a in (np.arange(500_000, dtype=np.uint64), np.arange(500_000, dtype=np.uint64)[::-1].copy(),
              np.full(300_000, 7, np.uint64), np.zeros(0, np.uint64), np.array([5], np.uint64)):
        d = _dev(a) if a.size else torch.empty(0, dtype=torch.int64, device="cuda")
        ctx.sort_classic(d)
        assert np.array_equal(d.cpu().numpy().view(np.uint64), np.sort(a))
    x = O.generate("normal", 400_000, 7)
    x[1234] = np.nan
    d = _dev(x)
    with pytest.raises(L.NanError) as e:
        ctx.sort_classic(d)
    assert e.value.index == 1234
    h = O.generate("exponential2", 1_000_000, 7)
    ctx.sort_classic(h)  # host memory
    assert np.all(np.diff(h) >= 0)
