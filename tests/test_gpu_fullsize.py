"""BASELINE.json configs at full size on one B200, checked through
size-independent properties (the oracle would take minutes at these sizes):
device verify_sorted + multiset_hash (verify.hpp:17-29) before/after, plus a
bit-exact comparison against numpy on a random window and on the extremes.
C5 (4e9 keys over 8 GPUs) runs its 5e8-key per-GPU shard."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2307_08637_b200 as L  # noqa: E402

CASES = [
    ("C1", "uniform", 42, 10_000_000),
    ("C2-normal", "normal", 7, 100_000_000),
    ("C2-lognormal", "lognormal05", 7, 100_000_000),
    ("C2-exponential", "exponential2", 7, 100_000_000),
    ("C3", "mixgauss", 11, 200_000_000),
    ("C4-rootdups", "rootdups", 3, 100_000_000),
    ("C4-twodups", "twodups", 3, 100_000_000),
    ("C4-zipf", "zipf", 3, 100_000_000),
    ("C5-shard", "lognormal2", 19, 500_000_000),
]


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    return L.Context(0)


@pytest.mark.parametrize("name,dist,seed,n", CASES, ids=[c[0] for c in CASES])
def test_full_size_config(ctx, name, dist, seed, n):
    if name == "C5-shard":
        h = L.generate(dist, 8 * n, seed, first=0, count=n)
    else:
        h = L.generate(dist, n, seed)
    t = torch.from_numpy(h if h.dtype == np.float64 else h.view(np.int64)).cuda()
    _, _, hash_before = ctx.verify(t)
    st = ctx.sort(t)
    ok, fv, hash_after = ctx.verify(t)
    assert ok, f"{name}: unsorted at {fv}"
    assert hash_after == hash_before, f"{name}: multiset changed"
    # bit-exact spot checks: min, max, and a sorted window equal numpy's
    got = t.cpu().numpy()
    exp_first = np.partition(h, 1000)[:1000]
    if h.dtype == np.float64:
        assert np.array_equal(np.sort(exp_first).view(np.uint64)[:100], got[:100].view(np.uint64))
        assert got[-1] == h.max() and got[0] == h.min()
    else:
        assert np.array_equal(np.sort(exp_first)[:100], got[:100].view(np.uint64))
        assert got.view(np.uint64)[-1] == h.max()
    del t, got
    torch.cuda.empty_cache()
