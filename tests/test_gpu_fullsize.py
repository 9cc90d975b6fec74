"""BASELINE.json configs at full size on one B200, checked through
size-independent properties (device verify_sorted + multiset_hash,
verify.hpp:17-29, before/after) and a whole-array bit-exact comparison
against numpy's sort of the encoded keys.
C5 (4e9 keys over 8 GPUs) runs its 5e8-key per-GPU shard."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2307_08637_b200 as L  # noqa: E402
from oracle import oracle as O  # noqa: E402

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
    # whole-array bit-exact comparison against numpy (np.sort of the encoded
    # keys: a keys-only sort has a unique result)
    got = t.cpu().numpy()
    if h.dtype == np.float64:
        exp = O.decode(np.sort(O.encode(h)))
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64)), f"{name}: differs from numpy"
    else:
        exp = np.sort(h)
        assert np.array_equal(got.view(np.uint64), exp), f"{name}: differs from numpy"
    del exp
    del t, got
    torch.cuda.empty_cache()
