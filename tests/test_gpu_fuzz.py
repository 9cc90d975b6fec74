"""GPU fuzz regression: lsort_cuda_sort against torch.sort, bit-exact.

Inputs are drawn on the device by tools/fuzz_sort.py (24 distributions the
BASELINE configs do not cover: tight clusters, Cauchy / Pareto tails, exponents
over the whole double range, pre-sorted, few distinct values ...). The named
cases are the ones the fuzz run of round 2 caught:

* clusters 4e7 (default policy): level 1 mostly splitter trees with a few cell
  tables -- the one-pass level 1 classified the empty tiles of the exact
  kernels' segments through an uninitialised table pointer;
* clusters 2e8 (strict policy): depth-cap / no-progress segments
  (kSegForceRadix) left ModelHdr::flags unset, so reused model memory could
  mark the radix model as a cell table;
* clusters 4.5e6: the fused cluster level's sort batches bounded their keys but
  not their digits (empty sub-buckets take one digit each).
"""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2307_08637_b200 as L  # noqa: E402
from lsort_testutil import ROOT  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tools"))
import fuzz_sort as F  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return L.Context(0)


def run_case(ctx, name, n, seed, flags):
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    x = F.draw(g, name, n, dev) if n else torch.empty(
        0, device=dev, dtype=torch.float64 if name in F.FLOATS else torch.int64)
    exp = torch.sort(F.ordered_i64(x))[0]
    cfg = L.SortConfig()
    cfg.flags |= flags
    ctx.sort(x, cfg)
    assert torch.equal(F.ordered_i64(x), exp), (name, n, seed, flags)


def test_clusters_level1_mostly_trees(ctx):
    for _ in range(2):
        run_case(ctx, "clusters", 40_179_256, 1126352106, 0)


def test_clusters_strict_force_radix_after_cell_tables(ctx):
    # a default-policy sort first: its model records (cell tables) are the memory
    # the strict sort's radix fallback models then reuse
    run_case(ctx, "clusters", 201_660_944, 383816745, 0)
    for _ in range(3):
        run_case(ctx, "clusters", 201_660_944, 383816745, L._native.FLAG_STRICT_POLICY)


def test_clusters_fused_cluster_level_digit_bound(ctx):
    """Auto-selected fused cluster level (cluster.cu) over segments whose sub-buckets
    are mostly empty: a sort batch of ~4096 keys plus its empty sub-buckets' digits
    exceeded the digit capacity ("work list overflow (64)")."""
    run_case(ctx, "clusters", 4_544_002, 1295304046, 0)


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_fuzz_short(ctx, seed):
    """40 random (distribution, size <= 3e7, policy) cases per seed."""
    rng = np.random.default_rng(seed)
    names = F.FLOATS + F.INTS
    for _ in range(40):
        name = names[rng.integers(len(names))]
        u = rng.random()
        if u < 0.3:
            n = int(F.EDGES[rng.integers(len(F.EDGES))] * rng.uniform(0.7, 1.5))
        elif u < 0.4:
            n = int(rng.integers(0, 20000))
        else:
            n = int(np.exp(rng.uniform(np.log(2), np.log(3e7))))
        n = min(n, 100_000_000)
        flags = L._native.FLAG_STRICT_POLICY if rng.random() < 0.15 else 0
        run_case(ctx, name, n, int(rng.integers(1 << 31)), flags)


def test_fuzz_entries_and_virtual_ranks():
    """150 cases of tools/fuzz_sort.py with 20% on 2-8 virtual ranks and 40% through the
    other entries (host memory, sort_many, sort_batch, classic path, NaN error path)."""
    import subprocess
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_sort.py"), "--seed", "21", "--cases", "150",
                        "--seconds", "600", "--max-keys", "3e7", "--dist", "0.2", "--api", "0.4"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "fuzz: 150 cases bit-exact" in r.stdout
