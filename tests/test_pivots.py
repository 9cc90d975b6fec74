"""Pivot analysis (Alg. 4, §3.1, Table 1).

CPU: the oracle restatement against the SPEC's known answers and properties,
and the Table 1 trend (RMI pivots beat random-sampling pivots on uniform data).
GPU (-m gpu): lsort_cuda_learned_pivots / pivot_quality / eta through the
C-ABI, bit-exact against the oracle on the same RMI parameters, and the
lsort_cli pivot-quality report."""
import csv
import io
import math
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2307_08637_b200", "lsort_cli")


def _splitmix(x):
    x = (x + 0x9E3779B97F4A7C15) & (2**64 - 1)
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    return x ^ (x >> 31)


def random_pivots(keys, b, seed):
    """IPS4o-style: alpha*b random keys (alpha = 0.2 log2 n), every alpha-th."""
    n = keys.size
    alpha = max(1, int(0.2 * math.log2(n)))
    idx = np.array([_splitmix(seed + j) % n for j in range(alpha * b)], np.uint64)
    s = np.sort(keys[idx])
    p = s[alpha * np.arange(1, b) - 1]
    return np.unique(p)


def rmi_model(keys, b, seed):
    n = keys.size
    s = max(2, min((n + 99) // 100, 1 << 20))
    idx = np.array([_splitmix(seed + j) % n for j in range(s)], np.uint64)
    return O.rmi_train(np.sort(keys[idx]), b)


def rmi_pivots(keys, b, seed):
    return O.learned_pivots(keys, rmi_model(keys, b, seed), b, b)


def rmi_distance(srt, P, b, pivots):
    """Distance of Alg. 4's pivots against b (the CLI's scoring): an empty cell's
    boundary (g+1)/b takes the largest key with F < (g+1)/b, i.e. the last pivot
    of a cell <= g (rank 0 before the first)."""
    cells = O.learned_bucket(P, b, b, pivots)
    ranks = np.searchsorted(srt, pivots, side="right")
    d, j, r = 0.0, 0, 0
    for g in range(b - 1):
        while j < pivots.size and cells[j] <= g:
            r = int(ranks[j])
            j += 1
        d += abs(r / srt.size - (g + 1) / b)
    return d


# ------------------------------------------------------------------ CPU
def test_spec_examples():
    a = np.arange(1000, dtype=np.uint64)
    P = O.rmi_train(a, 4)
    assert list(O.learned_pivots(a, P, 4, 4)) == [249, 499, 749]
    assert O.pivot_quality(a, np.array([249, 499, 749], np.uint64), 4) == 0.0  # perfect splitters
    n = a.size
    assert O.eta(a, 499) == 0.0                                           # median
    assert abs(O.eta(a, 0) - 0.5) <= 1.0 / n + 1e-12                      # minimum
    assert O.eta(a, 749) == 0.25                                          # 75th percentile
    c = np.full(100, 7, np.uint64)
    assert O.learned_pivots(c, O.rmi_train(c, 4), 4, 4).size <= 1        # constant array


def test_pivot_count_must_match_b():
    a = np.arange(100, dtype=np.uint64)
    with pytest.raises(ValueError):
        O.pivot_quality(a, np.array([10, 20], np.uint64), 4)


@pytest.mark.parametrize("dist,seed", [("uniform", 42), ("normal", 7), ("zipf", 3), ("rootdups", 3)])
def test_properties(dist, seed):
    x = O.generate(dist, 200_000, seed)
    k = O.encode(x) if x.dtype == np.float64 else x
    srt = np.sort(k)
    for b in (4, 64, 256):
        p = rmi_pivots(k, b, seed)
        assert np.all(np.diff(p.astype(np.float64)) > 0) and np.all(np.isin(p, k))  # increasing, subset
        if p.size + 1 == b:
            assert O.pivot_quality(srt, p, b) >= 0.0
        for q in p[:: max(1, p.size // 8)]:
            assert 0.0 <= O.eta(srt, int(q)) <= 0.5


def test_table1_trend_uniform():
    """PAPER.md Table 1 (uniform, 255 pivots): RMI distance < random distance
    in >= 9 of 10 trials and RMI <= 0.7x random on the mean."""
    k = O.encode(O.generate("uniform", 1_000_000, 42))
    srt = np.sort(k)
    wins, dr, dm = 0, [], []
    for t in range(10):
        rp = random_pivots(k, 256, 1000 + t)
        P = rmi_model(k, 256, 2000 + t)
        lp = O.learned_pivots(k, P, 256, 256)
        r = O.pivot_quality(srt, rp, rp.size + 1)
        m = O.pivot_quality(srt, lp, 256) if lp.size == 255 else rmi_distance(srt, P, 256, lp)
        dr.append(r)
        dm.append(m)
        wins += m < r
    assert wins >= 9 and np.mean(dm) <= 0.7 * np.mean(dr), (dr, dm)


# ------------------------------------------------------------------ GPU
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import paper_2307_08637_b200 as L
    return L.Context(0)


@pytest.mark.gpu
@pytest.mark.parametrize("dist,seed,b", [("uniform", 42, 256), ("normal", 7, 1024), ("lognormal2", 19, 64),
                                         ("zipf", 3, 256), ("twodups", 3, 2048)])
def test_gpu_pivots_match_oracle(ctx, dist, seed, b):
    x = O.generate(dist, 1_000_000, seed)
    f64 = x.dtype == np.float64
    k = O.encode(x) if f64 else x
    s = np.sort(k[np.array([_splitmix(seed + j) % k.size for j in range(10_000)])])
    P = O.rmi_train(s, b)
    d = torch.from_numpy(x.view(np.int64) if not f64 else x).cuda()
    got, cells = ctx.learned_pivots(P, b, b, d, cells=True)
    exp = O.learned_pivots(k, P, b, b)
    got_enc = O.encode(got) if f64 else got
    assert np.array_equal(got_enc, exp)
    assert np.array_equal(cells, O.learned_bucket(P, b, b, exp))
    # quality and eta on the sorted keys, bit-exact with the oracle
    srt = np.sort(k)
    ds = torch.from_numpy(O.decode(srt) if f64 else srt.view(np.int64)).cuda()
    dist_gpu, ranks = ctx.pivot_quality(ds, got, got.size + 1)
    assert dist_gpu == O.pivot_quality(srt, exp, exp.size + 1)
    assert np.array_equal(ranks, np.searchsorted(srt, exp, side="right").astype(np.uint64))
    for q in range(0, got.size, max(1, got.size // 5)):
        assert ctx.eta(ds, got[q]) == O.eta(srt, int(exp[q]))


@pytest.mark.gpu
def test_gpu_pivot_quality_rejects_bad_count(ctx):
    d = torch.arange(100, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):  # LSORT_EINVAL mirrors std::invalid_argument
        ctx.pivot_quality(d, np.array([10, 20], np.uint64), 4)


@pytest.mark.gpu
def test_cli_pivot_quality(tmp_path):
    out = tmp_path / "pq.csv"
    r = subprocess.run([CLI, "pivot-quality", "uniform", "1000000", "255", "10", "42", str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(out.read_text())))
    per = [r for r in rows if r["trial"] != "mean"]
    assert len(per) == 20
    mean = {r["method"]: float(r["distance"]) for r in rows if r["trial"] == "mean"}
    wins = sum(float(a["distance"]) > float(b["distance"])
               for a, b in zip(per[0::2], per[1::2]))  # random row, then rmi row
    assert wins >= 9 and mean["rmi"] <= 0.7 * mean["random"], rows
