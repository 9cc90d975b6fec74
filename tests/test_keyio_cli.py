"""Key files and the command-line harness (SPEC.md data module :480-497,
bench-cli module :521-590). CPU tests: file format, generate, verify. GPU
tests: sort and bench through the CLI."""
import csv
import os
import subprocess

import numpy as np
import pytest

import paper_2307_08637_b200 as L
from lsort_testutil import ROOT

CLI = os.path.join(ROOT, "paper_2307_08637_b200", "lsort_cli")


def run(*args):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)


def test_write_read_examples(tmp_path):
    p = tmp_path / "e.bin"
    L.write_keys(p, np.array([], np.uint64))
    assert p.read_bytes() == b"\0" * 8                                      # [] -> 8-byte file of zeros
    L.write_keys(p, np.array([1, 5], np.uint64))
    assert p.read_bytes() == bytes([2] + [0] * 7 + [1] + [0] * 7 + [5] + [0] * 7)  # the 24-byte sequence
    assert list(L.read_keys(p)) == [1, 5]


def test_round_trip_random(tmp_path):
    a = np.random.default_rng(3).integers(0, 2**64 - 1, 100_000, dtype=np.uint64, endpoint=True)
    p = tmp_path / "r.bin"
    L.write_keys(p, a)
    assert np.array_equal(L.read_keys(p), a)


def test_structural_errors(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(bytes([2] + [0] * 7) + b"\1" * 9)          # 17 bytes, count 2
    with pytest.raises(OSError, match="needs 24 bytes"):
        L.read_keys(p)
    p.write_bytes(b"\1\2\3")
    with pytest.raises(OSError, match="count header"):
        L.read_keys(p)
    with pytest.raises(OSError, match="cannot open"):
        L.read_keys(tmp_path / "missing.bin")


def test_cli_generate(tmp_path):
    a, b = tmp_path / "a.bin", tmp_path / "b.bin"
    assert run("generate", "uniform", 1000000, 1, a).returncode == 0
    assert a.stat().st_size == 8 + 8 * 10**6                  # size arithmetic
    assert run("generate", "uniform", 1000000, 1, b).returncode == 0
    assert a.read_bytes() == b.read_bytes()                  # determinism
    # float datasets are written as encoded keys: same as the library's generator + encode
    k = L.read_keys(a)
    x = L.generate("uniform", 10**6, 1)
    enc = np.where(x.view(np.uint64) >> 63, ~x.view(np.uint64), x.view(np.uint64) ^ np.uint64(1 << 63))
    assert np.array_equal(k, enc)
    r = tmp_path / "rd.bin"
    assert run("generate", "rootdups", 16, 42, r).returncode == 0
    assert sorted(L.read_keys(r).tolist()) == sorted([i % 4 for i in range(16)])  # i mod sqrt(N), shuffled
    bad = run("generate", "chisquared", 10, 1, tmp_path / "x.bin")
    assert bad.returncode != 0 and "registry" in bad.stderr


def test_cli_verify(tmp_path):
    s, u = tmp_path / "s.bin", tmp_path / "u.bin"
    L.write_keys(s, np.arange(100, dtype=np.uint64))
    L.write_keys(u, np.array([2, 1], np.uint64))
    assert run("verify", s).returncode == 0
    r = run("verify", u)
    assert r.returncode == 1 and "violation at index 1" in r.stdout
    (tmp_path / "m.bin").write_bytes(b"\2" + b"\0" * 7 + b"\1" * 9)
    assert run("verify", tmp_path / "m.bin").returncode == 2


@pytest.mark.gpu
def test_cli_sort(tmp_path):
    src, dst = tmp_path / "in.bin", tmp_path / "out.bin"
    assert run("generate", "normal", 3_000_000, 7, src).returncode == 0
    assert run("sort", src, dst).returncode == 0
    assert np.array_equal(L.read_keys(dst), np.sort(L.read_keys(src)))
    assert run("verify", dst).returncode == 0


@pytest.mark.gpu
def test_cli_bench(tmp_path):
    out = tmp_path / "b.csv"
    r = run("bench", "--dataset", "lognormal", "--n", 2_000_000, "--runs", 3, "--csv", out)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "algorithm,dataset,n,workers,run,elapsed_ns,keys_per_second,verified"
    rows = list(csv.reader(lines[1:7]))
    assert [x[0] for x in rows] == ["gpu-aips2o"] * 3 + ["reference"] * 3
    assert all(x[7] == "true" for x in rows)
    assert lines[7] == "# summary"
    # a key file as dataset, device-resident timing
    f = tmp_path / "z.bin"
    assert run("generate", "zipf", 500_000, 3, f).returncode == 0
    r = run("bench", "--dataset", f, "--runs", 2, "--algo", "gpu-aips2o", "--resident")
    assert r.returncode == 0, r.stderr
