"""GPU fuzz of lsort_cuda_sort against torch.sort (bit-exact), inputs drawn on the device.

    python tools/fuzz_sort.py [--seconds 600] [--seed 1] [--max-keys 6e8]

Each case: a random (distribution, size, key type), sizes log-uniform in
[2, max-keys] with extra weight on the region boundaries of the engine (base
case capacity, one-pass thresholds, 2e7-3e7). The sorted result is compared
whole-array with torch.sort of the order-preserving int64 image of the keys.
Prints one line per case and a summary; exit code 1 on the first mismatch or
library error (the failing case's seed and parameters are printed)."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_08637_b200 as L  # noqa: E402
from paper_2307_08637_b200.dist import sort_emulated  # noqa: E402

SIGN = -(1 << 63)


def ordered_i64(t):
    """Order-preserving int64 image (the encode of keys.hpp:24-27 with the sign bit flipped)."""
    if t.dtype == torch.float64:
        b = t.view(torch.int64)
        return torch.where(b < 0, ~b ^ SIGN, b)  # negative floats: all bits flipped, then sign flipped back
    return t ^ SIGN  # uint64 stored as int64: flip the sign bit


def draw(g, name, n, dev):
    r = lambda *s: torch.rand(*s, generator=g, device=dev, dtype=torch.float64)
    rn = lambda *s: torch.randn(*s, generator=g, device=dev, dtype=torch.float64)
    if name == "uniform":
        return r(n)
    if name == "normal":
        return rn(n)
    if name.startswith("lognormal"):
        return torch.exp(rn(n) * float(name[9:]))
    if name == "exponential":
        return -torch.log1p(-r(n)) / 2
    if name == "mixgauss":
        k = 5
        mu = (torch.rand(k, generator=g, device=dev, dtype=torch.float64) * 200 - 100)
        sd = (torch.rand(k, generator=g, device=dev, dtype=torch.float64) * 4 + 1)
        c = torch.randint(0, k, (n,), generator=g, device=dev)
        return rn(n) * sd[c] + mu[c]
    if name == "pareto":
        return (1 - r(n)) ** (-1 / 0.7)
    if name == "cauchy":
        return torch.tan(3.141592653589793 * (r(n) - 0.5))
    if name == "wide_exp":  # exponents spread over the whole double range, both signs
        e = torch.randint(-300, 300, (n,), generator=g, device=dev).double()
        return (r(n) + 0.5) * torch.pow(torch.tensor(10.0, device=dev, dtype=torch.float64), e) * \
            (torch.randint(0, 2, (n,), generator=g, device=dev).double() * 2 - 1)
    if name == "sorted":
        return torch.sort(rn(n))[0]
    if name == "reverse":
        return torch.sort(rn(n), descending=True)[0]
    if name == "nearly_sorted":
        x = torch.arange(n, device=dev, dtype=torch.float64)
        return x + rn(n) * 50
    if name == "clusters":  # many tight clusters far apart
        c = torch.randint(0, 1000, (n,), generator=g, device=dev).double()
        return c * 1e6 + rn(n) * 1e-3
    if name == "heavy_hitter":
        x = rn(n)
        x[r(n) < 0.4] = 1.25
        return x
    if name == "zeros_mix":
        x = rn(n)
        m = r(n)
        x[m < 0.2] = 0.0
        x[(m >= 0.2) & (m < 0.3)] = -0.0
        x[(m >= 0.3) & (m < 0.31)] = float("inf")
        x[(m >= 0.31) & (m < 0.32)] = float("-inf")
        return x
    # ---- uint64 (held as int64 bit patterns)
    ri = lambda lo, hi: torch.randint(lo, hi, (n,), generator=g, device=dev, dtype=torch.int64)
    if name == "u64_full":
        return ri(-(1 << 63), (1 << 63) - 1)
    if name == "u64_small_range":
        return ri(0, 1 << int(torch.randint(1, 40, (1,), generator=g, device=dev)))
    if name == "u64_rootdups":
        return ri(0, max(2, int(n ** 0.5)))
    if name == "u64_few":
        return ri(0, 7) * 1234567891011
    if name == "u64_zipf":
        u = r(n)
        return (1e6 * u ** 4).long()
    if name == "u64_two_ends":
        x = ri(0, 1 << 20)
        m = r(n) < 0.5
        x[m] = -1 - x[m]  # near 2^64
        return x
    if name == "u64_const":
        return torch.full((n,), 42, device=dev, dtype=torch.int64)
    if name == "u64_shifted_normal":
        return (rn(n) * 1e12).long() + (1 << 62)
    raise KeyError(name)


FLOATS = ["uniform", "normal", "lognormal0.5", "lognormal2", "lognormal4", "exponential", "mixgauss", "pareto",
          "cauchy", "wide_exp", "sorted", "reverse", "nearly_sorted", "clusters", "heavy_hitter", "zeros_mix"]
INTS = ["u64_full", "u64_small_range", "u64_rootdups", "u64_few", "u64_zipf", "u64_two_ends", "u64_const",
        "u64_shifted_normal"]
EDGES = [16384, 65536, 4 << 20, 1 << 24, 20_000_000, 30_000_000, 1 << 25, 1 << 26]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=600)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--max-keys", type=float, default=6e8)
    ap.add_argument("--only", default="")
    ap.add_argument("--case", default="", help="replay one case: name:n:seed:flags[:world[:api]]")
    ap.add_argument("--dist", type=float, default=0.0, help="fraction of cases run on 2-8 virtual ranks")
    ap.add_argument("--strict", type=float, default=0.1, help="fraction of cases under LSORT_FLAG_STRICT_POLICY")
    ap.add_argument("--cases", type=int, default=0, help="stop after this many cases (0: run for --seconds)")
    ap.add_argument("--repeat", type=int, default=1, help="--case: run the case this many times in one process")
    ap.add_argument("--api", type=float, default=0.0,
                    help="fraction of cases through another entry: host memory, sort_many, sort_batch, classic, NaN")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(a.seed)
    ctx = L.Context(0)
    t_end = time.time() + a.seconds
    cases = 0
    names = [x for x in FLOATS + INTS if not a.only or x in a.only.split(",")]
    replay = a.case.split(":") if a.case else None
    while time.time() < t_end:
        name = names[rng.integers(len(names))]
        u = rng.random()
        if u < 0.25:
            n = int(EDGES[rng.integers(len(EDGES))] * rng.uniform(0.7, 1.5))
        elif u < 0.30:
            n = int(rng.integers(0, 20000))
        else:
            n = int(np.exp(rng.uniform(np.log(1e4), np.log(a.max_keys))))
        n = min(n, int(a.max_keys))
        seed = int(rng.integers(1 << 31))
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        flags = 0
        if rng.random() < a.strict:
            flags |= L._native.FLAG_STRICT_POLICY
        if replay:
            name, n, seed, flags = replay[0], int(replay[1]), int(replay[2]), int(replay[3])
            g.manual_seed(seed)
            a.repeat -= 1
            if a.repeat <= 0:
                t_end = 0
        # --dist P: with probability P the case runs the multi-rank driver on virtual
        # ranks (lsort_cuda_dist_emulate), shards cut at random points (some empty)
        world = 0
        if a.dist and not replay and rng.random() < a.dist and n <= 100_000_000:
            world = int(rng.choice([2, 3, 4, 8]))
        if replay and len(replay) > 4:
            world = int(replay[4])
        x = draw(g, name, n, dev) if n else torch.empty(0, device=dev, dtype=torch.float64 if name in FLOATS else torch.int64)
        exp = torch.sort(ordered_i64(x))[0]
        cfg = L.SortConfig()
        cfg.flags |= flags
        t0 = time.time()
        try:
            api = "sort"
            if a.api and not replay and not world and rng.random() < a.api:
                api = str(rng.choice(["host", "many", "batch", "classic", "nan"]))
            if replay and len(replay) > 5:
                api = replay[5]
            if api != "sort" and (world or n > 60_000_000 or n < 2):
                api = "sort"
            if api == "host":  # LSORT_MEM_HOST: copies in / out inside the call
                h = x.cpu().numpy()
                st = ctx.sort(h, cfg)
                x = torch.from_numpy(h).to(dev)
                name += "/host"
            elif api in ("many", "batch"):  # three pieces sorted in one call (device: concurrently; host: pipelined)
                c1, c2 = sorted(int(v) for v in np.random.default_rng(seed).integers(0, n + 1, 2))
                parts = [x[:c1].clone(), x[c1:c2].clone(), x[c2:].clone()]
                exps = [torch.sort(ordered_i64(q))[0] for q in parts]
                if api == "batch":
                    hs = [q.cpu().numpy() for q in parts]
                    st = ctx.sort_batch(hs, cfg)
                    parts = [torch.from_numpy(q).to(dev) for q in hs]
                else:
                    st = ctx.sort_batch(parts, cfg)
                x = torch.cat(parts)
                exp = torch.cat(exps)
                name += "/" + api
            elif api == "classic":  # LearnedSort 2.0 path (one model, two rounds, counting sort + fix-up)
                st = ctx.sort_classic(x, cfg)
                name += "/classic"
            elif api == "nan" and x.dtype == torch.float64:  # NaN: error with its first index, input untouched
                idx = sorted(int(v) for v in np.random.default_rng(seed).integers(0, n, 3))
                x[idx] = float("nan")
                before = x.clone()
                try:
                    ctx.sort(x, cfg)
                    raise AssertionError("NaN input sorted without error")
                except L.NanError as e:
                    if e.index != idx[0]:
                        raise AssertionError(f"NaN index {e.index} != {idx[0]}")
                if not torch.equal(before.view(torch.int64), x.view(torch.int64)):
                    raise AssertionError("NaN input modified")
                st = {"levels": -1, "level0_kind": -1, "ms_total": 0.0}
                x = None  # (nothing to compare: the call must fail)
                name += "/nan"
            elif world:
                crng = np.random.default_rng(seed)
                cuts = np.sort(crng.integers(0, n + 1, world - 1)) if crng.random() < 0.5 else \
                    (np.arange(1, world) * n) // world
                cuts = [0] + [int(c) for c in cuts] + [n]
                shards = [x[cuts[r]:cuts[r + 1]] for r in range(world)]
                outs, sts = sort_emulated(shards, cfg)
                st = sts[0]
                x = torch.cat(outs)
                name = f"{name}@{world}"
            else:
                st = ctx.sort(x, cfg)
        except Exception as e:  # noqa: BLE001
            print(f"FAIL {name} n={n} seed={seed} flags={flags} world={world} api={api}: {type(e).__name__}: {e}", flush=True)
            sys.exit(1)
        got = exp if x is None else ordered_i64(x)
        same = bool(torch.equal(got, exp))
        cases += 1
        print(f"{'ok  ' if same else 'DIFF'} {name:18s} n={n:>11d} seed={seed:>10d} flags={flags} levels={st['levels']} "
              f"root={st['level0_kind']} {st['ms_total']:.3f} ms ({time.time() - t0:.2f} s)", flush=True)
        if not same:
            bad = torch.nonzero(got != exp)[:5].flatten().tolist()
            print(f"first mismatches at {bad}", flush=True)
            sys.exit(1)
        del x, exp, got
        if a.cases and cases >= a.cases:
            break
        if n > 20_000_000:  # torch's cached blocks are invisible to the library's own cudaMalloc
            torch.cuda.empty_cache()
    print(f"fuzz: {cases} cases bit-exact", flush=True)


if __name__ == "__main__":
    main()
