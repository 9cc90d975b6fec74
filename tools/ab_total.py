"""A/B of whole-sort device time over configs and SortConfig variants, one process.

    python tools/ab_total.py --dists lognormal2:5e8,normal:1e8 --variants "bucket_target=4096;bucket_target=2048" [--reps 5]

Prints, per (dist, variant): median / min device ms of lsort_cuda_sort (no per-phase
events), Gkeys/s, and one phase-timed breakdown."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_08637_b200 as L  # noqa: E402

SEEDS = {"uniform": 42, "normal": 7, "lognormal05": 7, "exponential2": 7, "mixgauss": 11,
         "lognormal2": 19, "rootdups": 3, "twodups": 3, "zipf": 3}


def parse_variant(v):
    kw = {}
    for item in filter(None, v.split(",")):
        k, x = item.split("=")
        kw[k.strip()] = float(x) if k.strip() == "sample_fraction" else int(float(x))
    return kw


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dists", default="lognormal2:5e8")
    ap.add_argument("--variants", default="")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    variants = [v for v in a.variants.split(";")] if a.variants else [""]
    ctx = L.Context(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for item in a.dists.split(","):
        d, n = item.split(":")
        n = int(float(n))
        h = L.generate(d, n, SEEDS[d])
        p = torch.from_numpy(h.view(np.int64) if h.dtype == np.uint64 else h).cuda()
        w = torch.empty_like(p)
        for v in variants:
            cfg = L.SortConfig(**parse_variant(v))
            ts = []
            for r in range(a.reps + 1):
                w.copy_(p)
                flush.fill_(1)
                torch.cuda.synchronize()
                st = ctx.sort(w, cfg)
                if r:
                    ts.append(st["ms_total"])
            ok, _, _ = ctx.verify(w)
            cfg.flags |= L._native.FLAG_PHASE_TIMING
            w.copy_(p)
            torch.cuda.synchronize()
            ph = ctx.sort(w, cfg)
            print(f"{d:12s} n={n:.0e} [{v or 'default'}] median {np.median(ts):.3f} ms min {min(ts):.3f} ms "
                  f"-> {n / np.median(ts) / 1e6:.2f} Gkeys/s sorted={ok} levels={ph['levels']} root={ph['level0_kind']} | models "
                  f"{ph['ms_models']:.3f} classify {ph['ms_classify']:.3f} scatter {ph['ms_scatter']:.3f} "
                  f"base {ph['ms_base']:.3f} fill {ph['ms_fill']:.3f} base_keys={ph['base_case_keys']}", flush=True)
        del p, w
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
