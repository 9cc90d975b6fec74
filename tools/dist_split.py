"""Rank split of the multi-GPU driver at full BASELINE sizes, on ONE GPU:
lsort_cuda_dist_emulate runs p virtual ranks (contiguous shards of the config
input) through the real driver -- global model, rank cuts, the exchange fused
into the scatter, local sorts -- and reports each rank's key range, the
global model kind, and whether the concatenation is sorted (device verify).
Timing of the emulation is meaningless (the ranks share one GPU).

    python tools/dist_split.py c3 [p ...]      # C3: 2e8 MixGauss, strong split
    python tools/dist_split.py c5 [p ...]      # C5: p x 5e8 LogNormal(0,2) would not fit: 1/p of 5e8 per rank
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_08637_b200 as L  # noqa: E402
from paper_2307_08637_b200.dist import sort_emulated  # noqa: E402

CFG = {"c3": ("mixgauss", 11, 200_000_000), "c5": ("lognormal2", 19, 500_000_000),
       "c2n": ("normal", 7, 100_000_000)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    ps = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
    dist, seed, n = CFG[name]
    h = L.generate(dist, n, seed)
    x = torch.from_numpy(h).cuda()
    ctx = L.Context(0)
    _, _, h0 = ctx.verify(x)
    for p in ps:
        shards = [t.contiguous() for t in torch.tensor_split(x, p)]
        outs, stats = sort_emulated(shards, out_caps=[n // p + n // (4 * p) + 65536] * p)
        loads = [o.numel() for o in outs]
        cat = torch.cat(outs)
        ok, fv, h1 = ctx.verify(cat)
        print(json.dumps({"config": name, "dist": dist, "n": n, "p": p, "loads": loads,
                          "max_over_mean": max(loads) * p / n, "global_model": "learned" if stats[0]["level0_kind"] == 0
                          else "splitter tree", "sorted": ok, "multiset_equal": h0 == h1}), flush=True)
        del outs, cat, shards
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
