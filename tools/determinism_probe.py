"""Same input sorted several times in one process: the statistics that depend on the
partition models (levels, segments, base-case segments, fill keys) must repeat.

    python tools/determinism_probe.py name:n:seed:flags [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2307_08637_b200 as L  # noqa: E402
import fuzz_sort as F  # noqa: E402

name, n, seed, flags = sys.argv[1].split(":")[:4]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dev = torch.device("cuda:0")
g = torch.Generator(device=dev)
g.manual_seed(int(seed))
x0 = F.draw(g, name, int(n), dev)
ctx = L.Context(0)
keys = ("levels", "level0_kind", "segments", "base_segments", "base_case_keys", "fill_keys", "partitioned_keys",
        "direct_keys")
seen = set()
for r in range(reps):
    x = x0.clone()
    cfg = L.SortConfig()
    cfg.flags |= int(flags)
    st = ctx.sort(x, cfg)
    sig = tuple(st[k] for k in keys)
    seen.add(sig)
    print(r, dict(zip(keys, sig)), f"{st['ms_total']:.3f} ms", flush=True)
print("deterministic" if len(seen) == 1 else f"NOT deterministic: {len(seen)} distinct statistics")
