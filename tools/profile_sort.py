"""Run the sort on one config distribution and print per-level traces / stats.

    LSORT_TRACE=1 python tools/profile_sort.py normal 100000000 [reps]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_08637_b200 as L  # noqa: E402

SEEDS = {"uniform": 42, "normal": 7, "lognormal05": 7, "exponential2": 7, "mixgauss": 11,
         "lognormal2": 19, "rootdups": 3, "twodups": 3, "zipf": 3}


def main():
    dist = sys.argv[1] if len(sys.argv) > 1 else "normal"
    n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 100_000_000
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    h = L.generate(dist, n, SEEDS[dist])
    p = torch.from_numpy(h.view(np.int64) if h.dtype == np.uint64 else h).cuda()
    w = torch.empty_like(p)
    ctx = L.Context(0)
    cfg = L.SortConfig(flags=L._native.FLAG_PHASE_TIMING)
    if os.environ.get("LSORT_TARGET"):
        cfg.bucket_target = int(os.environ["LSORT_TARGET"])
    if os.environ.get("LSORT_FLAGS"):
        cfg.flags |= int(os.environ["LSORT_FLAGS"])
    if os.environ.get("LSORT_RMI_B"):
        cfg.rmi_bucket_count = int(os.environ["LSORT_RMI_B"])
    for r in range(reps):
        w.copy_(p)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = ctx.sort(w, cfg)
        dt = time.perf_counter() - t0
        print(f"rep {r}: device {st['ms_total']:.3f} ms wall {dt*1e3:.3f} ms -> {n/st['ms_total']/1e6:.2f} Gkeys/s "
              f"levels={st['levels']} launches={st['kernel_launches']} models={st['ms_models']:.3f} "
              f"classify={st['ms_classify']:.3f} scatter={st['ms_scatter']:.3f} base={st['ms_base']:.3f} "
              f"L0 classify={st['ms_level0_classify']:.3f} L0 scatter={st['ms_level0_scatter']:.3f}",
              file=sys.stderr, flush=True)
    ok, fv, _ = ctx.verify(w)
    print("sorted:", ok, file=sys.stderr)


if __name__ == "__main__":
    main()
