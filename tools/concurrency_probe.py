"""Throughput of sorting the C2 arrays one after another vs concurrently
(one context + host thread per array). Device-resident inputs."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_08637_b200 as L  # noqa: E402

n = 100_000_000
src = [torch.from_numpy(L.generate(d, n, 7)).cuda() for d in ("normal", "lognormal05", "exponential2")]
work = [torch.empty_like(s) for s in src]
ctxs = [L.Context(0) for _ in src]


def run(concurrent: bool):
    for w, s in zip(work, src):
        w.copy_(s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if concurrent:
        with ThreadPoolExecutor(len(work)) as ex:
            list(ex.map(lambda i: ctxs[i].sort(work[i]), range(len(work))))
    else:
        for i in range(len(work)):
            ctxs[i].sort(work[i])
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


for mode in (False, True, False, True):
    ts = [run(mode) for _ in range(4)][1:]
    print("concurrent" if mode else "sequential", f"{np.mean(ts):.3f} ms per 3 sorts ->",
          f"{3 * n / (np.mean(ts) * 1e-3) / 1e9:.2f} Gkeys/s")
