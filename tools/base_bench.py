"""Base-case throughput in isolation: B segments of S keys each, every segment
a contiguous range of the sorted order shuffled in place (as a partition
level leaves them), sorted by lsort_cuda_sort_buckets (all buckets within the
base-case capacity: base-case kernels only). Prints ns/key and GB/s (16 B/key).

    python tools/base_bench.py [S ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_08637_b200 as L  # noqa: E402


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [512, 1024, 2048, 3000, 4096, 6000, 8192, 12000, 16384]
    ctx = L.Context(0)
    rng = np.random.default_rng(1)
    B = 2048
    P = np.zeros(4 + 4 * B)
    P[3] = 1.0
    P[4 + 1::4] = 0.5
    P[4 + 2::4] = 0.5
    P[4 + 3::4] = 0.5
    for S in sizes:
        n = B * S
        keys = np.sort(rng.integers(0, 2**62, n, dtype=np.uint64))
        keys = keys.reshape(B, S)
        keys = np.ascontiguousarray(rng.permuted(keys, axis=1)).reshape(-1)
        src = torch.from_numpy(keys.view(np.int64)).cuda()
        w = torch.empty_like(src)
        sizes_arr = np.full(B, S, np.uint64)
        ts = []
        for r in range(6):
            w.copy_(src)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.sort_buckets(w, P, B, 0, B, sizes_arr, None, L.SortConfig())
            e1.record()
            torch.cuda.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        ok, _, _ = ctx.verify(w)
        ms = float(np.median(ts))
        print(f"S={S:6d} n={n:9d} {ms:.3f} ms  {ms * 1e6 / n:.3f} ns/key  {16 * n / ms / 1e6:.0f} GB/s sorted={ok}",
              flush=True)


if __name__ == "__main__":
    main()
