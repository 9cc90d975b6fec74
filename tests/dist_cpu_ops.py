"""CPU stand-ins for the device steps of paper_2307_08637_b200.dist (TEST ONLY):
they let the distributed host logic (sample shares, all_gather, splitter
bounds, count exchange, all_to_all, ordering) run under gloo on CPU. They
use the oracle as the checker's arithmetic; the product never imports this."""
import numpy as np
import torch

from oracle import oracle as O


def _enc(keys):
    a = keys.numpy()
    return O.encode(a) if keys.dtype == torch.float64 else a.view(np.uint64)


class CpuOps:
    def sample(self, keys, s, seed):
        k = _enc(keys)
        n = k.size
        idx = np.array([O.lib().lso_rng_below(seed, j, n) for j in range(s)], np.uint64)
        return torch.from_numpy(k[idx.astype(np.int64)].view(np.int64).copy())

    def train(self, sample, B):
        s = np.sort(sample.numpy().view(np.uint64))
        return O.rmi_train(s, B)

    def histogram(self, keys, P, B):
        ids = O.learned_bucket(P, B, B, _enc(keys))
        return torch.from_numpy(np.bincount(ids, minlength=B).astype(np.int64))

    def partition(self, keys, P, B, bounds):
        k = _enc(keys)
        ids = O.learned_bucket(P, B, B, k)
        dest = np.searchsorted(bounds, ids, side="right") - 1
        order = np.argsort(dest, kind="stable")
        counts = np.bincount(dest, minlength=bounds.size - 1)
        return torch.from_numpy(k[order].view(np.int64).copy()), [int(c) for c in counts]

    bucket_major = True

    def partition_buckets(self, keys, P, B):
        k = _enc(keys)
        ids = O.learned_bucket(P, B, B, k)
        order = np.argsort(ids, kind="stable")
        return torch.from_numpy(k[order].view(np.int64).copy()), [int(c) for c in np.bincount(ids, minlength=B)]

    def copy_runs(self, src, dst, runs):
        s, d = src.numpy(), dst.numpy()
        for so, do, ln in np.asarray(runs, dtype=np.int64).reshape(-1, 3):
            d[do:do + ln] = s[so:so + ln]

    def sort_buckets(self, keys_u64, P, B, b_lo, b_hi, sizes, sample, cfg, to_f64=False):
        """Sorts each bucket segment on its own: the output is globally sorted
        only if the exchange put every key into its bucket's segment."""
        a = keys_u64.numpy().view(np.uint64)
        at = 0
        for j, ln in enumerate(np.asarray(sizes, dtype=np.int64)):
            seg = a[at:at + ln]
            if ln:  # every key of the segment must carry bucket b_lo + j
                assert np.all(O.learned_bucket(P, B, B, seg) == b_lo + j)
            seg.sort()
            at += ln
        assert at == a.size
        return {}

    def local_sort(self, keys_u64, cfg):
        a = keys_u64.numpy().view(np.uint64)
        a.sort()
        return {}

    def decode(self, keys_u64):
        return torch.from_numpy(O.decode(keys_u64.numpy().view(np.uint64)))


class CpuOpsRankMajor(CpuOps):
    """The destination-major exchange + whole local sort (dist.py steps 3-6)."""
    bucket_major = False
