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

    def local_sort(self, keys_u64, cfg):
        a = keys_u64.numpy().view(np.uint64)
        a.sort()
        return {}

    def decode(self, keys_u64):
        return torch.from_numpy(O.decode(keys_u64.numpy().view(np.uint64)))
