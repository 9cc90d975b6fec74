"""CPU stand-ins for the device steps of the multi-GPU driver (TEST ONLY):
they let the distributed host logic of paper_2307_08637_b200.dist (shard
sizes, sample shares, all_gather, the global model policy, the C++ rank plan,
the fused-scatter placement, equality fills) run under gloo on CPU. They use
the oracle as the checker's arithmetic; the product never imports this."""
import numpy as np
import torch

from oracle import oracle as O

GPU_MIN_RMI = 32768   # engine_core.cuh kGpuMinRmi (GPU policy)
DIST_TREE_K = 256     # dist.cu kDistTreeK
DIST_SHARE = 16       # dist.cu kDistShare
POOR_SHARE, POOR_MEAN = 16, 4  # kernels.cuh poor_model


class Model:
    def __init__(self, kind, nb, P=None, tree=None):
        self.kind, self.nb, self.P, self.tree = kind, nb, P, tree
        self.eq = np.zeros(nb, np.uint8)
        self.eqval = np.zeros(nb, np.uint64)
        if tree is not None:  # SplitterTree equality buckets (models.hpp:96-100)
            eqo = np.frombuffer(tree.eq_offset, np.uint32)
            spl = np.frombuffer(tree.splitters, np.uint64)
            for i in range(tree.nsplitters):
                if eqo[i + 1] - eqo[i] > 1 and eqo[i] + 1 < nb:
                    self.eq[eqo[i] + 1] = 1
                    self.eqval[eqo[i] + 1] = spl[i]

    def classify(self, k):
        if self.kind == 0:
            return O.learned_bucket(self.P, self.nb, self.nb, k).astype(np.int64)
        return O.tree_classify(self.tree, k).astype(np.int64)


class CpuOps:
    def encode(self, keys):
        a = keys.numpy()
        if keys.dtype == torch.float64:
            with np.errstate(invalid="ignore"):
                a = np.where(np.isnan(a), 0.0, a)  # (NaN reported by nan_index)
            return O.encode(a)
        return a.view(np.uint64).copy()

    def nan_index(self, keys):
        if keys.dtype != torch.float64:
            return -1
        bad = np.flatnonzero(np.isnan(keys.numpy()))
        return int(bad[0]) if bad.size else -1

    def sample(self, k, s, seed):
        n = k.size
        L = O.lib()
        idx = np.array([L.lso_rng_below(seed, j, n) for j in range(s)], np.int64)
        return k[idx] if s else np.zeros(0, np.uint64)

    def global_model(self, sample, N, cfg, world):
        """Alg. 5 on the global sample with the driver's GPU
        policy: RMI unless the first sample is duplicate-heavy or N is small;
        an RMI whose largest bucket is too big for balanced rank cuts is
        replaced by a splitter tree over the same sample."""
        s = sample.size
        s1 = min(s, cfg.first_sample_cap)
        first = sample[(np.arange(s1) * s) // s1]
        dup = O.duplicate_fraction(first)
        tk = max(DIST_TREE_K, cfg.tree_bucket_count) if world > 1 else cfg.tree_bucket_count
        if N >= min(cfg.min_rmi_input, GPU_MIN_RMI) and dup <= cfg.max_duplicate_fraction:
            B = cfg.rmi_bucket_count
            P = O.rmi_train(sample, B)
            mx = int(np.bincount(O.learned_bucket(P, B, B, sample), minlength=B).max())
            poor = (mx * POOR_SHARE > s and mx * B > POOR_MEAN * s) or (world > 1 and mx * DIST_SHARE * world > s)
            if not poor:
                return Model(0, B, P=P)
            t = O.tree_build(sample, tk, True)
        else:
            t = O.tree_build(first, tk, True)
        return Model(1, t.bucket_count, tree=t)

    def local_sort(self, seg, model, b):
        """Every key of a received bucket piece must belong to that bucket."""
        if seg.size:
            assert np.all(model.classify(seg) == b), "key delivered to the wrong bucket"
        seg.sort()

    def decode(self, buf):
        return torch.from_numpy(O.decode(buf))
