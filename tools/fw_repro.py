import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2307_08637_b200 as L
from oracle import oracle as O
n, B = 100_000_000, 2048
x = L.generate("normal", n, 7)
k = O.encode(x)
samp = np.sort(k[np.random.default_rng(1).integers(0, n, 1_000_000)])
ctx = L.Context(0)
ds = torch.from_numpy(samp.view(np.int64)).cuda()
P = ctx.rmi_train(ds, B)
ref = np.sort(k)
for it in range(4):
    for mode in ("fwd", "fwd_nosample", "plain"):
        d = torch.from_numpy(k.view(np.int64)).cuda()
        if mode == "fwd": st = ctx.sort_forward(d, P, B, 0, B, ds)
        elif mode == "fwd_nosample": st = ctx.sort_forward(d, P, B, 0, B, None)
        else: st = ctx.sort(d)
        got = d.cpu().numpy().view(np.uint64)
        bad = np.nonzero(got != ref)[0]
        print(it, mode, "ok" if bad.size == 0 else f"BAD first {bad[0]} count {bad.size}", st["levels"], flush=True)
