import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_08637_b200 as L
ctx = L.Context(0)
for dists, seed, kind in [(["normal","lognormal05","exponential2"], 7, "f64"), (["rootdups","twodups","zipf"], 3, "u64")]:
    hs = [L.generate(d, 100_000_000, seed) for d in dists]
    ps = [torch.from_numpy(h.view(np.int64) if h.dtype == np.uint64 else h).cuda() for h in hs]
    ws = [torch.empty_like(p) for p in ps]
    ts = []
    for r in range(4):
        for w, p in zip(ws, ps): w.copy_(p)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.sort_batch(ws)
        e1.record(); torch.cuda.synchronize()
        if r: ts.append(e0.elapsed_time(e1))
    print(dists[0], os.environ.get("LSORT_MANY_WAYS", "default"), "median ms", np.median(ts), "Gkeys/s", 3e8 / np.median(ts) / 1e6, flush=True)
