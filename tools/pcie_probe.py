import torch, time
n = 100_000_000
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True); h1.fill_(1)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.ones(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
a, b, c = t(h2d), t(d2h), t(both)
print(f"H2D {a:.1f} ms {8*n/a/1e6:.1f} GB/s | D2H {b:.1f} ms {8*n/b/1e6:.1f} GB/s | both {c:.1f} ms ({16*n/c/1e6:.1f} GB/s aggregate)")
