"""HBM probe for the read/write mixes of the benchmark kernels (torch's own kernels)."""
import torch

n = 1_000_000_000
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.rand(n, dtype=torch.float64, device="cuda")
z = torch.empty_like(x)


def t(fn, reps=8):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


for name, fn, byts in [
    ("copy 1R1W", lambda: z.copy_(x), 16 * n),
    ("add 2R1W (BS mix)", lambda: torch.add(x, y, out=z), 24 * n),
    ("sum 1R (reduction)", lambda: x.sum(), 8 * n),
    ("fill 1W", lambda: z.fill_(1.0), 8 * n),
]:
    ms = t(fn)
    print(f"{name}: {ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s")
