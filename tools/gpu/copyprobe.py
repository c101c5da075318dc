"""Copy-bandwidth probe for the stencil COPY's layout (torch's own kernels)."""
import torch

n = 32768
g = torch.zeros(n, n, dtype=torch.float64, device="cuda")
w = torch.ones(n - 2, n - 2, dtype=torch.float64, device="cuda")
flat_a = torch.ones((n - 2) * (n - 2), dtype=torch.float64, device="cuda")
flat_b = torch.zeros_like(flat_a)
byts = 2 * 8 * (n - 2) ** 2


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


for name, fn in [
    ("flat 1-D copy", lambda: flat_b.copy_(flat_a)),
    ("interior <- work (stencil COPY layout)", lambda: g[1:-1, 1:-1].copy_(w)),
    ("work <- interior", lambda: w.copy_(g[1:-1, 1:-1])),
    ("rows aligned: g[:, :n-2] <- w-ish", lambda: g[1:-1, 0:n - 2].copy_(w)),
]:
    ms = t(fn)
    print(f"{name}: {ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s")
