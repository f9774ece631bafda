"""Practical HBM ceilings for the two-kernel access patterns (torch, CUDA events)."""
import torch

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3

n = 1 << 30  # 8 GiB of doubles
x = torch.empty(n, dtype=torch.float64, device="cuda").uniform_()
y8 = torch.empty(n // 8, dtype=torch.float64, device="cuda")
big = torch.empty(n, dtype=torch.float64, device="cuda")
s = t(lambda: torch.sum(x.view(-1, 8), dim=1, out=y8))
print(f"read 8 / write 1 (evolve-like): {(n + n // 8) * 8 / s / 1e9:.0f} GB/s")
s = t(lambda: big.view(-1, 8).copy_(y8.view(-1, 1).expand(-1, 8)))
print(f"read 1 / write 8 (recon-like):  {(n + n // 8) * 8 / s / 1e9:.0f} GB/s")
s = t(lambda: big.copy_(x))
print(f"copy (read 1 / write 1):        {2 * n * 8 / s / 1e9:.0f} GB/s")
s = t(lambda: torch.sum(x))
print(f"read only (sum):                {n * 8 / s / 1e9:.0f} GB/s")
