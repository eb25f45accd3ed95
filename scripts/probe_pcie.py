"""PCIe copy rates on the box: H2D alone, D2H alone, both at once (pinned, 1 GiB)."""
import time

import torch

n = 256 * 1024 * 1024  # floats = 1 GiB
h1 = torch.empty(n, pin_memory=True)
h2 = torch.empty(n, pin_memory=True)
d1 = torch.empty(n, device="cuda")
d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def rate(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


def both():
    h2d()
    d2h()


GB = n * 4 / 1e9
t = rate(h2d); print(f"H2D alone {GB / t:.1f} GB/s")
t = rate(d2h); print(f"D2H alone {GB / t:.1f} GB/s")
t = rate(both); print(f"both at once: {2 * GB / t:.1f} GB/s total ({GB / t:.1f} each)")
