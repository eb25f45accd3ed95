"""HBM bandwidth by access mix: write-only (fill), read-only (sum), copy (read+write)."""
import torch

n = 256 * 1024 * 1024  # 1 GiB fp32
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
a.fill_(1.0)


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


GB = n * 4 / 1e9
print(f"write-only (fill_): {GB / t(lambda: b.fill_(2.0)):.0f} GB/s")
print(f"read-only (amax): {GB / t(lambda: a.amax()):.0f} GB/s")
print(f"copy (read+write): {2 * GB / t(lambda: b.copy_(a)):.0f} GB/s")
