"""HBM read-only / write-only / copy bandwidth on this GPU (torch kernels,
CUDA events, best of 10) — the denominators behind the write-heavy SDD."""
import torch

n = 1 << 30  # bytes
a = torch.empty(n // 2, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
a.normal_()


def t(fn, reps=10):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best / 1e3


w = t(lambda: b.fill_(1.0))
r = t(lambda: a.view(torch.int64).sum())
c = t(lambda: b.copy_(a))
print(f"write-only {n / w / 1e9:.0f} GB/s, read-only {n / r / 1e9:.0f} GB/s, copy {2 * n / c / 1e9:.0f} GB/s (read+write)")
