"""Pinned host <-> device copy bandwidth on this box (the ceiling of the e2e host-buffer path):
H2D alone, D2H alone, and both directions at once on two streams."""
import torch

n = 256 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1000.0


t = timed(lambda: d1.copy_(h1, non_blocking=True))
print(f"H2D {n / t / 1e9:.1f} GB/s")
t = timed(lambda: h2.copy_(d2, non_blocking=True))
print(f"D2H {n / t / 1e9:.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t = timed(both)
print(f"both directions {2 * n / t / 1e9:.1f} GB/s total ({n / t / 1e9:.1f} each)")
