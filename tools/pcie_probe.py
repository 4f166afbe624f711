"""PCIe transfer probe: pinned H2D alone, D2H alone, both at once on two
streams (the bound of the pipelined *_host smoother), 16 MiB x 2 in / 16 MiB out."""
import time

import torch

n = 2048383
hx = torch.empty(2 * n, dtype=torch.float64, pin_memory=True)
hy = torch.empty(n, dtype=torch.float64, pin_memory=True)
dx = torch.empty(2 * n, dtype=torch.float64, device="cuda")
dy = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(f, reps=20):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def h2d():
    with torch.cuda.stream(s1):
        dx.copy_(hx, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        hy.copy_(dy, non_blocking=True)


def both():
    h2d()
    d2h()


a, b, c = t(h2d), t(d2h), t(both)
print(f"H2D {2 * n * 8 / 1e6:.1f} MB: {a:.3f} ms ({2 * n * 8 / a / 1e6:.1f} GB/s); "
      f"D2H {n * 8 / 1e6:.1f} MB: {b:.3f} ms ({n * 8 / b / 1e6:.1f} GB/s); both concurrently {c:.3f} ms "
      f"(serial sum {a + b:.3f})")
