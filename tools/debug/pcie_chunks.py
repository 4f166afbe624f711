"""Chunked bidirectional PCIe pattern of the pipelined *_host smoother without
the compute: H2D (x, b) chunk i on one stream, D2H x chunk i on another after
an event, for several chunkings. Bounds what the pipeline can reach."""
import time

import torch

m = 127
pl = m * m
n = m * pl
hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
hb = torch.empty(n, dtype=torch.float64, pin_memory=True)
dx = torch.empty(n, dtype=torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(bounds, lag):
    # bounds: dof-plane boundaries of the H2D chunks; D2H of chunk i covers planes
    # up to bounds[i] - lag (the trailing colours), the last one everything
    evs = []
    with torch.cuda.stream(s1):
        for i in range(1, len(bounds)):
            a, b = bounds[i - 1] * pl, bounds[i] * pl
            dx[a:b].copy_(hx[a:b], non_blocking=True)
            db[a:b].copy_(hb[a:b], non_blocking=True)
            e = torch.cuda.Event()
            e.record(s1)
            evs.append(e)
    done = 0
    with torch.cuda.stream(s2):
        for i in range(1, len(bounds)):
            s2.wait_event(evs[i - 1])
            fin = m if i == len(bounds) - 1 else max(0, bounds[i] - lag)
            if fin > done:
                hx[done * pl:fin * pl].copy_(dx[done * pl:fin * pl], non_blocking=True)
                done = fin


def t(f, reps=20):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


for name, bounds in [("pipeline 6 (shrinking)", [0, 42, 76, 102, 122, 127]),
                     ("equal 4", [0, 32, 64, 96, 127]), ("equal 8", [0, 16, 32, 48, 64, 80, 96, 112, 127]),
                     ("equal 16", list(range(0, 127, 8)) + [127]), ("growing 6", [0, 8, 24, 48, 80, 127]),
                     ("one chunk", [0, 127])]:
    ms = t(lambda: run(bounds, 14))
    print(f"{name:26s} {ms:.3f} ms  -> {n / ms / 1e6:.2f} GDoF/s bound", flush=True)
