import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2405_19004_b200 as pmg
for (k, L, dt) in [(3, 7, "f64"), (4, 7, "f64"), (3, 7, "f32"), (4, 7, "f32"), (3, 5, "f64"), (4, 5, "f64")]:
    npdt = np.float64 if dt == "f64" else np.float32
    tdt = torch.float64 if dt == "f64" else torch.float32
    lev = pmg.make_level_context(pmg.build_hierarchy(3, k, L)[-1], dtype=npdt)
    n = lev.level.total_dofs
    x = torch.rand(n, dtype=tdt, device="cuda"); b = torch.rand(n, dtype=tdt, device="cuda"); r = torch.empty_like(x)
    for _ in range(3): pmg.compute_residual(lev, x, b, r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): pmg.compute_residual(lev, x, b, r)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    w = 8 if dt == "f64" else 4
    print(f"k={k} L={L} {dt} N={n:.3e} residual {t:.3f} ms  {3*n*w/t/1e6:.0f} GB/s  checksum {float(r.double().sum()):.10e}")
