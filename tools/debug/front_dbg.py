import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2405_19004_b200 as pmg
from paper_2405_19004_b200 import _lib
L = int(sys.argv[1])
ctx = pmg.make_multigrid_context(3, 1, L)
lev = ctx.levels[-1]
n = lev.level.total_dofs
x = torch.rand(n, dtype=torch.float64, device="cuda"); b = torch.rand(n, dtype=torch.float64, device="cuda")
lib = _lib.load()
out = (ctypes.c_int * 600)()
f = lib.pmg_front_debug
f.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.c_int]


def dump(tag):
    torch.cuda.synchronize()
    print(tag, "rc", f(lev.handle, out, 600), "ctl", list(out[:4]), flush=True)
    for i in range(min(out[3], 10)):
        print("  wait timeout: (c, j2, rb) =", list(out[4+8*i:7+8*i]), "on j2', rb' =", list(out[7+8*i:9+8*i]),
              "flag", out[9+8*i], "stamp", out[10+8*i], "tk", out[11+8*i], flush=True)


for i in range(3):
    pmg.smooth(lev, x, b, "fused")
    dump(f"smooth {i}")
pmg.smooth(lev, x, b, "boundary")
dump("boundary")
for i in range(2):
    pmg.v_cycle(ctx, L - 1, x, b, use_graph=False)
    dump(f"vcycle eager {i}")
for i in range(3):
    pmg.v_cycle(ctx, L - 1, x, b, use_graph=True)
    dump(f"vcycle graph {i}")
