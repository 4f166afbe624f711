import sys
sys.path.insert(0, '.')
sys.argv = ['x'] + sys.argv[1:]
import paper_2405_19004_b200 as pmg
from tools.vcycle_levels import vtime
k = int(sys.argv[1]); dt = sys.argv[2]
for impl in ["auto", "patch", "line", "plane"]:
    pmg.set_smoother_impl(impl)
    prev = 0
    out = []
    for L in range(1, 7):
        try:
            n, t = vtime(3, k, L, dt, 50)
        except Exception as e:
            out.append("err"); continue
        out.append(f"L{L}:+{(t-prev)*1e3:.1f}")
        prev = t
    print(impl, k, dt, " ".join(out), f"total {prev*1e3:.1f} us", flush=True)
