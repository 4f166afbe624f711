import sys
sys.path.insert(0, '.')
import paper_2405_19004_b200 as pmg
from tools.quick_time import run
for dt in ("f64", "f32"):
    for L in (4, 5, 6, 7, 8, 9):
        for impl in ("auto", "plane"):
            pmg.set_smoother_impl(impl)
            print(impl, end=" ")
            run(3, 1, L, dt, "fused")
pmg.set_smoother_impl("auto")
