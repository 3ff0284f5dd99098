"""Single-system SART plan (one folded system of config 3, as on each rank of a
2-GPU run, or sart_solve) — SSB_TILED=0/1 A/B; prints it/s and the layout."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_10559_b200 as P
from paper_1902_10559_b200.configs import CONFIGS
w = CONFIGS[int(os.environ.get("CFG", "3"))]
dtype = os.environ.get("DTYPE", "f32")
ctx = P.Context(0)
s = P.build_system(w.scan_config(), ctx=ctx)
f = P.rasterize(P.random_ellipses(w.seed(), 8), P.make_grid(w.scan_config()), ctx=ctx)
s.p = P.forward_project(s.a, f)
sp = P.split_system(s)
plan = P.SartPlan(sp.a1, None, P.SolveOptions(max_iters=w.iters, tol=0.0,
                                               relaxation=w.relaxation, dtype=dtype))
plan.set_rhs(0, sp.p1)
for _ in range(3):
    plan.run()
t = time.perf_counter()
n = 10
for _ in range(n):
    plan.launch()
plan.finish()
dt = time.perf_counter() - t
d = plan.describe()
fms, bms = plan.profile(20)
print(f"{d['layout']:16s} {n * w.iters / dt:9.1f} it/s  fwd {fms / 20 * 1e3:.1f} us  back {bms / 20 * 1e3:.1f} us  "
      f"{d['fwd_kernel']} / {d['back_kernel']}")
