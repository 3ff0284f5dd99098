"""CGLS on config 3 through solve_split (both folded branches concurrent):
iterations and device loop time per branch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_10559_b200 as P
from paper_1902_10559_b200.configs import CONFIGS
w = CONFIGS[int(os.environ.get("CFG", "3"))]
s = P.build_system(w.scan_config())
s.p = P.forward_project(s.a, P.rasterize(P.random_ellipses(w.seed(), 8), P.make_grid(w.scan_config())))
for dt in ("f32", "f64"):
    o = P.SolveOptions(method="cgls", max_iters=200, tol=1e-12, dtype=dt)
    P.solve_split(s, o)
    t = time.perf_counter()
    r = P.solve_split(s, o)
    wall = time.perf_counter() - t
    print(f"{dt}: iterations {r.iterations}, branches {r.branch1_seconds*1e3:.1f} / "
          f"{r.branch2_seconds*1e3:.1f} ms, call {wall*1e3:.1f} ms, "
          f"{r.iterations / max(r.branch1_seconds, r.branch2_seconds):.0f} CGLS it/s")
