"""CGLS 64x64 K=48 (acceptance criterion 7) direct vs split timings."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_10559_b200 as P
cfg64 = P.scan_config(k=48, grid_nx=64, grid_ny=64)
s = P.build_system(cfg64)
s.p = P.forward_project(s.a, P.rasterize(P.shepp_logan_ellipses(), P.make_grid(cfg64)))
cg = P.SolveOptions(method="cgls", tol=1e-8, max_iters=4000)
for _ in range(3):
    d = P.solve_direct(s, cg)
    sp = P.solve_split(s, cg)
print("direct", d.iterations, round(d.wall_time_seconds * 1e3, 2), "ms; split", sp.iterations,
      round(sp.wall_time_seconds * 1e3, 2), "ms", round(sp.branch1_seconds * 1e3, 2), round(sp.branch2_seconds * 1e3, 2))
