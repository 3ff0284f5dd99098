"""Phase timing of the dense min-norm path on the default 32x32 system (SSB_TRACE=1)."""
import os, sys, time
os.environ["SSB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_10559_b200 as P
cfg = P.scan_config()
s = P.build_system(cfg)
print("A", s.a.shape, file=sys.stderr)
s.p = P.forward_project(s.a, P.rasterize(P.shepp_logan_ellipses(), P.make_grid(cfg)))
o = P.SolveOptions(method="dense")
for mode in ("direct", "split", "direct", "split"):
    t = time.perf_counter()
    r = (P.solve_direct if mode == "direct" else P.solve_split)(s, o)
    print(f"--- {mode}: {1e3*(time.perf_counter()-t):.1f} ms wall {r.wall_time_seconds*1e3:.1f}", file=sys.stderr)
