"""Phase timing of ss_solve_split on config 3 (SSB_TRACE=1)."""
import os, sys, time
os.environ["SSB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa
import paper_1902_10559_b200 as P
w = P.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
ctx = P.Context(0)
s = P.build_system(w.scan_config(), ctx=ctx)
f = P.rasterize(P.random_ellipses(w.seed(), 8), P.make_grid(w.scan_config()), ctx=ctx)
p = P.forward_project(s.a, f)
opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype=w.dtypes[-1])
for rep in range(int(os.environ.get("REPS", "3"))):
    t = time.perf_counter()
    P.solve_split(P.CentroSystem(s.a, p, 0.0), opts)
    print(f"--- call {rep}: {1e3*(time.perf_counter()-t):.1f} ms", file=sys.stderr, flush=True)
