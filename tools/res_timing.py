import os, sys
sys.path.insert(0, "/root/repo")
import paper_1902_10559_b200 as P
idx = int(sys.argv[1]); dtype = sys.argv[2]
w = P.CONFIGS[idx]
ctx = P.Context(0)
s = P.build_system(w.scan_config(), ctx=ctx)
f = P.rasterize(P.random_ellipses(w.seed(), 8), P.make_grid(w.scan_config()), ctx=ctx)
p = P.forward_project(s.a, f)
sp = P.split_system(P.CentroSystem(s.a, p, 0.0))
opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype=dtype)
plan = P.SartPlan(sp.a1, sp.a2, opts)
plan.set_rhs(0, sp.p1); plan.set_rhs(1, sp.p2)
print(plan.describe()["persistent_kernel"], file=sys.stderr)
for _ in range(3):
    plan.run()
