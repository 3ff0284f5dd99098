"""SartPlan with tol > 0 (WHILE-node graph) vs the same solve without a graph:
identical iterations / history / solution; prints the replay time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1902_10559_b200 as P
from paper_1902_10559_b200.configs import CONFIGS
w = CONFIGS[int(os.environ.get('CFG', '2'))]
s = P.build_system(w.scan_config())
s.p = P.forward_project(s.a, P.rasterize(P.random_ellipses(w.seed(), 8), P.make_grid(w.scan_config())))
sp = P.split_system(s)
for tol in tuple(float(t) for t in os.environ.get('TOLS', '1e-3,1e-6,0').split(',')):
    o = P.SolveOptions(max_iters=400, tol=tol, relaxation=w.relaxation, dtype=os.environ.get("DT", "f32"))
    plan = P.SartPlan(sp.a1, sp.a2, o)
    plan.set_rhs(0, sp.p1); plan.set_rhs(1, sp.p2)
    r = plan.run()
    t = time.perf_counter(); r = plan.run(); dt = time.perf_counter() - t
    one = P.solve_split(P.CentroSystem(s.a, s.p, 0.0), o)  # direct enqueue, no graph
    f = np.concatenate([plan.solution(0), plan.solution(1)])
    fo = one.f
    print(f"tol={tol:g}: plan iterations={r.iterations} {dt*1e3:.2f} ms; solve_split iterations={one.iterations}"
          f" hist_equal={np.array_equal(plan.history(0), one.residual_history) if hasattr(one, 'residual_history') else None}")
