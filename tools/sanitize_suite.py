"""Small end-to-end run of every device kernel family, sized for
compute-sanitizer (one tool per gpurun call; run it plainly first):

  python tools/sanitize_suite.py && \
  compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_suite.py

Covers: Siddon build, rasterize, folded forward projection (+ noise), the
symmetry-checked fold, CSC, paired mirror-coded SART (fp64 / fp32, graph and
direct), tolerance-stopped WHILE-loop plans, single-system tiled plans,
multi-RHS plans, CGLS (paired and single), dense min-norm, recombine, and the
peer-exchange row-sharded kernels (emulated group of 3 ranks)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_10559_b200 as P  # noqa: E402
from paper_1902_10559_b200.configs import CONFIGS  # noqa: E402

w = CONFIGS[1]
cfg = w.scan_config()
s = P.build_system(cfg)
f_true = P.rasterize(P.random_ellipses(w.seed(), 8), P.make_grid(cfg))
p = P.forward_project(s.a, f_true, 0.01, 7)
sysm = P.CentroSystem(s.a, p, 0.0)
sp = P.split_system(sysm)
for dtype in ("f64", "f32"):
    o = P.SolveOptions(max_iters=12, tol=0.0, relaxation=w.relaxation, dtype=dtype)
    r = P.solve_split(sysm, o)                            # direct-enqueue paired loop
    plan = P.SartPlan(sp.a1, sp.a2, o)                    # graph-replayed paired loop
    plan.set_rhs(0, sp.p1)
    plan.set_rhs(1, sp.p2)
    plan.run()
    ot = P.SolveOptions(max_iters=40, tol=0.3, relaxation=w.relaxation, dtype=dtype)
    pt = P.SartPlan(sp.a1, sp.a2, ot)                     # WHILE-node loop, device stop
    pt.set_rhs(0, sp.p1)
    pt.set_rhs(1, sp.p2)
    pt.run()
    P.sart_solve(sp.a1, sp.p1, o)                         # single-system tiled plan
    mp = P.SartPlan(sp.a1, sp.a2, o, nrhs=4)              # multi-RHS
    mp.set_rhs(0, np.tile(sp.p1, 4))
    mp.set_rhs(1, np.tile(sp.p2, 4))
    mp.run()
    oc = P.SolveOptions(max_iters=12, tol=1e-12, method="cgls", dtype=dtype)
    P.solve_split(sysm, oc)
    P.cgls_solve(sp.a1, sp.p1, oc)
    grp = P.symsplit.ShardGroup(sp.a2, 3, o)              # peer exchange, 3 emulated ranks
    grp.set_rhs(sp.p2)
    grp.run()
small = P.Matrix.dense(np.array([[4.0, 1.0, 0.0], [2.0, 5.0, 1.0], [0.0, 1.0, 4.0]]))
P.pseudo_solve_dense(small, np.array([1.0, 2.0, 3.0]))
print("sanitize suite ok", r.iterations)
