import os, sys
sys.path.insert(0, "."); sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
import numpy as np, pyoracle as O
from helpers import oracle_workload, rel_err
import paper_1902_10559_b200 as P
w, cfg, a, csr, f_true, p = oracle_workload(1)
s = P.build_system(w.scan_config())
sp = O.split_system(a, p, 0.0)
gs = P.split_system(P.CentroSystem(s.a, p, 0.0))
for it in (1, 2, 3, 5, 10, 20, 30):
    o = O.cgls_solve(sp.a2, sp.p2, max_iters=it, tol=1e-10)
    g = P.cgls_solve(gs.a2, gs.p2, P.SolveOptions(method="cgls", max_iters=it, tol=1e-10))
    print(it, f"rel_err f {rel_err(g.f, o.f):.2e}  res {g.residual_norm:.6e} vs {o.residual_norm:.6e}")
