"""Cluster-persistent loop vs the two-launch loop with the same lane-group
widths (bitwise iterates) and vs the oracle; run under gpurun."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "oracle")
from helpers import oracle_workload, rel_err  # noqa: E402

import paper_1902_10559_b200 as P  # noqa: E402


def plan(sp, opts, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        pl = P.SartPlan(sp.a1, sp.a2, opts)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    pl.set_rhs(0, sp.p1)
    pl.set_rhs(1, sp.p2)
    return pl


for idx, dtype in [(1, "f64"), (1, "f32"), (2, "f32")]:
    w, cfg, a, csr, f_true, p = oracle_workload(idx, literal=False)
    s = P.build_system(w.scan_config())
    sp = P.split_system(P.CentroSystem(s.a, p, 0.0))
    opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype=dtype)
    cl = plan(sp, opts, {"SSB_PERSIST": "2"})
    d = cl.describe()
    vs = {"SSB_VS_FWD": str(d["vs_fwd"]), "SSB_VS_BACK": str(d["vs_back"])}
    ref = plan(sp, opts, dict(vs, SSB_PERSIST="0"))
    r1, r0 = cl.run(), ref.run()
    same = all(cl.solution(q).tobytes() == ref.solution(q).tobytes() for q in (0, 1))
    herr = max(float(np.max(np.abs(cl.history(q) - ref.history(q)) / np.abs(ref.history(q))))
               for q in (0, 1))
    import time
    for pl, name in ((cl, "cluster"), (ref, "two-launch")):
        pl.run()
        t = time.perf_counter()
        for _ in range(20):
            pl.run()
        dt = (time.perf_counter() - t) / 20
        print(f"cfg{idx} {dtype} {name:10s} {w.iters / dt:10.0f} it/s (wall)", flush=True)
    print(f"cfg{idx} {dtype} kernel={d['persistent_kernel']} grid={d['persistent_grid']} "
          f"bitwise={same} hist_rel={herr:.2e} iters={r1.iterations}/{r0.iterations}", flush=True)
