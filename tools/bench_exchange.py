"""Cost of the row-sharded exchange on one GPU (one folded system of config
CFG, as one group of a multi-GPU run holds it):

  unsharded      SartPlan on the whole system (no exchange at all)
  nccl G=1       ss_plan_create_sharded_x(NCCL): K2 partial + 1-rank ncclAllReduce + update
  peer G=1       ss_plan_create_sharded_x(PEER): fused exchange kernels, graph-captured
  peer emul G    ShardGroup: G ranks' kernels issued in rank order on one stream
                 (the per-iteration work of all G ranks serialised on one GPU,
                 so its time ~ unsharded + the exchange's extra passes)

Prints it/s per variant (CUDA-event loop time, min of REPS solves)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401,E402  (PyTorch's NCCL first)
import paper_1902_10559_b200 as P  # noqa: E402
from paper_1902_10559_b200.configs import CONFIGS  # noqa: E402

w = CONFIGS[int(os.environ.get("CFG", "3"))]
dtype = os.environ.get("DTYPE", "f32")
iters = int(os.environ.get("ITERS", str(w.iters)))
reps = int(os.environ.get("REPS", "5"))
ctx = P.Context(0)
s = P.build_system(w.scan_config(), ctx=ctx)
f = P.rasterize(P.random_ellipses(w.seed(), 8), P.make_grid(w.scan_config()), ctx=ctx)
s.p = P.forward_project(s.a, f)
sp = P.split_system(s)
opts = P.SolveOptions(max_iters=iters, tol=0.0, relaxation=w.relaxation, dtype=dtype)
rows = sp.a1.shape[0]
out = {"config": w.index, "dtype": dtype, "iters": iters, "rows": rows, "cols": sp.a1.shape[1]}


def timed(run, plans_ms):
    best = None
    for _ in range(reps + 1):
        run()
        ms = plans_ms()
        best = ms if best is None else min(best, ms)
    return round(iters / (best * 1e-3), 1)


only = os.environ.get("ONLY", "")
ref = P.SartPlan(sp.a1, None, opts)
ref.set_rhs(0, sp.p1)
out["unsharded"] = timed(lambda: ref.run(), lambda: ref.finish().wall_time_seconds * 1e3)
f_ref = ref.solution(0)
fms, bms = ref.profile(20)
out["unsharded_fwd_back_us"] = [round(fms / 20 * 1e3, 1), round(bms / 20 * 1e3, 1)]

P.symsplit.attach_nccl(ctx, P.symsplit.nccl_unique_id(), 1, 0)
for name, x in (("nccl_g1", "nccl"), ("peer_g1", "peer")):
    if only and name not in only.split(","):
        continue
    pl = P.symsplit.ShardedSartPlan(ctx, sp.a1, 0, rows, opts, exchange=x)
    pl.set_rhs(0, sp.p1)
    out[name] = timed(lambda: pl.run(), lambda: pl.finish().wall_time_seconds * 1e3)
    d = P.symsplit.np.linalg.norm(pl.solution(0) - f_ref) / P.symsplit.np.linalg.norm(f_ref)
    out[name + "_rel_err"] = float(d)
    fms, bms = pl.profile(20)
    out[name + "_fwd_back_us"] = [round(fms / 20 * 1e3, 1), round(bms / 20 * 1e3, 1)]
    del pl

groups = [int(v) for v in os.environ.get("GROUPS", "2,4").split(",") if v]
for g in groups:
    if only and f"peer_emul_g{g}" not in only.split(","):
        continue
    grp = P.symsplit.ShardGroup(sp.a1, g, opts)
    grp.set_rhs(sp.p1)
    out[f"peer_emul_g{g}"] = timed(lambda: grp.run(),
                                   lambda: grp.ranks[0].finish().wall_time_seconds * 1e3)
    d = P.symsplit.np.linalg.norm(grp.solution(0) - f_ref) / P.symsplit.np.linalg.norm(f_ref)
    out[f"peer_emul_g{g}_rel_err"] = float(d)
    del grp
print(json.dumps(out))
