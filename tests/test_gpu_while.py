"""Reusable plans with tol > 0 run the SART loop as a CUDA-graph WHILE node
(8 unrolled passes per body, the loop ends on the device). When no system
reaches the tolerance the loop must still apply all max_iters updates, like
sart_solve (proj/src/solvers.cpp:178-191: check-before-update, then update, on
every iteration): the final pass's back-projection runs after K1 has ended the
loop. Checked against the oracle for the two-launch plans (the WHILE path) and
the persistent kernels, for max_iters on and off the 8-pass body boundary."""
import os

import numpy as np
import pytest

import pyoracle as O
from helpers import oracle_workload, rel_err

import paper_1902_10559_b200 as P

pytestmark = pytest.mark.gpu

_cache = {}


def folded(idx):
    if idx not in _cache:
        w, cfg, a, csr, f_true, p = oracle_workload(idx, literal=False)
        s = P.build_system(w.scan_config())
        sp = P.split_system(P.CentroSystem(s.a, p, 0.0))
        f1, f2 = O.fold_rows_csr(csr)
        _cache[idx] = (w, sp, f1.to_matrix(), f2.to_matrix())
    return _cache[idx]


def plan_with(env, sp, opts):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        plan = P.SartPlan(sp.a1, sp.a2, opts)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    plan.set_rhs(0, sp.p1)
    plan.set_rhs(1, sp.p2)
    return plan


@pytest.mark.parametrize("idx,iters", [(1, 8), (1, 13), (1, 40), (2, 17)])
@pytest.mark.parametrize("persist", ["0", "1", "-1"])
def test_tolerance_not_reached_runs_every_update(idx, iters, persist):
    w, sp, m1, m2 = folded(idx)
    tol = 1e-9  # far below what these iteration counts reach
    opts = P.SolveOptions(max_iters=iters, tol=tol, relaxation=w.relaxation, dtype="f64")
    plan = plan_with({"SSB_PERSIST": persist}, sp, opts)
    rep = plan.run()
    assert rep.iterations == iters
    for which, (m, p) in enumerate(((m1, sp.p1), (m2, sp.p2))):
        want = O.sart_solve(m, p, iters, tol, w.relaxation)
        assert want.iterations == iters
        assert rel_err(plan.solution(which), want.f) <= 1e-10
        h = plan.history(which)
        assert len(h) == len(want.residual_history) == iters
        assert np.allclose(h, want.residual_history, rtol=1e-10, atol=0)


@pytest.mark.parametrize("staged", ["1", "0"])
def test_multi_rhs_tolerance_not_reached_runs_every_update(staged):
    """the same for a multi-RHS plan (staged or per-vector kernels): every
    slice equals its own oracle solve after all max_iters updates"""
    w, sp, m1, m2 = folded(1)
    S, iters, tol = 32, 11, 1e-9
    rng = np.random.default_rng(5)
    scale = rng.uniform(0.5, 1.5, size=S)
    p1 = np.concatenate([np.asarray(sp.p1) * c for c in scale])
    p2 = np.concatenate([np.asarray(sp.p2) * c for c in scale])
    opts = P.SolveOptions(max_iters=iters, tol=tol, relaxation=w.relaxation, dtype="f64")
    env = {"SSB_STAGED": staged, "SSB_BLOCKED": "0"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        plan = P.SartPlan(sp.a1, sp.a2, opts, nrhs=S)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    d = plan.describe()
    assert ("stage" in d["fwd_kernel"]) == (staged == "1"), d
    plan.set_rhs(0, p1)
    plan.set_rhs(1, p2)
    assert plan.run().iterations == iters
    x1 = plan.solution(0).reshape(S, -1)
    x2 = plan.solution(1).reshape(S, -1)
    for sl in (0, 13, S - 1):
        want1 = O.sart_solve(m1, np.asarray(sp.p1) * scale[sl], iters, tol, w.relaxation)
        want2 = O.sart_solve(m2, np.asarray(sp.p2) * scale[sl], iters, tol, w.relaxation)
        assert rel_err(x1[sl], want1.f) <= 1e-10
        assert rel_err(x2[sl], want2.f) <= 1e-10
        assert len(plan.history(0, sl)) == iters
