"""Persistent paired loop (sart_persistent_pair_kernel: one cooperative launch
per solve, grid barriers between the K1 and K2 phases) against the two
launches per pass it replaces on the L2-resident configs (SSB_PERSIST=0) and
against the oracle. Each row / column is reduced in the same tile order as the
pair kernels, so the iterates are bitwise identical; the per-CTA ||r||^2
partials group rows differently, so the history agrees to rounding."""
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
        _cache[idx] = (w, sp, csr, p)
    return _cache[idx]


def run_plan(sp, opts, persist):
    old = os.environ.get("SSB_PERSIST")
    os.environ["SSB_PERSIST"] = str(persist)
    try:
        plan = P.SartPlan(sp.a1, sp.a2, opts)
    finally:
        if old is None:
            os.environ.pop("SSB_PERSIST", None)
        else:
            os.environ["SSB_PERSIST"] = old
    plan.set_rhs(0, sp.p1)
    plan.set_rhs(1, sp.p2)
    return plan, plan.run()


@pytest.mark.parametrize("idx,dtype", [(1, "f64"), (2, "f64"), (2, "f32")])
def test_persistent_equals_two_launch_loop(idx, dtype):
    w, sp, csr, p = folded(idx)
    opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype=dtype)
    ref, rref = run_plan(sp, opts, 0)
    per, rper = run_plan(sp, opts, 1)
    assert per.describe()["persistent_kernel"].startswith("sart_persistent_pair_kernel")
    assert ref.describe()["persistent_kernel"] == ""
    assert rper.iterations == rref.iterations == w.iters
    for which in (0, 1):
        assert per.solution(which).tobytes() == ref.solution(which).tobytes()
        assert np.allclose(per.history(which), ref.history(which), rtol=1e-13, atol=0)


@pytest.mark.parametrize("tol", [0.3, 0.05])
def test_persistent_tolerance_stop(tol):
    """the stop test runs inside the kernel: same iteration, same iterate"""
    w, sp, csr, p = folded(2)
    opts = P.SolveOptions(max_iters=300, tol=tol, relaxation=w.relaxation, dtype="f64")
    ref, rref = run_plan(sp, opts, 0)
    per, rper = run_plan(sp, opts, 1)
    assert rper.iterations == rref.iterations < 300
    for which in (0, 1):
        assert per.solution(which).tobytes() == ref.solution(which).tobytes()
        assert len(per.history(which)) == len(ref.history(which))


def test_persistent_matches_oracle_and_repeats():
    w, sp, csr, p = folded(1)
    f1, f2 = O.fold_rows_csr(csr)
    p1, p2 = O.split_rhs(p)
    want, it, _ = O.solve_split_prepared(f1.to_matrix(), f2.to_matrix(), p1, p2, w.iters, 0.0,
                                         w.relaxation, True)
    opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype="f64")
    per, _ = run_plan(sp, opts, 1)
    f = per.recombine()
    assert rel_err(f, want) <= 1e-10
    for _ in range(3):  # the barrier words carry over between solves
        per.run()
        assert per.recombine().tobytes() == f.tobytes()


def test_solve_split_uses_persistent_loop_on_small_configs():
    w, sp, csr, p = folded(1)
    s = P.build_system(w.scan_config())
    r = P.solve_split(P.CentroSystem(s.a, p, 0.0),
                      P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation))
    f1, f2 = O.fold_rows_csr(csr)
    p1, p2 = O.split_rhs(p)
    want, it, _ = O.solve_split_prepared(f1.to_matrix(), f2.to_matrix(), p1, p2, w.iters, 0.0,
                                         w.relaxation, True)
    assert rel_err(r.f, want) <= 1e-10
