"""Stream-resident persistent loop (sart_resident_pair_kernel: one CTA per SM,
each CTA's share of both mirror-coded streams staged in shared memory once per
launch, grid barriers between the K1 and K2 phases) against the two launches
per pass (SSB_PERSIST=0), the L2-streamed grid kernel (SSB_PERSIST=1) and the
oracle. Rows and columns keep the pair kernels' tile order, so the iterates
are bitwise identical; the per-CTA ||r||^2 partials group rows differently, so
the history agrees to rounding."""
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


def run_plan(sp, opts, persist, **env):
    env = dict(env, SSB_PERSIST=str(persist))
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
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
    return plan, plan.run()


@pytest.mark.parametrize("idx,dtype,env", [
    (1, "f64", {}), (1, "f32", {}), (2, "f32", {}), (2, "f64", {}),
    (2, "f64", {"SSB_VS_FWD": 16, "SSB_VS_BACK": 8}),
    (2, "f32", {"SSB_VS_FWD": 16, "SSB_VS_BACK": 8}),
    (2, "f32", {"SSB_VS_FWD": 32, "SSB_VS_BACK": 16}),
])
def test_resident_equals_two_launch_loop(idx, dtype, env):
    w, sp, csr, p = folded(idx)
    opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype=dtype)
    ref, rref = run_plan(sp, opts, 0, **env)
    res, rres = run_plan(sp, opts, 3, **env)
    d = res.describe()
    assert d["persistent_kernel"].startswith("sart_resident_pair_kernel"), d
    assert ref.describe()["persistent_kernel"] == ""
    assert rres.iterations == rref.iterations == w.iters
    for which in (0, 1):
        assert res.solution(which).tobytes() == ref.solution(which).tobytes()
        assert np.allclose(res.history(which), ref.history(which), rtol=1e-13, atol=0)


def test_resident_is_the_default_for_config2():
    """auto selection: config 2's fp32 streams fit the GPU's shared memory
    (both staged); of the fp64 streams only K1's fits (K2 streams from L2)"""
    w, sp, csr, p = folded(2)
    for dtype, tail in (("f32", ", 2, true>"), ("f64", ", 2, false>")):
        opts = P.SolveOptions(max_iters=5, tol=0.0, relaxation=w.relaxation, dtype=dtype)
        plan, _ = run_plan(sp, opts, -1)
        name = plan.describe()["persistent_kernel"]
        assert name.startswith("sart_resident_pair_kernel") and name.endswith(tail), name


@pytest.mark.parametrize("tol,dtype", [(0.3, "f32"), (0.05, "f32"), (0.05, "f64")])
def test_resident_tolerance_stop(tol, dtype):
    """the stop test runs inside the kernel: same iteration, same iterate"""
    w, sp, csr, p = folded(2)
    opts = P.SolveOptions(max_iters=300, tol=tol, relaxation=w.relaxation, dtype=dtype)
    ref, rref = run_plan(sp, opts, 0)
    res, rres = run_plan(sp, opts, 3)
    assert res.describe()["persistent_kernel"].startswith("sart_resident_pair_kernel")
    assert rres.iterations == rref.iterations < 300
    for which in (0, 1):
        assert res.solution(which).tobytes() == ref.solution(which).tobytes()
        assert len(res.history(which)) == len(ref.history(which))


def test_resident_matches_oracle_and_repeats():
    w, sp, csr, p = folded(2)
    f1, f2 = O.fold_rows_csr(csr)
    p1, p2 = O.split_rhs(p)
    want, it, _ = O.solve_split_prepared(f1.to_matrix(), f2.to_matrix(), p1, p2, w.iters, 0.0,
                                         w.relaxation, True)
    opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype="f32")
    res, _ = run_plan(sp, opts, 3)
    assert res.describe()["persistent_kernel"].startswith("sart_resident_pair_kernel")
    first = np.concatenate([res.solution(0), res.solution(1)])
    res.set_rhs(0, sp.p1)
    res.set_rhs(1, sp.p2)
    res.run()  # a reusable plan replays its graph: the streams are staged again, same result
    again = np.concatenate([res.solution(0), res.solution(1)])
    assert first.tobytes() == again.tobytes()
    got = P.recombine_solution(res.solution(0), res.solution(1))
    assert rel_err(got, want) <= 1e-4


def plan_with(sp, opts, persist, p1=None, p2=None):
    old = os.environ.get("SSB_PERSIST")
    os.environ["SSB_PERSIST"] = str(persist)
    try:
        plan = P.SartPlan(sp.a1, sp.a2, opts)
    finally:
        if old is None:
            os.environ.pop("SSB_PERSIST", None)
        else:
            os.environ["SSB_PERSIST"] = old
    plan.set_rhs(0, sp.p1 if p1 is None else p1)
    plan.set_rhs(1, sp.p2 if p2 is None else p2)
    return plan


def test_resident_one_system_stops_first():
    """system 2 gets a zero right-hand side: ||r|| = 0 <= tol * 0 stops it at
    iteration 0 while system 1 runs on (independent stop state per system)"""
    w, sp, csr, p = folded(2)
    opts = P.SolveOptions(max_iters=40, tol=1e-3, relaxation=w.relaxation, dtype="f32")
    z = np.zeros_like(np.asarray(sp.p2))
    res, ref = plan_with(sp, opts, 3, p2=z), plan_with(sp, opts, 0, p2=z)
    assert res.describe()["persistent_kernel"].startswith("sart_resident_pair_kernel")
    r1, r0 = res.run(), ref.run()
    assert r1.iterations == r0.iterations > 1
    assert len(res.history(1)) == 1
    for which in (0, 1):
        assert res.solution(which).tobytes() == ref.solution(which).tobytes()
        assert len(res.history(which)) == len(ref.history(which))


def test_resident_divergence_reported_like_two_launch_loop():
    """a non-finite update seen by one CTA turns that system off in every CTA
    (its -1 partial in the next pass's exchange); the report names the same
    iteration as the two-launch loop's"""
    w, sp, csr, p = folded(2)
    opts = P.SolveOptions(max_iters=10, tol=0.0, relaxation=w.relaxation, dtype="f32")
    bad = np.array(sp.p1, dtype=np.float64)
    bad[7] = np.nan
    msgs = []
    for persist in (3, 0):
        plan = plan_with(sp, opts, persist, p1=bad)
        with pytest.raises(P.Error) as e:
            plan.run()
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1] and "diverged (non-finite iterate at iteration" in msgs[0], msgs
