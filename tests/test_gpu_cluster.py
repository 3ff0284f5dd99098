"""Cluster-persistent paired loop (sart_cluster_pair_kernel: one 16-CTA
thread-block cluster, streams staged in shared memory, x / w replicas and the
||r||^2 partials exchanged with st.async + mbarriers) against the two-launch
loop with the same lane-group widths (bitwise iterates: each row / column is
reduced in the same tile order) and against the oracle. Config 1 is the
shape it serves by default."""
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


def make_plan(sp, opts, env, p1=None, p2=None):
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
    plan.set_rhs(0, sp.p1 if p1 is None else p1)
    plan.set_rhs(1, sp.p2 if p2 is None else p2)
    return plan


def pair(sp, opts, **rhs):
    """(cluster plan, two-launch plan with the cluster plan's lane groups)"""
    cl = make_plan(sp, opts, {}, **rhs)
    d = cl.describe()
    ref = make_plan(sp, opts, {"SSB_PERSIST": "0", "SSB_VS_FWD": str(d["vs_fwd"]),
                               "SSB_VS_BACK": str(d["vs_back"])}, **rhs)
    return cl, ref


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_cluster_equals_two_launch_loop(dtype):
    w, sp, csr, p = folded(1)
    opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype=dtype)
    cl, ref = pair(sp, opts)
    d = cl.describe()
    assert d["persistent_kernel"].startswith("sart_cluster_pair_kernel"), d
    assert d["persistent_grid"] in (8, 16)
    assert ref.describe()["persistent_kernel"] == ""
    r1, r0 = cl.run(), ref.run()
    assert r1.iterations == r0.iterations == w.iters
    for which in (0, 1):
        assert cl.solution(which).tobytes() == ref.solution(which).tobytes()
        assert np.allclose(cl.history(which), ref.history(which), rtol=1e-13, atol=0)


@pytest.mark.parametrize("tol", [0.3, 0.05])
def test_cluster_tolerance_stop(tol):
    """the stop test runs in every CTA: same iteration, same iterate"""
    w, sp, csr, p = folded(1)
    opts = P.SolveOptions(max_iters=300, tol=tol, relaxation=w.relaxation, dtype="f64")
    cl, ref = pair(sp, opts)
    r1, r0 = cl.run(), ref.run()
    assert r1.iterations == r0.iterations < 300
    for which in (0, 1):
        assert cl.solution(which).tobytes() == ref.solution(which).tobytes()
        assert len(cl.history(which)) == len(ref.history(which))


def test_cluster_one_system_stops_first():
    """system 2 gets a zero right-hand side: ||r|| = 0 <= tol * 0 stops it at
    iteration 0 while system 1 runs on (independent stop state per system)"""
    w, sp, csr, p = folded(1)
    opts = P.SolveOptions(max_iters=40, tol=1e-3, relaxation=w.relaxation, dtype="f64")
    z = np.zeros_like(np.asarray(sp.p2))
    cl, ref = pair(sp, opts, p2=z)
    r1, r0 = cl.run(), ref.run()
    assert r1.iterations == r0.iterations > 1
    assert len(cl.history(1)) == 1
    for which in (0, 1):
        assert cl.solution(which).tobytes() == ref.solution(which).tobytes()
        assert len(cl.history(which)) == len(ref.history(which))


def test_cluster_divergence_reported_like_two_launch_loop():
    w, sp, csr, p = folded(1)
    opts = P.SolveOptions(max_iters=10, tol=0.0, relaxation=w.relaxation, dtype="f64")
    bad = np.array(sp.p1, dtype=np.float64)
    bad[7] = np.nan
    msgs = []
    for plan in pair(sp, opts, p1=bad):
        with pytest.raises(P.Error) as e:
            plan.run()
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1] and "diverged (non-finite iterate at iteration" in msgs[0], msgs


def test_cluster_matches_oracle_and_repeats():
    w, sp, csr, p = folded(1)
    f1, f2 = O.fold_rows_csr(csr)
    p1, p2 = O.split_rhs(p)
    want, it, _ = O.solve_split_prepared(f1.to_matrix(), f2.to_matrix(), p1, p2, w.iters, 0.0,
                                         w.relaxation, True)
    opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype="f64")
    cl = make_plan(sp, opts, {})
    cl.run()
    f = cl.recombine()
    assert rel_err(f, want) <= 1e-10
    for _ in range(3):  # mbarriers are re-initialised per launch
        cl.run()
        assert cl.recombine().tobytes() == f.tobytes()
    opts32 = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype="f32")
    c32 = make_plan(sp, opts32, {})
    c32.run()
    assert rel_err(c32.recombine(), want) <= 1e-4


def test_cluster_not_chosen_when_a_pass_does_not_fit():
    """config 2 (6,144 rows x 32,768 columns per system) stays on the grid-wide
    persistent kernel even when the cluster kernel is requested"""
    w, sp, csr, p = folded(2)
    opts = P.SolveOptions(max_iters=5, tol=0.0, relaxation=w.relaxation, dtype="f32")
    plan = make_plan(sp, opts, {"SSB_PERSIST": "2"})
    assert not plan.describe()["persistent_kernel"].startswith("sart_cluster")
    plan.run()
