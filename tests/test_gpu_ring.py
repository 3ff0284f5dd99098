"""TMA-fed ring kernels (csrc/ring.cuh) against the register-streamed paired
kernels they replace (SSB_RING=0) and against the oracle.

Both kernel families reduce every row / column in the same tile order with the
same butterfly, so a ring plan must reproduce the pair plan bit for bit
(fp32 and fp64), including the residual history and a tolerance stop on the
device (WHILE-loop graph). Small slot capacities and 2-3 stages force many
chunks per CTA and consumer groups running several chunks ahead of the
slowest one (the slot-ownership check of the ring protocol)."""
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


def run_plan(sp, opts, env):
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
    rep = plan.run()
    return plan, rep


@pytest.mark.parametrize("idx,dtype", [(1, "f64"), (2, "f64"), (2, "f32"), (3, "f32"),
                                       (3, "f64")])
def test_ring_equals_pair_kernels(idx, dtype):
    w, sp, csr, p = folded(idx)
    iters = min(w.iters, 40)
    opts = P.SolveOptions(max_iters=iters, tol=0.0, relaxation=w.relaxation, dtype=dtype)
    ref, rref = run_plan(sp, opts, {"SSB_RING": 0})
    ring, rring = run_plan(sp, opts, {"SSB_RING": 1})
    d = ring.describe()
    # shapes without a ring instantiation (4-lane groups) keep the pair kernel
    assert "sart_ring_kernel" in d["fwd_kernel"]
    assert ("sart_ring_kernel" in d["back_kernel"]) == (d["vs_back"] >= 8)
    assert "sart_ring_kernel" not in ref.describe()["fwd_kernel"]
    assert rring.iterations == rref.iterations == iters
    for which in (0, 1):
        assert ring.solution(which).tobytes() == ref.solution(which).tobytes()
        # ||r|| sums per-CTA partials: the ring grid (one CTA per SM) changes
        # the order of that fp64 reduction only
        assert np.allclose(ring.history(which), ref.history(which), rtol=1e-13, atol=0)


@pytest.mark.parametrize("env", [{"SSB_RING_CAP": 64, "SSB_RING_STAGES": 2},
                                 {"SSB_RING_CAP": 64, "SSB_RING_STAGES": 2, "SSB_RING_IL": 0},
                                 {"SSB_RING_CAP": 256, "SSB_RING_STAGES": 3},
                                 {"SSB_RING_CAP": 1024, "SSB_RING_STAGES": 8,
                                  "SSB_RING_UF_FWD": 2, "SSB_RING_UF_BACK": 2}])
def test_ring_protocol_small_slots(env):
    """Many small chunks per CTA: the producer recycles every slot many times
    per pass; the result must not change."""
    w, sp, csr, p = folded(2)
    opts = P.SolveOptions(max_iters=20, tol=0.0, relaxation=w.relaxation, dtype="f32")
    ref, _ = run_plan(sp, opts, {"SSB_RING": 0})
    ring, _ = run_plan(sp, opts, dict(env, SSB_RING=1))
    assert ring.describe()["ring_chunks"][0] > 148
    for which in (0, 1):
        assert ring.solution(which).tobytes() == ref.solution(which).tobytes()


def test_ring_tolerance_stop_on_device():
    """tol > 0: the WHILE-loop graph stops at the pair plan's iteration."""
    w, sp, csr, p = folded(2)
    opts = P.SolveOptions(max_iters=200, tol=0.2, relaxation=w.relaxation, dtype="f64")
    ref, rref = run_plan(sp, opts, {"SSB_RING": 0})
    ring, rring = run_plan(sp, opts, {"SSB_RING": 1})
    assert rref.iterations < 200
    assert rring.iterations == rref.iterations
    for which in (0, 1):
        assert ring.solution(which).tobytes() == ref.solution(which).tobytes()


def test_ring_plan_matches_oracle_config2():
    w, sp, csr, p = folded(2)
    f1, f2 = O.fold_rows_csr(csr)
    p1, p2 = O.split_rhs(p)
    want, it, _ = O.solve_split_prepared(f1.to_matrix(), f2.to_matrix(), p1, p2, w.iters, 0.0,
                                         w.relaxation, True)
    for dtype, tol in (("f64", 1e-10), ("f32", 1e-4)):
        opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype=dtype)
        ring, _ = run_plan(sp, opts, {"SSB_RING": 1})
        assert rel_err(ring.recombine(), want) <= tol


def test_ring_repeated_runs_bitwise():
    w, sp, csr, p = folded(3)
    opts = P.SolveOptions(max_iters=10, tol=0.0, relaxation=w.relaxation, dtype="f32")
    ring, _ = run_plan(sp, opts, {"SSB_RING": 1})
    a = ring.solution(0).copy()
    ring.run()
    assert ring.solution(0).tobytes() == a.tobytes()


@pytest.mark.parametrize("idx,dtype", [(1, "f64"), (2, "f32"), (3, "f32")])
def test_dynamic_schedule_equals_grid_stride(idx, dtype):
    """SSB_DYN=1 (contiguous nnz-balanced vector runs per CTA, grabbed by the
    lane groups from a shared counter) only changes who computes a vector,
    never how: bitwise identical to the grid-stride schedule."""
    w, sp, csr, p = folded(idx)
    opts = P.SolveOptions(max_iters=min(w.iters, 30), tol=0.0, relaxation=w.relaxation,
                          dtype=dtype)
    a, _ = run_plan(sp, opts, {"SSB_DYN": 0})
    b, _ = run_plan(sp, opts, {"SSB_DYN": 1})
    for which in (0, 1):
        assert a.solution(which).tobytes() == b.solution(which).tobytes()
        # the per-CTA ||r||^2 partials group rows differently (fp64 order only)
        assert np.allclose(a.history(which), b.history(which), rtol=1e-13, atol=0)
