"""Multi-RHS SART (S slices sharing the folded pair): the block-merged kernels
(sart_*_block_kernel: kBlockR neighbouring rays / voxels per warp, each
gathered S-wide record applied to all of them and both systems, union entries
staged in shared memory) against the per-vector multi kernels (SSB_BLOCKED=0)
and against single-slice solves. A block's union holds each vector's entries
in its own ascending order and adds exact zeros elsewhere, so the iterates are
bitwise those of the per-vector kernels."""
import os

import numpy as np
import pytest

import paper_1902_10559_b200 as P
from paper_1902_10559_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu

_cache = {}


def slices(idx, S):
    key = (idx, S)
    if key not in _cache:
        w = CONFIGS[idx]
        cfg = w.scan_config()
        s = P.build_system(cfg)
        grid = P.make_grid(cfg)
        split = P.split_system(P.CentroSystem(s.a, np.zeros(w.m), 0.0))
        p1s, p2s = [], []
        for sl in range(S):
            f = P.rasterize(P.random_ellipses(7000 + sl, 8), grid)
            a, b = P.split_rhs(P.forward_project(s.a, f))
            p1s.append(a)
            p2s.append(b)
        _cache[key] = (w, split, np.concatenate(p1s), np.concatenate(p2s))
    return _cache[key]


def plan_with(split, opts, S, blocked, staged=0):
    env = {"SSB_BLOCKED": str(blocked), "SSB_STAGED": str(staged)}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        pl = P.SartPlan(split.a1, split.a2, opts, nrhs=S)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return pl


@pytest.mark.parametrize("idx,S,dtype", [(2, 5, "f64"), (2, 64, "f32"), (4, 128, "f32"),
                                         (1, 3, "f64")])
def test_blocked_equals_per_vector(idx, S, dtype):
    w, split, p1, p2 = slices(idx, S)
    opts = P.SolveOptions(max_iters=12, tol=0.0, relaxation=w.relaxation, dtype=dtype)
    runs = []
    for blocked in (0, 1):
        pl = plan_with(split, opts, S, blocked)
        assert ("block" in pl.describe()["fwd_kernel"]) == bool(blocked)
        pl.set_rhs(0, p1)
        pl.set_rhs(1, p2)
        assert pl.run().iterations == 12
        runs.append(pl)
    a, b = runs
    for which in (0, 1):
        assert a.solution(which).tobytes() == b.solution(which).tobytes()
        for sl in (0, S - 1):
            assert np.allclose(a.history(which, sl), b.history(which, sl), rtol=1e-13, atol=0)


def test_blocked_equals_single_slice_solves():
    w, split, p1, p2 = slices(2, 4)
    opts = P.SolveOptions(max_iters=15, tol=0.0, relaxation=w.relaxation, dtype="f64")
    pl = plan_with(split, opts, 4, 1)
    pl.set_rhs(0, p1)
    pl.set_rhs(1, p2)
    pl.run()
    x1 = pl.solution(0).reshape(4, -1)
    m = len(p1) // 4
    for sl in range(4):
        one = P.SartPlan(split.a1, split.a2, opts)
        one.set_rhs(0, p1[sl * m:(sl + 1) * m])
        one.set_rhs(1, p2[sl * m:(sl + 1) * m])
        one.run()
        ref = one.solution(0)
        assert np.linalg.norm(x1[sl] - ref) <= 1e-12 * np.linalg.norm(ref)


def test_blocked_tolerance_stop_per_slice():
    """tol > 0: slices stop independently (per-slice state), as the per-vector kernels."""
    w, split, p1, p2 = slices(2, 5)
    opts = P.SolveOptions(max_iters=100, tol=0.05, relaxation=w.relaxation, dtype="f64")
    its = []
    for blocked in (0, 1):
        pl = plan_with(split, opts, 5, blocked)
        pl.set_rhs(0, p1)
        pl.set_rhs(1, p2)
        its.append((pl.run().iterations, [len(pl.history(0, s)) for s in range(5)],
                    pl.solution(1).tobytes()))
    assert its[0] == its[1]
