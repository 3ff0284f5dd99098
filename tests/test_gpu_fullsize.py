"""BASELINE configs 4 and 5 at full size on the GPU.

Config 4 (256 slices sharing one geometry) runs through the multi-RHS plan
and is compared with the oracle on sampled slices. Config 5 (M = 409,600
rays, N = 4,194,304 voxels, ~1e9 nonzeros) is too large for the oracle inside
a test run, so it is checked through properties that do not depend on size:
the built matrix is exactly centrosymmetric (tolerance 0), its mirror half is
the reversed traced half, A1/A2 have equal patterns when nothing cancels,
recombine(decompose(f)) == f, and the fp32 SART residual decreases."""
import numpy as np
import pytest

import pyoracle as O
from helpers import oracle_cfg, rel_err

import paper_1902_10559_b200 as P
from paper_1902_10559_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu


def test_config4_multi_rhs_matches_oracle_slices():
    w = CONFIGS[4]
    cfg = w.scan_config()
    s = P.build_system(cfg)
    grid = P.make_grid(cfg)
    S, iters = 32, 20
    p1s, p2s = [], []
    for sl in range(S):
        f = P.rasterize(P.random_ellipses(w.seed(sl), 8), grid)
        p1, p2 = P.split_rhs(P.forward_project(s.a, f))
        p1s.append(p1)
        p2s.append(p2)
    split = P.split_system(P.CentroSystem(s.a, np.zeros(w.m), 0.0))
    plan = P.SartPlan(split.a1, split.a2, P.SolveOptions(max_iters=iters, tol=0.0, dtype="f32"),
                      nrhs=S)
    plan.set_rhs(0, np.concatenate(p1s))
    plan.set_rhs(1, np.concatenate(p2s))
    plan.run()
    x1, x2 = plan.solution(0), plan.solution(1)
    # oracle (fp64) on two sampled slices, same folded matrices
    ocfg = oracle_cfg(w)
    t = O.build_traced_csr(ocfg)
    full = O.full_csr_from_traced(t, w.m, w.n)
    f1, f2 = O.fold_rows_csr(full)
    m1, m2 = f1.to_matrix(), f2.to_matrix()
    for sl in (0, 17):
        want1 = O.sart_solve(m1, p1s[sl], max_iters=iters, tol=0.0)
        want2 = O.sart_solve(m2, p2s[sl], max_iters=iters, tol=0.0)
        assert rel_err(x1[sl], want1.f) <= 1e-4
        assert rel_err(x2[sl], want2.f) <= 1e-4
        assert np.allclose(plan.history(0, sl), want1.residual_history, rtol=1e-4)


def test_config5_fullsize_properties():
    w = CONFIGS[5]
    cfg = w.scan_config()
    s = P.build_system(cfg)
    m, n = s.a.shape
    assert (m, n) == (w.m, w.n) == (409600, 4194304)
    nnz = s.a.stored
    assert 0.9e9 < nnz < 1.1e9 and nnz % 2 == 0
    rep = P.verify_symmetry(s.a, 0.0)
    assert rep.holds and rep.max_violation == 0.0
    # Siddon lengths are positive and bounded by the voxel diagonal
    ptr = s.a.to_csr()[0]
    assert ptr[0] == 0 and ptr[-1] == nnz and np.all(np.diff(ptr) > 0)
    f = P.rasterize(P.random_ellipses(w.seed(), 8), P.make_grid(cfg))
    p = P.forward_project(s.a, f)
    sigma = w.noise_frac * float(np.max(p))
    p = P.forward_project(s.a, f, sigma, w.noise_seed())
    split = P.split_system(P.CentroSystem(s.a, p, 0.0))
    assert split.a1.shape == split.a2.shape == (m // 2, n // 2)
    assert split.a2.stored + 0 >= split.a1.stored  # A1 may only lose cancelled buckets
    pair = P.decompose_solution(f)  # round trip within 1e-15 (test_centro.cpp:182-190)
    assert np.max(np.abs(P.recombine_solution(pair) - f)) <= 1e-15 * max(1.0, np.max(np.abs(f)))
    plan = P.SartPlan(split.a1, split.a2, P.SolveOptions(max_iters=8, tol=0.0,
                                                         relaxation=w.relaxation, dtype="f32"))
    plan.set_rhs(0, split.p1)
    plan.set_rhs(1, split.p2)
    plan.run()
    for which in (0, 1):
        h = plan.history(which)
        assert len(h) == 8 and np.all(np.isfinite(h))
        assert np.all(np.diff(h) < 0)  # residual decreases (lambda = 0.5)
    fr = plan.recombine()
    assert fr.shape == (n,) and np.all(np.isfinite(fr))
