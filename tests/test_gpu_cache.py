"""solve_split's per-matrix cache (the fold of A and the SART plan over A1/A2
kept on the immutable matrix handle): results are those of a fresh matrix,
bit for bit, for new right-hand sides, changed options and changed
symmetry tolerances; the reference's symmetry error is raised from the cache."""
import numpy as np
import pytest

import paper_1902_10559_b200 as P
from paper_1902_10559_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu


def fresh_solve(cfg, p, opts, tol=0.0):
    s = P.build_system(cfg)
    return P.solve_split(P.CentroSystem(s.a, p, tol), opts)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_cached_solves_equal_fresh_matrix(dtype):
    w = CONFIGS[2]
    cfg = w.scan_config()
    s = P.build_system(cfg)
    grid = P.make_grid(cfg)
    opts = P.SolveOptions(max_iters=30, tol=0.0, relaxation=w.relaxation, dtype=dtype)
    for seed in (11, 12, 13):
        p = P.forward_project(s.a, P.rasterize(P.random_ellipses(seed, 8), grid))
        got = P.solve_split(P.CentroSystem(s.a, p, 0.0), opts)
        want = fresh_solve(cfg, p, opts)
        assert got.f.tobytes() == want.f.tobytes()
        assert got.iterations == want.iterations == 30
        assert got.residual_norm == want.residual_norm


def test_cache_follows_option_changes():
    w = CONFIGS[1]
    cfg = w.scan_config()
    s = P.build_system(cfg)
    p = P.forward_project(s.a, P.rasterize(P.random_ellipses(w.seed(), 8), P.make_grid(cfg)))
    variants = [P.SolveOptions(max_iters=20, tol=0.0, dtype="f64"),
                P.SolveOptions(max_iters=35, tol=0.0, relaxation=0.7, dtype="f64"),
                P.SolveOptions(max_iters=20, tol=0.0, dtype="f32"),
                P.SolveOptions(max_iters=200, tol=1e-3, dtype="f64"),
                P.SolveOptions(max_iters=20, tol=0.0, dtype="f64")]
    for o in variants:
        got = P.solve_split(P.CentroSystem(s.a, p, 0.0), o)
        want = fresh_solve(cfg, p, o)
        assert got.f.tobytes() == want.f.tobytes()
        assert got.iterations == want.iterations
    s.a.release_cache()
    again = P.solve_split(P.CentroSystem(s.a, p, 0.0), variants[0])
    assert again.f.tobytes() == fresh_solve(cfg, p, variants[0]).f.tobytes()


def test_symmetry_tolerance_applies_per_call():
    """A perturbed (not exactly centrosymmetric) matrix: a call with a loose
    tolerance folds and caches it, a later call with tolerance 0 must still
    raise the reference's SymmetryError with the same report."""
    # 4 x 6 Example-1 matrix (reference oracles.hpp:165-178), one entry perturbed
    ex1 = np.array([1, 2, 7, 1, 3, 4, 3, 9, 5, 6, 8, 7, 7, 8, 6, 5, 9, 3, 4, 3, 1, 7, 2, 1],
                   dtype=float).reshape(6, 4).T
    bad = ex1.copy()
    bad[0, 0] += 1e-6
    a = P.Matrix.dense(bad)
    p = np.array([5.0, 6.0, 8.0, 7.0])
    opts = P.SolveOptions(max_iters=5, tol=0.0)
    with pytest.raises(P.SymmetryError) as e0:
        P.solve_split(P.CentroSystem(a, p, 0.0), opts)
    r = P.solve_split(P.CentroSystem(a, p, 1e-3), opts)  # folds and caches
    assert r.iterations == 5
    with pytest.raises(P.SymmetryError) as e1:
        P.solve_split(P.CentroSystem(a, p, 0.0), opts)
    assert str(e1.value) == str(e0.value)
    assert e1.value.report.max_violation == e0.value.report.max_violation
