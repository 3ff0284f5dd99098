"""Oracle CGLS (restating solvers.cpp:99-146) against the reference's CGLS pins
(tests/unit/test_solvers.cpp:84-151). CPU only."""
import numpy as np
import pytest

import pyoracle as O


def test_identity(pins):
    p = O.rng_uniform(2003, 6, -1.0, 1.0)
    r = O.cgls_solve(O.Matrix.dense(np.eye(6)), p, tol=1e-12)
    assert r.iterations <= 2 and np.max(np.abs(r.f - p)) <= 1e-12


def test_published_min_norm(pins):
    a2 = np.array(pins["example1_split"]["a2"], float)
    r = O.cgls_solve(O.Matrix.dense(a2), pins["example1_split"]["p2"], max_iters=50, tol=1e-12)
    assert np.max(np.abs(r.f - [0.3542, 0.3373, 0.6036])) <= 1e-4


def test_full_rank_least_squares():
    rng = np.random.default_rng(2004)
    m, n = 50, 30
    d = np.where(rng.random((m, n)) < 0.2, rng.uniform(-1, 1, (m, n)), 0.0)
    d[np.arange(n), np.arange(n)] += 2.0
    p = rng.uniform(-1, 1, m)
    r = O.cgls_solve(O.Matrix.dense(d), p, max_iters=500, tol=1e-14)
    want = np.linalg.lstsq(d, p, rcond=None)[0]
    assert np.linalg.norm(r.f - want) <= 1e-8 * max(1.0, np.linalg.norm(want))


def test_residual_non_increasing():
    rng = np.random.default_rng(2005)
    for _ in range(10):
        m, n = int(rng.integers(5, 40)), int(rng.integers(2, 20))
        r = O.cgls_solve(O.Matrix.dense(rng.uniform(-1, 1, (m, n))), rng.uniform(-1, 1, m),
                         max_iters=200, tol=1e-13)
        h = r.residual_history
        assert all(h[k] <= h[k - 1] * (1 + 1e-12) + 1e-14 for k in range(1, len(h)))


def test_errors_and_split():
    a = O.Matrix.dense(np.eye(2))
    with pytest.raises(O.OracleError, match="tol must be positive"):
        O.cgls_solve(a, np.ones(2), tol=0.0)
    with pytest.raises(O.OracleError, match="max_iters must be >= 1"):
        O.cgls_solve(a, np.ones(2), max_iters=0)
    # split CGLS equals direct CGLS in the limit (consistent centrosymmetric system)
    h1 = np.array([[2.0, 0.3], [0.1, 1.5], [0.2, 0.4]])
    h2 = np.array([[1.8, 0.2], [0.3, 2.1], [0.1, 0.5]])
    c = O.reconstruct_matrix(O.Matrix.dense(h1), O.Matrix.dense(h2))
    f = np.array([0.3, -0.2, 0.5, 0.1])
    p = c.apply(f)
    full = O.cgls_solve(c, p, max_iters=200, tol=1e-14)
    split, it, res = O.solve_split_method(c, p, "cgls", 1e-12, 200, 1e-14)
    assert np.linalg.norm(split - full.f) <= 1e-10
