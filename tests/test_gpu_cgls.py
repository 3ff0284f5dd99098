"""CGLS (reference cgls_solve, solvers.cpp:99-146) on the device vs the oracle
and the reference's own CGLS pins (tests/unit/test_solvers.cpp:84-151)."""
import numpy as np
import pytest

import pyoracle as O
from helpers import oracle_workload, rel_err

import paper_1902_10559_b200 as P

pytestmark = pytest.mark.gpu


def test_cgls_identity_one_iteration():
    # test_solvers.cpp:84-94
    p = O.rng_uniform(2003, 6, -1.0, 1.0)
    r = P.cgls_solve(P.Matrix.dense(np.eye(6)), p, P.SolveOptions(method="cgls", tol=1e-12))
    assert r.iterations <= 2
    assert np.max(np.abs(r.f - p)) <= 1e-12


def test_cgls_published_min_norm(pins):
    # test_solvers.cpp:96-109: the Example-1 quarter system A2
    a2 = np.array(pins["example1_split"]["a2"], float)
    r = P.cgls_solve(P.Matrix.dense(a2), pins["example1_split"]["p2"],
                     P.SolveOptions(method="cgls", tol=1e-12, max_iters=50))
    assert np.max(np.abs(r.f - [0.3542, 0.3373, 0.6036])) <= 1e-4


def test_cgls_sparse_full_rank_matches_min_norm():
    # test_solvers.cpp:111-132 (numpy least squares as the dense checker)
    rng = np.random.default_rng(2004)
    m, n = 50, 30
    d = np.where(rng.random((m, n)) < 0.2, rng.uniform(-1, 1, (m, n)), 0.0)
    d[np.arange(n), np.arange(n)] += 2.0
    p = rng.uniform(-1, 1, m)
    r = P.cgls_solve(P.Matrix.dense(d), p, P.SolveOptions(method="cgls", tol=1e-14, max_iters=500))
    want = np.linalg.lstsq(d, p, rcond=None)[0]
    assert np.linalg.norm(r.f - want) <= 1e-8 * max(1.0, np.linalg.norm(want))
    o = O.cgls_solve(O.Matrix.dense(d), p, max_iters=500, tol=1e-14)
    assert rel_err(r.f, o.f) <= 1e-10


def test_cgls_residual_non_increasing():
    # test_solvers.cpp:134-151
    rng = np.random.default_rng(2005)
    for _ in range(5):
        m, n = int(rng.integers(5, 40)), int(rng.integers(2, 20))
        d = rng.uniform(-1, 1, (m, n))
        p = rng.uniform(-1, 1, m)
        r = P.cgls_solve(P.Matrix.dense(d), p, P.SolveOptions(method="cgls", tol=1e-13,
                                                              max_iters=200))
        h = r.residual_history
        for k in range(1, len(h)):
            assert h[k] <= h[k - 1] * (1 + 1e-12) + 1e-14


def test_cgls_errors():
    a = P.Matrix.dense(np.eye(2))
    with pytest.raises(P.Error, match="cgls_solve: tol must be positive"):
        P.cgls_solve(a, np.ones(2), P.SolveOptions(method="cgls", tol=0.0))
    with pytest.raises(P.Error, match="cgls_solve: max_iters must be >= 1"):
        P.cgls_solve(a, np.ones(2), P.SolveOptions(method="cgls", max_iters=0))
    with pytest.raises(P.Error, match="cgls_solve: rhs length 3 does not match rows 2"):
        P.cgls_solve(a, np.ones(3), P.SolveOptions(method="cgls"))


@pytest.mark.parametrize("paired", ["1", "0"])  # one paired loop / two concurrent streams
def test_cgls_split_config1_matches_oracle(paired, monkeypatch):
    """Unlike SART (a contraction), CG loses orthogonality in finite precision:
    a summation-order difference of 1e-16 grows ~10x per iteration on this
    ill-conditioned underdetermined system (measured: 3e-16 after 3 iterations,
    8e-15 after 5, 1e-10 after 10, 4e-6 after 20). So f is compared where CG is
    stable (5 iterations, 1e-12) and, after 30 iterations, the residual norm —
    the quantity CGLS minimises — to 1e-3 relative. That residual moves with
    the summation order too: measured 2.9e-5 with 4-lane groups per vector and
    6.0e-4 with the 32 / 16-lane groups the paired streams use on this small
    system since they widen to fill the SMs (equally valid orders)."""
    monkeypatch.setenv("SSB_CGLS_PAIRED", paired)
    w, cfg, a, csr, f_true, p = oracle_workload(1)
    s = P.build_system(w.scan_config())
    for iters, f_tol in ((5, 1e-12), (30, None)):
        want_f, it, res = O.solve_split_method(a, p, "cgls", 0.0, iters, 1e-10)
        got = P.solve_split(P.CentroSystem(s.a, p, 0.0),
                            P.SolveOptions(method="cgls", max_iters=iters, tol=1e-10))
        assert got.method == "cgls" and got.iterations == it == iters
        if f_tol is not None:
            assert rel_err(got.f, want_f) <= f_tol
        assert abs(got.residual_norm - res) <= 1e-3 * res
    got32 = P.solve_split(P.CentroSystem(s.a, p, 0.0),
                          P.SolveOptions(method="cgls", max_iters=5, tol=1e-10, dtype="f32"))
    want_f, it, res = O.solve_split_method(a, p, "cgls", 0.0, 5, 1e-10)
    assert rel_err(got32.f, want_f) <= 1e-4
    direct = P.solve_direct(P.CentroSystem(s.a, p, 0.0),
                            P.SolveOptions(method="cgls", max_iters=30, tol=1e-10))
    assert direct.iterations == 30 and len(direct.residual_history) == 30


@pytest.mark.parametrize("paired", ["1", "0"])
def test_cgls_split_stops_independently_per_branch(paired, monkeypatch):
    """The two folded systems stop at their own iterations (the reference runs
    them as independent solves): compare each branch with the oracle's CGLS."""
    monkeypatch.setenv("SSB_CGLS_PAIRED", paired)
    rng = np.random.default_rng(41)
    h1 = 3 * np.eye(40, 30) + rng.uniform(0, 0.1, (40, 30))
    h2 = rng.uniform(0.1, 1.0, (40, 30))
    a = O.reconstruct_matrix(O.Matrix.dense(h1), O.Matrix.dense(h2)).to_dense()
    p = a @ rng.uniform(0.5, 1.5, 60)
    sys_ = P.CentroSystem(P.Matrix.dense(a), p, 0.0)
    split = P.split_system(sys_)
    got = P.solve_split(sys_, P.SolveOptions(method="cgls", max_iters=500, tol=1e-9))
    o1 = O.cgls_solve(O.Matrix.dense(h1), split.p1, max_iters=500, tol=1e-9)
    o2 = O.cgls_solve(O.Matrix.dense(h2), split.p2, max_iters=500, tol=1e-9)
    assert o1.iterations != o2.iterations
    assert got.iterations == max(o1.iterations, o2.iterations)
    want = O.recombine_solution(o1.f, o2.f)
    assert rel_err(got.f, want) <= 1e-8
