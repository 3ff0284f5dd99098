"""Dense minimum-norm path: reference pseudo_solve_dense
(solvers.cpp:81-97) and Method::dense_minnorm in solve_direct / solve_split,
pinned the way the reference pins it: published quarter solutions
(test_solvers.cpp:35-50), basic actions (:52-70), the SVD pseudo-inverse oracle
on random rank-deficient matrices (:72-84, tests/support/oracles.hpp:101-113),
solve_split against the pinv of the full system (:239-251) and branch-failure
aggregation (:290-303)."""
import os
import subprocess

import numpy as np
import pytest

import pyoracle as O
from helpers import oracle_workload

import paper_1902_10559_b200 as P

# published quarter systems of Example 1 (test_solvers.cpp:35-50)
A1 = np.array([[0, -6, -2], [-5, 1, -2]], float)
A2 = np.array([[2, 12, 12], [9, 7, 14]], float)
P1, P2 = np.array([-2.0, -2.0]), np.array([12.0, 14.0])
E1 = np.array([0.3512, 0.2508, 0.2475])
E2 = np.array([0.3542, 0.3373, 0.6036])


# ------------------------------------------------------------------ oracle pins (CPU)
def test_pinv_oracle_published_and_basic():
    assert np.max(np.abs(O.pinv_solve(A1, P1) - E1)) <= 1e-4
    assert np.max(np.abs(O.pinv_solve(A2, P2) - E2)) <= 1e-4
    p = np.random.default_rng(2001).uniform(-1, 1, 5)
    assert np.max(np.abs(O.pinv_solve(np.eye(5), p) - p)) <= 1e-14
    assert np.allclose(O.pinv_solve(np.array([[1.0, 1.0]]), [2.0]), [1.0, 1.0])
    assert np.all(O.pinv_solve(np.zeros((4, 4)), np.ones(4)) == 0.0)


def test_random_with_rank_oracle():
    rng = np.random.default_rng(2002)
    a = O.random_with_rank(7, 5, 3, rng)
    assert np.linalg.matrix_rank(a) == 3


# ------------------------------------------------------------------ device
@pytest.mark.gpu
def test_pseudo_solve_dense_published_quarter_solutions():
    f1 = P.pseudo_solve_dense(P.Matrix.dense(A1), P1)
    f2 = P.pseudo_solve_dense(P.Matrix.dense(A2), P2)
    assert np.max(np.abs(f1 - E1)) <= 1e-4
    assert np.max(np.abs(f2 - E2)) <= 1e-4
    assert np.linalg.norm(f1 - O.pinv_solve(A1, P1)) <= 1e-12
    assert np.linalg.norm(f2 - O.pinv_solve(A2, P2)) <= 1e-12


@pytest.mark.gpu
def test_pseudo_solve_dense_basic_actions():
    p = np.random.default_rng(2001).uniform(-1, 1, 5)
    assert np.max(np.abs(P.pseudo_solve_dense(P.Matrix.dense(np.eye(5)), p) - p)) <= 1e-14
    f = P.pseudo_solve_dense(P.Matrix.dense(np.array([[1.0, 1.0]])), [2.0])
    assert np.allclose(f, [1.0, 1.0], rtol=0, atol=1e-14)
    with pytest.raises(P.Error, match=r"pseudo_solve_dense: 4x4 exceeds the dense cap of 8 entries"):
        P.pseudo_solve_dense(P.Matrix.from_triplets(4, 4, [], [], []), np.zeros(4), dense_cap=8)
    assert np.all(P.pseudo_solve_dense(P.Matrix.from_triplets(4, 4, [], [], []), np.ones(4)) == 0)
    with pytest.raises(P.Error, match=r"pseudo_solve_dense: rhs length 3 does not match rows 4"):
        P.pseudo_solve_dense(P.Matrix.dense(np.eye(4)), np.ones(3))
    with pytest.raises(P.Error, match="pseudo_solve_dense: non-finite rhs"):
        P.pseudo_solve_dense(P.Matrix.dense(np.eye(2)), [1.0, np.nan])


@pytest.mark.gpu
def test_pseudo_solve_dense_matches_svd_oracle():
    rng = np.random.default_rng(2002)
    for _ in range(30):
        m, n = int(rng.integers(1, 13)), int(rng.integers(1, 13))
        rank = int(rng.integers(1, min(m, n) + 1))
        a = O.random_with_rank(m, n, rank, rng)
        b = rng.uniform(-1, 1, m)
        got = P.pseudo_solve_dense(P.Matrix.dense(a), b)
        want = O.pinv_solve(a, b)
        assert np.linalg.norm(got - want) <= 1e-10 * max(1.0, np.linalg.norm(want))


def _random_centro(m, n, rng, rank_deficient, consistent):
    """test_solvers.cpp:15-31 with numpy draws: A from two random folded halves."""
    mh, nh = m // 2, n // 2
    k = min(mh, nh)
    r1 = int(rng.integers(1, k + 1)) if rank_deficient and k > 1 else k
    r2 = int(rng.integers(1, k + 1)) if rank_deficient and k > 1 else k
    h1, h2 = O.random_with_rank(mh, nh, r1, rng), O.random_with_rank(mh, nh, r2, rng)
    a = O.reconstruct_matrix(O.Matrix.dense(h1), O.Matrix.dense(h2)).to_dense()
    p = a @ rng.uniform(-1, 1, n) if consistent else rng.uniform(-1, 1, m)
    return a, p


@pytest.mark.gpu
def test_solve_split_dense_matches_pinv_of_full_system():
    rng = np.random.default_rng(2009)
    opts = P.SolveOptions(method="dense")
    for trial in range(30):
        m, n = 2 * int(rng.integers(1, 11)), 2 * int(rng.integers(1, 11))
        a, p = _random_centro(m, n, rng, trial % 2 == 1, trial % 3 == 0)
        sys_ = P.CentroSystem(P.Matrix.dense(a), p, 1e-10)
        rep = P.solve_split(sys_, opts)
        want = O.pinv_solve(a, p)
        assert np.linalg.norm(rep.f - want) <= 1e-9 * max(1.0, np.linalg.norm(want))
        assert rep.method == "dense" and rep.mode == "split"
        direct = P.solve_direct(sys_, opts)
        assert np.linalg.norm(direct.f - want) <= 1e-9 * max(1.0, np.linalg.norm(want))
        assert abs(direct.residual_norm - np.linalg.norm(a @ direct.f - p)) <= 1e-12 * max(
            1.0, np.linalg.norm(p))


@pytest.mark.gpu
def test_solve_split_dense_reports_both_branch_failures():
    rng = np.random.default_rng(2012)
    a, p = _random_centro(8, 6, rng, False, False)
    with pytest.raises(P.Error) as ei:
        P.solve_split(P.CentroSystem(P.Matrix.dense(a), p, 1e-10),
                      P.SolveOptions(method="dense", dense_cap=1))
    msg = str(ei.value)
    assert msg.startswith("solve_split: branch failure:")
    assert "[system 1] pseudo_solve_dense: 4x3 exceeds the dense cap of 1 entries" in msg
    assert "[system 2]" in msg


@pytest.mark.gpu
def test_dense_split_on_config1_matches_oracle():
    """Config 1's folded systems (640 x 2048 each) through the dense path."""
    w, cfg, a, csr, f_true, p = oracle_workload(1)
    sys_ = P.build_system(w.scan_config())
    sys_.p = p
    rep = P.solve_split(sys_, P.SolveOptions(method="dense"))
    s = O.split_system(a, p, 0.0)
    f1 = O.pinv_solve(s.a1.to_dense(), s.p1)
    f2 = O.pinv_solve(s.a2.to_dense(), s.p2)
    want = O.recombine_solution(f1, f2)
    assert np.linalg.norm(rep.f - want) <= 1e-9 * np.linalg.norm(want)


@pytest.mark.gpu
def test_cli_solve_method_dense(tmp_path):
    cli = os.path.join(os.path.dirname(P.__file__), "symsplit_b200")
    a = P.Matrix.dense(O.reconstruct_matrix(O.Matrix.dense(A1), O.Matrix.dense(A2)).to_dense())
    P.write_matrix_market(a, str(tmp_path / "a.mtx"))
    rhs = O.reconstruct_matrix(O.Matrix.dense(A1), O.Matrix.dense(A2)).to_dense() @ np.arange(6.0)
    P.write_vector_csv(rhs, str(tmp_path / "p.csv"))
    r = subprocess.run([cli, "solve", "--matrix", str(tmp_path / "a.mtx"), "--rhs",
                        str(tmp_path / "p.csv"), "--mode", "split", "--method", "dense",
                        "--out", str(tmp_path / "f.csv")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("method=dense mode=split")
    dense = O.reconstruct_matrix(O.Matrix.dense(A1), O.Matrix.dense(A2)).to_dense()
    want = O.pinv_solve(dense, rhs)
    got = P.read_vector_csv(str(tmp_path / "f.csv"))
    assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)
