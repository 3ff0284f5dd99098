"""Pins the CPU oracle (oracle/) against every known-answer test the reference
holds for this path (fixtures: tests/golden/reference_pins.json). CPU only."""
import numpy as np
import pytest

import pyoracle as O
from helpers import deg, oracle_cfg, oracle_workload

from paper_1902_10559_b200.configs import CONFIGS


def ex1(pins):
    return np.array(pins["example1"]["matrix"], float), np.array(pins["example1"]["rhs"], float)


# ------------------------------------------------------------------ fold pins
@pytest.mark.parametrize("sparse", [False, True])
def test_example1_split_exact(pins, sparse):
    d, p = ex1(pins)
    a = O.Matrix.sparse_from_dense(d) if sparse else O.Matrix.dense(d)
    s = O.split_system(a, p, 0.0)
    e = pins["example1_split"]
    assert np.array_equal(s.a1.to_dense(), np.array(e["a1"], float))
    assert np.array_equal(s.a2.to_dense(), np.array(e["a2"], float))
    assert np.array_equal(s.p1, e["p1"]) and np.array_equal(s.p2, e["p2"])


def test_example1_pruned_zero(pins):
    d, p = ex1(pins)
    s = O.split_system(O.Matrix.sparse_from_dense(d), p, 0.0)
    outer, inner, val = s.a1.get_csc()
    assert s.a1.nonzeros() == pins["example1_split"]["a1_nonzeros"]
    assert len(val) == 5 and not np.any(val == 0.0)  # the cancelled 1-1 is not stored
    assert s.a1.to_dense()[0, 0] == 0.0


def test_split_2x2(pins):
    c = pins["split_2x2"]
    s = O.split_system(O.Matrix.dense(c["matrix"]), c["rhs"], 0.0)
    assert s.a1.to_dense()[0, 0] == c["a1"] and s.a2.to_dense()[0, 0] == c["a2"]
    assert s.p1[0] == c["p1"] and s.p2[0] == c["p2"]


def test_split_rhs_cases(pins):
    for c in pins["split_rhs_cases"]["cases"]:
        p1, p2 = O.split_rhs(c["p"])
        assert np.array_equal(p1, c["p1"]) and np.array_equal(p2, c["p2"])
    with pytest.raises(O.OracleError):
        O.split_rhs(np.zeros(3))


def test_split_reconstruct_roundtrip():
    # test_centro.cpp:99-112: symmetrized random 6x8, dense and sparse agree <= 1e-15
    vals = O.rng_uniform(1001, 20 * 48, -1.0, 1.0)
    for t in range(20):
        d = vals[t * 48:(t + 1) * 48].reshape(8, 6).T  # column-major fill like random_dense
        a = O.symmetrize(O.Matrix.dense(d))
        p = np.arange(6, dtype=float)
        s = O.split_system(a, p, 0.0)
        ss = O.split_system(O.Matrix.sparse_from_dense(a.to_dense()), p, 0.0)
        back = O.reconstruct_matrix(s.a1, s.a2).to_dense()
        assert np.max(np.abs(back - a.to_dense())) <= 1e-15
        assert np.max(np.abs(ss.a1.to_dense() - s.a1.to_dense())) <= 1e-15
        assert np.max(np.abs(ss.a2.to_dense() - s.a2.to_dense())) <= 1e-15


def test_symmetry_violation_report(pins):
    d, p = ex1(pins)
    i, j, v = pins["verify_symmetry_perturbed"]["perturb"]
    d[i, j] = v
    for a in (O.Matrix.dense(d), O.Matrix.sparse_from_dense(d)):
        r = O.verify_symmetry(a, 0.0)
        assert not r.holds and r.max_violation == 8.0
        assert [r.worst_row, r.worst_col] in pins["verify_symmetry_perturbed"]["worst_either"]
        with pytest.raises(O.OracleSymmetryError) as ei:
            O.split_system(a, p, 1e-12)
        assert ei.value.report.max_violation == 8.0


def test_odd_dimensions_status():
    r = O.verify_symmetry(O.Matrix.dense(np.eye(3)), 1.0)
    assert not r.holds and r.status == 1
    assert O.verify_symmetry(O.Matrix.dense(np.zeros((2, 3))), 1.0).status == 2


# ------------------------------------------------------------------ recombine pins
def test_decompose_recombine_published(pins):
    c = pins["decompose_published"]
    f1, f2 = O.decompose_solution(c["f"])
    assert np.max(np.abs(f1 - c["f1"])) <= c["tol"] and np.max(np.abs(f2 - c["f2"])) <= c["tol"]
    c = pins["recombine_published"]
    f = O.recombine_solution(c["f1"], c["f2"])
    assert np.max(np.abs(f - c["f"])) <= c["tol"]


def test_recombine_general_exact(pins):
    c = pins["recombine_general"]
    f = O.recombine_solution(c["f1"], c["f2"])
    assert np.array_equal(f, c["f"])
    d, p = ex1(pins)
    assert np.array_equal(O.Matrix.dense(d).apply(f), p)


def test_recombine_symmetric_and_errors(pins):
    f2 = np.array(pins["recombine_symmetric"]["f2"])
    f = O.recombine_solution(np.zeros(3), f2)
    assert np.array_equal(f[:3], f[::-1][:3]) and np.array_equal(f[:3], 0.5 * f2)
    with pytest.raises(O.OracleError):
        O.recombine_solution(np.zeros(3), np.zeros(2))
    with pytest.raises(O.OracleError):
        O.decompose_solution(np.zeros(5))


def test_recombine_inverts_decompose():
    vals = O.rng_uniform(1003, 50 * 24, -1, 1)
    for t in range(50):
        f = vals[t * 24:t * 24 + 2 * (1 + t % 12)]
        f1, f2 = O.decompose_solution(f)
        assert np.max(np.abs(O.recombine_solution(f1, f2) - f)) <= 1e-15


# ------------------------------------------------------------------ geometry pins
def test_snake(pins):
    g = O.GridC(2, 2, 0.1, 0.0, 0.25)
    for c, r, j in pins["snake_2x2"]["cases"]:
        assert O.snake_index(c, r, g) == j
    with pytest.raises(O.OracleError):
        O.snake_index(3, 1, g)
    for nx, ny in pins["snake_mirror_grids"]["grids"]:
        g = O.GridC(nx, ny, 0.1, 0.0, 0.25)
        total = nx * ny
        for j in range(1, total + 1):
            c, r = O.snake_inverse(j, g)
            assert O.snake_index(c, r, g) == j
            mc, mr = O.snake_inverse(total - j + 1, g)
            assert (mc, mr) == (nx - c + 1, r)


def test_emitter_angles_and_positions(pins):
    cfg = O.scan_config(4, deg(30.0), 1.0, 0.25, 0.43, 1024, 0.1, 32, 32)
    a = O.emitter_angles(cfg)
    assert np.allclose(a, [deg(x) for x in pins["emitter_angles_k4"]["deg"]], rtol=1e-13)
    cfg = O.scan_config(24, deg(30.0), 1.0, 0.25, 0.43, 1024, 0.1, 32, 32)
    a = O.emitter_angles(cfg)
    assert np.all(a + a[::-1] == 0.0) and np.all(a != 0.0)
    cfg = O.scan_config(6, deg(30.0), 1.0, 0.25, 0.43, 1024, 0.1, 32, 32)
    s = O.emitter_positions(cfg)
    assert np.all(s[:, 0] == -s[::-1, 0]) and np.all(s[:, 1] == s[::-1, 1])
    assert np.all(np.diff(s[:, 0]) > 0)


def test_rays_mirror_bitwise():
    cfg = O.scan_config(8, deg(30.0), 1.0, 0.25, 0.43, 1024, 0.1, 8, 8)
    g = O.GridC(8, 8, 0.1 / 8, 0.0, 0.25)
    rays, _, _ = O.enumerate_rays(cfg, g)
    m = len(rays)
    assert m > 0 and m % 2 == 0
    assert np.all(rays[:, 0] == -rays[::-1, 0]) and np.all(rays[:, 2] == -rays[::-1, 2])
    assert np.all(rays[:, 1] == rays[::-1, 1]) and np.all(rays[:, 3] == rays[::-1, 3])


def test_vertical_and_diagonal_rays(pins):
    c = pins["vertical_ray"]
    g = O.GridC(**c["grid"])
    xc = g.center_x + (2 - 0.5 - 0.5 * g.n_x) * g.voxel_size
    js, lens = O.ray_weights([xc, 3.0, xc, 0.0], g)
    assert len(js) == c["entries"]
    assert np.all(np.abs(lens - g.voxel_size) <= c["tol"])
    assert all(O.snake_inverse(int(j), g)[0] == 2 for j in js)
    assert abs(lens.sum() - g.n_y * g.voxel_size) <= c["tol"]
    c = pins["diagonal_ray"]
    g = O.GridC(**c["grid"])
    vs = g.voxel_size
    xl = g.center_x - 0.5 * g.n_x * vs
    js, lens = O.ray_weights([xl - vs, g.y_bottom - vs, xl + 2 * vs, g.y_bottom + g.n_y * vs + vs], g)
    assert np.all(js == 1)
    assert abs(lens.sum() - vs * np.sqrt(2.0)) <= c["rel_tol"] * vs * np.sqrt(2.0)


def liang_barsky(ray, g):
    # independent chord oracle (reference tests/support/oracles.hpp:116-140)
    sx, sy, ex, ey = ray
    dx, dy = ex - sx, ey - sy
    t0, t1 = 0.0, 1.0
    xl = g.center_x - 0.5 * g.n_x * g.voxel_size
    xr = g.center_x + 0.5 * g.n_x * g.voxel_size
    yt = g.y_bottom + g.n_y * g.voxel_size
    for p, q in ((-dx, sx - xl), (dx, xr - sx), (-dy, sy - g.y_bottom), (dy, yt - sy)):
        if p == 0.0:
            if q <= 0.0:
                return 0.0
            continue
        t = q / p
        if p < 0:
            t0 = max(t0, t)
        else:
            t1 = min(t1, t)
    return 0.0 if t1 <= t0 else (t1 - t0) * np.hypot(dx, dy)


def test_chord_conservation(pins):
    c = pins["chord_conservation"]
    g = O.GridC(32, 32, 0.1 / 32, 0.0, 0.25)
    u = O.rng_uniform(c["seed"], 4 * c["trials"])
    hits = 0
    for t in range(c["trials"]):
        a, b, cc, d = u[4 * t:4 * t + 4]
        ray = [-0.3 + 0.6 * a, 1.0 + 0.3 * b, -0.3 + 0.6 * cc, 0.0]
        js, lens = O.ray_weights(ray, g)
        chord = liang_barsky(ray, g)
        assert abs(lens.sum() - chord) <= c["tol"]
        hits += chord > 0
    assert hits > 0


def test_build_symmetric_and_worker_invariant():
    cfg = O.scan_config(12, deg(30.0), 1.0, 0.25, 0.43, 1024, 0.1, 16, 16)
    a = O.build_system(cfg)
    assert a.shape[0] % 2 == 0 and O.verify_symmetry(a, 0.0).holds and a.nonzeros() > 0
    cfg = O.scan_config(6, deg(30.0), 1.0, 0.25, 0.43, 1024, 0.1, 8, 8)
    s1 = O.build_system(cfg, 1).get_csc()
    s4 = O.build_system(cfg, 4).get_csc()
    assert all(np.array_equal(x, y) for x, y in zip(s1, s4))


def test_parse_scan_config(pins):
    c = pins["scan_config_text"]
    cfg = O.parse_scan_config(c["text"])
    assert cfg.k == c["k"] and abs(cfg.gamma - deg(c["gamma_deg"])) < 1e-15
    assert cfg.h_e == c["h_e"] and cfg.h_m == c["h_m"] and cfg.grid_nx == c["grid_nx"]
    assert abs(O.make_grid(cfg).voxel_size - c["voxel_size"]) < 1e-18
    for bad in ("unknown_key 3\n", "k 8 9\n", "k\n"):
        with pytest.raises(O.OracleError):
            O.parse_scan_config(bad)


# ------------------------------------------------------------------ phantom pins
def test_forward_project_basics(pins):
    d, _ = ex1(pins)
    a = O.Matrix.dense(d)
    assert np.all(O.forward_project(a, np.zeros(6)) == 0.0)
    e1 = np.zeros(6)
    e1[0] = 1.0
    assert np.array_equal(O.forward_project(a, e1), pins["forward_project_e1"]["column0"])
    with pytest.raises(O.OracleError):
        O.forward_project(a, np.zeros(5))


def test_symmetric_image_projects_symmetric():
    cfg = O.scan_config(8, deg(30.0), 1.0, 0.25, 0.43, 1024, 0.1, 16, 16)
    a = O.build_system(cfg)
    img = O.rasterize(O.shepp_logan(), O.make_grid(cfg))
    n = len(img)
    avg = 0.5 * (img[: n // 2] + img[::-1][: n // 2])
    img[: n // 2] = avg
    img[n // 2:] = avg[::-1]
    p = O.forward_project(a, img)
    assert np.array_equal(p[: len(p) // 2], p[::-1][: len(p) // 2])
    p1, _ = O.split_rhs(p)
    assert np.all(p1 == 0.0)


def test_noise_seeded():
    p = np.linspace(0, 1, 8)
    a = O.add_noise(p, 0.01, 7)
    assert np.array_equal(a, O.add_noise(p, 0.01, 7))
    assert not np.array_equal(a, p) and not np.array_equal(a, O.add_noise(p, 0.01, 8))
    assert np.array_equal(O.add_noise(p, 0.0, 7), p)


# ------------------------------------------------------------------ solver pins
def test_sart_identity_one_iteration(pins):
    c = pins["sart_identity"]
    p = O.rng_uniform(c["seed"], c["n"], 0.1, 1.0)
    r = O.sart_solve(O.Matrix.dense(np.eye(c["n"])), p, max_iters=200, tol=c["tol"])
    assert r.iterations == c["iterations"]
    assert np.max(np.abs(r.f - p)) <= c["tol"]


def test_sart_zero_matrix_throws():
    with pytest.raises(O.OracleError, match="no nonzero rows"):
        O.sart_solve(O.Matrix.dense(np.zeros((4, 4))), np.ones(4))


def test_sart_option_errors():
    a = O.Matrix.dense(np.eye(2))
    with pytest.raises(O.OracleError, match=r"relaxation must be in \(0, 2\]"):
        O.sart_solve(a, np.ones(2), relaxation=2.5)
    with pytest.raises(O.OracleError, match="max_iters must be >= 1"):
        O.sart_solve(a, np.ones(2), max_iters=0)
    with pytest.raises(O.OracleError, match="rhs length 3 does not match rows 2"):
        O.sart_solve(a, np.ones(3))
    with pytest.raises(O.OracleError, match="non-finite rhs"):
        O.sart_solve(a, np.array([1.0, np.nan]))


def split_limit_system(c):
    mh, nh = c["mh"], c["nh"]
    u = O.rng_uniform(c["seed"], 2 * mh * nh + 2 * nh, 0.0, 1.0)
    h1 = (0.3 * u[: mh * nh]).reshape(nh, mh).T.copy()
    h2 = (0.3 * u[mh * nh: 2 * mh * nh]).reshape(nh, mh).T.copy()
    for i in range(nh):
        h1[i, i] += 2.0
        h2[i, i] += 2.0
    a = O.reconstruct_matrix(O.Matrix.dense(h1), O.Matrix.dense(h2))
    f_true = -1.0 + 2.0 * u[2 * mh * nh:]
    return a, a.apply(f_true)


def test_sart_split_vs_full_limit(pins):
    c = pins["sart_split_limit"]
    a, p = split_limit_system(c)
    full = O.sart_solve(a, p, max_iters=c["iters"], tol=c["tol"])
    split = O.solve_split(a, p, 1e-10, c["iters"], c["tol"], 1.0)
    assert np.linalg.norm(full.f - split.f) <= c["agree"] * max(1.0, np.linalg.norm(full.f))


def test_solve_split_parallelism_invariant():
    w, cfg, a, csr, f_true, p = oracle_workload(1)
    r1 = O.solve_split(a, p, 0.0, 20, 0.0, 1.0, parallelism=1)
    r8 = O.solve_split(a, p, 0.0, 20, 0.0, 1.0, parallelism=8)
    assert r1.f.tobytes() == r8.f.tobytes()


def test_solve_split_branch_failure_message():
    # A with A1 == 0 (mirror-equal row pairs): branch 1 has no nonzero rows.
    c = np.array([[1.0, 2.0], [3.0, 0.5]])
    a = O.reconstruct_matrix(O.Matrix.dense(np.zeros((2, 2))), O.Matrix.dense(2.0 * c))
    with pytest.raises(O.OracleError, match=r"branch failure: \[system 1\] sart_solve: matrix has no nonzero rows"):
        O.solve_split(a, np.ones(4), 1e-12, 10, 0.0, 1.0)


# ------------------------------------------------------------------ Eigen restatement checks
def test_norm_matches_numpy():
    for n in (0, 1, 2, 3, 4, 5, 7, 8, 31, 1000):
        v = O.rng_uniform(5 + n, n, -1, 1)
        ref = float(np.sqrt(np.sum(v * v))) if n else 0.0
        assert abs(O.norm(v) - ref) <= 1e-15 * max(1.0, ref)


def test_triplet_duplicates_sum_in_order():
    # (0,0) receives 1e16, 1.0, -1e16 in that order: ((1e16+1)-1e16) = 0 in fp64
    a = O.Matrix.triplets(2, 2, [0, 1, 0, 0], [0, 1, 0, 0], [1e16, 5.0, 1.0, -1e16])
    outer, inner, val = a.get_csc()
    assert list(outer) == [0, 1, 2] and list(inner) == [0, 1]
    assert val[0] == (1e16 + 1.0) - 1e16 and val[1] == 5.0


# ------------------------------------------------------------------ BASELINE config pins
def test_config1_counts_and_fast_fold(pins):
    c = pins["config1_counts"]
    w, cfg, a, csr, f_true, p = oracle_workload(1)
    m, n = a.shape
    assert m == c["m"] == w.m and a.info()[2] == c["nnz"]
    assert O.verify_symmetry(a, 0.0).holds
    s = O.split_system(a, p, 0.0)
    assert s.a2.nonzeros() == c["nnz_a2"]
    # fast path (what the GPU does) == literal setFromTriplets path, bit for bit
    t = O.build_traced_csr(cfg)
    full = O.full_csr_from_traced(t, m, n)
    for x, y in zip(full.arrays(), csr.arrays()):
        assert x.tobytes() == y.tobytes()
    f1, f2 = O.fold_rows_csr(full)
    for got, want in ((f1, s.a1), (f2, s.a2)):
        for x, y in zip(got.arrays(), want.to_csr().arrays()):
            assert x.tobytes() == y.tobytes()


@pytest.mark.parametrize("idx", [2, 4])
def test_baseline_ray_counts_full(idx):
    w = CONFIGS[idx]
    cfg = oracle_cfg(w)
    rays, samples, pitch = O.enumerate_rays(cfg, O.make_grid(cfg))
    assert samples == w.bins and len(rays) == w.m


def test_config2_fast_fold_equals_literal():
    w, cfg, a, csr, f_true, p = oracle_workload(2)
    s = O.split_system(a, p, 0.0)
    t = O.build_traced_csr(cfg)
    full = O.full_csr_from_traced(t, w.m, w.n)
    for x, y in zip(full.arrays(), csr.arrays()):
        assert x.tobytes() == y.tobytes()
    f1, f2 = O.fold_rows_csr(full)
    for got, want in ((f1, s.a1), (f2, s.a2)):
        for x, y in zip(got.arrays(), want.to_csr().arrays()):
            assert x.tobytes() == y.tobytes()
