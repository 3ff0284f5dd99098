"""GPU path vs the CPU oracle, through the C ABI. Bit-exact for the build,
fold, split_rhs, recombine, rasterize and forward projection (fp64); f and
||Af - p||/||p|| within 1e-10 relative (fp64) / 1e-4 relative (fp32, against
the fp64 oracle) after the fixed iteration count (north-star tolerances)."""
import numpy as np
import pytest

import pyoracle as O
from helpers import oracle_workload, rel_err

import paper_1902_10559_b200 as P
from paper_1902_10559_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu

TOL_F64 = 1e-10
TOL_F32 = 1e-4

_cache = {}


def workload(idx):
    if idx not in _cache:
        w, cfg, a, csr, f_true, p = oracle_workload(idx, literal=idx <= 2)
        sys_ = P.build_system(w.scan_config())
        _cache[idx] = (w, cfg, a, csr, f_true, p, sys_)
    return _cache[idx]


def same_bytes(x, y):
    x, y = np.asarray(x), np.asarray(y)
    return x.dtype == y.dtype and x.shape == y.shape and x.tobytes() == y.tobytes()


# ------------------------------------------------------------------ build / fold
@pytest.mark.parametrize("idx", [1, 2])
def test_build_system_bitexact(idx):
    w, cfg, a, csr, f_true, p, s = workload(idx)
    assert s.a.shape == (w.m, w.n) and s.symmetry_tol == 0.0 and np.all(s.p == 0)
    got = s.a.to_csr()
    want = csr.arrays()
    assert all(same_bytes(g, e) for g, e in zip(got, want))
    got_c = s.a.to_csc()
    want_c = a.get_csc()
    assert all(same_bytes(g, e) for g, e in zip(got_c, want_c))


def test_build_system_config3_bitexact():
    w, cfg, a, csr, f_true, p, s = workload(3)
    got = s.a.to_csr()
    assert all(same_bytes(g, e) for g, e in zip(got, csr.arrays()))


@pytest.mark.parametrize("idx", [1, 2])
def test_split_system_bitexact(idx):
    w, cfg, a, csr, f_true, p, s = workload(idx)
    want = O.split_system(a, p, 0.0)
    got = P.split_system(P.CentroSystem(s.a, p, 0.0))
    for g, e in ((got.a1, want.a1), (got.a2, want.a2)):
        assert all(same_bytes(x, y) for x, y in zip(g.to_csr(), e.to_csr().arrays()))
        assert all(same_bytes(x, y) for x, y in zip(g.to_csc(), e.get_csc()))
    assert same_bytes(got.p1, want.p1) and same_bytes(got.p2, want.p2)
    assert got.parent_fill == want.parent_fill
    assert got.fill1 == want.fill1 and got.fill2 == want.fill2


def test_fold_config3_bitexact():
    w, cfg, a, csr, f_true, p, s = workload(3)
    f1, f2 = O.fold_rows_csr(csr)
    got = P.split_system(P.CentroSystem(s.a, p, 0.0))
    for g, e in ((got.a1, f1), (got.a2, f2)):
        assert all(same_bytes(x, y) for x, y in zip(g.to_csr(), e.arrays()))


@pytest.mark.parametrize("idx", [1, 2])
def test_phantom_and_projection_bitexact(idx):
    w, cfg, a, csr, f_true, p, s = workload(idx)
    grid = P.make_grid(w.scan_config())
    ell = P.random_ellipses(w.seed(), 8)
    assert same_bytes(ell, O.random_ellipses(w.seed(), 8))
    img = P.rasterize(ell, grid)
    assert same_bytes(img, f_true)
    pg = P.forward_project(s.a, img)
    if w.noise_frac:
        pg = P.forward_project(s.a, img, w.noise_frac * float(np.max(pg)), w.noise_seed())
    assert same_bytes(pg, p)


def test_verify_symmetry_built():
    w, cfg, a, csr, f_true, p, s = workload(1)
    r = P.verify_symmetry(s.a, 0.0)
    assert r.holds and r.max_violation == 0.0 and (r.worst_row, r.worst_col) == (1, 1)


# ------------------------------------------------------------------ SART parity
# config 3 at its full 200 iterations (and configs 4, 5): tests/test_golden_large.py
@pytest.mark.parametrize("idx", [1, 2])
def test_solve_split_f64(idx):
    w, cfg, a, csr, f_true, p, s = workload(idx)
    iters = w.iters
    if a is None:
        f1, f2 = O.fold_rows_csr(csr)
        p1, p2 = O.split_rhs(p)
        want_f, it, _ = O.solve_split_prepared(f1.to_matrix(), f2.to_matrix(), p1, p2, iters,
                                               0.0, w.relaxation)
        want_res = np.linalg.norm(csr_apply(csr, want_f) - p)
        want_sn = np.linalg.norm(want_f)
    else:
        want = O.solve_split(a, p, 0.0, iters, 0.0, w.relaxation)
        assert want.iterations == iters
        want_f, want_res, want_sn = want.f, want.residual_norm, want.solution_norm
    got = P.solve_split(P.CentroSystem(s.a, p, 0.0),
                        P.SolveOptions(max_iters=iters, tol=0.0, relaxation=w.relaxation))
    assert got.iterations == iters
    assert rel_err(got.f, want_f) <= TOL_F64
    pn = np.linalg.norm(p)
    assert abs(got.residual_norm - want_res) / pn <= TOL_F64
    assert abs(got.solution_norm - want_sn) <= TOL_F64 * want_sn


@pytest.mark.parametrize("idx", [2])
def test_solve_split_f32(idx):
    w, cfg, a, csr, f_true, p, s = workload(idx)
    iters = w.iters
    if a is None:
        f1, f2 = O.fold_rows_csr(csr)
        p1, p2 = O.split_rhs(p)
        want_f, it, _ = O.solve_split_prepared(f1.to_matrix(), f2.to_matrix(), p1, p2, iters,
                                               0.0, w.relaxation)  # recombined f
        want_res = np.linalg.norm(csr_apply(csr, want_f) - p)
    else:
        want = O.solve_split(a, p, 0.0, iters, 0.0, w.relaxation)
        want_f, want_res = want.f, want.residual_norm
    got = P.solve_split(P.CentroSystem(s.a, p, 0.0),
                        P.SolveOptions(max_iters=iters, tol=0.0, relaxation=w.relaxation,
                                       dtype="f32"))
    assert rel_err(got.f, want_f) <= TOL_F32
    assert abs(got.residual_norm - want_res) / np.linalg.norm(p) <= TOL_F32


def csr_apply(csr, x):
    ptr, idx, val = csr.arrays()
    rows = np.repeat(np.arange(len(ptr) - 1), np.diff(ptr))
    return np.bincount(rows, weights=val * x[idx], minlength=len(ptr) - 1)


def test_sart_solve_history_f64():
    w, cfg, a, csr, f_true, p, s = workload(1)
    sp = O.split_system(a, p, 0.0)
    want = O.sart_solve(sp.a1, sp.p1, max_iters=30, tol=0.0, relaxation=1.0)
    gs = P.split_system(P.CentroSystem(s.a, p, 0.0))
    got = P.sart_solve(gs.a1, gs.p1, P.SolveOptions(max_iters=30, tol=0.0))
    assert got.iterations == want.iterations == 30
    assert len(got.residual_history) == len(want.residual_history) == 30
    assert np.max(np.abs(np.array(got.residual_history) - want.residual_history) /
                  want.residual_history) <= TOL_F64
    assert rel_err(got.f, want.f) <= TOL_F64


def test_sart_tolerance_stop_matches():
    w, cfg, a, csr, f_true, p, s = workload(1)
    sp = O.split_system(a, p, 0.0)
    want = O.sart_solve(sp.a2, sp.p2, max_iters=200, tol=0.05)
    gs = P.split_system(P.CentroSystem(s.a, p, 0.0))
    got = P.sart_solve(gs.a2, gs.p2, P.SolveOptions(max_iters=200, tol=0.05))
    assert got.iterations == want.iterations < 200
    assert len(got.residual_history) == want.iterations + 1
    assert rel_err(got.f, want.f) <= TOL_F64


def test_determinism_and_parallelism_invariance():
    w, cfg, a, csr, f_true, p, s = workload(2)
    sysg = P.CentroSystem(s.a, p, 0.0)
    r1 = P.solve_split(sysg, P.SolveOptions(max_iters=20, tol=0.0, parallelism=1))
    r8 = P.solve_split(sysg, P.SolveOptions(max_iters=20, tol=0.0, parallelism=8))
    r8b = P.solve_split(sysg, P.SolveOptions(max_iters=20, tol=0.0, parallelism=8))
    assert r1.f.tobytes() == r8.f.tobytes() == r8b.f.tobytes()


@pytest.mark.parametrize("S", [5, 64, 128, 200])  # 1, 2 and 4 slices per lane (+ a 2nd pass)
def test_multi_rhs_plan_matches_single(S):
    w, cfg, a, csr, f_true, p, s = workload(1)
    gs = P.split_system(P.CentroSystem(s.a, p, 0.0))
    rng = np.random.default_rng(7)
    ps1 = np.stack([gs.p1 * (1 + 0.1 * k) + rng.standard_normal(len(gs.p1)) * 0.01 for k in range(S)])
    ps2 = np.stack([gs.p2 * (1 - 0.05 * k) for k in range(S)])
    opts = P.SolveOptions(max_iters=25, tol=0.0)
    multi = P.SartPlan(gs.a1, gs.a2, opts, nrhs=S)
    multi.set_rhs(0, ps1.reshape(-1))
    multi.set_rhs(1, ps2.reshape(-1))
    multi.run()
    m1, m2 = multi.solution(0), multi.solution(1)
    for k in sorted({0, 1, S // 2, S - 1}):
        single = P.SartPlan(gs.a1, gs.a2, opts)
        single.set_rhs(0, ps1[k])
        single.set_rhs(1, ps2[k])
        single.run()
        assert rel_err(m1[k], single.solution(0)) <= 1e-12
        assert rel_err(m2[k], single.solution(1)) <= 1e-12
        want = O.sart_solve(O.split_system(a, p, 0.0).a1, ps1[k], max_iters=25, tol=0.0)
        assert rel_err(m1[k], want.f) <= TOL_F64
        assert np.allclose(multi.history(0, k), want.residual_history, rtol=TOL_F64, atol=0)


@pytest.mark.parametrize("bands", [2, 3, 5])
def test_multi_rhs_column_bands(bands, monkeypatch):
    """K1 over column bands (partial dots accumulated in w, the last pass forms
    r): the same solution as one pass within 1e-12 (only the in-row summation
    splits at band edges), and the oracle within the north-star tolerance."""
    w, cfg, a, csr, f_true, p, s = workload(1)
    gs = P.split_system(P.CentroSystem(s.a, p, 0.0))
    S = 64
    ps1 = np.stack([gs.p1 * (1 + 0.01 * k) for k in range(S)])
    ps2 = np.stack([gs.p2 * (1 - 0.01 * k) for k in range(S)])
    opts = P.SolveOptions(max_iters=25, tol=0.0)

    def solve():
        pl = P.SartPlan(gs.a1, gs.a2, opts, nrhs=S)
        pl.set_rhs(0, ps1.reshape(-1))
        pl.set_rhs(1, ps2.reshape(-1))
        pl.run()
        return pl.solution(0), pl.solution(1), pl.history(1, S - 1)

    monkeypatch.setenv("SSB_BANDS", "1")
    one = solve()
    monkeypatch.setenv("SSB_BANDS", str(bands))
    banded = solve()
    assert rel_err(banded[0], one[0]) <= 1e-12 and rel_err(banded[1], one[1]) <= 1e-12
    assert np.allclose(banded[2], one[2], rtol=1e-12, atol=0)
    want = O.sart_solve(O.split_system(a, p, 0.0).a2, ps2[S - 1], max_iters=25, tol=0.0)
    assert rel_err(banded[1][S - 1], want.f) <= TOL_F64


# ------------------------------------------------------------------ reference pins on the GPU
def ex1(pins):
    return np.array(pins["example1"]["matrix"], float), np.array(pins["example1"]["rhs"], float)


def test_example1_split_pins(pins):
    d, p = ex1(pins)
    s = P.split_system(P.CentroSystem(P.Matrix.dense(d), p, 0.0))
    e = pins["example1_split"]
    assert np.array_equal(s.a1.to_dense(), e["a1"]) and np.array_equal(s.a2.to_dense(), e["a2"])
    assert np.array_equal(s.p1, e["p1"]) and np.array_equal(s.p2, e["p2"])
    assert s.a1.nonzeros() == e["a1_nonzeros"] and s.a1.stored == 5
    c = pins["split_2x2"]
    s = P.split_system(P.CentroSystem(P.Matrix.dense(c["matrix"]), c["rhs"], 0.0))
    assert s.a1.to_dense()[0, 0] == c["a1"] and s.a2.to_dense()[0, 0] == c["a2"]
    assert s.p1[0] == c["p1"] and s.p2[0] == c["p2"]


def test_symmetry_errors(pins):
    d, p = ex1(pins)
    i, j, v = pins["verify_symmetry_perturbed"]["perturb"]
    d[i, j] = v
    a = P.Matrix.dense(d)
    r = P.verify_symmetry(a, 0.0)
    assert not r.holds and r.max_violation == 8.0 and (r.worst_row, r.worst_col) == (1, 1)
    with pytest.raises(P.SymmetryError) as ei:
        P.split_system(P.CentroSystem(a, p, 1e-12))
    assert ei.value.report.max_violation == 8.0
    assert "not centrosymmetric (max violation 8 at (1,1), tol 1e-12)" in str(ei.value)
    with pytest.raises(P.SymmetryError) as ei:
        P.solve_split(P.CentroSystem(a, p, 1e-12), P.SolveOptions(tol=0.0))
    r = ei.value.report
    assert r.max_violation == 8.0 and (r.worst_row, r.worst_col) == (1, 1)
    r = P.verify_symmetry(P.Matrix.dense(np.eye(3)), 1.0)
    assert not r.holds and r.status == 1
    assert P.verify_symmetry(P.Matrix.dense(np.ones((2, 3))), 1.0).status == 2


def test_rhs_and_recombine_pins(pins):
    for c in pins["split_rhs_cases"]["cases"]:
        p1, p2 = P.split_rhs(c["p"])
        assert np.array_equal(p1, c["p1"]) and np.array_equal(p2, c["p2"])
    with pytest.raises(P.Error):
        P.split_rhs(np.zeros(3))
    c = pins["recombine_general"]
    assert np.array_equal(P.recombine_solution(c["f1"], c["f2"]), c["f"])
    c = pins["recombine_published"]
    assert np.max(np.abs(P.recombine_solution(c["f1"], c["f2"]) - c["f"])) <= c["tol"]
    c = pins["decompose_published"]
    pair = P.decompose_solution(c["f"])
    assert np.max(np.abs(pair.f1 - c["f1"])) <= c["tol"]
    with pytest.raises(P.Error, match="component lengths differ"):
        P.recombine_solution(np.zeros(3), np.zeros(2))
    with pytest.raises(P.Error, match="non-finite component"):
        P.recombine_solution(np.array([np.inf]), np.zeros(1))


def test_forward_project_pin(pins):
    d, _ = ex1(pins)
    a = P.Matrix.dense(d)
    e1 = np.zeros(6)
    e1[0] = 1.0
    assert np.array_equal(P.forward_project(a, e1), pins["forward_project_e1"]["column0"])
    with pytest.raises(P.Error):
        P.forward_project(a, np.zeros(5))


def test_sart_identity_and_errors(pins):
    c = pins["sart_identity"]
    p = O.rng_uniform(c["seed"], c["n"], 0.1, 1.0)
    r = P.sart_solve(P.Matrix.dense(np.eye(c["n"])), p, P.SolveOptions(tol=c["tol"]))
    assert r.iterations == 1 and np.max(np.abs(r.f - p)) <= c["tol"]
    a = P.Matrix.dense(np.eye(2))
    with pytest.raises(P.Error, match="no nonzero rows"):
        P.sart_solve(P.Matrix.from_triplets(4, 4, [], [], []), np.ones(4))
    with pytest.raises(P.Error, match=r"relaxation must be in \(0, 2\]"):
        P.sart_solve(a, np.ones(2), P.SolveOptions(relaxation=2.5))
    with pytest.raises(P.Error, match="max_iters must be >= 1"):
        P.sart_solve(a, np.ones(2), P.SolveOptions(max_iters=0))
    with pytest.raises(P.Error, match="rhs length 3 does not match rows 2"):
        P.sart_solve(a, np.ones(3))
    with pytest.raises(P.Error, match="non-finite rhs"):
        P.sart_solve(a, np.array([1.0, np.nan]))


def test_split_limit_and_branch_failure(pins):
    from test_oracle_pins import split_limit_system
    c = pins["sart_split_limit"]
    ao, p = split_limit_system(c)
    outer, inner, val = ao.get_csc() if ao.is_sparse else (None, None, None)
    a = P.Matrix.dense(ao.to_dense())
    opts = P.SolveOptions(max_iters=c["iters"], tol=c["tol"])
    full = P.sart_solve(a, p, opts)
    split = P.solve_split(P.CentroSystem(a, p, 1e-10), opts)
    assert np.linalg.norm(full.f - split.f) <= c["agree"] * max(1.0, np.linalg.norm(full.f))
    cc = np.array([[1.0, 2.0], [3.0, 0.5]])
    z = O.reconstruct_matrix(O.Matrix.dense(np.zeros((2, 2))), O.Matrix.dense(2.0 * cc))
    with pytest.raises(P.Error, match=r"branch failure: \[system 1\] sart_solve: matrix has no nonzero rows"):
        P.solve_split(P.CentroSystem(P.Matrix.dense(z.to_dense()), np.ones(4), 1e-12),
                      P.SolveOptions(max_iters=10, tol=0.0))


def test_triplets_and_csc_roundtrip():
    a = P.Matrix.from_triplets(2, 2, [0, 1, 0, 0], [0, 1, 0, 0], [1e16, 5.0, 1.0, -1e16])
    outer, inner, val = a.to_csc()
    assert list(outer) == [0, 1, 2] and list(inner) == [0, 1]
    assert val[0] == (1e16 + 1.0) - 1e16 and val[1] == 5.0
    w, cfg, ao, csr, f_true, p, s = workload(1)
    o, i, v = ao.get_csc()
    b = P.Matrix.from_csc(w.m, w.n, o, i, v)
    assert all(same_bytes(x, y) for x, y in zip(b.to_csr(), csr.arrays()))
    x = np.linspace(-1, 1, w.n)
    assert rel_err(b.apply(x), ao.apply(x)) <= 1e-14
    y = np.linspace(0, 1, w.m)
    assert rel_err(b.apply_transpose(y), ao.apply_transpose(y)) <= 1e-14


def test_sharded_plan_single_rank_nccl():
    """Row-sharded plan (ss_plan_create_sharded: K1 on local rows, partial
    back-projection, ncclAllReduce of [A^T w | ||r||^2], shared update) on a
    1-rank NCCL communicator must equal the unsharded plan."""
    import torch  # noqa: F401  (loads PyTorch's NCCL first, like bench.py)
    w, cfg, a, csr, f_true, p, s = workload(2)
    gs = P.split_system(P.CentroSystem(s.a, p, 0.0))
    ctx = P.Context(0)
    P.symsplit.attach_nccl(ctx, P.symsplit.nccl_unique_id(), 1, 0)
    for dtype in ("f64", "f32"):
        opts = P.SolveOptions(max_iters=20, tol=0.0, relaxation=w.relaxation, dtype=dtype)
        ref = P.SartPlan(gs.a2, None, opts)
        ref.set_rhs(0, gs.p2)
        ref.run()
        rows = gs.a2.shape[0]
        sh = P.symsplit.ShardedSartPlan(ctx, gs.a2, 0, rows, opts)
        sh.set_rhs(0, gs.p2)
        sh.run()
        tol = 1e-12 if dtype == "f64" else 1e-5
        assert rel_err(sh.solution(0), ref.solution(0)) <= tol
        assert np.allclose(sh.history(0), ref.history(0), rtol=tol)


# ------------------------------------------------------------------ paired-stream layouts
def _wide_centro(seed, mh, nh, per_row, span):
    """Random centrosymmetric sparse system whose rows reach `span` columns apart
    (forces the 16-bit tiled index stream back to int32 when span >= 65536)."""
    rng = np.random.default_rng(seed)
    m, n = 2 * mh, 2 * nh
    r, c, v = [], [], []
    for i in range(mh):
        lo = int(rng.integers(0, max(1, n - span)))
        cols = np.unique(rng.integers(lo, min(n, lo + span), per_row))
        vals = rng.uniform(0.1, 1.0, len(cols))
        r += [i] * len(cols) + [m - 1 - i] * len(cols)
        c += list(cols) + list(n - 1 - cols)
        v += list(vals) + list(vals)
    p = rng.uniform(0.5, 1.5, m)
    return m, n, np.array(r), np.array(c), np.array(v), p


@pytest.mark.parametrize("span,per_row", [(3000, 150), (200000, 8)])
def test_paired_tiled_layouts_match_oracle(span, per_row, monkeypatch):
    m, n, r, c, v, p = _wide_centro(7 + span, 96, 120000, per_row, span)
    a = P.Matrix.from_triplets(m, n, r, c, v)
    sys_ = P.CentroSystem(a, p, 0.0)
    split = P.split_system(sys_)
    plan = P.SartPlan(split.a1, split.a2, P.SolveOptions(max_iters=12, tol=0.0))
    d = plan.describe()
    assert d["layout"] == "paired-tiled-u16-mirror"
    # K2 (columns list rows < 96) always fits 16 bits (mirror-coded); K1 keeps
    # int32 indices for wide rows (mirror-coded values, layout mode 6)
    assert d["back_kernel"].endswith(", 4>")
    assert d["fwd_kernel"].endswith(", 4>" if span < 65536 else ", 6>")
    # the same system through the interleaved (non-mirror) streams
    monkeypatch.setenv("SSB_MIRROR", "0")
    d0 = P.SartPlan(split.a1, split.a2, P.SolveOptions(max_iters=12, tol=0.0)).describe()
    assert d0["fwd_kernel"].endswith(", 2>" if span < 65536 else ", 1>")
    plain = P.solve_split(sys_, P.SolveOptions(max_iters=12, tol=0.0))
    monkeypatch.setenv("SSB_MIRROR", "1")
    got = P.solve_split(sys_, P.SolveOptions(max_iters=12, tol=0.0))
    ref = O.solve_split(O.Matrix.triplets(m, n, r, c, v), p, 0.0, 12, 0.0, 1.0)
    assert rel_err(got.f, ref.f) <= TOL_F64
    assert rel_err(got.f, plain.f) <= 1e-13
    got32 = P.solve_split(sys_, P.SolveOptions(max_iters=12, tol=0.0, dtype="f32"))
    assert rel_err(got32.f, ref.f) <= TOL_F32


def test_paired_lane_groups_narrow_to_fit_16bit(monkeypatch):
    """Rows of ~110 entries ~2.6K columns apart: 32-entry tiles (8-lane groups)
    span > 65535 columns, 16-entry tiles fit. The paired plan narrows its lane
    groups to keep 16-bit offsets (config 5's K2 case) and still matches the
    oracle; pinning the lane groups at 8 falls back to int32 indices."""
    rng = np.random.default_rng(31)
    mh, nh = 96, 300000
    m, n = 2 * mh, 2 * nh
    r, c, v = [], [], []
    for i in range(mh):
        cols = int(rng.integers(0, 14000)) + np.arange(110) * 2600 + rng.integers(0, 50, 110)
        vals = rng.uniform(0.1, 1.0, len(cols))
        r += [i] * len(cols) + [m - 1 - i] * len(cols)
        c += list(cols) + list(n - 1 - cols)
        v += list(vals) + list(vals)
    r, c, v = np.array(r), np.array(c), np.array(v)
    p = rng.uniform(0.5, 1.5, m)
    a = P.Matrix.from_triplets(m, n, r, c, v)
    sys_ = P.CentroSystem(a, p, 0.0)
    split = P.split_system(sys_)
    monkeypatch.delenv("SSB_VS_FWD", raising=False)
    d = P.SartPlan(split.a1, split.a2, P.SolveOptions(max_iters=12, tol=0.0)).describe()
    assert d["vs_fwd"] == 4 and d["fwd_kernel"].endswith(", 4>")
    got = P.solve_split(sys_, P.SolveOptions(max_iters=12, tol=0.0))
    got32 = P.solve_split(sys_, P.SolveOptions(max_iters=12, tol=0.0, dtype="f32"))
    monkeypatch.setenv("SSB_VS_FWD", "8")
    d8 = P.SartPlan(split.a1, split.a2, P.SolveOptions(max_iters=12, tol=0.0)).describe()
    assert d8["vs_fwd"] == 8 and d8["fwd_kernel"].endswith(", 6>")
    wide = P.solve_split(sys_, P.SolveOptions(max_iters=12, tol=0.0))
    ref = O.solve_split(O.Matrix.triplets(m, n, r, c, v), p, 0.0, 12, 0.0, 1.0)
    assert rel_err(got.f, ref.f) <= TOL_F64
    assert rel_err(wide.f, ref.f) <= TOL_F64
    assert rel_err(got32.f, ref.f) <= TOL_F32


def _mirror_rich_centro(seed, mh, nh, per_row, frac):
    """Centrosymmetric system whose rows also meet the point mirror of a
    fraction `frac` of their columns with a different value: those buckets fold
    to a1 != +-a2 (the mirror-coded stream's exception lists)."""
    rng = np.random.default_rng(seed)
    m, n = 2 * mh, 2 * nh
    r, c, v = [], [], []
    for i in range(mh):
        lo = int(rng.integers(0, n - 4000))
        cols = np.unique(rng.integers(lo, lo + 4000, per_row))
        k = max(1, int(frac * len(cols)))
        extra = n - 1 - cols[:k]  # mirror columns in the same row
        cols = np.unique(np.concatenate([cols, extra]))
        vals = rng.uniform(0.1, 1.0, len(cols))
        r += [i] * len(cols) + [m - 1 - i] * len(cols)
        c += list(cols) + list(n - 1 - cols)
        v += list(vals) + list(vals)
    p = rng.uniform(0.5, 1.5, m)
    return m, n, np.array(r), np.array(c), np.array(v), p


@pytest.mark.parametrize("frac", [0.05, 0.5])
def test_mirror_coded_exceptions_match_oracle(frac, monkeypatch):
    """Mirror-coded pair streams: a1 = +-a2 buckets as one value + sign bit,
    4-term buckets through the per-vector exception lists (both kernels)."""
    m, n, r, c, v, p = _mirror_rich_centro(31, 80, 20000, 200, frac)
    a = P.Matrix.from_triplets(m, n, r, c, v)
    sys_ = P.CentroSystem(a, p, 0.0)
    split = P.split_system(sys_)
    opts = P.SolveOptions(max_iters=15, tol=0.0)
    d = P.SartPlan(split.a1, split.a2, opts).describe()
    assert d["layout"] == "paired-tiled-u16-mirror"
    assert d["exceptions"][0] > 0 and d["exceptions"][1] == d["exceptions"][0]
    ref = O.solve_split(O.Matrix.triplets(m, n, r, c, v), p, 0.0, 15, 0.0, 1.0)
    got = P.solve_split(sys_, opts)
    assert rel_err(got.f, ref.f) <= TOL_F64
    got32 = P.solve_split(sys_, P.SolveOptions(max_iters=15, tol=0.0, dtype="f32"))
    assert rel_err(got32.f, ref.f) <= TOL_F32
    # the interleaved 16-bit stream gives the same iterates up to summation order
    monkeypatch.setenv("SSB_MIRROR", "0")
    assert P.SartPlan(split.a1, split.a2, opts).describe()["layout"] == "paired-tiled-u16"
    plain = P.solve_split(sys_, opts)
    assert rel_err(got.f, plain.f) <= 1e-12
    # CGLS over the same mirror-coded streams
    monkeypatch.setenv("SSB_MIRROR", "1")
    monkeypatch.setenv("SSB_CGLS_PAIRED", "1")
    cg = P.solve_split(sys_, P.SolveOptions(method="cgls", max_iters=5, tol=1e-10))
    want_f, it, res = O.solve_split_method(O.Matrix.triplets(m, n, r, c, v), p, "cgls", 0.0, 5,
                                           1e-10)
    assert cg.iterations == it and rel_err(cg.f, want_f) <= 1e-10
    assert abs(cg.residual_norm - res) <= 1e-10 * res


@pytest.mark.parametrize("span,per_row", [(3000, 150), (200000, 8)])
def test_single_tiled_layouts_match_oracle(span, per_row):
    """sart_solve on one system: single-system tiled streams (16-bit or int32)."""
    m, n, r, c, v, p = _wide_centro(11 + span, 64, 90000, per_row, span)
    a = P.Matrix.from_triplets(m, n, r, c, v)
    plan = P.SartPlan(a, None, P.SolveOptions(max_iters=9, tol=0.0))
    d = plan.describe()
    assert d["layout"] == "single-tiled"
    assert d["fwd_kernel"].endswith("true>" if span < 65536 else "false>")
    got = P.sart_solve(a, p, P.SolveOptions(max_iters=9, tol=0.0))
    ref = O.sart_solve(O.Matrix.triplets(m, n, r, c, v), p, max_iters=9, tol=0.0)
    assert rel_err(got.f, ref.f) <= TOL_F64
    h, hr = np.asarray(got.residual_history), np.asarray(ref.residual_history)
    # late residuals are differences of O(|p|) quantities: compare at |p|*1e-12
    assert h.shape == hr.shape and np.allclose(h, hr, rtol=1e-10, atol=1e-12 * hr[0])


def test_reusable_plan_stops_on_device_like_the_oracle():
    """tol > 0: the captured graph is a WHILE loop whose condition K1's last block
    sets; it must stop at the oracle's iteration with the oracle's history."""
    rng = np.random.default_rng(31)
    h1 = 3 * np.eye(40, 30) + rng.uniform(0, 0.1, (40, 30))  # well conditioned: stops
    h2 = 2 * np.eye(40, 30) + rng.uniform(0, 0.2, (40, 30))  # at ~30 / ~100 passes
    a = O.reconstruct_matrix(O.Matrix.dense(h1), O.Matrix.dense(h2)).to_dense()
    p = a @ rng.uniform(0.5, 1.5, 60)
    split = P.split_system(P.CentroSystem(P.Matrix.dense(a), p, 0.0))
    opts = P.SolveOptions(max_iters=5000, tol=1e-6)
    plan = P.SartPlan(split.a1, split.a2, opts)
    plan.set_rhs(0, split.p1)
    plan.set_rhs(1, split.p2)
    for rep in range(2):  # replays reset the loop state
        r = plan.run()
        o1 = O.sart_solve(O.Matrix.dense(h1), split.p1, max_iters=5000, tol=1e-6)
        o2 = O.sart_solve(O.Matrix.dense(h2), split.p2, max_iters=5000, tol=1e-6)
        assert 0 < o1.iterations < 5000 and 0 < o2.iterations < 5000
        assert r.iterations == max(o1.iterations, o2.iterations)
        assert np.allclose(plan.history(0), o1.residual_history, rtol=1e-9, atol=0)
        assert np.allclose(plan.history(1), o2.residual_history, rtol=1e-9, atol=0)
        assert rel_err(plan.solution(0), o1.f) <= TOL_F64
        assert rel_err(plan.solution(1), o2.f) <= TOL_F64


def test_fused_fold_symmetry_report_matches_verify_symmetry():
    """split_system checks symmetry inside the fold's count pass; its report
    (value, first column-major arg-max, 1-based) must equal verify_symmetry's,
    including ties, missing mirrors and stored zeros."""
    rng = np.random.default_rng(77)
    for trial in range(40):
        mh, nh = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        h1, h2 = rng.uniform(-1, 1, (mh, nh)), rng.uniform(-1, 1, (mh, nh))
        a = O.reconstruct_matrix(O.Matrix.dense(h1), O.Matrix.dense(h2)).to_dense()
        a[np.abs(a) < 0.3] = 0.0
        r, c = np.nonzero(a)
        v = a[r, c].copy()
        kind = trial % 4
        if kind == 0 and len(v):      # one perturbed entry
            v[int(rng.integers(len(v)))] += 0.25
        elif kind == 1 and len(v) > 1:  # two equal violations (tie -> column-major first)
            idx = rng.choice(len(v), 2, replace=False)
            v[idx] += 0.5
        elif kind == 2 and len(v):    # a stored zero where the mirror is non-zero
            v[int(rng.integers(len(v)))] = 0.0
        else:                         # an entry whose mirror is absent
            zr, zc = np.nonzero(a == 0)
            if len(zr):
                t = int(rng.integers(len(zr)))
                r, c, v = np.append(r, zr[t]), np.append(c, zc[t]), np.append(v, 0.75)
        m = P.Matrix.from_triplets(2 * mh, 2 * nh, r, c, v)
        want = P.verify_symmetry(m, 0.0)
        p = np.ones(2 * mh)
        if want.holds:
            P.split_system(P.CentroSystem(m, p, 0.0))
            continue
        with pytest.raises(P.SymmetryError) as ei:
            P.split_system(P.CentroSystem(m, p, 0.0))
        got = ei.value.report
        assert (got.max_violation, got.worst_row, got.worst_col, got.status) == \
            (want.max_violation, want.worst_row, want.worst_col, want.status)
        ref = O.verify_symmetry(O.Matrix.triplets(2 * mh, 2 * nh, r, c, v), 0.0)
        assert (ref.max_violation, ref.worst_row, ref.worst_col) == \
            (want.max_violation, want.worst_row, want.worst_col)
