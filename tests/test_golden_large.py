"""BASELINE configs 3, 4 and 5 at their stated iteration counts.

Committed fixtures tests/golden/oracle_cfg{3,4,5}.json (made offline by
tests/golden/make_golden_large.py from the CPU oracle): SHA-256 of the CSR of
A, A1 and A2 (bit-exact build and fold), of the seeded phantom, p (with noise)
and p1 / p2, and the fp64 solve_split f (norm, sum, values at a seeded sample
of indices) and ||A f - p|| after the config's own iteration count.

CPU half: the oracle still reproduces the config-3 fixture and two config-4
slices (config 5 needs ~40 GB of host RAM and minutes: SSB_GOLDEN_SLOW=1).

GPU half (the parity tests proper, through the C ABI):
  * config 3 (the benched workload): build / fold / projection digests; the
    benched SartPlan (paired mirror-coded streams, CUDA graph) in fp32 at 200
    iterations and solve_split in fp64 at 200 iterations against the live
    oracle's full f (1e-4 / 1e-10 relative) and against the fixture;
  * config 4: digests; all 256 slices as the bench runs them (two multi-RHS
    plans of 128 slices) at 100 iterations; 8 slices (0 and 255 included)
    against the live oracle's full f and the fixture (1e-4);
  * config 5 (1.017G nonzeros): digests of A, A1, A2, p; the benched plan at 50
    iterations against the fixture: f norm and sum, the relative error of f
    estimated from the sampled entries, and ||A f - p|| / ||p|| (1e-4).
"""
import hashlib
import json
import math
import os
import sys

import numpy as np
import pytest

import pyoracle as O
from helpers import oracle_cfg, oracle_workload, rel_err

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

TOL_F32 = 1e-4
TOL_F64 = 1e-10


def load(idx):
    with open(os.path.join(HERE, "golden", f"oracle_cfg{idx}.json")) as f:
        return json.load(f)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        mv = memoryview(a).cast("B")
        for o in range(0, len(mv), 1 << 28):
            h.update(mv[o:o + (1 << 28)])
    return h.hexdigest()


def check_f_against_fixture(f, fix, sample_idx, tol):
    """f norm / sum and the relative error of f estimated from the sampled
    entries (sqrt(N / n_samples * sum of squared sample errors) / ||f_want||)."""
    f = np.asarray(f)
    want = np.asarray(fix["sample_f"])
    got = f[np.asarray(sample_idx)]
    est = math.sqrt(len(f) / len(want) * float(np.sum((got - want) ** 2))) / fix["f_norm"]
    assert est <= tol, f"sampled relative error of f {est:.3e} > {tol}"
    assert abs(float(np.linalg.norm(f)) - fix["f_norm"]) <= tol * fix["f_norm"]
    assert abs(float(np.sum(f)) - fix["f_sum"]) <= tol * float(np.sum(np.abs(f)))
    return est


# ------------------------------------------------------------------ CPU: fixtures reproduce
def test_oracle_reproduces_cfg3_fixture():
    import make_golden_large as G
    got = G.golden(3)
    want = load(3)
    assert got == want


def test_oracle_reproduces_cfg4_fixture_slices():
    import make_golden_large as G
    want = load(4)
    got = G.golden(4, slices=(0, 255))
    for k in ("m", "n", "nnz", "csr_sha256", "a1_csr_sha256", "a2_csr_sha256", "nnz_a1",
              "nnz_a2", "iters", "relaxation", "sample_idx"):
        assert got[k] == want[k], k
    by_slice = {d["slice"]: d for d in want["solves"]}
    for d in got["solves"]:
        assert d == by_slice[d["slice"]]


@pytest.mark.skipif(os.environ.get("SSB_GOLDEN_SLOW") != "1",
                    reason="config 5 oracle: ~40 GB host RAM, minutes (SSB_GOLDEN_SLOW=1)")
def test_oracle_reproduces_cfg5_fixture():
    import make_golden_large as G
    assert G.golden(5) == load(5)


def test_fixtures_are_complete():
    """Every fixture pins the config's own iteration count and the shapes of
    BASELINE.json; config 4 pins 8 slices including 0 and 255."""
    from paper_1902_10559_b200.configs import CONFIGS
    for c in (3, 4, 5):
        g = load(c)
        w = CONFIGS[c]
        assert (g["m"], g["n"], g["iters"], g["relaxation"]) == (w.m, w.n, w.iters, w.relaxation)
        assert g["nnz_a1"] == g["nnz_a2"] and len(g["sample_idx"]) >= 2000
    slices = [d["slice"] for d in load(4)["solves"]]
    assert len(slices) == 8 and 0 in slices and 255 in slices
    assert load(5)["nnz"] == 1016766514


# ------------------------------------------------------------------ GPU parity
_c3 = {}


def cfg3_oracle():
    """Live oracle of config 3: the folded pair and the fp64 solve_split f at
    200 iterations (~20 s of host time)."""
    if not _c3:
        w, cfg, _, csr, f_true, p = oracle_workload(3, literal=False)
        f1, f2 = O.fold_rows_csr(csr)
        m1, m2 = f1.to_matrix(), f2.to_matrix()
        p1, p2 = O.split_rhs(p)
        f, it, _ = O.solve_split_prepared(m1, m2, p1, p2, w.iters, 0.0, w.relaxation, True)
        assert it == w.iters
        res = float(np.linalg.norm(O.forward_project_csr(csr, f) - p))
        _c3.update(w=w, p=p, f=f, res=res)
    return _c3


@pytest.mark.gpu
def test_cfg3_digests():
    import paper_1902_10559_b200 as P
    from paper_1902_10559_b200.configs import CONFIGS
    g, w = load(3), CONFIGS[3]
    s = P.build_system(w.scan_config())
    assert s.a.shape == (g["m"], g["n"]) and s.a.stored == g["nnz"]
    assert sha(*s.a.to_csr()) == g["csr_sha256"]
    fix = g["solves"][0]
    f_true = P.rasterize(P.random_ellipses(w.seed(), 8), P.make_grid(w.scan_config()))
    assert sha(f_true) == fix["f_true_sha256"]
    p = P.forward_project(s.a, f_true)
    assert sha(p) == fix["p_sha256"]
    sp = P.split_system(P.CentroSystem(s.a, p, 0.0))
    assert sha(*sp.a1.to_csr()) == g["a1_csr_sha256"]
    assert sha(*sp.a2.to_csr()) == g["a2_csr_sha256"]
    assert sha(sp.p1, sp.p2) == fix["p1_p2_sha256"]


@pytest.mark.gpu
def test_cfg3_benched_plan_f32_200_iterations():
    """The bench's own path (SartPlan over the paired mirror-coded streams,
    one CUDA graph of 200 passes) at the bench's iteration count."""
    import paper_1902_10559_b200 as P
    o = cfg3_oracle()
    w, p = o["w"], o["p"]
    g = load(3)
    s = P.build_system(w.scan_config())
    sp = P.split_system(P.CentroSystem(s.a, p, 0.0))
    plan = P.SartPlan(sp.a1, sp.a2, P.SolveOptions(max_iters=w.iters, tol=0.0,
                                                   relaxation=w.relaxation, dtype="f32"))
    assert plan.describe()["layout"].startswith("paired")
    plan.set_rhs(0, sp.p1)
    plan.set_rhs(1, sp.p2)
    rep = plan.run()
    assert rep.iterations == w.iters
    f = plan.recombine()
    err = rel_err(f, o["f"])
    assert err <= TOL_F32, f"cfg3 fp32 200 iterations: rel err {err:.3e}"
    res = float(np.linalg.norm(s.a.apply(f) - p))
    assert abs(res - o["res"]) / np.linalg.norm(p) <= TOL_F32
    check_f_against_fixture(f, g["solves"][0], g["sample_idx"], TOL_F32)
    assert abs(res - g["solves"][0]["residual_norm"]) / g["solves"][0]["p_norm"] <= TOL_F32


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [("f64", TOL_F64), ("f32", TOL_F32)])
def test_cfg3_solve_split_200_iterations(dtype, tol):
    """ss_solve_split (the reference-facing one-shot call, the e2e path)."""
    import paper_1902_10559_b200 as P
    o = cfg3_oracle()
    w, p = o["w"], o["p"]
    s = P.build_system(w.scan_config())
    r = P.solve_split(P.CentroSystem(s.a, p, 0.0),
                      P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation,
                                     dtype=dtype))
    assert r.iterations == w.iters
    err = rel_err(r.f, o["f"])
    assert err <= tol, f"cfg3 {dtype} solve_split 200 iterations: rel err {err:.3e}"
    assert abs(r.residual_norm - o["res"]) / np.linalg.norm(p) <= tol


@pytest.mark.gpu
def test_cfg4_all_slices_100_iterations():
    import paper_1902_10559_b200 as P
    from paper_1902_10559_b200.configs import CONFIGS
    from concurrent.futures import ThreadPoolExecutor
    g, w = load(4), CONFIGS[4]
    cfg = w.scan_config()
    s = P.build_system(cfg)
    assert s.a.stored == g["nnz"] and sha(*s.a.to_csr()) == g["csr_sha256"]
    grid = P.make_grid(cfg)
    split = P.split_system(P.CentroSystem(s.a, np.zeros(w.m), 0.0))
    assert sha(*split.a1.to_csr()) == g["a1_csr_sha256"]
    assert sha(*split.a2.to_csr()) == g["a2_csr_sha256"]
    fixes = {d["slice"]: d for d in g["solves"]}
    p1 = np.empty((w.slices, w.m // 2))
    p2 = np.empty((w.slices, w.m // 2))
    ps = {}
    for sl in range(w.slices):
        f = P.rasterize(P.random_ellipses(w.seed(sl), 8), grid)
        p = P.forward_project(s.a, f)
        p1[sl], p2[sl] = P.split_rhs(p)
        if sl in fixes:
            assert sha(f) == fixes[sl]["f_true_sha256"]
            assert sha(p) == fixes[sl]["p_sha256"]
            assert sha(p1[sl], p2[sl]) == fixes[sl]["p1_p2_sha256"]
            ps[sl] = p
    # the bench's layout: two multi-RHS plans of 128 slices
    S = 128
    x1 = np.empty((w.slices, w.n // 2))
    x2 = np.empty((w.slices, w.n // 2))
    opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype="f32")
    for b in range(w.slices // S):
        plan = P.SartPlan(split.a1, split.a2, opts, nrhs=S)
        plan.set_rhs(0, p1[b * S:(b + 1) * S].reshape(-1))
        plan.set_rhs(1, p2[b * S:(b + 1) * S].reshape(-1))
        assert plan.run().iterations == w.iters
        x1[b * S:(b + 1) * S] = plan.solution(0).reshape(S, -1)
        x2[b * S:(b + 1) * S] = plan.solution(1).reshape(S, -1)
    # live oracle (fp64) on the 8 pinned slices, concurrently on the host cores
    t = O.build_traced_csr(oracle_cfg(w))
    full = O.full_csr_from_traced(t, w.m, w.n)
    f1c, f2c = O.fold_rows_csr(full)
    m1, m2 = f1c.to_matrix(), f2c.to_matrix()

    def solve(sl):
        return O.solve_split_prepared(m1, m2, p1[sl], p2[sl], w.iters, 0.0, w.relaxation,
                                      True)[0]

    with ThreadPoolExecutor(4) as ex:
        wants = dict(zip(fixes, ex.map(solve, list(fixes))))
    for sl, fix in fixes.items():
        f = P.recombine_solution(P.SolutionPair(x1[sl], x2[sl]))
        err = rel_err(f, wants[sl])
        assert err <= TOL_F32, f"cfg4 slice {sl}: rel err {err:.3e}"
        check_f_against_fixture(f, fix, g["sample_idx"], TOL_F32)
        res = float(np.linalg.norm(s.a.apply(f) - ps[sl]))
        assert abs(res - fix["residual_norm"]) / fix["p_norm"] <= TOL_F32


@pytest.mark.gpu
def test_cfg5_fullsize_50_iterations():
    """1.017G nonzeros in A: bit-exact build / fold / projection digests and the
    benched plan at 50 iterations against the oracle fixture."""
    import gc
    import paper_1902_10559_b200 as P
    from paper_1902_10559_b200.configs import CONFIGS
    g, w = load(5), CONFIGS[5]
    fix = g["solves"][0]
    cfg = w.scan_config()
    s = P.build_system(cfg)
    assert s.a.shape == (g["m"], g["n"]) and s.a.stored == g["nnz"]
    assert sha(*s.a.to_csr()) == g["csr_sha256"]
    gc.collect()
    rep = P.verify_symmetry(s.a, 0.0)
    assert rep.holds and rep.max_violation == 0.0
    f_true = P.rasterize(P.random_ellipses(w.seed(), 8), P.make_grid(cfg))
    assert sha(f_true) == fix["f_true_sha256"]
    p = P.forward_project(s.a, f_true)
    p = P.forward_project(s.a, f_true, w.noise_frac * float(np.max(p)), w.noise_seed())
    assert sha(p) == fix["p_sha256"]
    sp = P.split_system(P.CentroSystem(s.a, p, 0.0))
    assert sp.a1.stored == g["nnz_a1"] and sp.a2.stored == g["nnz_a2"]
    assert sha(*sp.a1.to_csr()) == g["a1_csr_sha256"]
    gc.collect()
    assert sha(*sp.a2.to_csr()) == g["a2_csr_sha256"]
    gc.collect()
    assert sha(sp.p1, sp.p2) == fix["p1_p2_sha256"]
    plan = P.SartPlan(sp.a1, sp.a2, P.SolveOptions(max_iters=w.iters, tol=0.0,
                                                   relaxation=w.relaxation, dtype="f32"))
    plan.set_rhs(0, sp.p1)
    plan.set_rhs(1, sp.p2)
    assert plan.run().iterations == w.iters
    for which in (0, 1):
        h = plan.history(which)
        assert len(h) == w.iters and np.all(np.isfinite(h)) and np.all(np.diff(h) < 0)
    f = plan.recombine()
    check_f_against_fixture(f, fix, g["sample_idx"], TOL_F32)
    res = float(np.linalg.norm(s.a.apply(f) - p))
    assert abs(res - fix["residual_norm"]) / fix["p_norm"] <= TOL_F32
