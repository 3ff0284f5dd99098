"""Fused peer-memory exchange of the row-sharded SART (SS_XCHG_PEER, SURVEY §8e
level 3) on one GPU.

The multi-GPU kernels (K1x waits for the previous iteration's x chunks, K2x
stores each column chunk into its owner's receive row, the last rank to arrive
reduces in rank order, updates and broadcasts x) run here as an emulated group:
G ranks' plans on one device whose exchange regions are linked directly, every
launch issued in rank order on one stream, so a wait is always on chunks that
launches already completed have reduced (never on a concurrently running
kernel). A single-rank NCCL communicator covers the real (non-emulated) setup.
Parity bar: the unsharded plan within 1e-12 (fp64) / 1e-5 (fp32) and the fp64
oracle within the north-star 1e-10."""
import numpy as np
import pytest

import pyoracle as O
from helpers import oracle_workload, rel_err

import paper_1902_10559_b200 as P

pytestmark = pytest.mark.gpu

_cache = {}


def folded(idx=2):
    if idx not in _cache:
        w, cfg, a, csr, f_true, p = oracle_workload(idx, literal=idx <= 2)
        s = P.build_system(w.scan_config())
        gs = P.split_system(P.CentroSystem(s.a, p, 0.0))
        _cache[idx] = (w, gs, a, p)
    return _cache[idx][:2]


def unsharded(gs, opts):
    ref = P.SartPlan(gs.a2, None, opts)
    ref.set_rhs(0, gs.p2)
    rep = ref.run()
    return ref.solution(0), ref.history(0), rep.iterations


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("parts", [1, 2, 3, 4])
def test_group_matches_unsharded(dtype, parts):
    w, gs = folded(2)
    opts = P.SolveOptions(max_iters=20, tol=0.0, relaxation=w.relaxation, dtype=dtype)
    f_ref, h_ref, _ = unsharded(gs, opts)
    grp = P.symsplit.ShardGroup(gs.a2, parts, opts)
    grp.set_rhs(gs.p2)
    reps = grp.run()
    tol = 1e-12 if dtype == "f64" else 1e-5
    assert all(r.iterations == 20 for r in reps)
    f0 = grp.solution(0)
    assert rel_err(f0, f_ref) <= tol
    for g in range(parts):  # every replica holds the same iterate, bit for bit
        assert grp.solution(g).tobytes() == f0.tobytes()
        h = grp.history(g)
        assert len(h) == 20 and np.allclose(h, h_ref, rtol=tol, atol=0)


def test_group_repeat_is_bitwise_and_epochs_advance():
    """Counters are monotone over solves: a second and third solve on the same
    plans (epoch base advanced on the device) give the identical bits."""
    w, gs = folded(2)
    opts = P.SolveOptions(max_iters=7, tol=0.0, relaxation=w.relaxation, dtype="f64")
    grp = P.symsplit.ShardGroup(gs.a2, 4, opts)
    grp.set_rhs(gs.p2)
    grp.run()
    a = grp.solution(0)
    for _ in range(2):
        grp.run()
        assert grp.solution(0).tobytes() == a.tobytes()
        assert grp.solution(3).tobytes() == a.tobytes()


def test_group_matches_oracle_fp64():
    """Full config-1 iteration count on the folded system A2 against the oracle
    sart_solve (north-star 1e-10)."""
    w, gs = folded(1)
    opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype="f64")
    grp = P.symsplit.ShardGroup(gs.a2, 4, opts)
    grp.set_rhs(gs.p2)
    grp.run()
    a, p = _cache[1][2:]
    sp = O.split_system(a, p, 0.0)
    want = O.sart_solve(sp.a2, sp.p2, max_iters=w.iters, tol=0.0, relaxation=w.relaxation)
    assert rel_err(grp.solution(0), want.f) <= 1e-10
    assert np.allclose(grp.history(0), want.residual_history, rtol=1e-10, atol=0)


def test_group_tolerance_stop():
    """tol > 0: the stop test is settled by every rank from the same rank-order
    ||r||^2, at the same iteration as the unsharded plan (check before update)."""
    w, gs = folded(2)
    probe = P.SolveOptions(max_iters=40, tol=0.0, relaxation=w.relaxation, dtype="f64")
    _, h, _ = unsharded(gs, probe)
    pn = float(np.linalg.norm(gs.p2))
    tol = float(h[12]) / pn * (1 + 1e-9)  # stops at iteration 12
    opts = P.SolveOptions(max_iters=40, tol=tol, relaxation=w.relaxation, dtype="f64")
    f_ref, h_ref, it_ref = unsharded(gs, opts)
    grp = P.symsplit.ShardGroup(gs.a2, 3, opts)
    grp.set_rhs(gs.p2)
    reps = grp.run()
    assert it_ref == 12
    assert all(r.iterations == it_ref for r in reps)
    assert rel_err(grp.solution(1), f_ref) <= 1e-12
    assert len(grp.history(2)) == len(h_ref) == 13
    assert np.allclose(grp.history(2), h_ref, rtol=1e-12, atol=0)


def test_peer_plan_single_rank_nccl():
    """The real (non-emulated) setup path: a one-rank communicator, the region
    and kernels of SS_XCHG_PEER, captured into a CUDA graph (fixed count)."""
    import torch  # noqa: F401  (PyTorch's NCCL first, like bench.py)
    w, gs = folded(2)
    ctx = P.Context(0)
    P.symsplit.attach_nccl(ctx, P.symsplit.nccl_unique_id(), 1, 0)
    for dtype in ("f64", "f32"):
        opts = P.SolveOptions(max_iters=20, tol=0.0, relaxation=w.relaxation, dtype=dtype)
        f_ref, h_ref, _ = unsharded(gs, opts)
        rows = gs.a2.shape[0]
        sh = P.symsplit.ShardedSartPlan(ctx, gs.a2, 0, rows, opts, exchange="peer")
        sh.set_rhs(0, gs.p2)
        sh.run()
        first = sh.solution(0)
        sh.run()  # second solve: epoch base advanced by the first
        tol = 1e-12 if dtype == "f64" else 1e-5
        assert sh.solution(0).tobytes() == first.tobytes()
        sh.profile(7)  # a partial pass count (7 of 20): the last reduce is announced
        sh.run()       # by the final kernel; the next solve must not time out
        assert sh.solution(0).tobytes() == first.tobytes()
        assert rel_err(first, f_ref) <= tol
        assert np.allclose(sh.history(0), h_ref, rtol=tol)


# ---------------------------------------------------------------- the row-sharded pair
def unsharded_pair(gs, opts):
    ref = P.SartPlan(gs.a1, gs.a2, opts)
    ref.set_rhs(0, gs.p1)
    ref.set_rhs(1, gs.p2)
    rep = ref.run()
    return ref, rep.iterations


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("parts", [1, 2, 3, 4])
def test_pair_group_matches_unsharded_pair(dtype, parts):
    """Both folded systems row-sharded over G ranks on the paired streams:
    the unsharded paired plan within 1e-12 (fp64) / 1e-5 (fp32), every rank's
    replica bitwise identical."""
    w, gs = folded(2)
    opts = P.SolveOptions(max_iters=20, tol=0.0, relaxation=w.relaxation, dtype=dtype)
    ref, _ = unsharded_pair(gs, opts)
    grp = P.symsplit.ShardPairGroup(gs.a1, gs.a2, parts, opts)
    grp.set_rhs(gs.p1, gs.p2)
    reps = grp.run()
    tol = 1e-12 if dtype == "f64" else 1e-5
    assert all(r.iterations == 20 for r in reps)
    for which in (0, 1):
        f0 = grp.solution(which)
        assert rel_err(f0, ref.solution(which)) <= tol
        for g in range(parts):
            assert grp.solution(which, g).tobytes() == f0.tobytes()
            h = grp.history(which, g)
            assert len(h) == 20 and np.allclose(h, ref.history(which), rtol=tol, atol=0)
    assert rel_err(grp.recombine(parts - 1), ref.recombine()) <= tol


def test_pair_group_matches_oracle_and_repeats():
    """config 1 at its full 50 iterations against the oracle solve_split
    (north-star 1e-10); repeated solves are bitwise identical."""
    w, gs = folded(1)
    opts = P.SolveOptions(max_iters=w.iters, tol=0.0, relaxation=w.relaxation, dtype="f64")
    grp = P.symsplit.ShardPairGroup(gs.a1, gs.a2, 4, opts)
    grp.set_rhs(gs.p1, gs.p2)
    grp.run()
    a, p = _cache[1][2:]
    want = O.solve_split(a, p, 0.0, w.iters, 0.0, w.relaxation)
    f = grp.recombine(0)
    assert rel_err(f, want.f) <= 1e-10
    for _ in range(2):
        grp.run()
        assert grp.recombine(3).tobytes() == f.tobytes()


def test_pair_group_independent_stops():
    """tol > 0: each system stops at its own iteration (check before update),
    as in the unsharded pair plan; the other system keeps iterating."""
    w, gs = folded(2)
    probe = P.SolveOptions(max_iters=60, tol=0.0, relaxation=w.relaxation, dtype="f64")
    ref, _ = unsharded_pair(gs, probe)
    h1, h2 = ref.history(0), ref.history(1)
    # a tolerance between the two systems' relative residual curves
    r1, r2 = h1 / np.linalg.norm(gs.p1), h2 / np.linalg.norm(gs.p2)
    tol = float(max(r1[9], r2[9]))
    opts = P.SolveOptions(max_iters=60, tol=tol, relaxation=w.relaxation, dtype="f64")
    ref, it_ref = unsharded_pair(gs, opts)
    grp = P.symsplit.ShardPairGroup(gs.a1, gs.a2, 3, opts)
    grp.set_rhs(gs.p1, gs.p2)
    reps = grp.run()
    assert all(r.iterations == it_ref for r in reps)
    for which in (0, 1):
        assert len(grp.history(which, 1)) == len(ref.history(which))
        assert rel_err(grp.solution(which, 2), ref.solution(which)) <= 1e-12


def test_pair_plan_single_rank_nccl():
    """The real setup path of the row-sharded pair with a one-rank communicator."""
    import torch  # noqa: F401
    w, gs = folded(2)
    ctx = P.Context(0)
    P.symsplit.attach_nccl(ctx, P.symsplit.nccl_unique_id(), 1, 0)
    for dtype in ("f64", "f32"):
        opts = P.SolveOptions(max_iters=20, tol=0.0, relaxation=w.relaxation, dtype=dtype)
        ref, _ = unsharded_pair(gs, opts)
        rows = gs.a1.shape[0]
        sh = P.symsplit.ShardedPairPlan(ctx, gs.a1, gs.a2, 0, rows, opts)
        sh.set_rhs(0, gs.p1)
        sh.set_rhs(1, gs.p2)
        sh.run()
        first = sh.recombine()
        sh.run()
        tol = 1e-12 if dtype == "f64" else 1e-5
        assert sh.recombine().tobytes() == first.tobytes()
        assert rel_err(first, ref.recombine()) <= tol
