"""Staged multi-RHS kernels (sart_stage_kernel: blocks of 16 rays (K1) /
voxels (K2), their index union streamed chunk by chunk into a shared-memory
ring by bulk copies, neighbouring vector pairs merged, each entry applied from
the staged S-wide X / W record) against the per-vector multi kernels
(SSB_STAGED=0 SSB_BLOCKED=0). Both sum every vector and slice in CSR / CSC
order, one product at a time (the pair merge adds exact zeros), so the
iterates are bitwise equal."""
import numpy as np
import pytest

import paper_1902_10559_b200 as P
from test_gpu_multi import plan_with, slices

pytestmark = pytest.mark.gpu


def run(split, opts, S, p1, p2, staged):
    pl = plan_with(split, opts, S, blocked=0, staged=staged)
    d = pl.describe()
    for name in (d["fwd_kernel"], d["back_kernel"]):
        assert ("stage" in name) == bool(staged), d
    pl.set_rhs(0, p1)
    pl.set_rhs(1, p2)
    rep = pl.run()
    return pl, rep


@pytest.mark.parametrize("idx,S,dtype", [(2, 64, "f32"), (4, 128, "f32"), (2, 32, "f64"),
                                         (1, 128, "f64"), (1, 32, "f32")])
def test_staged_equals_per_row(idx, S, dtype):
    w, split, p1, p2 = slices(idx, S)
    opts = P.SolveOptions(max_iters=7, tol=0.0, relaxation=w.relaxation, dtype=dtype)
    a, ra = run(split, opts, S, p1, p2, 1)
    b, rb = run(split, opts, S, p1, p2, 0)
    assert ra.iterations == rb.iterations == 7
    for which in (0, 1):
        assert a.solution(which).tobytes() == b.solution(which).tobytes()
        for sl in (0, S // 2, S - 1):
            assert np.allclose(a.history(which, sl), b.history(which, sl), rtol=1e-13, atol=0)


def test_staged_tolerance_stop_per_slice():
    """slices stop independently (per-slice state), as with the per-row kernel"""
    w, split, p1, p2 = slices(2, 32)
    opts = P.SolveOptions(max_iters=100, tol=0.05, relaxation=w.relaxation, dtype="f64")
    out = []
    for staged in (1, 0):
        pl, rep = run(split, opts, 32, p1, p2, staged)
        out.append((rep.iterations, [len(pl.history(0, s)) for s in range(32)],
                    pl.solution(1).tobytes()))
    assert out[0] == out[1]
    assert len(set(out[0][1])) > 1  # the slices really stopped at different passes


def test_staged_not_used_for_other_slice_counts():
    w, split, p1, p2 = slices(2, 5)
    opts = P.SolveOptions(max_iters=3, tol=0.0, relaxation=w.relaxation, dtype="f64")
    pl = plan_with(split, opts, 5, blocked=0, staged=1)
    assert "stage" not in pl.describe()["fwd_kernel"] + pl.describe()["back_kernel"]
