"""Committed oracle fixtures (tests/golden/oracle_cfg*.json, made by
tests/golden/make_golden.py): the CPU oracle must reproduce them exactly (CPU),
and the device path must match them (GPU: bit-exact build / fold / phantom /
projection digests; solve_split f within the north-star tolerances)."""
import hashlib
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))


def load(idx):
    with open(os.path.join(HERE, "golden", f"oracle_cfg{idx}.json")) as f:
        return json.load(f)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("idx", [1, 2])
def test_oracle_reproduces_golden(idx):
    import make_golden
    got, f = make_golden.golden(idx)
    assert got == load(idx)
    if idx == 1:
        assert f.tobytes() == np.load(os.path.join(HERE, "golden", "oracle_cfg1_f.npy")).tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("idx", [1, 2])
def test_device_path_matches_golden(idx):
    import paper_1902_10559_b200 as P
    from paper_1902_10559_b200.configs import CONFIGS
    g = load(idx)
    w = CONFIGS[idx]
    s = P.build_system(w.scan_config())
    assert s.a.shape == (g["m"], g["n"]) and sha(*s.a.to_csr()) == g["csr_sha256"]
    f_true = P.rasterize(P.random_ellipses(w.seed(), 8), P.make_grid(w.scan_config()))
    assert sha(f_true) == g["f_true_sha256"]
    p = P.forward_project(s.a, f_true)
    if w.noise_frac:
        p = P.forward_project(s.a, f_true, w.noise_frac * float(np.max(p)), w.noise_seed())
    assert sha(p) == g["p_sha256"]
    sp = P.split_system(P.CentroSystem(s.a, p, 0.0))
    assert sha(*sp.a1.to_csr()) == g["a1_csr_sha256"]
    assert sha(*sp.a2.to_csr()) == g["a2_csr_sha256"]
    assert sha(sp.p1, sp.p2) == g["p1_p2_sha256"]
    for dtype, tol in (("f64", 1e-10), ("f32", 1e-4)):
        r = P.solve_split(P.CentroSystem(s.a, p, 0.0),
                          P.SolveOptions(max_iters=g["iters"], tol=0.0,
                                         relaxation=g["relaxation"], dtype=dtype))
        assert abs(np.linalg.norm(r.f) - g["f_norm"]) <= tol * g["f_norm"]
        # ||Af - p|| / ||p|| to the same tolerance (as tests/test_gpu_parity.py)
        assert abs(r.residual_norm - g["residual_norm"]) <= tol * np.linalg.norm(p)
        if idx == 1:
            want = np.load(os.path.join(HERE, "golden", "oracle_cfg1_f.npy"))
            assert np.linalg.norm(r.f - want) <= tol * np.linalg.norm(want)
