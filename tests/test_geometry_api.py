"""Row A1 / A3 entry points on their own: emitter_angles / emitter_positions
(host, libm — reference geometry.cpp:107-130) and ray_weights for one ray on
the device tracer (geometry.cpp:175-225), against the oracle bit for bit and
the reference's geometry pins (tests/unit/test_geometry.cpp:44-183)."""
import numpy as np
import pytest

import pyoracle as O
from helpers import deg
from test_oracle_pins import liang_barsky

import paper_1902_10559_b200 as P


def _grid(g):
    return P.make_grid(P.scan_config()) if g is None else g


def test_emitter_angles_and_positions_match_oracle(pins):
    for k, gamma_deg in ((4, 30.0), (10, 18.0), (50, 24.5), (100, 24.75)):
        cfg = P.scan_config(k=k, gamma_deg=gamma_deg, h_e=2.0, h_m=1e-4)
        ocfg = O.scan_config(k, deg(gamma_deg), 2.0, 1e-4, 0.43, 1024, 0.1, 32, 32)
        a = P.emitter_angles(cfg)
        assert a.tobytes() == O.emitter_angles(ocfg).tobytes()
        assert np.all(a[::-1] == -a)  # exact sign flips (test_geometry.cpp:44-63)
        for cx in (0.0, 0.125):
            xy = P.emitter_positions(cfg, cx)
            assert xy.tobytes() == O.emitter_positions(ocfg, cx).tobytes()
            h = k // 2  # upper half = lower half reflected (as computed, bit for bit)
            assert np.all(xy[::-1][:h, 0] == 2.0 * cx - xy[:h, 0])
            assert np.all(xy[::-1][:h, 1] == xy[:h, 1])
    a4 = P.emitter_angles(P.scan_config(k=4, gamma_deg=30.0))
    assert np.allclose(a4, np.radians(pins["emitter_angles_k4"]["deg"]), rtol=0, atol=1e-15)
    with pytest.raises(P.Error, match="geometry: k must be even"):
        P.emitter_angles(P.scan_config(k=5))


@pytest.mark.gpu
def test_ray_weights_pins(pins):
    c = pins["vertical_ray"]
    g = P.symsplit.N.GridSpec(**c["grid"])
    xc = g.center_x + (2 - 0.5 - 0.5 * g.n_x) * g.voxel_size
    js, lens = P.ray_weights([xc, 3.0, xc, 0.0], g)
    assert len(js) == c["entries"] and np.all(np.abs(lens - g.voxel_size) <= c["tol"])
    assert all(P.snake_inverse(int(j), g)[0] == 2 for j in js)
    c = pins["diagonal_ray"]
    g = P.symsplit.N.GridSpec(**c["grid"])
    vs, xl = g.voxel_size, g.center_x - 0.5 * g.n_x * g.voxel_size
    js, lens = P.ray_weights([xl - vs, g.y_bottom - vs, xl + 2 * vs,
                              g.y_bottom + g.n_y * vs + vs], g)
    assert np.all(js == 1) and abs(lens.sum() - vs * np.sqrt(2.0)) <= c["rel_tol"] * vs * np.sqrt(2)
    with pytest.raises(P.Error, match="ray_weights: degenerate ray"):
        P.ray_weights([0.1, 0.2, 0.1, 0.2], g)
    assert len(P.ray_weights([5.0, 5.0, 6.0, 6.0], g)[0]) == 0  # misses the grid


@pytest.mark.gpu
def test_ray_weights_bitexact_and_chord_conservation(pins):
    c = pins["chord_conservation"]
    g = P.symsplit.N.GridSpec(32, 32, 0.1 / 32, 0.0, 0.25)
    og = O.GridC(32, 32, 0.1 / 32, 0.0, 0.25)
    u = O.rng_uniform(c["seed"], 4 * c["trials"])
    hits = 0
    for t in range(c["trials"]):
        a, b, cc, d = u[4 * t:4 * t + 4]
        ray = [-0.3 + 0.6 * a, 1.0 + 0.3 * b, -0.3 + 0.6 * cc, 0.0]
        js, lens = P.ray_weights(ray, g)
        ojs, olens = O.ray_weights(ray, og)
        assert js.tobytes() == ojs.astype(np.int32).tobytes()
        assert lens.tobytes() == olens.tobytes()
        chord = liang_barsky(ray, og)
        assert abs(lens.sum() - chord) <= c["tol"]
        hits += chord > 0
    assert hits > 0
