"""CPU-only checks of the product library: it loads, exports every symbol the
C ABI header declares, and its host-side logic (scan config, snake numbering,
ray enumeration, phantom parameters, noise, row partition) matches the oracle
bit for bit. No compute call needs a GPU here; on a GPU-less host, device
entry points must fail loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import pyoracle as O
from helpers import deg, oracle_cfg

import paper_1902_10559_b200 as P
from paper_1902_10559_b200 import _native as N
from paper_1902_10559_b200.configs import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "symsplit_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\*]+\s+\**(ss_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.load()
    names = declared_symbols()
    assert len(names) >= 50
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.SIGNATURES), set(names) ^ set(N.SIGNATURES)


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.DeviceError):
        P.Context(0)


def test_default_options_match_reference():
    o = N.SolveOptionsC()
    # a C caller's stack struct holds garbage: every field must be written
    C.memset(C.byref(o), 0x5A, C.sizeof(o))
    N.load().ss_default_options(C.byref(o))
    assert (o.max_iters, o.tol, o.relaxation, o.parallelism, o.dtype) == (200, 1e-10, 1.0, 0, 0)
    assert o.method == 0 and o.dense_cap == 0  # 0 = the reference's 5e7 cap
    d = P.SolveOptions()
    assert (d.max_iters, d.tol, d.relaxation, d.parallelism) == (200, 1e-10, 1.0, 0)


def test_parse_scan_config(pins):
    c = pins["scan_config_text"]
    cfg = P.parse_scan_config(c["text"])
    ocfg = O.parse_scan_config(c["text"])
    for f in ("k", "gamma", "h_e", "h_m", "l_m", "n_p", "obj_size", "grid_nx", "grid_ny"):
        assert getattr(cfg, f) == getattr(ocfg, f), f
    g = P.make_grid(cfg)
    og = O.make_grid(ocfg)
    assert (g.n_x, g.n_y, g.voxel_size, g.center_x, g.y_bottom) == \
        (og.n_x, og.n_y, og.voxel_size, og.center_x, og.y_bottom)
    for bad, msg in (("unknown_key 3\n", "unknown key 'unknown_key'"),
                     ("k 8 9\n", "trailing content '9'"),
                     ("k\n", "missing numeric value for key 'k'")):
        with pytest.raises(P.Error, match=msg):
            P.parse_scan_config(bad)


def test_snake(pins):
    g = P.make_grid(P.scan_config(grid_nx=2, grid_ny=2))
    for c, r, j in pins["snake_2x2"]["cases"]:
        assert P.snake_index(c, r, g) == j
    with pytest.raises(P.Error):
        P.snake_index(3, 1, g)
    with pytest.raises(P.Error):
        P.snake_inverse(5, g)
    for nx, ny in pins["snake_mirror_grids"]["grids"]:
        g = P.make_grid(P.scan_config(grid_nx=nx, grid_ny=ny))
        for j in range(1, nx * ny + 1):
            c, r = P.snake_inverse(j, g)
            assert P.snake_index(c, r, g) == j
            assert P.snake_inverse(nx * ny - j + 1, g) == (nx - c + 1, r)


@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
def test_enumerate_rays_bitexact(idx):
    w = CONFIGS[idx]
    rays, samples, pitch = P.enumerate_rays(w.scan_config())
    cfg = oracle_cfg(w)
    orays, osamples, opitch = O.enumerate_rays(cfg, O.make_grid(cfg))
    assert (samples, pitch) == (osamples, opitch) and samples == w.bins
    assert rays.tobytes() == orays.tobytes()
    assert len(rays) == w.m  # every BASELINE ray hits the grid (h_m = 1e-4)


def test_enumerate_rays_reference_scan():
    # test_geometry.cpp:98-105: default scan, 32x32 grid
    rays, _, _ = P.enumerate_rays(P.scan_config())
    assert len(rays) % 2 == 0 and 1000 <= len(rays) <= 5000
    with pytest.raises(P.Error, match="k must be even"):
        P.enumerate_rays(P.scan_config(k=7))


def test_random_ellipses_and_noise_bitexact():
    for seed in (1000, 2000, 4007):
        assert P.random_ellipses(seed, 8).tobytes() == O.random_ellipses(seed, 8).tobytes()
    p = np.linspace(0.0, 3.0, 1001)
    got = p.copy()
    N.load().ss_add_noise(got.ctypes.data_as(N.dp), len(got), C.c_double(0.03), C.c_uint64(77))
    assert got.tobytes() == O.add_noise(p, 0.03, 77).tobytes()


def test_partition_rows_balanced():
    rng = np.random.default_rng(0)
    lens = rng.integers(0, 300, size=5000)
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    for parts in (1, 2, 3, 4, 7):
        b = P.symsplit.partition_rows(ptr, parts)
        assert b[0] == 0 and b[-1] == 5000 and np.all(np.diff(b) >= 0)
        w = [(ptr[b[i + 1]] - ptr[b[i]]) + (b[i + 1] - b[i]) for i in range(parts)]
        assert max(w) - min(w) <= 2 * (lens.max() + 1)


def test_configs_match_baseline_wording():
    # BASELINE.json configs: K, angle range/step, bins, grid, iterations, lambda
    c = CONFIGS
    assert (c[1].grid_nx, c[1].grid_ny, c[1].k, c[1].bins, c[1].m, c[1].iters) == (64, 64, 10, 128, 1280, 50)
    assert (c[2].n, c[2].m, c[2].iters, c[2].relaxation) == (65536, 12288, 100, 0.8)
    assert (c[3].grid_nx, c[3].grid_ny, c[3].m, c[3].iters) == (1024, 512, 102400, 200)
    assert (c[4].m, c[4].slices, c[4].iters) == (30720, 256, 100)
    assert (c[5].n, c[5].m, c[5].iters, c[5].relaxation) == (4194304, 409600, 50, 0.5)
    for w, first, step in ((c[1], 2.0, 4.0), (c[2], 1.0, 2.0), (c[3], 0.5, 1.0), (c[4], 1.0, 2.0),
                           (c[5], 0.25, 0.5)):
        a = np.degrees(O.emitter_angles(oracle_cfg(w)))
        assert abs(a[len(a) // 2] - first) < 1e-9 and abs(np.diff(a)[0] - step) < 1e-9
