"""Shared test helpers: BASELINE workloads through the oracle (CPU checker)."""
from __future__ import annotations

import numpy as np

import pyoracle as O
from paper_1902_10559_b200.configs import CONFIGS

kPi = 3.14159265358979323846


def deg(d):
    return d * kPi / 180.0


def oracle_cfg(w):
    return O.scan_config(w.k, deg(w.gamma_deg), w.h_e, w.h_m, w.l_m, w.bins, w.obj_size,
                         w.grid_nx, w.grid_ny)


def oracle_workload(idx, literal=True, slice_=0):
    """Oracle build of a BASELINE config: A (literal setFromTriplets path or the
    fast traced path), f_true, p (with the config's seeded noise)."""
    w = CONFIGS[idx]
    cfg = oracle_cfg(w)
    grid = O.make_grid(cfg)
    if literal:
        a = O.build_system(cfg)
        csr = a.to_csr()
    else:
        t = O.build_traced_csr(cfg)
        csr = O.full_csr_from_traced(t, 2 * t.info()[0], w.n)
        a = None
    ell = O.random_ellipses(w.seed(slice_), 8)
    f_true = O.rasterize(ell, grid)
    p = O.forward_project_csr(csr, f_true)
    if w.noise_frac:
        p = O.add_noise(p, w.noise_frac * float(np.max(p)), w.noise_seed())
    return w, cfg, a, csr, f_true, p


def rel_err(got, want):
    d = np.linalg.norm(np.asarray(want))
    return float(np.linalg.norm(np.asarray(got) - np.asarray(want)) / (d if d > 0 else 1.0))
