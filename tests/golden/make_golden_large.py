"""Regenerates tests/golden/oracle_cfg{3,4,5}.json from the CPU oracle (test
infrastructure; run from the repo root, ~62 GB of host RAM for config 5:
`python tests/golden/make_golden_large.py [3] [4] [5]`).

The oracle is too slow / too large to run inside the GPU test session at
BASELINE configs 4 and 5 (1.017G nonzeros in A at config 5), so this script
pins them once, offline, at each config's own iteration count:

  * SHA-256 of the CSR (row pointer, column index, fp64 value bytes) of A and
    of the folded A1 / A2 (bit-exact build and fold, reference
    geometry.cpp:227-275, centro.cpp:103-130);
  * SHA-256 of the seeded phantom, of p (with the config's seeded noise) and of
    p1 / p2 (split_rhs, centro.cpp:89-99);
  * the fp64 solve_split f (solvers.cpp:207-269, SART per branch
    solvers.cpp:148-199) after the fixed iteration count: exactly rounded
    norm and sum (math.fsum), the values at a seeded sample of indices (the
    GPU test estimates the relative error of the whole f from them), and
    ||A f - p|| (config 5 through the exact fold identity
    ||A f - p||^2 = (||A1 f1 - p1||^2 + ||A2 f2 - p2||^2) / 2).

Config 4 pins 8 of its 256 slices (0 and 255 included) at 100 iterations.
"""
import gc
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import pyoracle as O  # noqa: E402
from helpers import oracle_cfg  # noqa: E402
from paper_1902_10559_b200.configs import CONFIGS  # noqa: E402

SLICES_C4 = (0, 37, 74, 111, 148, 185, 222, 255)
N_SAMPLES = {3: 4096, 4: 2048, 5: 4096}


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        mv = memoryview(a).cast("B")
        for o in range(0, len(mv), 1 << 28):  # chunked: config 5 arrays are GBs
            h.update(mv[o:o + (1 << 28)])
    return h.hexdigest()


def csr_sha(c):
    ptr, idx, val = c.arrays()
    s = sha(ptr, idx, val)
    del ptr, idx, val
    gc.collect()
    return s


def sample_indices(n, count, seed):
    """Seeded sample of f indices: the first / last entries, the centre pair
    (mirror partners), and a uniform draw."""
    rng = np.random.default_rng(seed)
    fixed = np.array([0, 1, n // 2 - 1, n // 2, n - 2, n - 1], dtype=np.int64)
    draw = rng.choice(n, size=count - len(fixed), replace=False).astype(np.int64)
    return np.unique(np.concatenate([fixed, draw]))


def f_summary(f, idx):
    return {"f_norm": math.sqrt(math.fsum(float(v) * float(v) for v in f)),
            "f_sum": math.fsum(float(v) for v in f),
            "sample_f": [float(v) for v in f[idx]]}


def log(*a):
    print(*a, flush=True)


def golden(c, slices=None):
    w = CONFIGS[c]
    cfg = oracle_cfg(w)
    grid = O.make_grid(cfg)
    t0 = time.time()
    t = O.build_traced_csr(cfg)
    csr = O.full_csr_from_traced(t, 2 * t.info()[0], w.n)
    del t
    gc.collect()
    m, n, nnz = csr.info()
    log(f"cfg{c}: built A {m}x{n} nnz={nnz} in {time.time() - t0:.1f}s")
    out = {"config": c, "m": m, "n": n, "nnz": nnz, "csr_sha256": csr_sha(csr),
           "iters": w.iters, "relaxation": w.relaxation}
    if slices is None:
        slices = SLICES_C4 if w.slices > 1 else (0,)
    rhs = []
    for s in slices:
        f_true = O.rasterize(O.random_ellipses(w.seed(s), 8), grid)
        p = O.forward_project_csr(csr, f_true)
        if w.noise_frac:
            p = O.add_noise(p, w.noise_frac * float(np.max(p)), w.noise_seed())
        rhs.append((s, f_true, p))
    a1c, a2c = O.fold_rows_csr(csr)
    keep_full = c != 5  # config 5: the residual comes from the fold identity
    if not keep_full:
        del csr
        gc.collect()
    out["nnz_a1"], out["nnz_a2"] = a1c.info()[2], a2c.info()[2]
    out["a1_csr_sha256"] = csr_sha(a1c)
    out["a2_csr_sha256"] = csr_sha(a2c)
    m1 = a1c.to_matrix()
    del a1c
    gc.collect()
    m2 = a2c.to_matrix()
    del a2c
    gc.collect()
    log(f"cfg{c}: folded nnz(A1)={out['nnz_a1']} nnz(A2)={out['nnz_a2']} "
        f"({time.time() - t0:.1f}s)")
    idx = sample_indices(n, N_SAMPLES[c], 7000 + c)
    out["sample_idx"] = [int(i) for i in idx]
    out["solves"] = []
    for s, f_true, p in rhs:
        p1, p2 = O.split_rhs(p)
        t1 = time.time()
        f, it, _ = O.solve_split_prepared(m1, m2, p1, p2, w.iters, 0.0, w.relaxation, True)
        assert it == w.iters
        if keep_full:
            res = float(np.linalg.norm(O.forward_project_csr(csr, f) - p))
        else:
            f1, f2 = O.decompose_solution(f)
            r1 = m1.apply(f1) - p1
            r2 = m2.apply(f2) - p2
            res = math.sqrt((math.fsum(r1 * r1) + math.fsum(r2 * r2)) / 2.0)
        d = {"slice": s, "f_true_sha256": sha(f_true), "p_sha256": sha(p),
             "p1_p2_sha256": sha(p1, p2), "p_norm": float(np.linalg.norm(p)),
             "residual_norm": res}
        d.update(f_summary(f, idx))
        out["solves"].append(d)
        log(f"cfg{c} slice {s}: {w.iters} iters in {time.time() - t1:.1f}s, "
            f"|f|={d['f_norm']:.6g}, res/|p|={res / d['p_norm']:.4g}")
    return out


if __name__ == "__main__":
    which = [int(a) for a in sys.argv[1:]] or [3, 4, 5]
    for c in which:
        g = golden(c)
        with open(os.path.join(HERE, f"oracle_cfg{c}.json"), "w") as fh:
            json.dump(g, fh, indent=0)
        gc.collect()
