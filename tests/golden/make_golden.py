"""Regenerates tests/golden/oracle_cfg{1,2}.json + oracle_cfg1_f.npy from the CPU
oracle (test infrastructure; run from the repo root:
`python tests/golden/make_golden.py`). The digests pin the build, the fold,
the seeded phantom / projection and the fixed-count solve_split of BASELINE
configs 1 and 2 (config 2: 20 iterations, bounded oracle time), so a change
in either the oracle or the product shows up against committed values."""
import hashlib
import math
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import pyoracle as O  # noqa: E402
from helpers import oracle_workload  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


ITERS = {1: None, 2: 20}  # None: the config's own iteration count


def golden(idx):
    w, cfg, a, csr, f_true, p = oracle_workload(idx, literal=True)
    ptr, ind, val = csr.arrays()
    sp = O.split_system(a, p, 0.0)
    iters = ITERS[idx] or w.iters
    r = O.solve_split(a, p, 0.0, iters, 0.0, w.relaxation)
    return {
        "config": idx,
        "m": int(len(ptr) - 1), "n": int(w.n), "nnz": int(len(val)),
        "csr_sha256": sha(ptr, ind, val),
        "a1_csr_sha256": sha(*sp.a1.to_csr().arrays()),
        "a2_csr_sha256": sha(*sp.a2.to_csr().arrays()),
        "f_true_sha256": sha(f_true),
        "p_sha256": sha(p),
        "p1_p2_sha256": sha(sp.p1, sp.p2),
        "iters": iters, "relaxation": w.relaxation,
        # exactly rounded sums (math.fsum): no BLAS / CPU dependence
        "f_norm": math.sqrt(math.fsum(float(v) * float(v) for v in r.f)),
        "f_sum": math.fsum(float(v) for v in r.f),
        "residual_norm": float(r.residual_norm),
        "f_sha256": sha(r.f),
    }, r.f


if __name__ == "__main__":
    for idx in (1, 2):
        g, f = golden(idx)
        with open(os.path.join(HERE, f"oracle_cfg{idx}.json"), "w") as fh:
            json.dump(g, fh, indent=1)
        if idx == 1:
            np.save(os.path.join(HERE, "oracle_cfg1_f.npy"), f)
        print(idx, g["nnz"], g["f_sha256"][:16])
