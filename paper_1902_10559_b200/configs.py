"""BASELINE.json configs mapped onto the reference ScanConfig.

Mapping: K positions -> k; "+-a..+-b" -> gamma_deg = b (the reference step
2b/(K-1) equals the stated step); emitter height 2.0 -> h_e = 2.0; grid lower
edge h_m = 1e-4 (every ray hits, so M = K*bins); detector l_m = 1.0 with
n_p = bins; unit-width object obj_size = 1.0. Phantoms: 8 seeded ellipses,
seed 1000*c (slice s of config 4: 4000 + s); noise sigma = frac * max(p) with
seed 1000*c + 1. These synthetic inputs stand in for the BASELINE data.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Workload:
    name: str
    grid_nx: int
    grid_ny: int
    k: int
    gamma_deg: float
    bins: int
    iters: int
    relaxation: float
    dtypes: tuple
    noise_frac: float = 0.0
    slices: int = 1
    h_e: float = 2.0
    h_m: float = 1e-4
    l_m: float = 1.0
    obj_size: float = 1.0

    @property
    def index(self) -> int:
        return int(self.name[-1])

    @property
    def m(self) -> int:
        return self.k * self.bins

    @property
    def n(self) -> int:
        return self.grid_nx * self.grid_ny

    def seed(self, slice_: int = 0) -> int:
        return 4000 + slice_ if self.slices > 1 else 1000 * self.index

    def noise_seed(self) -> int:
        return 1000 * self.index + 1

    def scan_config(self):
        from . import symsplit as S
        return S.scan_config(k=self.k, gamma_deg=self.gamma_deg, h_e=self.h_e, h_m=self.h_m,
                             l_m=self.l_m, n_p=self.bins, obj_size=self.obj_size,
                             grid_nx=self.grid_nx, grid_ny=self.grid_ny)


CONFIGS = {
    1: Workload("cfg1", 64, 64, 10, 18.0, 128, 50, 1.0, ("f64",)),
    2: Workload("cfg2", 256, 256, 24, 23.0, 512, 100, 0.8, ("f64", "f32"), noise_frac=0.01),
    3: Workload("cfg3", 1024, 512, 50, 24.5, 2048, 200, 1.0, ("f32",)),
    4: Workload("cfg4", 512, 512, 30, 29.0, 1024, 100, 1.0, ("f32",), slices=256),
    5: Workload("cfg5", 2048, 2048, 100, 24.75, 4096, 50, 0.5, ("f32",), noise_frac=0.005),
}
