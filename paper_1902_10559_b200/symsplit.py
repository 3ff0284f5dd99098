"""Python mirror of the reference `symsplit` API for the folded-SART path.

Same names, argument meaning and error behaviour as the reference C++/pybind11
surface (proj/include/symsplit/*.hpp, proj/python/bindings.cpp), backed by the
sm_100a library through its C ABI (include/symsplit_b200.h). Matrices live on
the GPU; vectors cross the boundary as numpy float64 arrays.

Differences from the reference, all deliberate:
  * Method.sart is the default (the reference defaults to dense_minnorm);
    Method.cgls and Method.dense_minnorm also run on the device;
  * Matrix storage is always sparse on the device — `Matrix.dense(d)` stores
    the nonzero entries, so its fold follows the sparse (4-term) semantics
    (centro.cpp:109-130); for exactly centrosymmetric inputs both agree;
  * SolveOptions.dtype selects fp64 (reference) or fp32 device arithmetic.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N

kPi = 3.14159265358979323846


# ----------------------------------------------------------------- errors
class Error(RuntimeError):
    """symsplit::Error (matrix.hpp:22-25); pybind name SymsplitError."""


SymsplitError = Error


class SymmetryError(Error):
    """symsplit::SymmetryError carrying its SymmetryReport (centro.hpp:73-78)."""

    def __init__(self, what, report):
        super().__init__(what)
        self.report = report


class DeviceError(Error):
    """CUDA / NCCL / out-of-memory failure inside the library."""


class IoError(Error):
    """symsplit::IoError (io.hpp:14-20): file open / parse failures, path and line in the message."""


def _lib():
    return N.load()


def _check(rc, report=None):
    if rc == N.SS_OK:
        return
    msg = _lib().ss_last_error().decode()
    if rc == N.SS_ERR_SYMMETRY:
        raise SymmetryError(msg, report)
    if rc in (N.SS_ERR_CUDA, N.SS_ERR_NCCL, N.SS_ERR_OOM):
        raise DeviceError(msg)
    if rc == N.SS_ERR_IO:
        raise IoError(msg)
    raise Error(msg)


def _f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _i32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def _dp(a):
    return a.ctypes.data_as(N.dp)


def _ip(a):
    return a.ctypes.data_as(N.i32p)


def degrees_to_radians(deg):
    return deg * kPi / 180.0


# ----------------------------------------------------------------- context
class Context:
    """One CUDA stream + workspace on one device (ss_ctx_t)."""

    def __init__(self, device: int = 0):
        h = N.vp()
        _check(_lib().ss_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            _lib().ss_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(_lib().ss_ctx_synchronize(self.h))

    @property
    def stream(self) -> int:
        return _lib().ss_ctx_stream(self.h) or 0

    @property
    def launch_count(self) -> int:
        return int(_lib().ss_ctx_launch_count(self.h))


_ctx_lock = threading.Lock()
_contexts: dict = {}


def default_context(device: int = 0) -> Context:
    with _ctx_lock:
        if device not in _contexts:
            _contexts[device] = Context(device)
        return _contexts[device]


# ----------------------------------------------------------------- matrix
class Matrix:
    """Device sparse matrix (reference Matrix, matrix.hpp:34-87)."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx

    def __del__(self):
        try:
            if getattr(self, "h", None) and N._lib is not None:
                N._lib.ss_matrix_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # -- construction
    @classmethod
    def from_csc(cls, rows, cols, outer, inner, values, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        outer, inner, values = _i32(outer), _i32(inner), _f64(values)
        h = N.vp()
        _check(_lib().ss_matrix_from_csc(ctx.h, rows, cols, len(values), _ip(outer), _ip(inner),
                                         _dp(values), C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_triplets(cls, rows, cols, row, col, values, ctx: Optional[Context] = None):
        """Matrix::from_triplets (matrix.cpp:12-18): repeats summed in order."""
        ctx = ctx or default_context()
        row, col, values = _i32(row), _i32(col), _f64(values)
        h = N.vp()
        _check(_lib().ss_matrix_from_triplets(ctx.h, rows, cols, len(values), _ip(row), _ip(col),
                                              _dp(values), C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def dense(cls, d, ctx: Optional[Context] = None):
        d = np.asarray(d, dtype=np.float64)
        if not np.all(np.isfinite(d)):
            raise Error("matrix contains non-finite values")
        cols_, rows_ = np.nonzero(d.T)  # column-major order of the nonzeros
        return cls.from_triplets(d.shape[0], d.shape[1], rows_, cols_, d[rows_, cols_], ctx)

    # -- queries
    @property
    def shape(self):
        r, c, s = N.i64(), N.i64(), N.i64()
        _check(_lib().ss_matrix_shape(self.h, C.byref(r), C.byref(c), C.byref(s)))
        return r.value, c.value

    def rows(self):
        return self.shape[0]

    def cols(self):
        return self.shape[1]

    @property
    def stored(self) -> int:
        r, c, s = N.i64(), N.i64(), N.i64()
        _check(_lib().ss_matrix_shape(self.h, C.byref(r), C.byref(c), C.byref(s)))
        return s.value

    def is_sparse(self):
        return True

    def nonzeros(self) -> int:
        out = N.i64()
        _check(_lib().ss_matrix_nonzeros(self.h, C.byref(out)))
        return out.value

    def fill_ratio(self) -> float:
        out = C.c_double()
        _check(_lib().ss_matrix_fill_ratio(self.h, C.byref(out)))
        return out.value

    def to_csr(self):
        rows, cols = self.shape
        nnz = self.stored
        ptr = np.empty(rows + 1, np.int32)
        idx = np.empty(nnz, np.int32)
        val = np.empty(nnz, np.float64)
        _check(_lib().ss_matrix_download_csr(self.h, _ip(ptr), _ip(idx), _dp(val)))
        return ptr, idx, val

    def to_csc(self):
        rows, cols = self.shape
        nnz = self.stored
        outer = np.empty(cols + 1, np.int32)
        inner = np.empty(nnz, np.int32)
        val = np.empty(nnz, np.float64)
        _check(_lib().ss_matrix_download_csc(self.h, _ip(outer), _ip(inner), _dp(val)))
        return outer, inner, val

    def to_dense(self):
        rows, cols = self.shape
        ptr, idx, val = self.to_csr()
        d = np.zeros((rows, cols))
        for i in range(rows):
            d[i, idx[ptr[i]:ptr[i + 1]]] = val[ptr[i]:ptr[i + 1]]
        return d

    def coeff(self, i, j):
        """matrix.cpp:44-50: stored value at 0-based (i, j), or 0."""
        out = C.c_double()
        _check(_lib().ss_matrix_coeff(self.h, int(i), int(j), C.byref(out)))
        return out.value

    def release_cache(self):
        """Free the fold and SART plan solve_split keeps on this matrix."""
        _check(_lib().ss_matrix_release_cache(self.h))

    def for_each(self, f):
        """matrix.hpp:76-87: f(row, col, value) over the stored entries in
        compressed-column order."""
        outer, inner, val = self.to_csc()
        for j in range(len(outer) - 1):
            for k in range(outer[j], outer[j + 1]):
                f(int(inner[k]), j, float(val[k]))

    def apply(self, x):
        x = _f64(x)
        rows, cols = self.shape
        if x.shape != (cols,):
            raise Error("matrix-vector size mismatch")
        y = np.empty(rows)
        _check(_lib().ss_matrix_apply(self.h, _dp(x), _dp(y)))
        return y

    def apply_transpose(self, y):
        y = _f64(y)
        rows, cols = self.shape
        if y.shape != (rows,):
            raise Error("matrix-vector size mismatch")
        x = np.empty(cols)
        _check(_lib().ss_matrix_apply_transpose(self.h, _dp(y), _dp(x)))
        return x


# ----------------------------------------------------------------- value types
@dataclass
class SymmetryReport:
    holds: bool = False
    max_violation: float = 0.0
    worst_row: int = 1
    worst_col: int = 1
    status: int = 0  # 0 ok, 1 odd_row_count, 2 odd_col_count

    @classmethod
    def _from(cls, r: N.SymmetryReportC):
        return cls(bool(r.holds), r.max_violation, r.worst_row, r.worst_col, r.status)


@dataclass
class CentroSystem:
    a: Matrix
    p: np.ndarray
    symmetry_tol: float = 1e-12


@dataclass
class SplitSystem:
    a1: Matrix
    p1: np.ndarray
    a2: Matrix
    p2: np.ndarray
    parent_fill: float = 0.0
    fill1: float = 0.0
    fill2: float = 0.0


@dataclass
class SolutionPair:
    f1: np.ndarray
    f2: np.ndarray


@dataclass
class SolveOptions:
    """reference SolveOptions (solvers.hpp:19-27). The default method here is
    SART (the B200 product path); the reference's default is dense_minnorm."""
    max_iters: int = 200
    tol: float = 1e-10
    relaxation: float = 1.0
    parallelism: int = 0
    dtype: str = "f64"  # "f64" (reference arithmetic) or "f32"
    method: str = "sart"  # "sart", "cgls", "dense" / "dense_minnorm"
    dense_cap: int = 50_000_000

    def _c(self):
        codes = {"sart": 0, "cgls": 1, "dense": 2, "dense_minnorm": 2}
        if self.method not in codes:
            raise Error(f"unknown method name: {self.method}")  # solvers.cpp:73-78
        if self.dtype not in ("f64", "f32"):
            raise Error("dtype must be 'f64' or 'f32'")
        return N.SolveOptionsC(int(self.max_iters), float(self.tol), float(self.relaxation),
                               int(self.parallelism), N.SS_F64 if self.dtype == "f64" else N.SS_F32,
                               codes[self.method], int(self.dense_cap))


@dataclass
class SolveReport:
    f: np.ndarray
    residual_norm: float = 0.0
    solution_norm: float = 0.0
    iterations: int = 0
    wall_time_seconds: float = 0.0
    method: str = "sart"
    mode: str = "direct"
    residual_history: list = field(default_factory=list)
    split_seconds: float = 0.0
    recombine_seconds: float = 0.0
    branch1_seconds: float = 0.0
    branch2_seconds: float = 0.0


def _report(f, r: N.SolveReportC, mode, hist=()):
    return SolveReport(f=f, residual_norm=r.residual_norm, solution_norm=r.solution_norm,
                       iterations=r.iterations, wall_time_seconds=r.wall_time_seconds,
                       mode=mode, residual_history=list(hist), split_seconds=r.split_seconds,
                       recombine_seconds=r.recombine_seconds, branch1_seconds=r.branch1_seconds,
                       branch2_seconds=r.branch2_seconds)


# ----------------------------------------------------------------- centro
def verify_symmetry(a: Matrix, tol: float) -> SymmetryReport:
    """centro.cpp:46-66"""
    r = N.SymmetryReportC()
    _check(_lib().ss_verify_symmetry(a.h, C.c_double(tol), C.byref(r)))
    return SymmetryReport._from(r)


def split_rhs(p, ctx: Optional[Context] = None):
    """centro.cpp:89-99"""
    ctx = ctx or default_context()
    p = _f64(p)
    p1 = np.empty(len(p) // 2)
    p2 = np.empty(len(p) // 2)
    _check(_lib().ss_split_rhs(ctx.h, _dp(p), len(p), _dp(p1), _dp(p2)))
    return p1, p2


def split_system(sys: CentroSystem) -> SplitSystem:
    """centro.cpp:144-156 (sparse fold :109-130), bit-exact on the device."""
    a = sys.a
    p = _f64(sys.p)
    m = len(p)
    a1, a2 = N.vp(), N.vp()
    p1 = np.empty(m // 2)
    p2 = np.empty(m // 2)
    fills = np.empty(3)
    rep = N.SymmetryReportC()
    rc = _lib().ss_split_system(a.h, _dp(p), m, C.c_double(sys.symmetry_tol), C.byref(a1),
                                C.byref(a2), _dp(p1), _dp(p2), _dp(fills), C.byref(rep))
    _check(rc, SymmetryReport._from(rep))
    return SplitSystem(Matrix(a1, a.ctx), p1, Matrix(a2, a.ctx), p2, *fills)


def decompose_solution(f, ctx: Optional[Context] = None) -> SolutionPair:
    ctx = ctx or default_context()
    f = _f64(f)
    f1 = np.empty(len(f) // 2)
    f2 = np.empty(len(f) // 2)
    _check(_lib().ss_decompose_solution(ctx.h, _dp(f), len(f), _dp(f1), _dp(f2)))
    return SolutionPair(f1, f2)


def recombine_solution(pair, f2=None, ctx: Optional[Context] = None):
    """centro.cpp:170-185; accepts a SolutionPair or (f1, f2)."""
    ctx = ctx or default_context()
    f1 = pair.f1 if isinstance(pair, SolutionPair) else pair
    f2 = pair.f2 if isinstance(pair, SolutionPair) else f2
    f1, f2 = _f64(f1), _f64(f2)
    if len(f1) != len(f2):
        raise Error("recombine_solution: component lengths differ")
    f = np.empty(2 * len(f1))
    _check(_lib().ss_recombine_solution(ctx.h, _dp(f1), _dp(f2), len(f1), _dp(f)))
    return f


# ----------------------------------------------------------------- solvers
def sart_solve(a: Matrix, p, opts: Optional[SolveOptions] = None) -> SolveReport:
    """solvers.cpp:148-199"""
    opts = opts or SolveOptions()
    p = _f64(p)
    rows, cols = a.shape
    f = np.empty(cols)
    hist = np.empty(int(opts.max_iters) + 1)
    r = N.SolveReportC()
    o = opts._c()
    _check(_lib().ss_sart_solve(a.h, _dp(p), len(p), C.byref(o), _dp(f), cols, C.byref(r),
                                _dp(hist)))
    return _report(f, r, "direct", hist[:r.history_len])


def cgls_solve(a: Matrix, p, opts: Optional[SolveOptions] = None) -> SolveReport:
    """solvers.cpp:99-146 on the device."""
    opts = opts or SolveOptions(method="cgls")
    p = _f64(p)
    rows, cols = a.shape
    f = np.empty(cols)
    hist = np.empty(int(opts.max_iters) + 1)
    r = N.SolveReportC()
    o = opts._c()
    _check(_lib().ss_cgls_solve(a.h, _dp(p), len(p), C.byref(o), _dp(f), cols, C.byref(r),
                                _dp(hist)))
    rep = _report(f, r, "direct", hist[:r.history_len])
    rep.method = "cgls"
    return rep


def pseudo_solve_dense(a: Matrix, p, dense_cap: int = 50_000_000):
    """solvers.cpp:81-97: minimum-norm solution (device SVD pseudo-inverse at the
    reference threshold max(m,n)*eps); refuses rows*cols > dense_cap."""
    p = _f64(p)
    f = np.empty(a.shape[1])
    _check(_lib().ss_pseudo_solve_dense(a.h, _dp(p), len(p), int(dense_cap), _dp(f), len(f)))
    return f


def solve_direct(sys: CentroSystem, opts: Optional[SolveOptions] = None) -> SolveReport:
    """solvers.cpp:201-205 (method = sart, cgls or dense)"""
    opts = opts or SolveOptions()
    if opts.method == "cgls":
        return cgls_solve(sys.a, sys.p, opts)
    if opts.method in ("dense", "dense_minnorm"):
        p = _f64(sys.p)
        f = np.empty(sys.a.shape[1])
        r = N.SolveReportC()
        o = opts._c()
        _check(_lib().ss_solve_direct(sys.a.h, _dp(p), len(p), C.byref(o), _dp(f), len(f),
                                      C.byref(r)))
        rep = _report(f, r, "direct")
        rep.method = "dense"
        return rep
    return sart_solve(sys.a, sys.p, opts)


def solve_split(sys: CentroSystem, opts: Optional[SolveOptions] = None) -> SolveReport:
    """solvers.cpp:207-269 (method = sart): fold, both branches, recombine."""
    opts = opts or SolveOptions()
    p = _f64(sys.p)
    rows, cols = sys.a.shape
    f = np.empty(cols)
    r = N.SolveReportC()
    o = opts._c()
    rc = _lib().ss_solve_split(sys.a.h, _dp(p), len(p), C.c_double(sys.symmetry_tol),
                               C.byref(o), _dp(f), cols, C.byref(r))
    if rc == N.SS_ERR_SYMMETRY:
        msg = _lib().ss_last_error().decode()
        raise SymmetryError(msg, verify_symmetry(sys.a, sys.symmetry_tol))
    _check(rc)
    rep = _report(f, r, "split")
    rep.method = "dense" if opts.method == "dense_minnorm" else opts.method
    return rep


# ----------------------------------------------------------------- geometry
def scan_config(k=24, gamma=None, gamma_deg=30.0, h_e=1.0, h_m=0.25, l_m=0.43, n_p=1024,
                a_e=7e-4, obj_size=0.1, grid_nx=32, grid_ny=32) -> N.ScanConfig:
    g = degrees_to_radians(gamma_deg) if gamma is None else gamma
    return N.ScanConfig(k, g, h_e, h_m, l_m, n_p, a_e, obj_size, grid_nx, grid_ny)


def parse_scan_config(text: str) -> N.ScanConfig:
    out = N.ScanConfig()
    _check(_lib().ss_parse_scan_config(text.encode(), C.byref(out)))
    return out


def make_grid(cfg: N.ScanConfig) -> N.GridSpec:
    g = N.GridSpec()
    _check(_lib().ss_make_grid(C.byref(cfg), C.byref(g)))
    return g


def snake_index(c, r, grid: N.GridSpec) -> int:
    j = C.c_int()
    _check(_lib().ss_snake_index(c, r, C.byref(grid), C.byref(j)))
    return j.value


def snake_inverse(j, grid: N.GridSpec):
    c, r = C.c_int(), C.c_int()
    _check(_lib().ss_snake_inverse(j, C.byref(grid), C.byref(c), C.byref(r)))
    return c.value, r.value


def emitter_angles(cfg: N.ScanConfig):
    """geometry.cpp:107-117 (host, libm): k angles, most negative first."""
    out = np.empty(cfg.k)
    _check(_lib().ss_emitter_angles(C.byref(cfg), _dp(out)))
    return out


def emitter_positions(cfg: N.ScanConfig, center_x: float = 0.0):
    """geometry.cpp:119-130: k sources as rows (x, y), mirrored bitwise about center_x."""
    out = np.empty((cfg.k, 2))
    _check(_lib().ss_emitter_positions(C.byref(cfg), C.c_double(center_x), _dp(out)))
    return out


def ray_weights(ray4, grid: N.GridSpec, ctx: Optional[Context] = None):
    """geometry.cpp:175-225 for one ray (source x, y, detector x, y) on the
    device tracer: (1-based snake columns, lengths) in path order."""
    ctx = ctx or default_context()
    r = _f64(ray4).reshape(4)
    n = N.i64()
    _check(_lib().ss_ray_weights(ctx.h, _dp(r), C.byref(grid), 0, None, None, C.byref(n)))
    cols = np.empty(n.value, np.int32)
    lens = np.empty(n.value)
    _check(_lib().ss_ray_weights(ctx.h, _dp(r), C.byref(grid), n.value, _ip(cols), _dp(lens),
                                 C.byref(n)))
    return cols, lens


def enumerate_rays(cfg: N.ScanConfig, grid: Optional[N.GridSpec] = None):
    """geometry.cpp:132-173 -> (rays[M,4] as (sx,sy,dx,dy), samples, pitch);
    with `grid` the reference's enumerate_rays(geometry, grid)."""
    cnt, samples, pitch = N.i64(), C.c_int(), C.c_double()

    def call(out):
        if grid is None:
            return _lib().ss_enumerate_rays(C.byref(cfg), out, C.byref(cnt), C.byref(samples),
                                            C.byref(pitch))
        return _lib().ss_enumerate_rays_grid(C.byref(cfg), C.byref(grid), out, C.byref(cnt),
                                             C.byref(samples), C.byref(pitch))
    _check(call(None))
    rays = np.empty((cnt.value, 4))
    _check(call(_dp(rays)))
    return rays, samples.value, pitch.value


def build_system(geometry: N.ScanConfig, grid: Optional[N.GridSpec] = None,
                 parallelism: int = 0, ctx: Optional[Context] = None) -> CentroSystem:
    """geometry.cpp:227-275 on the GPU: A with p = 0 and symmetry_tol = 0.

    build_system(geometry, grid, parallelism=0) is the reference signature
    (geometry.hpp:118, bindings.cpp:246): `geometry`'s k / gamma / h_e / h_m /
    l_m / n_p / obj_size with the caller's grid. build_system(cfg) uses
    make_grid(cfg)."""
    ctx = ctx or default_context()
    if isinstance(grid, int) and not isinstance(grid, bool):  # build_system(cfg, parallelism)
        grid, parallelism = None, grid
    h = N.vp()
    if grid is None:
        _check(_lib().ss_build_system(ctx.h, C.byref(geometry), parallelism, C.byref(h)))
    else:
        _check(_lib().ss_build_system_grid(ctx.h, C.byref(geometry), C.byref(grid), parallelism,
                                           C.byref(h)))
    a = Matrix(h, ctx)
    return CentroSystem(a, np.zeros(a.shape[0]), 0.0)


# ----------------------------------------------------------------- file formats
def read_matrix_market(path: str, ctx: Optional[Context] = None) -> Matrix:
    """io.cpp:83-187: coordinate real general -> device CSR; IoError names path:line."""
    ctx = ctx or default_context()
    h = N.vp()
    _check(_lib().ss_read_matrix_market(ctx.h, os.fsencode(path), C.byref(h)))
    return Matrix(h, ctx)


def write_matrix_market(a: Matrix, path: str) -> None:
    """io.cpp:189-210: stored non-zeros, 1-based, %.17g."""
    _check(_lib().ss_write_matrix_market(a.h, os.fsencode(path)))


def read_vector_csv(path: str):
    """io.cpp:212-230: one value per line, blank lines and '#' comments skipped."""
    n = C.c_int64(0)
    _check(_lib().ss_read_vector_csv(os.fsencode(path), None, 0, C.byref(n)))
    out = np.empty(n.value)
    _check(_lib().ss_read_vector_csv(os.fsencode(path), _dp(out), n.value, C.byref(n)))
    return out


def write_vector_csv(v, path: str) -> None:
    """io.cpp:232-238."""
    v = _f64(v)
    _check(_lib().ss_write_vector_csv(os.fsencode(path), _dp(v), len(v)))


# ----------------------------------------------------------------- phantom
def shepp_logan_ellipses():
    """phantom.cpp:18-32: the 10-ellipse Shepp-Logan table, rows
    (x0, y0, a, b, angle [rad], density)."""
    t = [(0.0, 0.0, 0.69, 0.92, 0.0, 2.0), (0.0, -0.0184, 0.6624, 0.874, 0.0, -0.98),
         (0.22, 0.0, 0.11, 0.31, -18.0, -0.02), (-0.22, 0.0, 0.16, 0.41, 18.0, -0.02),
         (0.0, 0.35, 0.21, 0.25, 0.0, 0.01), (0.0, 0.1, 0.046, 0.046, 0.0, 0.01),
         (0.0, -0.1, 0.046, 0.046, 0.0, 0.01), (-0.08, -0.605, 0.046, 0.023, 0.0, 0.01),
         (0.0, -0.606, 0.023, 0.023, 0.0, 0.01), (0.06, -0.605, 0.023, 0.046, 0.0, 0.01)]
    return np.array([(x, y, a, b, degrees_to_radians(d), rho) for x, y, a, b, d, rho in t])


def random_ellipses(seed: int, count: int = 8):
    out = np.empty((count, 6))
    _check(_lib().ss_random_ellipses(seed, count, _dp(out)))
    return out


def rasterize(ellipses, grid: N.GridSpec, ctx: Optional[Context] = None):
    """phantom.cpp:34-58 on the GPU; ellipses rows (x0, y0, a, b, angle, density)."""
    ctx = ctx or default_context()
    e = _f64(np.asarray(ellipses, dtype=np.float64).reshape(-1, 6))
    out = np.empty(grid.n_x * grid.n_y)
    _check(_lib().ss_rasterize(ctx.h, _dp(e), len(e), C.byref(grid), _dp(out)))
    return out


def forward_project(a: Matrix, f, noise_sigma: float = 0.0, seed: int = 0):
    """phantom.cpp:108-149: folded row sums on the GPU, seeded noise on the host."""
    f = _f64(f)
    rows, cols = a.shape
    if f.shape != (cols,):
        raise Error("forward_project: image length does not match columns")
    p = np.empty(rows)
    _check(_lib().ss_forward_project(a.h, _dp(f), _dp(p)))
    if noise_sigma != 0.0 or noise_sigma < 0:
        _check(_lib().ss_add_noise(_dp(p), rows, C.c_double(noise_sigma), C.c_uint64(seed)))
    return p


# ----------------------------------------------------------------- plans
class SartPlan:
    """Device-resident SART loop over one system or the folded pair (ss_plan_t).

    Normalisers are computed at construction (the reference computes them
    before its timer). `run()` = one full solve from x0 = 0.
    """

    def __init__(self, a1: Matrix, a2: Optional[Matrix] = None,
                 opts: Optional[SolveOptions] = None, nrhs: int = 1):
        self.opts = opts or SolveOptions()
        self.ctx = a1.ctx
        self.nsys = 2 if a2 is not None else 1
        self.nrhs = nrhs
        self.a = (a1, a2)  # keep the matrices alive
        h = N.vp()
        o = self.opts._c()
        _check(_lib().ss_plan_create(self.ctx.h, a1.h, a2.h if a2 is not None else None,
                                     C.byref(o), nrhs, C.byref(h)))
        self.h = h
        self.rows, self.cols = a1.shape

    def __del__(self):
        try:
            if getattr(self, "h", None) and N._lib is not None:
                N._lib.ss_plan_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def set_rhs(self, which, p):
        p = _f64(p)
        if p.size != self.rows * self.nrhs:
            raise Error("plan: rhs size mismatch")
        _check(_lib().ss_plan_set_rhs(self.h, which, _dp(p)))

    def set_rhs_device(self, which, ptr: int):
        _check(_lib().ss_plan_set_rhs_device(self.h, which, N.vp(ptr)))

    def launch(self):
        _check(_lib().ss_plan_launch(self.h))

    def finish(self) -> N.SolveReportC:
        r = N.SolveReportC()
        _check(_lib().ss_plan_finish(self.h, C.byref(r)))
        return r

    def run(self) -> N.SolveReportC:
        self.launch()
        return self.finish()

    def solution(self, which=0):
        f = np.empty(self.cols * self.nrhs)
        _check(_lib().ss_plan_get_solution(self.h, which, _dp(f)))
        return f if self.nrhs == 1 else f.reshape(self.nrhs, self.cols)

    def history(self, which=0, slice_=0):
        h = np.empty(int(self.opts.max_iters) + 1)
        n = C.c_int()
        _check(_lib().ss_plan_get_history(self.h, which, slice_, _dp(h), C.byref(n)))
        return h[:n.value].copy()

    def recombine(self):
        f = np.empty(2 * self.cols * self.nrhs)
        _check(_lib().ss_plan_recombine(self.h, _dp(f)))
        return f if self.nrhs == 1 else f.reshape(self.nrhs, 2 * self.cols)

    def solution_device_ptr(self, which=0) -> int:
        return _lib().ss_plan_solution_device(self.h, which) or 0

    def stats(self):
        mb, vb, k = N.i64(), N.i64(), C.c_int()
        _check(_lib().ss_plan_stats(self.h, C.byref(mb), C.byref(vb), C.byref(k)))
        return mb.value, vb.value, k.value

    def kernel_bytes(self):
        f, b = N.i64(), N.i64()
        _check(_lib().ss_plan_kernel_bytes(self.h, C.byref(f), C.byref(b)))
        return f.value, b.value

    def describe(self) -> dict:
        """Kernel layout, VS/UF, grid and the kernel names ncu reports."""
        import json
        buf = C.create_string_buffer(2048)
        _check(_lib().ss_plan_describe(self.h, buf, len(buf)))
        return json.loads(buf.value.decode())

    def profile(self, iters):
        a, b = C.c_float(), C.c_float()
        _check(_lib().ss_plan_profile(self.h, iters, C.byref(a), C.byref(b)))
        return a.value, b.value

    def time_kernel(self, fwd: bool, reps: int = 50) -> float:
        """In-loop milliseconds per launch of K1 (fwd) or K2: `reps` launches
        back to back, CUDA events around the batch. Resets the plan."""
        ms = C.c_float()
        _check(_lib().ss_plan_time_kernel(self.h, 1 if fwd else 0, reps, C.byref(ms)))
        return ms.value


# ----------------------------------------------------------------- multi-GPU helpers
def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib().ss_nccl_unique_id(C.cast(buf, N.vp)))
    return buf.raw


def attach_nccl(ctx: Context, unique_id: bytes, nranks: int, rank: int):
    buf = C.create_string_buffer(bytes(unique_id), 128)
    _check(_lib().ss_ctx_attach_nccl(ctx.h, C.cast(buf, N.vp), nranks, rank))


def partition_rows(rowptr, parts: int):
    """Balanced row blocks of a CSR row pointer by nnz (host logic, no GPU)."""
    rowptr = _i32(rowptr)
    bounds = np.empty(parts + 1, np.int64)
    _check(_lib().ss_partition_rows(_ip(rowptr), len(rowptr) - 1, parts,
                                    bounds.ctypes.data_as(N.i64p)))
    return bounds


XCHG_NCCL, XCHG_PEER = 0, 1  # SS_XCHG_* of symsplit_b200.h


def exchange_owned_columns(cols: int, parts: int, rank: int):
    """Columns [begin, end) rank `rank` reduces and pushes in the peer
    exchange (host logic, no GPU)."""
    b, e = N.i64(), N.i64()
    _check(_lib().ss_exchange_owned_columns(cols, parts, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


class ShardedSartPlan(SartPlan):
    """Rows [row_begin, row_end) of one folded system on this rank. exchange
    "nccl": the back-projection is all-reduced over the context's NCCL
    communicator; "peer": the fused peer-memory exchange (K2 stores each
    column's partial into its owner's receive row over NVLink; each owner sums
    the ranks' partials of its own columns in rank order, applies the update
    and pushes its x range into every replica; no NCCL on the data path)."""

    def __init__(self, ctx: Context, a: Matrix, row_begin: int, row_end: int,
                 opts: Optional[SolveOptions] = None, exchange: str = "nccl"):
        self.opts = opts or SolveOptions()
        self.ctx = ctx
        self.nsys = 1
        self.nrhs = 1
        self.a = (a, None)
        h = N.vp()
        o = self.opts._c()
        x = {"nccl": XCHG_NCCL, "peer": XCHG_PEER}[exchange]
        _check(_lib().ss_plan_create_sharded_x(ctx.h, a.h, row_begin, row_end, C.byref(o), x,
                                               C.byref(h)))
        self.h = h
        self.rows = row_end - row_begin
        self.cols = a.shape[1]


class ShardedPairPlan(SartPlan):
    """Rows [row_begin, row_end) of BOTH folded systems on this rank (the
    row-sharded pair: every rank streams 1/N of the paired mirror-coded
    streams); {u1, u2} back-projection pairs travel through the fused
    peer-memory exchange. solution(0 / 1) and recombine() give the full
    iterates (every rank holds a replica)."""

    def __init__(self, ctx: Context, a1: Matrix, a2: Matrix, row_begin: int, row_end: int,
                 opts: Optional[SolveOptions] = None):
        self.opts = opts or SolveOptions()
        self.ctx = ctx
        self.nsys = 2
        self.nrhs = 1
        self.a = (a1, a2)
        h = N.vp()
        o = self.opts._c()
        _check(_lib().ss_plan_create_sharded_pair(ctx.h, a1.h, a2.h, row_begin, row_end,
                                                  C.byref(o), C.byref(h)))
        self.h = h
        self.rows = row_end - row_begin
        self.cols = a1.shape[1]


class _GroupMember(SartPlan):
    """One emulated rank of a ShardGroup (owns its ss_plan_t)."""

    def __init__(self, ctx, a, h, rows, opts, a2=None):
        self.opts = opts
        self.ctx = ctx
        self.nsys = 2 if a2 is not None else 1
        self.nrhs = 1
        self.a = (a, a2)
        self.h = h
        self.rows = rows
        self.cols = a.shape[1]


class ShardGroup:
    """One-device emulation of `parts` peer-exchange ranks of a row-sharded
    system (ss_plan_create_sharded_group / ss_plan_group_run): the same
    kernels, chunk ownership, arrival counters and rank-order reductions as
    the multi-GPU path, with every rank's launches issued in rank order on one
    stream. Used by the parity tests and the single-GPU exchange measurement."""

    def __init__(self, a: Matrix, parts: int, opts: Optional[SolveOptions] = None,
                 bounds=None):
        self.opts = opts or SolveOptions()
        self.parts = parts
        if bounds is None:
            bounds = partition_rows(a.to_csr()[0], parts)
        self.bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        hs = (N.vp * parts)()
        o = self.opts._c()
        _check(_lib().ss_plan_create_sharded_group(a.ctx.h, a.h, parts,
                                                   self.bounds.ctypes.data_as(N.i64p),
                                                   C.byref(o), hs))
        self.hs = hs
        self.ranks = [_GroupMember(a.ctx, a, N.vp(hs[g]),
                                   int(self.bounds[g + 1] - self.bounds[g]), self.opts)
                      for g in range(parts)]

    def set_rhs(self, p):
        p = _f64(p)
        for g, r in enumerate(self.ranks):
            r.set_rhs(0, p[self.bounds[g]:self.bounds[g + 1]])

    def run(self):
        _check(_lib().ss_plan_group_run(self.hs, self.parts))
        return [r.finish() for r in self.ranks]

    def solution(self, rank=0):
        return self.ranks[rank].solution(0)

    def history(self, rank=0):
        return self.ranks[rank].history(0)


class ShardPairGroup:
    """One-device emulation of `parts` ranks of the row-sharded PAIR
    (ss_plan_create_sharded_pair_group / ss_plan_group_run): both folded
    systems row-sharded over all ranks on the paired streams, {u1, u2}
    exchanged through the same arrival counters and rank-order reductions as
    on real ranks."""

    def __init__(self, a1: Matrix, a2: Matrix, parts: int,
                 opts: Optional[SolveOptions] = None, bounds=None):
        self.opts = opts or SolveOptions()
        self.parts = parts
        if bounds is None:
            bounds = partition_rows(a1.to_csr()[0], parts)
        self.bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        hs = (N.vp * parts)()
        o = self.opts._c()
        _check(_lib().ss_plan_create_sharded_pair_group(a1.ctx.h, a1.h, a2.h, parts,
                                                        self.bounds.ctypes.data_as(N.i64p),
                                                        C.byref(o), hs))
        self.hs = hs
        self.ranks = [_GroupMember(a1.ctx, a1, N.vp(hs[g]),
                                   int(self.bounds[g + 1] - self.bounds[g]), self.opts, a2)
                      for g in range(parts)]

    def set_rhs(self, p1, p2):
        p1, p2 = _f64(p1), _f64(p2)
        for g, r in enumerate(self.ranks):
            r.set_rhs(0, p1[self.bounds[g]:self.bounds[g + 1]])
            r.set_rhs(1, p2[self.bounds[g]:self.bounds[g + 1]])

    def run(self):
        _check(_lib().ss_plan_group_run(self.hs, self.parts))
        return [r.finish() for r in self.ranks]

    def solution(self, which, rank=0):
        return self.ranks[rank].solution(which)

    def history(self, which, rank=0):
        return self.ranks[rank].history(which)

    def recombine(self, rank=0):
        return self.ranks[rank].recombine()
