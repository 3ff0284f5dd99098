"""TEST INFRASTRUCTURE ONLY — ctypes view of the C++ oracle (oracle/*.cpp).

Used by tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs as the
checker / CPU baseline; never by the product package. See oracle/oracle.hpp
for what is restated and where in the reference it comes from.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_symsplit.so")

_i64 = C.c_int64
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p


class OracleError(RuntimeError):
    pass


class OracleSymmetryError(OracleError):
    def __init__(self, msg, report):
        super().__init__(msg)
        self.report = report


class ScanConfigC(C.Structure):
    _fields_ = [("k", C.c_int), ("gamma", C.c_double), ("h_e", C.c_double),
                ("h_m", C.c_double), ("l_m", C.c_double), ("n_p", C.c_int),
                ("a_e", C.c_double), ("obj_size", C.c_double),
                ("grid_nx", C.c_int), ("grid_ny", C.c_int)]


class GridC(C.Structure):
    _fields_ = [("n_x", C.c_int), ("n_y", C.c_int), ("voxel_size", C.c_double),
                ("center_x", C.c_double), ("y_bottom", C.c_double)]


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.or_last_error.restype = C.c_char_p
        for name in ("or_mat_dense", "or_mat_csc", "or_mat_triplets", "or_reconstruct",
                     "or_symmetrize", "or_build_system", "or_build_traced_csr",
                     "or_full_csr_from_traced", "or_csr_from_mat", "or_mat_from_csr",
                     "or_csr_make"):
            getattr(_lib, name).restype = _vp
        _lib.or_mat_nonzeros.restype = _i64
        _lib.or_mat_fill_ratio.restype = C.c_double
        _lib.or_norm.restype = C.c_double
        _lib.or_norm.argtypes = [_dp, _i64]
        _lib.or_mat_dense.argtypes = [_i64, _i64, _dp]
        _lib.or_mat_csc.argtypes = [_i64, _i64, _i64, _ip, _ip, _dp]
        _lib.or_mat_triplets.argtypes = [_i64, _i64, _i64, _ip, _ip, _dp]
        _lib.or_csr_make.argtypes = [_i64, _i64, _i64, _ip, _ip, _dp]
        for name in ("or_mat_free", "or_csr_free"):
            getattr(_lib, name).argtypes = [_vp]
        _lib.or_rng_uniform.argtypes = [C.c_uint64, _i64, C.c_double, C.c_double, _dp]
        _lib.or_random_ellipses.argtypes = [C.c_uint64, C.c_int, _dp]
        _lib.or_add_noise.argtypes = [_dp, _i64, C.c_double, C.c_uint64]
    return _lib


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _check(rc):
    if rc == 0:
        return
    msg = lib().or_last_error().decode()
    raise OracleError(msg)


def f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def i32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


# ----------------------------------------------------------------- matrices
class Matrix:
    """Owning handle to an oracle Matrix (dense col-major or CSC)."""

    def __init__(self, handle):
        if not handle:
            raise OracleError(lib().or_last_error().decode())
        self.h = _vp(handle)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_mat_free(self.h)
            self.h = None

    @classmethod
    def dense(cls, d):
        d = np.asarray(d, dtype=np.float64)
        cm = f64(d.T.reshape(-1))  # column-major
        return cls(lib().or_mat_dense(d.shape[0], d.shape[1], _d(cm)))

    @classmethod
    def csc(cls, rows, cols, outer, inner, val):
        outer, inner, val = i32(outer), i32(inner), f64(val)
        return cls(lib().or_mat_csc(rows, cols, len(val), _i(outer), _i(inner), _d(val)))

    @classmethod
    def triplets(cls, rows, cols, r, c, v):
        r, c, v = i32(r), i32(c), f64(v)
        return cls(lib().or_mat_triplets(rows, cols, len(v), _i(r), _i(c), _d(v)))

    @classmethod
    def sparse_from_dense(cls, d, keep_zeros=False):
        d = np.asarray(d, dtype=np.float64)
        rr, cc, vv = [], [], []
        for j in range(d.shape[1]):
            for i in range(d.shape[0]):
                if keep_zeros or d[i, j] != 0.0:
                    rr.append(i); cc.append(j); vv.append(d[i, j])
        return cls.triplets(d.shape[0], d.shape[1], rr, cc, vv)

    def info(self):
        r, c, s, sp = _i64(), _i64(), _i64(), C.c_int()
        lib().or_mat_info(self.h, C.byref(r), C.byref(c), C.byref(s), C.byref(sp))
        return r.value, c.value, s.value, bool(sp.value)

    @property
    def shape(self):
        r, c, _, _ = self.info()
        return r, c

    @property
    def is_sparse(self):
        return self.info()[3]

    def nonzeros(self):
        return lib().or_mat_nonzeros(self.h)

    def fill_ratio(self):
        return lib().or_mat_fill_ratio(self.h)

    def get_csc(self):
        rows, cols, nnz, sp = self.info()
        assert sp
        outer = np.empty(cols + 1, np.int32)
        inner = np.empty(nnz, np.int32)
        val = np.empty(nnz, np.float64)
        lib().or_mat_get_csc(self.h, _i(outer), _i(inner), _d(val))
        return outer, inner, val

    def to_dense(self):
        rows, cols, _, _ = self.info()
        cm = np.empty(rows * cols, np.float64)
        lib().or_mat_get_dense(self.h, _d(cm))
        return cm.reshape(cols, rows).T.copy()

    def apply(self, x):
        x = f64(x)
        y = np.empty(self.shape[0])
        _check(lib().or_mat_apply(self.h, _d(x), _d(y)))
        return y

    def apply_transpose(self, y):
        y = f64(y)
        x = np.empty(self.shape[1])
        _check(lib().or_mat_apply_t(self.h, _d(y), _d(x)))
        return x

    def to_csr(self):
        return Csr(lib().or_csr_from_mat(self.h))


class Csr:
    def __init__(self, handle):
        if not handle:
            raise OracleError(lib().or_last_error().decode())
        self.h = _vp(handle)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_csr_free(self.h)
            self.h = None

    @classmethod
    def make(cls, rows, cols, ptr, idx, val):
        ptr, idx, val = i32(ptr), i32(idx), f64(val)
        return cls(lib().or_csr_make(rows, cols, len(val), _i(ptr), _i(idx), _d(val)))

    def info(self):
        r, c, n = _i64(), _i64(), _i64()
        lib().or_csr_info(self.h, C.byref(r), C.byref(c), C.byref(n))
        return r.value, c.value, n.value

    def arrays(self):
        rows, cols, nnz = self.info()
        ptr = np.empty(rows + 1, np.int32)
        idx = np.empty(nnz, np.int32)
        val = np.empty(nnz, np.float64)
        lib().or_csr_get(self.h, _i(ptr), _i(idx), _d(val))
        return ptr, idx, val

    def to_matrix(self):
        return Matrix(lib().or_mat_from_csr(self.h))


def norm(v):
    v = f64(v)
    return lib().or_norm(_d(v), len(v))


# ----------------------------------------------------------------- centro
@dataclass
class SymmetryReport:
    holds: bool
    max_violation: float
    worst_row: int
    worst_col: int
    status: int


def verify_symmetry(a: Matrix, tol: float) -> SymmetryReport:
    h, mv, wr, wc, st = C.c_int(), C.c_double(), _i64(), _i64(), C.c_int()
    _check(lib().or_verify_symmetry(a.h, C.c_double(tol), C.byref(h), C.byref(mv),
                                    C.byref(wr), C.byref(wc), C.byref(st)))
    return SymmetryReport(bool(h.value), mv.value, wr.value, wc.value, st.value)


@dataclass
class SplitSystem:
    a1: Matrix
    p1: np.ndarray
    a2: Matrix
    p2: np.ndarray
    parent_fill: float
    fill1: float
    fill2: float


def split_system(a: Matrix, p, tol: float) -> SplitSystem:
    p = f64(p)
    m = a.shape[0]
    a1, a2 = _vp(), _vp()
    p1 = np.empty(max(m // 2, 0))
    p2 = np.empty(max(m // 2, 0))
    fills = np.empty(3)
    mv, wr, wc, st = C.c_double(), _i64(), _i64(), C.c_int()
    rc = lib().or_split_system(a.h, _d(p), _i64(len(p)), C.c_double(tol), C.byref(a1), C.byref(a2),
                               _d(p1), _d(p2), _d(fills), C.byref(mv), C.byref(wr),
                               C.byref(wc), C.byref(st))
    if rc == 2:
        raise OracleSymmetryError(lib().or_last_error().decode(),
                                  SymmetryReport(False, mv.value, wr.value, wc.value, st.value))
    _check(rc)
    return SplitSystem(Matrix(a1.value), p1, Matrix(a2.value), p2, *fills)


def split_matrix(a: Matrix):
    a1, a2 = _vp(), _vp()
    _check(lib().or_split_matrix(a.h, C.byref(a1), C.byref(a2)))
    return Matrix(a1.value), Matrix(a2.value)


def split_rhs(p):
    p = f64(p)
    p1 = np.empty(len(p) // 2)
    p2 = np.empty(len(p) // 2)
    _check(lib().or_split_rhs(_d(p), _i64(len(p)), _d(p1), _d(p2)))
    return p1, p2


def recombine_solution(f1, f2):
    f1, f2 = f64(f1), f64(f2)
    f = np.empty(2 * len(f1))
    _check(lib().or_recombine(_d(f1), _i64(len(f1)), _d(f2), _i64(len(f2)), _d(f)))
    return f


def decompose_solution(f):
    f = f64(f)
    f1 = np.empty(len(f) // 2)
    f2 = np.empty(len(f) // 2)
    _check(lib().or_decompose(_d(f), _i64(len(f)), _d(f1), _d(f2)))
    return f1, f2


def reconstruct_matrix(a1: Matrix, a2: Matrix) -> Matrix:
    return Matrix(lib().or_reconstruct(a1.h, a2.h))


def symmetrize(a: Matrix) -> Matrix:
    return Matrix(lib().or_symmetrize(a.h))


def fold_rows_csr(a: Csr):
    a1, a2 = _vp(), _vp()
    _check(lib().or_fold_rows_csr(a.h, C.byref(a1), C.byref(a2)))
    return Csr(a1.value), Csr(a2.value)


# ----------------------------------------------------------------- solvers
@dataclass
class SolveReport:
    f: np.ndarray
    iterations: int
    residual_norm: float
    solution_norm: float
    wall_time_seconds: float
    residual_history: np.ndarray
    split_seconds: float = 0.0
    recombine_seconds: float = 0.0
    branch1_seconds: float = 0.0
    branch2_seconds: float = 0.0


def sart_solve(a: Matrix, p, max_iters=200, tol=1e-10, relaxation=1.0) -> SolveReport:
    p = f64(p)
    f = np.empty(a.shape[1])
    hist = np.empty(max_iters + 1)
    it, rn, sn, wall, hl = C.c_int(), C.c_double(), C.c_double(), C.c_double(), C.c_int()
    _check(lib().or_sart_solve(a.h, _d(p), _i64(len(p)), max_iters, C.c_double(tol),
                               C.c_double(relaxation), _d(f), C.byref(it), C.byref(rn),
                               C.byref(sn), C.byref(wall), _d(hist), C.byref(hl)))
    return SolveReport(f, it.value, rn.value, sn.value, wall.value, hist[:hl.value].copy())


def cgls_solve(a: Matrix, p, max_iters=200, tol=1e-10) -> SolveReport:
    p = f64(p)
    f = np.empty(a.shape[1])
    hist = np.empty(max_iters + 1)
    it, rn, sn, hl = C.c_int(), C.c_double(), C.c_double(), C.c_int()
    _check(lib().or_cgls_solve(a.h, _d(p), _i64(len(p)), max_iters, C.c_double(tol), _d(f),
                               C.byref(it), C.byref(rn), C.byref(sn), _d(hist), C.byref(hl)))
    return SolveReport(f, it.value, rn.value, sn.value, 0.0, hist[:hl.value].copy())


def solve_split_method(a: Matrix, p, method="cgls", symmetry_tol=1e-12, max_iters=200,
                       tol=1e-10, relaxation=1.0):
    p = f64(p)
    f = np.empty(a.shape[1])
    it, rn = C.c_int(), C.c_double()
    _check(lib().or_solve_split_method(a.h, _d(p), _i64(len(p)), C.c_double(symmetry_tol),
                                       1 if method == "cgls" else 0, max_iters, C.c_double(tol),
                                       C.c_double(relaxation), _d(f), C.byref(it), C.byref(rn)))
    return f, it.value, rn.value


def solve_split(a: Matrix, p, symmetry_tol=1e-12, max_iters=200, tol=1e-10, relaxation=1.0,
                parallelism=0) -> SolveReport:
    p = f64(p)
    f = np.empty(a.shape[1])
    t4 = np.empty(4)
    it, rn, sn, wall = C.c_int(), C.c_double(), C.c_double(), C.c_double()
    _check(lib().or_solve_split(a.h, _d(p), _i64(len(p)), C.c_double(symmetry_tol), max_iters,
                                C.c_double(tol), C.c_double(relaxation), parallelism, _d(f),
                                C.byref(it), C.byref(rn), C.byref(sn), C.byref(wall), _d(t4)))
    return SolveReport(f, it.value, rn.value, sn.value, wall.value, np.empty(0), *t4)


def solve_split_prepared(a1: Matrix, a2: Matrix, p1, p2, max_iters, tol, relaxation,
                         parallel=True):
    p1, p2 = f64(p1), f64(p2)
    f = np.empty(2 * a1.shape[1])
    t4 = np.empty(4)
    it = C.c_int()
    _check(lib().or_solve_split_prepared(a1.h, a2.h, _d(p1), _d(p2), max_iters,
                                         C.c_double(tol), C.c_double(relaxation),
                                         1 if parallel else 0, _d(f), C.byref(it), _d(t4)))
    return f, it.value, t4


# ----------------------------------------------------------------- dense min-norm
def pinv_solve(a, b):
    """tests/support/oracles.hpp:101-113 restated with numpy's SVD: the reference's
    own oracle for pseudo_solve_dense (test_solvers.cpp:72-84 pins the
    implementation to it within 1e-10). Cutoff max(m,n)*eps*s_0."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m, n = a.shape
    if m == 0 or n == 0:
        return np.zeros(n)
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    cutoff = max(m, n) * np.finfo(np.float64).eps * (s[0] if s.size else 0.0)
    y = u.T @ b
    y = np.where(s > cutoff, y / np.where(s > cutoff, s, 1.0), 0.0)
    return vt.T @ y


def random_with_rank(m, n, rank, rng):
    """tests/support/oracles.hpp:70-85 (numpy Generator instead of the Rng):
    Q_u diag(sigma, sigma ~ U[0.5,1.5] on `rank` entries) Q_v^T."""
    qu, _ = np.linalg.qr(rng.uniform(-1, 1, (m, m)))
    qv, _ = np.linalg.qr(rng.uniform(-1, 1, (n, n)))
    k = min(m, n)
    s = np.zeros((m, n))
    r = min(rank, k)
    s[np.arange(r), np.arange(r)] = rng.uniform(0.5, 1.5, r)
    return qu @ s @ qv.T


# ----------------------------------------------------------------- geometry
def scan_config(k, gamma, h_e, h_m, l_m, n_p, obj_size, grid_nx, grid_ny, a_e=7e-4):
    return ScanConfigC(k, gamma, h_e, h_m, l_m, n_p, a_e, obj_size, grid_nx, grid_ny)


def parse_scan_config(text: str) -> ScanConfigC:
    out = ScanConfigC()
    _check(lib().or_parse_scan_config(text.encode(), C.byref(out)))
    return out


def make_grid(cfg: ScanConfigC) -> GridC:
    g = GridC()
    _check(lib().or_make_grid(C.byref(cfg), C.byref(g)))
    return g


def snake_index(c, r, grid: GridC) -> int:
    j = C.c_int()
    _check(lib().or_snake_index(c, r, C.byref(grid), C.byref(j)))
    return j.value


def snake_inverse(j, grid: GridC):
    c, r = C.c_int(), C.c_int()
    _check(lib().or_snake_inverse(j, C.byref(grid), C.byref(c), C.byref(r)))
    return c.value, r.value


def emitter_angles(cfg):
    out = np.empty(cfg.k)
    _check(lib().or_emitter_angles(C.byref(cfg), _d(out)))
    return out


def emitter_positions(cfg, center_x=0.0):
    out = np.empty((cfg.k, 2))
    _check(lib().or_emitter_positions(C.byref(cfg), C.c_double(center_x), _d(out)))
    return out


def enumerate_rays(cfg, grid):
    cnt, samples, pitch = _i64(), C.c_int(), C.c_double()
    _check(lib().or_enumerate_rays(C.byref(cfg), C.byref(grid), None, C.byref(cnt),
                                   C.byref(samples), C.byref(pitch)))
    out = np.empty((cnt.value, 4))
    _check(lib().or_enumerate_rays(C.byref(cfg), C.byref(grid), _d(out), C.byref(cnt),
                                   C.byref(samples), C.byref(pitch)))
    return out, samples.value, pitch.value


def ray_weights(ray4, grid):
    ray4 = f64(ray4)
    cap = grid.n_x + grid.n_y + 4
    js = np.empty(cap, np.int32)
    lens = np.empty(cap)
    cnt = _i64()
    _check(lib().or_ray_weights(_d(ray4), C.byref(grid), _i(js), _d(lens), _i64(cap), C.byref(cnt)))
    return js[:cnt.value].copy(), lens[:cnt.value].copy()


def build_system(cfg, parallelism=0) -> Matrix:
    return Matrix(lib().or_build_system(C.byref(cfg), parallelism))


def build_traced_csr(cfg, parallelism=0) -> Csr:
    return Csr(lib().or_build_traced_csr(C.byref(cfg), parallelism))


def full_csr_from_traced(t: Csr, m, n) -> Csr:
    return Csr(lib().or_full_csr_from_traced(t.h, _i64(m), _i64(n)))


# ----------------------------------------------------------------- phantom
def random_ellipses(seed, count=8):
    out = np.empty((count, 6))
    _check(lib().or_random_ellipses(seed, count, _d(out)))
    return out


def shepp_logan():
    out = np.empty((10, 6))
    _check(lib().or_shepp_logan(_d(out)))
    return out


def rasterize(ellipses, grid):
    e = f64(np.asarray(ellipses).reshape(-1, 6))
    out = np.empty(grid.n_x * grid.n_y)
    _check(lib().or_rasterize(_d(e), len(e), C.byref(grid), _d(out)))
    return out


def forward_project(a: Matrix, f):
    f = f64(f)
    p = np.empty(a.shape[0])
    _check(lib().or_forward_project(a.h, _d(f), _i64(len(f)), _d(p)))
    return p


def forward_project_csr(a: Csr, f):
    f = f64(f)
    p = np.empty(a.info()[0])
    _check(lib().or_forward_project_csr(a.h, _d(f), _d(p)))
    return p


def add_noise(p, sigma, seed):
    p = f64(p).copy()
    _check(lib().or_add_noise(_d(p), len(p), C.c_double(sigma), seed))
    return p


def rng_uniform(seed, n, lo=0.0, hi=1.0):
    out = np.empty(n)
    _check(lib().or_rng_uniform(seed, n, C.c_double(lo), C.c_double(hi), _d(out)))
    return out
