"""ctypes declarations of the C ABI in include/symsplit_b200.h.

The shared library is built in-tree (paper_1902_10559_b200/libsymsplit_b200.so,
see csrc/Makefile). There is no fallback: if it is missing, importing the
compute entry points raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSB_LIB") or os.path.join(HERE, "libsymsplit_b200.so")  # SSB_LIB: A/B builds

(SS_OK, SS_ERR_INVALID, SS_ERR_SYMMETRY, SS_ERR_DIVERGED, SS_ERR_CUDA, SS_ERR_NCCL, SS_ERR_OOM,
 SS_ERR_IO) = (0, 1, 2, 3, 4, 5, 6, 7)
SS_F64, SS_F32 = 0, 1

i64 = C.c_int64
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
dp = C.POINTER(C.c_double)
fp = C.POINTER(C.c_float)
vp = C.c_void_p


class ScanConfig(C.Structure):
    """ss_scan_config — reference ScanConfig/ScanGeometry (geometry.hpp:54-68, 137-141)."""
    _fields_ = [("k", C.c_int), ("gamma", C.c_double), ("h_e", C.c_double),
                ("h_m", C.c_double), ("l_m", C.c_double), ("n_p", C.c_int),
                ("a_e", C.c_double), ("obj_size", C.c_double),
                ("grid_nx", C.c_int), ("grid_ny", C.c_int)]


class GridSpec(C.Structure):
    """ss_grid_spec — reference GridSpec (geometry.hpp:22-37)."""
    _fields_ = [("n_x", C.c_int), ("n_y", C.c_int), ("voxel_size", C.c_double),
                ("center_x", C.c_double), ("y_bottom", C.c_double)]


class SolveOptionsC(C.Structure):
    _fields_ = [("max_iters", C.c_int), ("tol", C.c_double), ("relaxation", C.c_double),
                ("parallelism", C.c_int), ("dtype", C.c_int), ("method", C.c_int),
                ("dense_cap", C.c_int64)]


class SolveReportC(C.Structure):
    _fields_ = [("residual_norm", C.c_double), ("solution_norm", C.c_double),
                ("iterations", C.c_int), ("wall_time_seconds", C.c_double),
                ("split_seconds", C.c_double), ("recombine_seconds", C.c_double),
                ("branch1_seconds", C.c_double), ("branch2_seconds", C.c_double),
                ("history_len", C.c_int)]


class SymmetryReportC(C.Structure):
    _fields_ = [("holds", C.c_int), ("max_violation", C.c_double), ("worst_row", C.c_int64),
                ("worst_col", C.c_int64), ("status", C.c_int)]


# name -> (restype, argtypes); every symbol the header declares
SIGNATURES = {
    "ss_last_error": (C.c_char_p, []),
    "ss_version": (C.c_int, []),
    "ss_default_options": (None, [C.POINTER(SolveOptionsC)]),
    "ss_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "ss_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "ss_ctx_destroy": (C.c_int, [vp]),
    "ss_ctx_synchronize": (C.c_int, [vp]),
    "ss_ctx_stream": (vp, [vp]),
    "ss_ctx_launch_count": (i64, [vp]),
    "ss_matrix_from_csc": (C.c_int, [vp, i64, i64, i64, i32p, i32p, dp, C.POINTER(vp)]),
    "ss_matrix_from_triplets": (C.c_int, [vp, i64, i64, i64, i32p, i32p, dp, C.POINTER(vp)]),
    "ss_matrix_destroy": (C.c_int, [vp]),
    "ss_matrix_shape": (C.c_int, [vp, i64p, i64p, i64p]),
    "ss_matrix_nonzeros": (C.c_int, [vp, i64p]),
    "ss_matrix_fill_ratio": (C.c_int, [vp, dp]),
    "ss_matrix_download_csr": (C.c_int, [vp, i32p, i32p, dp]),
    "ss_matrix_download_csc": (C.c_int, [vp, i32p, i32p, dp]),
    "ss_matrix_apply": (C.c_int, [vp, dp, dp]),
    "ss_matrix_coeff": (C.c_int, [vp, C.c_int64, C.c_int64, dp]),
    "ss_matrix_release_cache": (C.c_int, [vp]),
    "ss_matrix_apply_transpose": (C.c_int, [vp, dp, dp]),
    "ss_parse_scan_config": (C.c_int, [C.c_char_p, C.POINTER(ScanConfig)]),
    "ss_make_grid": (C.c_int, [C.POINTER(ScanConfig), C.POINTER(GridSpec)]),
    "ss_snake_index": (C.c_int, [C.c_int, C.c_int, C.POINTER(GridSpec), C.POINTER(C.c_int)]),
    "ss_snake_inverse": (C.c_int, [C.c_int, C.POINTER(GridSpec), C.POINTER(C.c_int),
                                   C.POINTER(C.c_int)]),
    "ss_enumerate_rays": (C.c_int, [C.POINTER(ScanConfig), dp, i64p, C.POINTER(C.c_int), dp]),
    "ss_build_system": (C.c_int, [vp, C.POINTER(ScanConfig), C.c_int, C.POINTER(vp)]),
    "ss_build_system_grid": (C.c_int, [vp, C.POINTER(ScanConfig), C.POINTER(GridSpec), C.c_int,
                                       C.POINTER(vp)]),
    "ss_enumerate_rays_grid": (C.c_int, [C.POINTER(ScanConfig), C.POINTER(GridSpec), dp, i64p,
                                         C.POINTER(C.c_int), dp]),
    "ss_verify_symmetry": (C.c_int, [vp, C.c_double, C.POINTER(SymmetryReportC)]),
    "ss_split_rhs": (C.c_int, [vp, dp, i64, dp, dp]),
    "ss_split_system": (C.c_int, [vp, dp, i64, C.c_double, C.POINTER(vp), C.POINTER(vp), dp, dp,
                                  dp, C.POINTER(SymmetryReportC)]),
    "ss_decompose_solution": (C.c_int, [vp, dp, i64, dp, dp]),
    "ss_recombine_solution": (C.c_int, [vp, dp, dp, i64, dp]),
    "ss_sart_solve": (C.c_int, [vp, dp, i64, C.POINTER(SolveOptionsC), dp, i64,
                                C.POINTER(SolveReportC), dp]),
    "ss_pseudo_solve_dense": (C.c_int, [vp, dp, i64, i64, dp, i64]),
    "ss_emitter_angles": (C.c_int, [C.POINTER(ScanConfig), dp]),
    "ss_emitter_positions": (C.c_int, [C.POINTER(ScanConfig), C.c_double, dp]),
    "ss_ray_weights": (C.c_int, [vp, dp, C.POINTER(GridSpec), i64, i32p, dp, i64p]),
    "ss_cgls_solve": (C.c_int, [vp, dp, i64, C.POINTER(SolveOptionsC), dp, i64,
                                C.POINTER(SolveReportC), dp]),
    "ss_solve_split": (C.c_int, [vp, dp, i64, C.c_double, C.POINTER(SolveOptionsC), dp, i64,
                                 C.POINTER(SolveReportC)]),
    "ss_solve_direct": (C.c_int, [vp, dp, i64, C.POINTER(SolveOptionsC), dp, i64,
                                  C.POINTER(SolveReportC)]),
    "ss_random_ellipses": (C.c_int, [C.c_uint64, C.c_int, dp]),
    "ss_rasterize": (C.c_int, [vp, dp, C.c_int, C.POINTER(GridSpec), dp]),
    "ss_forward_project": (C.c_int, [vp, dp, dp]),
    "ss_add_noise": (C.c_int, [dp, i64, C.c_double, C.c_uint64]),
    "ss_plan_create": (C.c_int, [vp, vp, vp, C.POINTER(SolveOptionsC), C.c_int, C.POINTER(vp)]),
    "ss_plan_destroy": (C.c_int, [vp]),
    "ss_plan_set_rhs": (C.c_int, [vp, C.c_int, dp]),
    "ss_plan_set_rhs_device": (C.c_int, [vp, C.c_int, vp]),
    "ss_plan_launch": (C.c_int, [vp]),
    "ss_plan_finish": (C.c_int, [vp, C.POINTER(SolveReportC)]),
    "ss_plan_get_solution": (C.c_int, [vp, C.c_int, dp]),
    "ss_plan_get_history": (C.c_int, [vp, C.c_int, C.c_int, dp, C.POINTER(C.c_int)]),
    "ss_plan_recombine": (C.c_int, [vp, dp]),
    "ss_plan_solution_device": (vp, [vp, C.c_int]),
    "ss_plan_stats": (C.c_int, [vp, i64p, i64p, C.POINTER(C.c_int)]),
    "ss_plan_profile": (C.c_int, [vp, C.c_int, fp, fp]),
    "ss_plan_time_kernel": (C.c_int, [vp, C.c_int, C.c_int, fp]),
    "ss_plan_kernel_bytes": (C.c_int, [vp, i64p, i64p]),
    "ss_plan_describe": (C.c_int, [vp, C.c_char_p, i64]),
    "ss_nccl_unique_id": (C.c_int, [vp]),
    "ss_ctx_attach_nccl": (C.c_int, [vp, vp, C.c_int, C.c_int]),
    "ss_partition_rows": (C.c_int, [i32p, i64, C.c_int, i64p]),
    "ss_plan_create_sharded": (C.c_int, [vp, vp, i64, i64, C.POINTER(SolveOptionsC),
                                         C.POINTER(vp)]),
    "ss_exchange_owned_columns": (C.c_int, [i64, C.c_int, C.c_int, i64p, i64p]),
    "ss_plan_create_sharded_x": (C.c_int, [vp, vp, i64, i64, C.POINTER(SolveOptionsC), C.c_int,
                                           C.POINTER(vp)]),
    "ss_plan_create_sharded_group": (C.c_int, [vp, vp, C.c_int, i64p, C.POINTER(SolveOptionsC),
                                               C.POINTER(vp)]),
    "ss_plan_create_sharded_pair": (C.c_int, [vp, vp, vp, i64, i64, C.POINTER(SolveOptionsC),
                                              C.POINTER(vp)]),
    "ss_plan_create_sharded_pair_group": (C.c_int, [vp, vp, vp, C.c_int, i64p,
                                                    C.POINTER(SolveOptionsC), C.POINTER(vp)]),
    "ss_plan_group_run": (C.c_int, [C.POINTER(vp), C.c_int]),
    "ss_read_matrix_market": (C.c_int, [vp, C.c_char_p, C.POINTER(vp)]),
    "ss_write_matrix_market": (C.c_int, [vp, C.c_char_p]),
    "ss_read_vector_csv": (C.c_int, [C.c_char_p, dp, i64, i64p]),
    "ss_write_vector_csv": (C.c_int, [C.c_char_p, dp, i64]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def load():
    """Load the in-tree CUDA library; raises (no fallback) if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} is missing: build it with `make -C paper_1902_10559_b200/csrc` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
