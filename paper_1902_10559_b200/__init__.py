"""B200-native folded SART for arXiv 1902.10559 (reference `symsplit`).

The product is the CUDA library libsymsplit_b200.so (C ABI in
include/symsplit_b200.h, C++ facade include/symsplit_b200.hpp); this package
is its Python mirror of the reference API. No CPU fallback exists.
"""
from .symsplit import (  # noqa: F401
    CentroSystem, Context, DeviceError, Error, Matrix, SartPlan, SolutionPair, SolveOptions,
    IoError, cgls_solve, emitter_angles, emitter_positions, pseudo_solve_dense, ray_weights,
    shepp_logan_ellipses, read_matrix_market, read_vector_csv, write_matrix_market,
    write_vector_csv,
    SolveReport, SplitSystem, SymmetryError, SymmetryReport, SymsplitError, build_system,
    decompose_solution, default_context, degrees_to_radians, enumerate_rays, forward_project,
    make_grid, parse_scan_config, random_ellipses, rasterize, recombine_solution, sart_solve,
    scan_config, snake_index, snake_inverse, solve_direct, solve_split, split_rhs,
    split_system, verify_symmetry)
from .configs import CONFIGS, Workload  # noqa: F401
