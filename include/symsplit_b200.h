/*
 * symsplit_b200 — C ABI of the B200-native folded-SART path.
 *
 * This is the drop-in boundary for the reference library `symsplit`
 * (/root/reference/proj). The reference exposes a C++ value API over Eigen
 * types (no plugin registry; method dispatch is the switch in run_method,
 * proj/src/solvers.cpp:38-57). Every entry point below replaces one reference
 * function, cited as "replaces <file>:<line>". Plain pointers and sizes only:
 * host buffers are caller-owned, device data lives behind opaque handles that
 * the caller destroys explicitly. Errors are status codes plus a thread-local
 * message (ss_last_error) carrying the reference's exception text; the C++
 * facade (symsplit_b200.hpp) turns them back into symsplit::Error /
 * SymmetryError. Calls on distinct contexts are thread-safe; a context (one
 * per device) serialises its own work on one CUDA stream.
 *
 * Index convention: 0-based at this interface, like the reference Matrix API
 * (matrix.hpp:29-31); reports carry the reference's 1-based worst_row/col.
 */
#ifndef SYMSPLIT_B200_H
#define SYMSPLIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
#define SS_OK 0
#define SS_ERR_INVALID 1   /* symsplit::Error (bad argument, shape, rank ...) */
#define SS_ERR_SYMMETRY 2  /* symsplit::SymmetryError (centro.hpp:73-78)       */
#define SS_ERR_DIVERGED 3  /* sart_solve: diverged (solvers.cpp:186-189)       */
#define SS_ERR_CUDA 4      /* CUDA runtime failure                            */
#define SS_ERR_NCCL 5      /* NCCL failure                                    */
#define SS_ERR_OOM 6       /* device allocation failed                        */
#define SS_ERR_IO 7        /* symsplit::IoError (io.hpp:14-20)                 */

/* arithmetic type of a SART plan */
#define SS_F64 0
#define SS_F32 1

typedef struct ss_context* ss_ctx_t;
typedef struct ss_matrix* ss_matrix_t; /* device sparse matrix, fp64 master  */
typedef struct ss_plan* ss_plan_t;     /* prepared SART over 1 or 2 systems  */

/* replaces ScanConfig / ScanGeometry (geometry.hpp:54-68, 137-141) */
typedef struct {
  int k;            /* emitter positions (even)                    */
  double gamma;     /* half sweep, radians                         */
  double h_e;       /* emitter rotation radius                     */
  double h_m;       /* lower grid edge above the detector          */
  double l_m;       /* detector length                             */
  int n_p;          /* detector pixels                             */
  double a_e;       /* recorded only (pencil-ray model ignores it) */
  double obj_size;  /* lateral extent of the reconstruction region */
  int grid_nx;
  int grid_ny;
} ss_scan_config;

/* replaces GridSpec (geometry.hpp:22-37) */
typedef struct {
  int n_x, n_y;
  double voxel_size, center_x, y_bottom;
} ss_grid_spec;

/* iterative methods on the device (reference Method, solvers.hpp:14) */
#define SS_METHOD_SART 0
#define SS_METHOD_CGLS 1
#define SS_METHOD_DENSE 2 /* Method::dense_minnorm (pseudo_solve_dense) */

/* replaces SolveOptions (solvers.hpp:19-27) */
typedef struct {
  int max_iters;      /* default 200                           */
  double tol;         /* default 1e-10; 0 = fixed iteration count (SART) */
  double relaxation;  /* default 1.0, in (0, 2] (SART only)    */
  int parallelism;    /* accepted for parity; results never depend on it */
  int dtype;          /* SS_F64 (reference) or SS_F32          */
  int method;         /* SS_METHOD_SART (default), SS_METHOD_CGLS or SS_METHOD_DENSE */
  int64_t dense_cap;  /* rows*cols guard of the dense path; 0 = reference default 5e7 */
} ss_solve_options;

/* replaces SolveReport scalars (solvers.hpp:29-45) */
typedef struct {
  double residual_norm;
  double solution_norm;
  int iterations;
  double wall_time_seconds;
  double split_seconds;
  double recombine_seconds;
  double branch1_seconds;
  double branch2_seconds;
  int history_len;
} ss_solve_report;

/* replaces SymmetryReport (centro.hpp:16-22) */
typedef struct {
  int holds;
  double max_violation;
  int64_t worst_row; /* 1-based */
  int64_t worst_col; /* 1-based */
  int status;        /* 0 ok, 1 odd_row_count, 2 odd_col_count */
} ss_symmetry_report;

/* ------------------------------------------------------------ runtime */
const char* ss_last_error(void);
int ss_version(void);
void ss_default_options(ss_solve_options* out); /* SolveOptions{} defaults */
int ss_device_count(int* out);
int ss_ctx_create(int device, ss_ctx_t* out);
int ss_ctx_destroy(ss_ctx_t ctx);
int ss_ctx_synchronize(ss_ctx_t ctx);
/* cudaStream_t the context launches on (for event timing by callers) */
void* ss_ctx_stream(ss_ctx_t ctx);
/* Number of kernels this context has launched so far (launch accounting). */
int64_t ss_ctx_launch_count(ss_ctx_t ctx);

/* ------------------------------------------------------------ matrices */
/* replaces Matrix(SparseStorage) (matrix.cpp:7-10): compressed CSC in, finite check */
int ss_matrix_from_csc(ss_ctx_t ctx, int64_t rows, int64_t cols, int64_t nnz,
                       const int32_t* outer, const int32_t* inner, const double* values,
                       ss_matrix_t* out);
/* replaces Matrix::from_triplets (matrix.cpp:12-18): duplicates summed in triplet order */
int ss_matrix_from_triplets(ss_ctx_t ctx, int64_t rows, int64_t cols, int64_t count,
                            const int32_t* row, const int32_t* col, const double* values,
                            ss_matrix_t* out);
int ss_matrix_destroy(ss_matrix_t a);
/* ss_solve_split keeps the fold of its matrix and the SART plan over it on the
 * (immutable) matrix handle for the next call; this frees them early */
int ss_matrix_release_cache(ss_matrix_t a);
int ss_matrix_shape(ss_matrix_t a, int64_t* rows, int64_t* cols, int64_t* stored);
/* replaces Matrix::nonzeros / fill_ratio (matrix.cpp:28-42) */
int ss_matrix_nonzeros(ss_matrix_t a, int64_t* out);
int ss_matrix_fill_ratio(ss_matrix_t a, double* out);
/* byte-parity downloads: CSR (columns ascending per row) and CSC (rows ascending per column) */
int ss_matrix_download_csr(ss_matrix_t a, int32_t* ptr, int32_t* idx, double* values);
int ss_matrix_download_csc(ss_matrix_t a, int32_t* outer, int32_t* inner, double* values);
/* replaces Matrix::apply / apply_transpose (matrix.cpp:67-76) */
int ss_matrix_apply(ss_matrix_t a, const double* x, double* y);
/* replaces Matrix::coeff (matrix.cpp:44-50): the stored value at 0-based
 * (i, j) or 0; "matrix index out of range" outside the shape */
int ss_matrix_coeff(ss_matrix_t a, int64_t i, int64_t j, double* out);
int ss_matrix_apply_transpose(ss_matrix_t a, const double* y, double* x);

/* ------------------------------------------------------------ geometry */
/* replaces parse_scan_config (geometry.cpp:352-401) and make_grid (:403-411) */
int ss_parse_scan_config(const char* text, ss_scan_config* out);
int ss_make_grid(const ss_scan_config* cfg, ss_grid_spec* out);
/* replaces snake_index / snake_inverse (geometry.cpp:76-92), 1-based */
int ss_snake_index(int c, int r, const ss_grid_spec* grid, int* j);
int ss_snake_inverse(int j, const ss_grid_spec* grid, int* c, int* r);
/* replaces enumerate_rays (geometry.cpp:132-173); rays as (sx,sy,dx,dy) rows,
 * pass rays4 = NULL to query the count */
int ss_enumerate_rays(const ss_scan_config* cfg, double* rays4, int64_t* count,
                      int* samples, double* pitch);
/* replaces emitter_angles (geometry.cpp:107-117): k angles, most negative first */
int ss_emitter_angles(const ss_scan_config* cfg, double* angles);
/* replaces emitter_positions (geometry.cpp:119-130): k sources as (x, y) pairs */
int ss_emitter_positions(const ss_scan_config* cfg, double center_x, double* xy);
/* replaces ray_weights (geometry.cpp:175-225) for one ray (source x, y,
 * detector x, y), walked on the device with the build's tracer: 1-based snake
 * columns and lengths in path order; pass capacity 0 to query the count */
int ss_ray_weights(ss_ctx_t ctx, const double ray4[4], const ss_grid_spec* grid, int64_t capacity,
                   int* cols, double* lens, int64_t* count);
/* replaces build_system (geometry.cpp:227-275): GPU Siddon trace of rays
 * 0..M/2-1, mirror rows by reflection; returns A (M x N) on the device */
int ss_build_system(ss_ctx_t ctx, const ss_scan_config* cfg, int parallelism,
                    ss_matrix_t* out);
/* replaces build_system(const ScanGeometry&, const GridSpec&, int parallelism)
 * (geometry.hpp:118, geometry.cpp:227-275) with a caller-supplied grid: the
 * geometry fields of `geom` are used, its grid_nx / grid_ny are ignored */
int ss_build_system_grid(ss_ctx_t ctx, const ss_scan_config* geom, const ss_grid_spec* grid,
                         int parallelism, ss_matrix_t* out);
/* replaces enumerate_rays(const ScanGeometry&, const GridSpec&)
 * (geometry.cpp:132-173) with a caller-supplied grid (as above) */
int ss_enumerate_rays_grid(const ss_scan_config* geom, const ss_grid_spec* grid, double* rays4,
                           int64_t* count, int* samples, double* pitch);

/* ------------------------------------------------------------ centro */
/* replaces verify_symmetry (centro.cpp:46-66) */
int ss_verify_symmetry(ss_matrix_t a, double tol, ss_symmetry_report* out);
/* replaces split_rhs (centro.cpp:89-99) */
int ss_split_rhs(ss_ctx_t ctx, const double* p, int64_t m, double* p1, double* p2);
/* replaces split_system (centro.cpp:144-156) + detail::split_matrix sparse fold
 * (:109-130): bit-exact A1/A2. p/p1/p2 are host vectors (m and m/2).
 * fills = {parent_fill, fill1, fill2}. On SS_ERR_SYMMETRY `report` holds the
 * violation. */
int ss_split_system(ss_matrix_t a, const double* p, int64_t m, double symmetry_tol,
                    ss_matrix_t* a1, ss_matrix_t* a2, double* p1, double* p2,
                    double* fills, ss_symmetry_report* report);
/* replaces decompose_solution / recombine_solution (centro.cpp:158-185) */
int ss_decompose_solution(ss_ctx_t ctx, const double* f, int64_t n, double* f1, double* f2);
int ss_recombine_solution(ss_ctx_t ctx, const double* f1, const double* f2, int64_t nh,
                          double* f);

/* ------------------------------------------------------------ solvers */
/* replaces sart_solve (solvers.cpp:148-199). history may be NULL, else room
 * for max_iters + 1 entries. */
int ss_sart_solve(ss_matrix_t a, const double* p, int64_t m, const ss_solve_options* opts,
                  double* f, int64_t n, ss_solve_report* report, double* history);
/* replaces cgls_solve (solvers.cpp:99-146); history may be NULL, else room
 * for max_iters entries */
int ss_cgls_solve(ss_matrix_t a, const double* p, int64_t m, const ss_solve_options* opts,
                  double* f, int64_t n, ss_solve_report* report, double* history);
/* replaces pseudo_solve_dense (solvers.cpp:81-97): minimum-norm solution via
 * the SVD pseudo-inverse at the reference threshold max(m,n)*eps; refuses
 * rows*cols > dense_cap with the reference message */
int ss_pseudo_solve_dense(ss_matrix_t a, const double* p, int64_t m, int64_t dense_cap,
                          double* f, int64_t n);
/* replaces solve_split (solvers.cpp:207-269) with method = sart, cgls or dense */
int ss_solve_split(ss_matrix_t a, const double* p, int64_t m, double symmetry_tol,
                   const ss_solve_options* opts, double* f, int64_t n,
                   ss_solve_report* report);
/* replaces solve_direct (solvers.cpp:201-205) with method = sart or cgls */
int ss_solve_direct(ss_matrix_t a, const double* p, int64_t m, const ss_solve_options* opts,
                    double* f, int64_t n, ss_solve_report* report);

/* ------------------------------------------------------------ phantom (input side) */
/* BASELINE synthetic ellipses from the reference Rng (oracles.hpp:29-50):
 * rows of (x0, y0, a, b, angle, density) */
int ss_random_ellipses(uint64_t seed, int count, double* out6);
/* replaces rasterize (phantom.cpp:34-58): GPU, bit-exact, snake order */
int ss_rasterize(ss_ctx_t ctx, const double* ellipses6, int count, const ss_grid_spec* grid,
                 double* values);
/* replaces forward_project (phantom.cpp:62-127): GPU, mirror-pair folded row sums */
int ss_forward_project(ss_matrix_t a, const double* f, double* p);
/* replaces the seeded noise of forward_project (phantom.cpp:129-149); host */
int ss_add_noise(double* p, int64_t m, double sigma, uint64_t seed);

/* ------------------------------------------------------------ file formats (ingestion) */
/* replaces read_matrix_market (io.cpp:83-187): validated, sorted, no duplicates */
int ss_read_matrix_market(ss_ctx_t ctx, const char* path, ss_matrix_t* out);
/* replaces write_matrix_market (io.cpp:189-210): canonical order, %.17g */
int ss_write_matrix_market(ss_matrix_t a, const char* path);
/* replaces read_vector_csv (io.cpp:212-230); pass values = NULL to query the length */
int ss_read_vector_csv(const char* path, double* values, int64_t capacity, int64_t* count);
/* replaces write_vector_csv (io.cpp:232-238) */
int ss_write_vector_csv(const char* path, const double* values, int64_t count);

/* ------------------------------------------------------------ plans (device-resident loop) */
/* A prepared SART over one system (a2 == NULL) or the folded pair (a1, a2),
 * both run by the same launches. Normalisers are computed here (the
 * reference computes them before its timer, solvers.cpp:156-172). nrhs > 1
 * makes a multi-right-hand-side plan (independent slices sharing A). */
int ss_plan_create(ss_ctx_t ctx, ss_matrix_t a1, ss_matrix_t a2, const ss_solve_options* opts,
                   int nrhs, ss_plan_t* out);
int ss_plan_destroy(ss_plan_t plan);
/* p for system `which` (0/1): host vector of rows*nrhs doubles, slice-major
 * (p[s*rows + i]). */
int ss_plan_set_rhs(ss_plan_t plan, int which, const double* p);
/* same from a device buffer of the plan dtype laid out [rows][nrhs] */
int ss_plan_set_rhs_device(ss_plan_t plan, int which, const void* p_dev);
/* enqueue one full solve (x0 = 0, max_iters iterations) on the context stream */
int ss_plan_launch(ss_plan_t plan);
/* wait, check divergence, fill the report (wall = device loop time) */
int ss_plan_finish(ss_plan_t plan, ss_solve_report* report);
/* solution of system `which`, host, slice-major like set_rhs */
int ss_plan_get_solution(ss_plan_t plan, int which, double* f);
int ss_plan_get_history(ss_plan_t plan, int which, int slice, double* hist, int* len);
/* recombined f (N = 2*cols, slice-major) of a two-system plan */
int ss_plan_recombine(ss_plan_t plan, double* f);
/* device pointer to the iterate of system `which` ([cols][nrhs], plan dtype) */
void* ss_plan_solution_device(ss_plan_t plan, int which);
/* algorithmic bytes per iteration (matrices + pointers), kernels per iteration */
int ss_plan_stats(ss_plan_t plan, int64_t* matrix_bytes_per_iter,
                  int64_t* vector_bytes_per_iter, int* kernels_per_iter);
/* matrix bytes each SART kernel streams per launch in this plan's format
 * (paired plans share one index stream between the two folded systems) */
int ss_plan_kernel_bytes(ss_plan_t plan, int64_t* fwd_bytes, int64_t* back_bytes);
/* one-line JSON description of the plan's kernels (layout, VS, UF, grid,
 * kernel names as ncu reports them); NUL-terminated, truncated to cap */
int ss_plan_describe(ss_plan_t plan, char* buf, int64_t cap);
/* time `iters` bare iterations of the loop with CUDA events on the context
 * stream (per-kernel split: fwd_ms = forward kernels, back_ms = back kernels) */
int ss_plan_profile(ss_plan_t plan, int iters, float* fwd_ms, float* back_ms);
/* in-loop time of one SART kernel (fwd != 0: K1, else K2): `reps` launches back
 * to back with the loop's launch configuration, events around the batch;
 * ms = time per launch. Resets the plan. */
int ss_plan_time_kernel(ss_plan_t plan, int fwd, int reps, float* ms);

/* ------------------------------------------------------------ row-sharded multi-GPU */
/* One process per GPU. Ranks r0..r0+n-1 of an NCCL communicator share one
 * folded system; each keeps rows [row_begin,row_end) of it and all-reduces
 * the back-projection once per iteration (SURVEY §8e level 3). */
int ss_nccl_unique_id(void* out128);
int ss_ctx_attach_nccl(ss_ctx_t ctx, const void* unique_id128, int nranks, int rank);
/* balanced row split of a CSR row pointer by nnz (host, no GPU needed) */
int ss_partition_rows(const int32_t* rowptr, int64_t rows, int parts, int64_t* bounds);
int ss_plan_create_sharded(ss_ctx_t ctx, ss_matrix_t a, int64_t row_begin, int64_t row_end,
                           const ss_solve_options* opts, ss_plan_t* out);

/* How the ranks of a row-sharded system combine their back-projections.
 * SS_XCHG_NCCL: K2 writes the partial A_g^T w_g, then ncclAllReduce + update.
 * SS_XCHG_PEER: fused exchange over NVLink peer memory. K2 stores each
 *   column's partial straight into its owner's receive row; each owner sums
 *   the G partials of its own columns in rank order, applies the update and
 *   stores its new x range into every rank's replica; the next K1 waits
 *   (device-side) for all ranges. No NCCL call on the data path; the
 *   regions are mapped with CUDA IPC (handles exchanged once over the
 *   context's NCCL communicator). Replaces the same reference loop as
 *   ss_plan_create_sharded (solvers.cpp:173-192). */
#define SS_XCHG_NCCL 0
#define SS_XCHG_PEER 1
/* columns [col_begin, col_end) whose partials rank `rank` of `parts` reduces
 * and whose x it pushes to every replica (host, no GPU needed) */
int ss_exchange_owned_columns(int64_t cols, int parts, int rank, int64_t* col_begin,
                              int64_t* col_end);
int ss_plan_create_sharded_x(ss_ctx_t ctx, ss_matrix_t a, int64_t row_begin, int64_t row_end,
                             const ss_solve_options* opts, int exchange, ss_plan_t* out);
/* The folded PAIR row-sharded over all ranks of the context's communicator
 * (the B200 layout for N >= 2): each rank keeps rows [row_begin, row_end) of
 * BOTH folded systems on the paired mirror-coded streams (one index stream,
 * both systems per launch) and exchanges {u1, u2} back-projection pairs through
 * the fused peer exchange (SS_XCHG_PEER); each system keeps its own stop /
 * divergence state. Replaces the reference's two-branch solve_split
 * (solvers.cpp:212-233) run over N devices. */
int ss_plan_create_sharded_pair(ss_ctx_t ctx, ss_matrix_t a1, ss_matrix_t a2, int64_t row_begin,
                                int64_t row_end, const ss_solve_options* opts, ss_plan_t* out);
/* one-device emulation of `parts` ranks of the row-sharded pair (tests) */
int ss_plan_create_sharded_pair_group(ss_ctx_t ctx, ss_matrix_t a1, ss_matrix_t a2, int parts,
                                      const int64_t* bounds, const ss_solve_options* opts,
                                      ss_plan_t* plans);
/* One-device emulation of `parts` peer-exchange ranks (tests and single-GPU
 * measurement of the fused exchange): plans[g] keeps rows
 * [bounds[g], bounds[g+1]) and the plans' regions are linked directly. Set
 * each plan's rhs slice with ss_plan_set_rhs, then ss_plan_group_run launches
 * every rank's kernels in rank order on the shared stream; ss_plan_finish /
 * get_solution / get_history work per plan. */
int ss_plan_create_sharded_group(ss_ctx_t ctx, ss_matrix_t a, int parts, const int64_t* bounds,
                                 const ss_solve_options* opts, ss_plan_t* plans);
int ss_plan_group_run(ss_plan_t* plans, int parts);

#ifdef __cplusplus
}
#endif

#endif /* SYMSPLIT_B200_H */
