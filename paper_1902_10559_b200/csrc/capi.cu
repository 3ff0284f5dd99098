// extern "C" surface (include/symsplit_b200.h). Each function validates like
// the reference function it replaces, runs on the device, and converts
// exceptions to status codes + a thread-local message.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <memory>
#include <sstream>
#include <string>

#include "nccl_dyn.hpp"
#include "io.hpp"
#include "plan.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SS_OK;
  } catch (const ssb::Failure& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return SS_ERR_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SS_ERR_INVALID;
  }
}

void need(const void* p, const char* what) {
  if (!p) ssb::fail(std::string(what) + " must not be null");
}

// The opaque ABI handles are the internal objects themselves.
ssb::Matrix* M(ss_matrix_t a) {
  need(a, "matrix");
  return reinterpret_cast<ssb::Matrix*>(a);
}
ssb::Context* CX(ss_ctx_t c) {
  need(c, "ctx");
  return reinterpret_cast<ssb::Context*>(c);
}
ssb::Plan* PL(ss_plan_t p) {
  need(p, "plan");
  return reinterpret_cast<ssb::Plan*>(p);
}
ss_matrix_t wrap(ssb::Matrix* a) { return reinterpret_cast<ss_matrix_t>(a); }
ss_plan_t wrap(ssb::Plan* p) { return reinterpret_cast<ss_plan_t>(p); }

void use_device(ssb::Context* c) {
  SSB_CUDA(cudaSetDevice(c->device));
  ssb::alloc_stream() = c->stream;
}

template <class T>
ssb::DBuf<T> to_device(ssb::Context* c, const T* h, std::int64_t n) {
  ssb::DBuf<T> d(n);
  if (n) {
    need(h, "host buffer");
    SSB_CUDA(cudaMemcpyAsync(d.get(), h, n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  }
  return d;
}

template <class T>
void to_host(ssb::Context* c, T* h, const T* d, std::int64_t n) {
  if (n) {
    need(h, "host buffer");
    SSB_CUDA(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
  }
  c->sync();
}

// reference solvers.cpp:28-36
void check_system(std::int64_t rows, const double* p, std::int64_t m, const char* op) {
  if (m != rows) {
    std::ostringstream msg;
    msg << op << ": rhs length " << m << " does not match rows " << rows;
    ssb::fail(msg.str());
  }
  for (std::int64_t i = 0; i < m; ++i) {
    if (!std::isfinite(p[i])) ssb::fail(std::string(op) + ": non-finite rhs");
  }
}

// reference SolveOptions::dense_cap default (solvers.hpp:26); 0 = that default
std::int64_t effective_dense_cap(const ss_solve_options& o) {
  return o.dense_cap > 0 ? o.dense_cap : 50000000;
}

void check_options(const ss_solve_options& o) {
  if (o.relaxation <= 0 || o.relaxation > 2) ssb::fail("sart_solve: relaxation must be in (0, 2]");
  if (o.max_iters < 1) ssb::fail("sart_solve: max_iters must be >= 1");
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Phase timing of the host-facing calls (SSB_TRACE=1 prints to stderr).
struct Trace {
  ssb::Context* ctx;
  bool on;
  double t;
  explicit Trace(ssb::Context* c) : ctx(c), on(std::getenv("SSB_TRACE") != nullptr), t(now()) {}
  void mark(const char* what) {
    if (!on) return;
    ctx->sync();
    const double n = now();
    std::fprintf(stderr, "[ssb] %-28s %9.3f ms\n", what, (n - t) * 1e3);
    t = n;
  }
};

// ||A f - p|| and ||f|| on the device in fp64, after the timed loop like the
// reference (solvers.cpp:194-197, :266-267).
void fill_report(ssb::Matrix& a, const double* f_dev, const double* p_dev, ss_solve_report* rep) {
  ssb::DBuf<double> r(a.rows);
  ssb::residual_dev(a, f_dev, p_dev, r.get());
  rep->residual_norm = std::sqrt(ssb::norm2_dev(a.ctx, r.get(), a.rows));
  rep->solution_norm = std::sqrt(ssb::norm2_dev(a.ctx, f_dev, a.cols));
}

// reference centro.cpp:27-42 message
std::string symmetry_message(const char* op, const ss_symmetry_report& r, double tol) {
  std::ostringstream msg;
  msg << op << ": matrix is not centrosymmetric";
  if (r.status == 1) {
    msg << " (odd row count)";
  } else if (r.status == 2) {
    msg << " (odd column count)";
  } else {
    msg << " (max violation " << r.max_violation << " at (" << r.worst_row << ","
        << r.worst_col << "), tol " << tol << ")";
  }
  return msg.str();
}

struct SplitOut {
  std::unique_ptr<ssb::Matrix> a1, a2;
  ssb::DBuf<double> p1, p2;
  double fills[3] = {0, 0, 0};
};

// reference split_system (centro.cpp:144-156) on the device
void split_device(ssb::Matrix& a, const double* p_dev, std::int64_t m, double tol, SplitOut& o,
                  ss_symmetry_report* rep) {
  if (m != a.rows) ssb::fail("split_system: right-hand side length does not match rows");
  Trace tr(a.ctx);
  ssb::Matrix *x = nullptr, *y = nullptr;
  const ss_symmetry_report r = ssb::fold_checked(a, tol, x, y);  // verify + fold, one pass
  tr.mark("  verify_symmetry + fold");
  if (!r.holds) {
    if (rep) *rep = r;
    throw ssb::Failure(SS_ERR_SYMMETRY, symmetry_message("split_system", r, tol));
  }
  o.a1.reset(x);
  o.a2.reset(y);
  o.p1.alloc(m / 2);
  o.p2.alloc(m / 2);
  ssb::split_rhs_dev(a.ctx, p_dev, o.p1.get(), o.p2.get(), m / 2);
  const double parent = static_cast<double>(a.rows) * static_cast<double>(a.cols);
  const double half = static_cast<double>(o.a1->rows) * static_cast<double>(o.a1->cols);
  o.fills[0] = parent > 0 ? static_cast<double>(ssb::nonzeros(a)) / parent : 0.0;
  // the fold stores no zeros (it prunes v != 0 like centro.cpp:127-128), so the
  // folded systems' nonzero counts are their stored counts
  o.fills[1] = half > 0 ? static_cast<double>(o.a1->nnz) / half : 0.0;
  o.fills[2] = half > 0 ? static_cast<double>(o.a2->nnz) / half : 0.0;
  tr.mark("  split_rhs + fills");
}

}  // namespace

namespace ssb {
// solve_split's per-matrix cache (Matrix::solve_cache). A matrix handle is
// immutable, so its fold (the reference recomputes it every call,
// centro.cpp:144-156) and the SART plan over A1/A2 (normalisers, CSC, paired
// streams, captured loop) are derived once and reused; a call with new options
// rebuilds the plan only. The symmetry report is kept independent of the
// tolerance (the fold is computed with an unbounded one) and each call applies
// its own symmetry_tol. Calls on one matrix serialise on `mu`.
struct SolveCache {
  std::mutex mu;
  bool folded = false;
  ss_symmetry_report rep{};
  std::unique_ptr<Matrix> a1, a2;
  std::unique_ptr<Plan> plan;
  ss_solve_options plan_opts{};
};
}  // namespace ssb

namespace {

bool same_plan_options(const ss_solve_options& a, const ss_solve_options& b) {
  return a.max_iters == b.max_iters && a.tol == b.tol && a.relaxation == b.relaxation &&
         a.dtype == b.dtype;
}

// fold of A for solve_split, from the matrix's cache (computed on first use)
ssb::SolveCache& folded_cache(ssb::Matrix& a, double tol, std::unique_lock<std::mutex>& lk) {
  if (!a.solve_cache) a.solve_cache = std::make_shared<ssb::SolveCache>();
  ssb::SolveCache& C = *a.solve_cache;
  lk = std::unique_lock<std::mutex>(C.mu);
  if (tol < 0) ssb::fail("verify_symmetry: tol must be non-negative");
  if (!C.folded) {
    ssb::Matrix *x = nullptr, *y = nullptr;
    const ss_symmetry_report r =
        ssb::fold_checked(a, std::numeric_limits<double>::max(), x, y);
    if (!r.holds) {  // odd shape (or a non-finite violation): nothing to cache
      ss_symmetry_report q = r;
      throw ssb::Failure(SS_ERR_SYMMETRY, symmetry_message("split_system", q, tol));
    }
    C.a1.reset(x);
    C.a2.reset(y);
    C.rep = r;
    C.folded = true;
  }
  if (!(C.rep.max_violation <= tol)) {
    ss_symmetry_report q = C.rep;
    q.holds = 0;
    throw ssb::Failure(SS_ERR_SYMMETRY, symmetry_message("split_system", q, tol));
  }
  return C;
}

ssb::Grid to_grid(const ss_grid_spec* g) {
  need(g, "grid");
  ssb::Grid o;
  o.n_x = g->n_x;
  o.n_y = g->n_y;
  o.voxel_size = g->voxel_size;
  o.center_x = g->center_x;
  o.y_bottom = g->y_bottom;
  return o;
}

}  // namespace

extern "C" {

const char* ss_last_error(void) { return g_err.c_str(); }

int ss_version(void) { return 1; }

void ss_default_options(ss_solve_options* o) {
  o->max_iters = 200;
  o->tol = 1e-10;
  o->relaxation = 1.0;
  o->parallelism = 0;
  o->dtype = SS_F64;
  o->method = SS_METHOD_SART;
  o->dense_cap = 0;  // 0 selects the reference default 5e7 (solvers.hpp:26)
}

int ss_device_count(int* out) {
  return guarded([&] { SSB_CUDA(cudaGetDeviceCount(out)); });
}

int ss_ctx_create(int device, ss_ctx_t* out) {
  return guarded([&] {
    need(out, "out");
    SSB_CUDA(cudaSetDevice(device));
    auto c = std::make_unique<ssb::Context>();
    c->device = device;
    SSB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    // keep freed pool memory for reuse instead of returning it to the driver
    cudaMemPool_t pool;
    SSB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    std::uint64_t keep = UINT64_MAX;
    SSB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    ssb::alloc_stream() = c->stream;
    SSB_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
    int l2 = 0;
    SSB_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
    c->l2_bytes = static_cast<std::size_t>(l2);
    *out = reinterpret_cast<ss_ctx_t>(c.release());
  });
}

int ss_ctx_destroy(ss_ctx_t h) {
  return guarded([&] {
    if (!h) return;
    ssb::Context* ctx = CX(h);
    cudaSetDevice(ctx->device);
    ssb::alloc_stream() = ctx->stream;
    cudaStreamSynchronize(ctx->stream);
    if (ctx->comm) ssb::nccl().CommDestroy(static_cast<ncclComm_t>(ctx->comm));
    ssb::release_solver(ctx);
    ctx->scratch.release();
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int ss_ctx_synchronize(ss_ctx_t h) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    use_device(ctx);
    ctx->sync();
  });
}

void* ss_ctx_stream(ss_ctx_t h) {
  return h ? static_cast<void*>(reinterpret_cast<ssb::Context*>(h)->stream) : nullptr;
}

int64_t ss_ctx_launch_count(ss_ctx_t h) {
  return h ? reinterpret_cast<ssb::Context*>(h)->launches : 0;
}

// ------------------------------------------------------------ matrices
int ss_matrix_from_csc(ss_ctx_t h, int64_t rows, int64_t cols, int64_t nnz, const int32_t* outer,
                       const int32_t* inner, const double* values, ss_matrix_t* out) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(out, "out");
    need(outer, "outer");
    use_device(ctx);
    *out = wrap(ssb::matrix_from_csc_host(ctx, rows, cols, nnz, outer, inner, values));
  });
}

int ss_matrix_from_triplets(ss_ctx_t h, int64_t rows, int64_t cols, int64_t count,
                            const int32_t* row, const int32_t* col, const double* values,
                            ss_matrix_t* out) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(out, "out");
    use_device(ctx);
    *out = wrap(ssb::matrix_from_triplets_host(ctx, rows, cols, count, row, col, values));
  });
}

int ss_matrix_release_cache(ss_matrix_t a) {
  return guarded([&] {
    ssb::Matrix* m = M(a);
    use_device(m->ctx);
    m->solve_cache.reset();
  });
}

int ss_matrix_destroy(ss_matrix_t a) {
  return guarded([&] {
    if (!a) return;
    ssb::Matrix* m = M(a);
    use_device(m->ctx);
    delete m;
  });
}

int ss_matrix_shape(ss_matrix_t a, int64_t* rows, int64_t* cols, int64_t* stored) {
  return guarded([&] {
    ssb::Matrix* m = M(a);
    if (rows) *rows = m->rows;
    if (cols) *cols = m->cols;
    if (stored) *stored = m->nnz;
  });
}

int ss_matrix_nonzeros(ss_matrix_t a, int64_t* out) {
  return guarded([&] {
    ssb::Matrix* m = M(a);
    use_device(m->ctx);
    *out = ssb::nonzeros(*m);
  });
}

int ss_matrix_fill_ratio(ss_matrix_t a, double* out) {
  return guarded([&] {
    ssb::Matrix* m = M(a);
    use_device(m->ctx);
    const double size = static_cast<double>(m->rows) * static_cast<double>(m->cols);
    *out = size > 0 ? static_cast<double>(ssb::nonzeros(*m)) / size : 0.0;
  });
}

int ss_matrix_download_csr(ss_matrix_t a, int32_t* ptr, int32_t* idx, double* values) {
  return guarded([&] {
    ssb::Matrix* m = M(a);
    use_device(m->ctx);
    if (ptr) to_host(m->ctx, ptr, m->rowptr.get(), m->rows + 1);
    if (idx) to_host(m->ctx, idx, m->colidx.get(), m->nnz);
    if (values) to_host(m->ctx, values, m->val.get(), m->nnz);
  });
}

int ss_matrix_download_csc(ss_matrix_t a, int32_t* outer, int32_t* inner, double* values) {
  return guarded([&] {
    ssb::Matrix* m = M(a);
    use_device(m->ctx);
    m->ensure_csc();
    if (outer) to_host(m->ctx, outer, m->colptr.get(), m->cols + 1);
    if (inner) to_host(m->ctx, inner, m->rowidx.get(), m->nnz);
    if (values) to_host(m->ctx, values, m->cval.get(), m->nnz);
  });
}

int ss_matrix_coeff(ss_matrix_t a, int64_t i, int64_t j, double* out) {
  return guarded([&] {
    ssb::Matrix* m = M(a);
    need(out, "out");
    if (i < 0 || i >= m->rows || j < 0 || j >= m->cols) ssb::fail("matrix index out of range");
    use_device(m->ctx);
    // row i of the CSR (columns ascending): its bounds, then a binary search
    // over its column indices
    int be[2] = {0, 0};
    to_host(m->ctx, be, m->rowptr.get() + i, 2);
    std::vector<int> cols(static_cast<std::size_t>(be[1] - be[0]));
    if (!cols.empty()) to_host(m->ctx, cols.data(), m->colidx.get() + be[0], cols.size());
    const auto it = std::lower_bound(cols.begin(), cols.end(), static_cast<int>(j));
    *out = 0.0;
    if (it != cols.end() && *it == j) {
      to_host(m->ctx, out, m->val.get() + be[0] + (it - cols.begin()), 1);
    }
  });
}

int ss_matrix_apply(ss_matrix_t a, const double* x, double* y) {
  return guarded([&] {
    ssb::Matrix* m = M(a);
    ssb::Context* c = m->ctx;
    use_device(c);
    auto dx = to_device(c, x, m->cols);
    ssb::DBuf<double> dy(m->rows);
    ssb::apply_dev(*m, dx.get(), dy.get());
    to_host(c, y, dy.get(), m->rows);
  });
}

int ss_matrix_apply_transpose(ss_matrix_t a, const double* y, double* x) {
  return guarded([&] {
    ssb::Matrix* m = M(a);
    ssb::Context* c = m->ctx;
    use_device(c);
    auto dy = to_device(c, y, m->rows);
    ssb::DBuf<double> dx(m->cols);
    ssb::apply_transpose_dev(*m, dy.get(), dx.get());
    to_host(c, x, dx.get(), m->cols);
  });
}

// ------------------------------------------------------------ geometry
int ss_parse_scan_config(const char* text, ss_scan_config* out) {
  return guarded([&] {
    need(text, "text");
    need(out, "out");
    *out = ssb::parse_scan_config(text);
  });
}

int ss_make_grid(const ss_scan_config* cfg, ss_grid_spec* out) {
  return guarded([&] {
    need(cfg, "cfg");
    const ssb::Grid g = ssb::make_grid(*cfg);
    *out = ss_grid_spec{g.n_x, g.n_y, g.voxel_size, g.center_x, g.y_bottom};
  });
}

int ss_snake_index(int c, int r, const ss_grid_spec* grid, int* j) {
  return guarded([&] { *j = ssb::snake_index(c, r, to_grid(grid)); });
}

int ss_snake_inverse(int j, const ss_grid_spec* grid, int* c, int* r) {
  return guarded([&] {
    auto [a, b] = ssb::snake_inverse(j, to_grid(grid));
    *c = a;
    *r = b;
  });
}

int ss_enumerate_rays(const ss_scan_config* cfg, double* rays4, int64_t* count, int* samples,
                      double* pitch) {
  return guarded([&] {
    need(cfg, "cfg");
    const ssb::Grid g = ssb::make_grid(*cfg);
    const ssb::RayTable t = ssb::enumerate_rays(*cfg, g, rays4 != nullptr);
    *count = t.m;
    if (samples) *samples = t.samples;
    if (pitch) *pitch = t.pitch;
    if (rays4) std::memcpy(rays4, t.all4.data(), t.all4.size() * sizeof(double));
  });
}

int ss_build_system(ss_ctx_t h, const ss_scan_config* cfg, int parallelism, ss_matrix_t* out) {
  (void)parallelism;  // the device build is identical for any worker count
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(cfg, "cfg");
    need(out, "out");
    use_device(ctx);
    *out = wrap(ssb::build_system(ctx, *cfg));
  });
}

int ss_build_system_grid(ss_ctx_t h, const ss_scan_config* geom, const ss_grid_spec* grid,
                         int parallelism, ss_matrix_t* out) {
  (void)parallelism;  // the device build is identical for any worker count
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(geom, "geom");
    need(out, "out");
    use_device(ctx);
    *out = wrap(ssb::build_system(ctx, *geom, to_grid(grid)));
  });
}

int ss_enumerate_rays_grid(const ss_scan_config* geom, const ss_grid_spec* grid, double* rays4,
                           int64_t* count, int* samples, double* pitch) {
  return guarded([&] {
    need(geom, "geom");
    need(count, "count");
    const ssb::RayTable t = ssb::enumerate_rays(*geom, to_grid(grid), rays4 != nullptr);
    *count = t.m;
    if (samples) *samples = t.samples;
    if (pitch) *pitch = t.pitch;
    if (rays4) std::memcpy(rays4, t.all4.data(), t.all4.size() * sizeof(double));
  });
}

// ------------------------------------------------------------ centro
int ss_verify_symmetry(ss_matrix_t a, double tol, ss_symmetry_report* out) {
  return guarded([&] {
    ssb::Matrix* m = M(a);
    use_device(m->ctx);
    *out = ssb::verify_symmetry(*m, tol);
  });
}

int ss_split_rhs(ss_ctx_t h, const double* p, int64_t m, double* p1, double* p2) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    if (m % 2 != 0) ssb::fail("split_rhs: vector length must be even");
    use_device(ctx);
    auto dp = to_device(ctx, p, m);
    ssb::DBuf<double> d1(m / 2), d2(m / 2);
    ssb::split_rhs_dev(ctx, dp.get(), d1.get(), d2.get(), m / 2);
    to_host(ctx, p1, d1.get(), m / 2);
    to_host(ctx, p2, d2.get(), m / 2);
  });
}

int ss_split_system(ss_matrix_t a, const double* p, int64_t m, double symmetry_tol,
                    ss_matrix_t* a1, ss_matrix_t* a2, double* p1, double* p2, double* fills,
                    ss_symmetry_report* report) {
  return guarded([&] {
    ssb::Matrix* A = M(a);
    ssb::Context* c = A->ctx;
    use_device(c);
    need(a1, "a1");
    need(a2, "a2");
    auto dp = to_device(c, p, m);
    SplitOut o;
    split_device(*A, dp.get(), m, symmetry_tol, o, report);
    to_host(c, p1, o.p1.get(), m / 2);
    to_host(c, p2, o.p2.get(), m / 2);
    if (fills) std::memcpy(fills, o.fills, sizeof o.fills);
    *a1 = wrap(o.a1.release());
    *a2 = wrap(o.a2.release());
  });
}

int ss_decompose_solution(ss_ctx_t h, const double* f, int64_t n, double* f1, double* f2) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    if (n % 2 != 0) ssb::fail("decompose_solution: vector length must be even");
    use_device(ctx);
    auto df = to_device(ctx, f, n);
    ssb::DBuf<double> d1(n / 2), d2(n / 2);
    ssb::decompose_dev(ctx, df.get(), d1.get(), d2.get(), n / 2);
    to_host(ctx, f1, d1.get(), n / 2);
    to_host(ctx, f2, d2.get(), n / 2);
  });
}

int ss_recombine_solution(ss_ctx_t h, const double* f1, const double* f2, int64_t nh,
                          double* f) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    use_device(ctx);
    auto d1 = to_device(ctx, f1, nh);
    auto d2 = to_device(ctx, f2, nh);
    if (!ssb::all_finite_dev(ctx, d1.get(), nh) || !ssb::all_finite_dev(ctx, d2.get(), nh)) {
      ssb::fail("recombine_solution: non-finite component");
    }
    ssb::DBuf<double> df(2 * nh);
    ssb::recombine_dev(ctx, d1.get(), d2.get(), df.get(), nh, 1);
    to_host(ctx, f, df.get(), 2 * nh);
  });
}

// ------------------------------------------------------------ solvers
int ss_sart_solve(ss_matrix_t a, const double* p, int64_t m, const ss_solve_options* opts,
                  double* f, int64_t n, ss_solve_report* report, double* history) {
  return guarded([&] {
    ssb::Matrix* A = M(a);
    ssb::Context* c = A->ctx;
    use_device(c);
    need(opts, "opts");
    check_system(A->rows, p, m, "sart_solve");
    check_options(*opts);
    if (n != A->cols) ssb::fail("sart_solve: solution length does not match columns");
    std::unique_ptr<ssb::Plan> P(ssb::make_plan(c, A, nullptr, *opts, 1, false));
    P->set_rhs_host(0, p);
    P->launch();
    ss_solve_report rep{};
    P->finish(&rep);
    P->get_solution(0, f);
    auto fd = to_device(c, f, n);
    auto dp = to_device(c, p, m);
    fill_report(*A, fd.get(), dp.get(), &rep);
    int len = 0;
    P->get_history(0, 0, history, &len);
    rep.history_len = len;
    if (report) *report = rep;
  });
}

int ss_cgls_solve(ss_matrix_t a, const double* p, int64_t m, const ss_solve_options* opts,
                  double* f, int64_t n, ss_solve_report* report, double* history) {
  return guarded([&] {
    ssb::Matrix* A = M(a);
    ssb::Context* c = A->ctx;
    use_device(c);
    need(opts, "opts");
    check_system(A->rows, p, m, "cgls_solve");
    if (n != A->cols) ssb::fail("cgls_solve: solution length does not match columns");
    auto dp = to_device(c, p, m);
    ssb::DBuf<double> fd(n);
    ss_solve_report rep{};
    ssb::cgls_device(*A, dp.get(), *opts, fd.get(), &rep, history);
    to_host(c, f, fd.get(), n);
    fill_report(*A, fd.get(), dp.get(), &rep);
    if (report) *report = rep;
  });
}

int ss_emitter_angles(const ss_scan_config* cfg, double* angles) {
  return guarded([&] {
    need(cfg, "cfg");
    need(angles, "angles");
    const std::vector<double> a = ssb::emitter_angles(*cfg);
    std::copy(a.begin(), a.end(), angles);
  });
}

int ss_emitter_positions(const ss_scan_config* cfg, double center_x, double* xy) {
  return guarded([&] {
    need(cfg, "cfg");
    need(xy, "xy");
    std::vector<double> x, y;
    ssb::emitter_positions(*cfg, center_x, x, y);
    for (std::size_t i = 0; i < x.size(); ++i) {
      xy[2 * i] = x[i];
      xy[2 * i + 1] = y[i];
    }
  });
}

int ss_ray_weights(ss_ctx_t h, const double ray4[4], const ss_grid_spec* grid, int64_t capacity,
                   int* cols, double* lens, int64_t* count) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(ray4, "ray4");
    need(count, "count");
    use_device(ctx);
    std::vector<int> c;
    std::vector<double> l;
    ssb::ray_weights_dev(ctx, ray4[0], ray4[1], ray4[2], ray4[3], to_grid(grid), c, l);
    *count = static_cast<int64_t>(c.size());
    if (capacity <= 0) return;
    if (capacity < *count) ssb::fail("ray_weights: capacity too small");
    need(cols, "cols");
    need(lens, "lens");
    std::copy(c.begin(), c.end(), cols);
    std::copy(l.begin(), l.end(), lens);
  });
}

int ss_pseudo_solve_dense(ss_matrix_t a, const double* p, int64_t m, int64_t dense_cap,
                          double* f, int64_t n) {
  return guarded([&] {
    ssb::Matrix* A = M(a);
    ssb::Context* c = A->ctx;
    use_device(c);
    need(f, "f");
    check_system(A->rows, p, m, "pseudo_solve_dense");
    if (n != A->cols) ssb::fail("pseudo_solve_dense: solution length does not match columns");
    auto dp = to_device(c, p, m);
    ssb::DBuf<double> fd(std::max<int64_t>(n, 1));
    ssb::pseudo_solve_dense_dev(*A, dp.get(), fd.get(), dense_cap);
    to_host(c, f, fd.get(), n);
  });
}

int ss_solve_direct(ss_matrix_t a, const double* p, int64_t m, const ss_solve_options* opts,
                    double* f, int64_t n, ss_solve_report* report) {
  if (opts && opts->method == SS_METHOD_CGLS) return ss_cgls_solve(a, p, m, opts, f, n, report, nullptr);
  if (opts && opts->method == SS_METHOD_DENSE) {
    // run_method's dense branch (solvers.cpp:40-48): f, wall time, residual, norms
    return guarded([&] {
      ssb::Matrix* A = M(a);
      ssb::Context* c = A->ctx;
      use_device(c);
      check_system(A->rows, p, m, "pseudo_solve_dense");
      if (n != A->cols) ssb::fail("pseudo_solve_dense: solution length does not match columns");
      auto dp = to_device(c, p, m);
      ssb::DBuf<double> fd(std::max<int64_t>(n, 1));
      const double t0 = now();
      ssb::pseudo_solve_dense_dev(*A, dp.get(), fd.get(), effective_dense_cap(*opts));
      ss_solve_report rep{};
      rep.wall_time_seconds = now() - t0;
      to_host(c, f, fd.get(), n);
      fill_report(*A, fd.get(), dp.get(), &rep);
      if (report) *report = rep;
    });
  }
  return ss_sart_solve(a, p, m, opts, f, n, report, nullptr);
}

int ss_solve_split(ss_matrix_t a, const double* p, int64_t m, double symmetry_tol,
                   const ss_solve_options* opts, double* f, int64_t n, ss_solve_report* report) {
  return guarded([&] {
    ssb::Matrix* A = M(a);
    ssb::Context* c = A->ctx;
    use_device(c);
    need(opts, "opts");
    Trace tr(c);
    const double t0 = now();
    auto dp = to_device(c, p, m);
    tr.mark("h2d p");
    if (m != A->rows) ssb::fail("split_system: right-hand side length does not match rows");
    // the fold of A comes from the matrix's cache (first call: computed and kept)
    std::unique_lock<std::mutex> lk;
    ssb::SolveCache& C = folded_cache(*A, symmetry_tol, lk);
    struct {
      ssb::Matrix* a1;
      ssb::Matrix* a2;
      ssb::DBuf<double> p1, p2;
    } o{C.a1.get(), C.a2.get(), {}, {}};
    o.p1.alloc(m / 2);
    o.p2.alloc(m / 2);
    ssb::split_rhs_dev(c, dp.get(), o.p1.get(), o.p2.get(), m / 2);
    c->sync();
    const double split_seconds = now() - t0;
    tr.mark("split_system");
    if (n != A->cols) ssb::fail("solve_split: solution length does not match columns");
    // Branch validation in the reference's order; failures of both branches
    // aggregate into one message (solvers.cpp:235-247).
    std::string errs[2];
    auto raise_if_failed = [&](int code) {
      if (errs[0].empty() && errs[1].empty()) return;
      std::ostringstream msg;
      msg << "solve_split: branch failure:";
      for (int s = 0; s < 2; ++s) {
        if (!errs[s].empty()) msg << " [system " << s + 1 << "] " << errs[s];
      }
      throw ssb::Failure(code, msg.str());
    };
    const std::int64_t mh = m / 2;
    const bool cgls = opts->method == SS_METHOD_CGLS;
    const bool dense = opts->method == SS_METHOD_DENSE;
    for (int s = 0; s < 2; ++s) {
      try {
        // check_system on the device-resident folded rhs (lengths match by construction)
        const char* op = cgls ? "cgls_solve" : (dense ? "pseudo_solve_dense" : "sart_solve");
        if (!ssb::all_finite_dev(c, (s ? o.p2 : o.p1).get(), mh)) {
          ssb::fail(std::string(op) + ": non-finite rhs");
        }
        if (dense) {
          // no options to validate (solvers.cpp:81-97)
        } else if (cgls) {
          if (opts->tol <= 0) ssb::fail("cgls_solve: tol must be positive");
          if (opts->max_iters < 1) ssb::fail("cgls_solve: max_iters must be >= 1");
        } else {
          check_options(*opts);
        }
      } catch (const ssb::Failure& e) {
        errs[s] = e.what();
      }
    }
    raise_if_failed(SS_ERR_INVALID);
    tr.mark("branch validation");
    if (cgls || dense) {
      // both branches on the device, failures aggregated like the reference
      ssb::DBuf<double> f1(std::max<int64_t>(n / 2, 1)), f2(std::max<int64_t>(n / 2, 1));
      ss_solve_report rb[2] = {};
      int code = SS_OK;
      if (dense) {  // the two branches concurrently (the reference's two threads)
        ssb::Matrix* am[2] = {o.a1, o.a2};
        const double* pm[2] = {o.p1.get(), o.p2.get()};
        double* fm[2] = {f1.get(), f2.get()};
        double secs[2] = {0.0, 0.0};
        int codes[2] = {SS_OK, SS_OK};
        ssb::pseudo_solve_dense_pair(am, pm, fm, effective_dense_cap(*opts), secs, errs, codes);
        for (int s = 0; s < 2; ++s) {
          rb[s].wall_time_seconds = secs[s];
          if (codes[s] != SS_OK) code = codes[s];
        }
      }
      if (cgls) {
        // both systems in one loop over the paired streams (independent scalars
        // and stop tests), or concurrent single-system solves on two streams
        ssb::Matrix* am[2] = {o.a1, o.a2};
        const double* pm[2] = {o.p1.get(), o.p2.get()};
        double* fm[2] = {f1.get(), f2.get()};
        int codes[2] = {SS_OK, SS_OK};
        // small systems are launch-latency bound: two concurrent streams win there
        const char* e = std::getenv("SSB_CGLS_PAIRED");
        const bool paired = e && *e ? *e != '0' : o.a1->nnz >= 1000000;
        if (paired) {
          ssb::cgls_device_paired(o.a1, o.a2, pm, *opts, fm, rb, errs, codes);
        } else {
          ssb::cgls_device_pair(am, pm, *opts, fm, rb, errs, codes);
        }
        for (int s = 0; s < 2; ++s) {
          if (codes[s] != SS_OK) code = codes[s];
        }
      }
      raise_if_failed(code == SS_OK ? SS_ERR_INVALID : code);
      const double t_rec0 = now();
      if (!ssb::all_finite_dev(c, f1.get(), n / 2) || !ssb::all_finite_dev(c, f2.get(), n / 2)) {
        ssb::fail("recombine_solution: non-finite component");
      }
      ssb::DBuf<double> fd(n);
      ssb::recombine_dev(c, f1.get(), f2.get(), fd.get(), n / 2, 1);
      to_host(c, f, fd.get(), n);
      ss_solve_report rep{};
      rep.recombine_seconds = now() - t_rec0;
      fill_report(*A, fd.get(), dp.get(), &rep);
      rep.iterations = std::max(rb[0].iterations, rb[1].iterations);
      rep.branch1_seconds = rb[0].wall_time_seconds;
      rep.branch2_seconds = rb[1].wall_time_seconds;
      rep.split_seconds = split_seconds;
      // the branches ran concurrently: their maximum counts (solvers.cpp:258-261)
      rep.wall_time_seconds = split_seconds + rep.recombine_seconds +
                              std::max(rep.branch1_seconds, rep.branch2_seconds);
      if (report) *report = rep;
      return;
    }
    // the SART plan over A1/A2 (normalisers, CSC, paired streams, captured
    // loop) is cached with the fold; new options rebuild it
    if (!C.plan || !same_plan_options(C.plan_opts, *opts)) {
      C.plan.reset();
      C.plan.reset(ssb::make_plan(c, o.a1, o.a2, *opts, 1, true));
      C.plan_opts = *opts;
    }
    ssb::Plan* P = C.plan.get();
    tr.mark("plan (csc, norms, graph)");
    for (int s = 0; s < 2; ++s) {
      if (P->empty_rows[s]) errs[s] = "sart_solve: matrix has no nonzero rows";
    }
    raise_if_failed(SS_ERR_INVALID);
    P->set_rhs_device_f64(0, o.p1.get());
    P->set_rhs_device_f64(1, o.p2.get());
    tr.mark("set rhs");
    P->launch();
    ss_solve_report rep{};
    try {
      P->finish(&rep);
      tr.mark("sart loop");
    } catch (const ssb::Failure& e) {
      if (e.code != SS_ERR_DIVERGED) throw;
      for (int s = 0; s < 2; ++s) {
        const int at = P->diverged_at(s);
        if (at) {
          errs[s] = "sart_solve: diverged (non-finite iterate at iteration " +
                    std::to_string(at) + ")";
        }
      }
      raise_if_failed(SS_ERR_DIVERGED);
    }
    const double t_rec0 = now();
    ssb::DBuf<double> fd(n);
    P->recombine_device(fd.get());
    to_host(c, f, fd.get(), n);
    const double recombine_seconds = now() - t_rec0;
    tr.mark("recombine + d2h f");
    fill_report(*A, fd.get(), dp.get(), &rep);
    tr.mark("residual");
    rep.split_seconds = split_seconds;
    rep.recombine_seconds = recombine_seconds;
    rep.wall_time_seconds = split_seconds + rep.branch1_seconds + recombine_seconds;
    rep.history_len = 0;  // solve_split's report carries no history
    if (report) *report = rep;
  });
}

// ------------------------------------------------------------ phantom
int ss_random_ellipses(uint64_t seed, int count, double* out6) {
  return guarded([&] {
    if (count < 0) ssb::fail("random_ellipses: count must be >= 0");
    ssb::random_ellipses(seed, count, out6);
  });
}

int ss_rasterize(ss_ctx_t h, const double* ellipses6, int count, const ss_grid_spec* grid,
                 double* values) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    use_device(ctx);
    const ssb::Grid g = to_grid(grid);
    g.validate();
    const std::int64_t n = static_cast<std::int64_t>(g.n_x) * g.n_y;
    ssb::DBuf<double> out(n);
    ssb::rasterize_dev(ctx, ellipses6, count, g, out.get());
    to_host(ctx, values, out.get(), n);
  });
}

int ss_forward_project(ss_matrix_t a, const double* f, double* p) {
  return guarded([&] {
    ssb::Matrix* A = M(a);
    ssb::Context* c = A->ctx;
    use_device(c);
    for (std::int64_t j = 0; j < A->cols; ++j) {
      if (!std::isfinite(f[j])) ssb::fail("forward_project: non-finite image");
    }
    auto df = to_device(c, f, A->cols);
    ssb::DBuf<double> dp(A->rows);
    ssb::forward_project_dev(*A, df.get(), dp.get());
    to_host(c, p, dp.get(), A->rows);
  });
}

int ss_add_noise(double* p, int64_t m, double sigma, uint64_t seed) {
  return guarded([&] { ssb::add_noise(p, m, sigma, seed); });
}

// ------------------------------------------------------------ file formats
int ss_read_matrix_market(ss_ctx_t h, const char* path, ss_matrix_t* out) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(path, "path");
    need(out, "out");
    use_device(ctx);
    const ssb::MmData d = ssb::read_matrix_market(path);
    *out = wrap(ssb::matrix_from_triplets_host(ctx, d.rows, d.cols,
                                               static_cast<int64_t>(d.v.size()), d.r.data(),
                                               d.c.data(), d.v.data()));
  });
}

int ss_write_matrix_market(ss_matrix_t a, const char* path) {
  return guarded([&] {
    ssb::Matrix* m = M(a);
    need(path, "path");
    use_device(m->ctx);
    std::vector<int> ptr(m->rows + 1), idx(m->nnz);
    std::vector<double> val(m->nnz);
    to_host(m->ctx, ptr.data(), m->rowptr.get(), m->rows + 1);
    to_host(m->ctx, idx.data(), m->colidx.get(), m->nnz);
    to_host(m->ctx, val.data(), m->val.get(), m->nnz);
    ssb::write_matrix_market(path, m->rows, m->cols, ptr, idx, val);
  });
}

int ss_read_vector_csv(const char* path, double* values, int64_t capacity, int64_t* count) {
  return guarded([&] {
    need(path, "path");
    need(count, "count");
    const std::vector<double> v = ssb::read_vector_csv(path);
    *count = static_cast<int64_t>(v.size());
    if (values) {
      if (capacity < *count) ssb::fail("read_vector_csv: buffer too small");
      std::memcpy(values, v.data(), v.size() * sizeof(double));
    }
  });
}

int ss_write_vector_csv(const char* path, const double* values, int64_t count) {
  return guarded([&] {
    need(path, "path");
    if (count) need(values, "values");
    ssb::write_vector_csv(path, values, count);
  });
}

// ------------------------------------------------------------ plans
int ss_plan_create(ss_ctx_t h, ss_matrix_t a1, ss_matrix_t a2, const ss_solve_options* opts,
                   int nrhs, ss_plan_t* out) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(opts, "opts");
    need(out, "out");
    use_device(ctx);
    check_options(*opts);
    *out = wrap(ssb::make_plan(ctx, M(a1), a2 ? M(a2) : nullptr, *opts, nrhs));
  });
}

int ss_plan_destroy(ss_plan_t plan) {
  return guarded([&] {
    if (!plan) return;
    ssb::Plan* P = PL(plan);
    use_device(P->ctx);
    delete P;
  });
}

int ss_plan_set_rhs(ss_plan_t plan, int which, const double* p) {
  return guarded([&] {
    ssb::Plan* P = PL(plan);
    use_device(P->ctx);
    need(p, "p");
    P->set_rhs_host(which, p);
  });
}

int ss_plan_set_rhs_device(ss_plan_t plan, int which, const void* p_dev) {
  return guarded([&] {
    ssb::Plan* P = PL(plan);
    use_device(P->ctx);
    need(p_dev, "p_dev");
    P->set_rhs_device(which, p_dev);
  });
}

int ss_plan_launch(ss_plan_t plan) {
  return guarded([&] {
    ssb::Plan* P = PL(plan);
    use_device(P->ctx);
    P->launch();
  });
}

int ss_plan_finish(ss_plan_t plan, ss_solve_report* report) {
  return guarded([&] {
    ssb::Plan* P = PL(plan);
    use_device(P->ctx);
    P->finish(report);
  });
}

int ss_plan_get_solution(ss_plan_t plan, int which, double* f) {
  return guarded([&] {
    ssb::Plan* P = PL(plan);
    use_device(P->ctx);
    need(f, "f");
    P->get_solution(which, f);
  });
}

int ss_plan_get_history(ss_plan_t plan, int which, int slice, double* hist, int* len) {
  return guarded([&] {
    ssb::Plan* P = PL(plan);
    use_device(P->ctx);
    need(len, "len");
    P->get_history(which, slice, hist, len);
  });
}

int ss_plan_recombine(ss_plan_t plan, double* f) {
  return guarded([&] {
    ssb::Plan* P = PL(plan);
    use_device(P->ctx);
    need(f, "f");
    P->recombine(f);
  });
}

void* ss_plan_solution_device(ss_plan_t plan, int which) {
  if (!plan) return nullptr;
  ssb::Plan* P = reinterpret_cast<ssb::Plan*>(plan);
  if (which < 0 || which >= P->nsys) return nullptr;
  return P->x[which].get();
}

int ss_plan_stats(ss_plan_t plan, int64_t* mb, int64_t* vb, int* kernels) {
  return guarded([&] { PL(plan)->stats(mb, vb, kernels); });
}

int ss_plan_kernel_bytes(ss_plan_t plan, int64_t* fwd_bytes, int64_t* back_bytes) {
  return guarded([&] { PL(plan)->kernel_bytes(fwd_bytes, back_bytes); });
}

int ss_plan_describe(ss_plan_t plan, char* buf, int64_t cap) {
  return guarded([&] {
    need(buf, "buf");
    if (cap < 1) ssb::fail("plan_describe: cap must be positive");
    const std::string d = PL(plan)->describe();
    const std::size_t n = std::min<std::size_t>(d.size(), static_cast<std::size_t>(cap - 1));
    std::memcpy(buf, d.data(), n);
    buf[n] = '\0';
  });
}

int ss_plan_profile(ss_plan_t plan, int iters, float* fwd_ms, float* back_ms) {
  return guarded([&] {
    ssb::Plan* P = PL(plan);
    use_device(P->ctx);
    need(fwd_ms, "fwd_ms");
    need(back_ms, "back_ms");
    P->profile(iters, fwd_ms, back_ms);
  });
}

int ss_plan_time_kernel(ss_plan_t plan, int fwd, int reps, float* ms) {
  return guarded([&] {
    ssb::Plan* P = PL(plan);
    use_device(P->ctx);
    need(ms, "ms");
    P->time_kernel(fwd != 0, reps, ms);
  });
}

// ------------------------------------------------------------ multi-GPU
int ss_nccl_unique_id(void* out128) {
  return guarded([&] {
    need(out128, "out");
    ncclUniqueId id;
    ssb::nccl_check(ssb::nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof id);
  });
}

int ss_ctx_attach_nccl(ss_ctx_t h, const void* uid, int nranks, int rank) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(uid, "unique_id");
    use_device(ctx);
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    ncclComm_t comm;
    ssb::nccl_check(ssb::nccl().CommInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
    // re-attaching (e.g. a fallback that builds a second plan) replaces the
    // communicator: release the old one instead of leaking it
    if (ctx->comm) ssb::nccl().CommDestroy(static_cast<ncclComm_t>(ctx->comm));
    ctx->comm = comm;
    ctx->nranks = nranks;
    ctx->rank = rank;
  });
}

int ss_partition_rows(const int32_t* rowptr, int64_t rows, int parts, int64_t* bounds) {
  return guarded([&] {
    need(rowptr, "rowptr");
    need(bounds, "bounds");
    ssb::partition_rows(rowptr, rows, parts, bounds);
  });
}

int ss_plan_create_sharded(ss_ctx_t h, ss_matrix_t a, int64_t row_begin, int64_t row_end,
                           const ss_solve_options* opts, ss_plan_t* out) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(opts, "opts");
    need(out, "out");
    use_device(ctx);
    *out = wrap(ssb::make_sharded_plan(ctx, M(a), row_begin, row_end, *opts));
  });
}

int ss_exchange_owned_columns(int64_t cols, int parts, int rank, int64_t* col_begin,
                              int64_t* col_end) {
  return guarded([&] {
    need(col_begin, "col_begin");
    need(col_end, "col_end");
    ssb::exchange_owned_columns(cols, parts, rank, col_begin, col_end);
  });
}

int ss_plan_create_sharded_pair(ss_ctx_t h, ss_matrix_t a1, ss_matrix_t a2, int64_t row_begin,
                                int64_t row_end, const ss_solve_options* opts, ss_plan_t* out) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(opts, "opts");
    need(out, "out");
    use_device(ctx);
    *out = wrap(ssb::make_sharded_pair_plan(ctx, M(a1), M(a2), row_begin, row_end, *opts));
  });
}

int ss_plan_create_sharded_pair_group(ss_ctx_t h, ss_matrix_t a1, ss_matrix_t a2, int parts,
                                      const int64_t* bounds, const ss_solve_options* opts,
                                      ss_plan_t* plans) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(opts, "opts");
    need(bounds, "bounds");
    need(plans, "plans");
    if (parts < 1) ssb::fail("plan: parts must be >= 1");
    use_device(ctx);
    std::vector<std::unique_ptr<ssb::Plan>> made;
    for (int g = 0; g < parts; ++g) {
      made.emplace_back(ssb::make_sharded_pair_plan(ctx, M(a1), M(a2), bounds[g], bounds[g + 1],
                                                    *opts, parts, g));
    }
    std::vector<ssb::Plan*> raw;
    for (auto& p : made) raw.push_back(p.get());
    ssb::link_group(raw.data(), parts);
    for (int g = 0; g < parts; ++g) plans[g] = wrap(made[g].release());
  });
}

int ss_plan_create_sharded_x(ss_ctx_t h, ss_matrix_t a, int64_t row_begin, int64_t row_end,
                             const ss_solve_options* opts, int exchange, ss_plan_t* out) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(opts, "opts");
    need(out, "out");
    use_device(ctx);
    *out = wrap(ssb::make_sharded_plan(ctx, M(a), row_begin, row_end, *opts, exchange));
  });
}

int ss_plan_create_sharded_group(ss_ctx_t h, ss_matrix_t a, int parts, const int64_t* bounds,
                                 const ss_solve_options* opts, ss_plan_t* plans) {
  return guarded([&] {
    ssb::Context* ctx = CX(h);
    need(opts, "opts");
    need(bounds, "bounds");
    need(plans, "plans");
    if (parts < 1) ssb::fail("plan: parts must be >= 1");
    use_device(ctx);
    std::vector<std::unique_ptr<ssb::Plan>> made;
    for (int g = 0; g < parts; ++g) {
      made.emplace_back(ssb::make_sharded_plan(ctx, M(a), bounds[g], bounds[g + 1], *opts,
                                               SS_XCHG_PEER, parts, g));
    }
    std::vector<ssb::Plan*> raw;
    for (auto& p : made) raw.push_back(p.get());
    ssb::link_group(raw.data(), parts);
    for (int g = 0; g < parts; ++g) plans[g] = wrap(made[g].release());
  });
}

int ss_plan_group_run(ss_plan_t* plans, int parts) {
  return guarded([&] {
    need(plans, "plans");
    if (parts < 1) ssb::fail("plan: parts must be >= 1");
    std::vector<ssb::Plan*> raw;
    for (int g = 0; g < parts; ++g) raw.push_back(PL(plans[g]));
    use_device(raw[0]->ctx);
    ssb::run_group(raw.data(), parts);
  });
}

}  // extern "C"
