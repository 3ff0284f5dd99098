// TEST INFRASTRUCTURE ONLY (see oracle.hpp): a flat C surface over the
// oracle so pytest (ctypes) and bench.py's CPU legs can drive it.
#include <cstring>
#include <string>

#include "oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const SymmetryError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <class T>
void* guarded_ptr(T&& make) {
  try {
    return make();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

Vector vec(const double* p, std::int64_t n) { return Vector(p, p + n); }
void put(const Vector& v, double* out) {
  if (out) std::memcpy(out, v.data(), v.size() * sizeof(double));
}
}  // namespace

extern "C" {

struct or_scan_config {
  int k;
  double gamma;
  double h_e, h_m, l_m;
  int n_p;
  double a_e;
  double obj_size;
  int grid_nx, grid_ny;
};

struct or_grid {
  int n_x, n_y;
  double voxel_size, center_x, y_bottom;
};

static ScanConfig to_cfg(const or_scan_config* c) {
  ScanConfig s;
  s.geom.k = c->k;
  s.geom.gamma = c->gamma;
  s.geom.h_e = c->h_e;
  s.geom.h_m = c->h_m;
  s.geom.l_m = c->l_m;
  s.geom.n_p = c->n_p;
  s.geom.a_e = c->a_e;
  s.geom.obj_size = c->obj_size;
  s.grid_nx = c->grid_nx;
  s.grid_ny = c->grid_ny;
  return s;
}

static GridSpec to_grid(const or_grid* g) {
  GridSpec s;
  s.n_x = g->n_x;
  s.n_y = g->n_y;
  s.voxel_size = g->voxel_size;
  s.center_x = g->center_x;
  s.y_bottom = g->y_bottom;
  return s;
}

const char* or_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- matrices
void* or_mat_dense(std::int64_t rows, std::int64_t cols, const double* cm) {
  return guarded_ptr([&] {
    return new Matrix(Matrix::dense(rows, cols, vec(cm, rows * cols)));
  });
}

void* or_mat_csc(std::int64_t rows, std::int64_t cols, std::int64_t nnz,
                 const int* outer, const int* inner, const double* val) {
  return guarded_ptr([&] {
    Csc s;
    s.rows = rows;
    s.cols = cols;
    s.outer.assign(outer, outer + cols + 1);
    s.inner.assign(inner, inner + nnz);
    s.values.assign(val, val + nnz);
    return new Matrix(Matrix::sparse(std::move(s)));
  });
}

void* or_mat_triplets(std::int64_t rows, std::int64_t cols, std::int64_t n,
                      const int* r, const int* c, const double* v) {
  return guarded_ptr([&] {
    std::vector<Triplet> ts(static_cast<std::size_t>(n));
    for (std::int64_t k = 0; k < n; ++k) ts[k] = {r[k], c[k], v[k]};
    return new Matrix(Matrix::from_triplets(rows, cols, ts));
  });
}

void or_mat_free(void* m) { delete static_cast<Matrix*>(m); }

void or_mat_info(void* m, std::int64_t* rows, std::int64_t* cols,
                 std::int64_t* stored, int* is_sparse) {
  const Matrix& a = *static_cast<Matrix*>(m);
  *rows = a.rows();
  *cols = a.cols();
  *stored = a.is_sparse() ? a.csc().nnz() : a.rows() * a.cols();
  *is_sparse = a.is_sparse() ? 1 : 0;
}

std::int64_t or_mat_nonzeros(void* m) { return static_cast<Matrix*>(m)->nonzeros(); }
double or_mat_fill_ratio(void* m) { return static_cast<Matrix*>(m)->fill_ratio(); }

void or_mat_get_csc(void* m, int* outer, int* inner, double* val) {
  const Csc& s = static_cast<Matrix*>(m)->csc();
  std::memcpy(outer, s.outer.data(), s.outer.size() * sizeof(int));
  std::memcpy(inner, s.inner.data(), s.inner.size() * sizeof(int));
  std::memcpy(val, s.values.data(), s.values.size() * sizeof(double));
}

void or_mat_get_dense(void* m, double* cm) { put(static_cast<Matrix*>(m)->to_dense(), cm); }

int or_mat_apply(void* m, const double* x, double* y) {
  return guarded([&] {
    const Matrix& a = *static_cast<Matrix*>(m);
    put(a.apply(vec(x, a.cols())), y);
  });
}

int or_mat_apply_t(void* m, const double* y, double* x) {
  return guarded([&] {
    const Matrix& a = *static_cast<Matrix*>(m);
    put(a.apply_transpose(vec(y, a.rows())), x);
  });
}

double or_norm(const double* v, std::int64_t n) { return norm(vec(v, n)); }

// ---------------------------------------------------------------- CSR
void or_csr_free(void* c) { delete static_cast<Csr*>(c); }
void or_csr_info(void* c, std::int64_t* rows, std::int64_t* cols, std::int64_t* nnz) {
  const Csr& a = *static_cast<Csr*>(c);
  *rows = a.rows;
  *cols = a.cols;
  *nnz = a.nnz();
}
void or_csr_get(void* c, int* ptr, int* idx, double* val) {
  const Csr& a = *static_cast<Csr*>(c);
  std::memcpy(ptr, a.ptr.data(), a.ptr.size() * sizeof(int));
  std::memcpy(idx, a.idx.data(), a.idx.size() * sizeof(int));
  std::memcpy(val, a.values.data(), a.values.size() * sizeof(double));
}
void* or_csr_from_mat(void* m) {
  return guarded_ptr([&] { return new Csr(csc_to_csr(static_cast<Matrix*>(m)->csc())); });
}
void* or_mat_from_csr(void* c) {
  return guarded_ptr(
      [&] { return new Matrix(Matrix::sparse(csr_to_csc(*static_cast<Csr*>(c)))); });
}
void* or_csr_make(std::int64_t rows, std::int64_t cols, std::int64_t nnz, const int* ptr,
                  const int* idx, const double* val) {
  return guarded_ptr([&] {
    auto* c = new Csr();
    c->rows = rows;
    c->cols = cols;
    c->ptr.assign(ptr, ptr + rows + 1);
    c->idx.assign(idx, idx + nnz);
    c->values.assign(val, val + nnz);
    return c;
  });
}

// ---------------------------------------------------------------- centro
int or_verify_symmetry(void* m, double tol, int* holds, double* maxv, std::int64_t* wr,
                       std::int64_t* wc, int* status) {
  return guarded([&] {
    const SymmetryReport r = verify_symmetry(*static_cast<Matrix*>(m), tol);
    *holds = r.holds ? 1 : 0;
    *maxv = r.max_violation;
    *wr = r.worst_row;
    *wc = r.worst_col;
    *status = static_cast<int>(r.status);
  });
}

int or_split_system(void* m, const double* p, std::int64_t plen, double tol, void** a1,
                    void** a2, double* p1, double* p2, double* fills3, double* maxv,
                    std::int64_t* wr, std::int64_t* wc, int* status) {
  try {
    CentroSystem sys{*static_cast<Matrix*>(m), vec(p, plen), tol};
    SplitSystem s = split_system(sys);
    *a1 = new Matrix(std::move(s.a1));
    *a2 = new Matrix(std::move(s.a2));
    put(s.p1, p1);
    put(s.p2, p2);
    fills3[0] = s.parent_fill;
    fills3[1] = s.fill1;
    fills3[2] = s.fill2;
    return 0;
  } catch (const SymmetryError& e) {
    g_err = e.what();
    *maxv = e.report.max_violation;
    *wr = e.report.worst_row;
    *wc = e.report.worst_col;
    *status = static_cast<int>(e.report.status);
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int or_split_matrix(void* m, void** a1, void** a2) {
  return guarded([&] {
    auto [x, y] = split_matrix(*static_cast<Matrix*>(m));
    *a1 = new Matrix(std::move(x));
    *a2 = new Matrix(std::move(y));
  });
}

int or_split_rhs(const double* p, std::int64_t m, double* p1, double* p2) {
  return guarded([&] {
    auto [a, b] = split_rhs(vec(p, m));
    put(a, p1);
    put(b, p2);
  });
}

int or_recombine(const double* f1, std::int64_t n1, const double* f2, std::int64_t n2,
                 double* f) {
  return guarded([&] { put(recombine_solution({vec(f1, n1), vec(f2, n2)}), f); });
}

int or_decompose(const double* f, std::int64_t n, double* f1, double* f2) {
  return guarded([&] {
    SolutionPair p = decompose_solution(vec(f, n));
    put(p.f1, f1);
    put(p.f2, f2);
  });
}

void* or_reconstruct(void* a1, void* a2) {
  return guarded_ptr([&] {
    return new Matrix(reconstruct_matrix(*static_cast<Matrix*>(a1), *static_cast<Matrix*>(a2)));
  });
}

void* or_symmetrize(void* a) {
  return guarded_ptr([&] { return new Matrix(symmetrize(*static_cast<Matrix*>(a))); });
}

int or_fold_rows_csr(void* a, void** a1, void** a2) {
  return guarded([&] {
    auto* x = new Csr();
    auto* y = new Csr();
    fold_rows_csr(*static_cast<Csr*>(a), *x, *y);
    *a1 = x;
    *a2 = y;
  });
}

// ---------------------------------------------------------------- solvers
int or_sart_solve(void* m, const double* p, std::int64_t plen, int max_iters, double tol,
                  double relax, double* f, int* iters, double* resnorm, double* solnorm,
                  double* wall, double* hist, int* hist_len) {
  return guarded([&] {
    SolveOptions o;
    o.max_iters = max_iters;
    o.tol = tol;
    o.relaxation = relax;
    SolveReport r = sart_solve(*static_cast<Matrix*>(m), vec(p, plen), o);
    put(r.f, f);
    *iters = r.iterations;
    *resnorm = r.residual_norm;
    *solnorm = r.solution_norm;
    *wall = r.wall_time_seconds;
    if (hist) std::memcpy(hist, r.residual_history.data(), r.residual_history.size() * 8);
    *hist_len = static_cast<int>(r.residual_history.size());
  });
}

int or_cgls_solve(void* m, const double* p, std::int64_t plen, int max_iters, double tol,
                  double* f, int* iters, double* resnorm, double* solnorm, double* hist,
                  int* hist_len) {
  return guarded([&] {
    SolveOptions o;
    o.method = Method::cgls;
    o.max_iters = max_iters;
    o.tol = tol;
    SolveReport r = cgls_solve(*static_cast<Matrix*>(m), vec(p, plen), o);
    put(r.f, f);
    *iters = r.iterations;
    *resnorm = r.residual_norm;
    *solnorm = r.solution_norm;
    if (hist) std::memcpy(hist, r.residual_history.data(), r.residual_history.size() * 8);
    *hist_len = static_cast<int>(r.residual_history.size());
  });
}

int or_solve_split_method(void* m, const double* p, std::int64_t plen, double sym_tol,
                          int method, int max_iters, double tol, double relax, double* f,
                          int* iters, double* resnorm) {
  return guarded([&] {
    SolveOptions o;
    o.method = method == 1 ? Method::cgls : Method::sart;
    o.max_iters = max_iters;
    o.tol = tol;
    o.relaxation = relax;
    CentroSystem sys{*static_cast<Matrix*>(m), vec(p, plen), sym_tol};
    SolveReport r = solve_split_sart(sys, o);
    put(r.f, f);
    *iters = r.iterations;
    *resnorm = r.residual_norm;
  });
}

int or_solve_split(void* m, const double* p, std::int64_t plen, double sym_tol, int max_iters,
                   double tol, double relax, int parallelism, double* f, int* iters,
                   double* resnorm, double* solnorm, double* wall, double* times4) {
  return guarded([&] {
    SolveOptions o;
    o.max_iters = max_iters;
    o.tol = tol;
    o.relaxation = relax;
    o.parallelism = parallelism;
    CentroSystem sys{*static_cast<Matrix*>(m), vec(p, plen), sym_tol};
    SolveReport r = solve_split_sart(sys, o);
    put(r.f, f);
    *iters = r.iterations;
    *resnorm = r.residual_norm;
    *solnorm = r.solution_norm;
    *wall = r.wall_time_seconds;
    times4[0] = r.split_seconds;
    times4[1] = r.recombine_seconds;
    times4[2] = r.branch1_seconds;
    times4[3] = r.branch2_seconds;
  });
}

// Branch solves on an already folded pair (CPU baseline: times only the
// SART loops, like the reference's branch wall times).
int or_solve_split_prepared(void* a1, void* a2, const double* p1, const double* p2,
                            int max_iters, double tol, double relax, int parallel, double* f,
                            int* iters, double* times4) {
  return guarded([&] {
    SplitSystem ss{*static_cast<Matrix*>(a1), vec(p1, static_cast<Matrix*>(a1)->rows()),
                   *static_cast<Matrix*>(a2), vec(p2, static_cast<Matrix*>(a2)->rows())};
    SolveOptions o;
    o.max_iters = max_iters;
    o.tol = tol;
    o.relaxation = relax;
    SolveReport r = solve_split_prepared(ss, o, parallel != 0);
    put(r.f, f);
    *iters = r.iterations;
    times4[0] = 0.0;
    times4[1] = r.recombine_seconds;
    times4[2] = r.branch1_seconds;
    times4[3] = r.branch2_seconds;
  });
}

// ---------------------------------------------------------------- geometry
int or_parse_scan_config(const char* text, or_scan_config* out) {
  return guarded([&] {
    ScanConfig c = parse_scan_config(text);
    out->k = c.geom.k;
    out->gamma = c.geom.gamma;
    out->h_e = c.geom.h_e;
    out->h_m = c.geom.h_m;
    out->l_m = c.geom.l_m;
    out->n_p = c.geom.n_p;
    out->a_e = c.geom.a_e;
    out->obj_size = c.geom.obj_size;
    out->grid_nx = c.grid_nx;
    out->grid_ny = c.grid_ny;
  });
}

int or_make_grid(const or_scan_config* c, or_grid* g) {
  return guarded([&] {
    GridSpec s = make_grid(to_cfg(c));
    g->n_x = s.n_x;
    g->n_y = s.n_y;
    g->voxel_size = s.voxel_size;
    g->center_x = s.center_x;
    g->y_bottom = s.y_bottom;
  });
}

int or_snake_index(int c, int r, const or_grid* g, int* j) {
  return guarded([&] { *j = snake_index(c, r, to_grid(g)); });
}

int or_snake_inverse(int j, const or_grid* g, int* c, int* r) {
  return guarded([&] {
    auto [a, b] = snake_inverse(j, to_grid(g));
    *c = a;
    *r = b;
  });
}

int or_emitter_angles(const or_scan_config* c, double* out) {
  return guarded([&] { put(emitter_angles(to_cfg(c).geom), out); });
}

int or_emitter_positions(const or_scan_config* c, double center_x, double* out2) {
  return guarded([&] {
    auto s = emitter_positions(to_cfg(c).geom, center_x);
    for (std::size_t i = 0; i < s.size(); ++i) {
      out2[2 * i] = s[i].x;
      out2[2 * i + 1] = s[i].y;
    }
  });
}

// rays as (sx, sy, dx, dy) rows; pass out4 = nullptr to query the count.
int or_enumerate_rays(const or_scan_config* c, const or_grid* g, double* out4,
                      std::int64_t* count, int* samples, double* pitch) {
  return guarded([&] {
    RaySet rs = enumerate_rays(to_cfg(c).geom, to_grid(g));
    *count = rs.count();
    *samples = rs.samples_per_position;
    *pitch = rs.sample_pitch;
    if (out4) {
      for (std::int64_t i = 0; i < rs.count(); ++i) {
        out4[4 * i] = rs.rays[i].source.x;
        out4[4 * i + 1] = rs.rays[i].source.y;
        out4[4 * i + 2] = rs.rays[i].detector.x;
        out4[4 * i + 3] = rs.rays[i].detector.y;
      }
    }
  });
}

int or_ray_weights(const double* ray4, const or_grid* g, int* js, double* lens,
                   std::int64_t cap, std::int64_t* count) {
  return guarded([&] {
    Ray r{{ray4[0], ray4[1]}, {ray4[2], ray4[3]}};
    auto w = ray_weights(r, to_grid(g));
    *count = static_cast<std::int64_t>(w.size());
    for (std::int64_t k = 0; k < *count && k < cap; ++k) {
      js[k] = w[k].first;
      lens[k] = w[k].second;
    }
  });
}

void* or_build_system(const or_scan_config* c, int parallelism) {
  return guarded_ptr([&] {
    ScanConfig s = to_cfg(c);
    CentroSystem sys = build_system(s.geom, make_grid(s), parallelism);
    return new Matrix(std::move(sys.a));
  });
}

void* or_build_traced_csr(const or_scan_config* c, int parallelism) {
  return guarded_ptr([&] {
    ScanConfig s = to_cfg(c);
    return new Csr(build_traced_csr(s.geom, make_grid(s), parallelism));
  });
}

void* or_full_csr_from_traced(void* traced, std::int64_t m, std::int64_t n) {
  return guarded_ptr(
      [&] { return new Csr(full_csr_from_traced(*static_cast<Csr*>(traced), m, n)); });
}

// ---------------------------------------------------------------- phantom
int or_random_ellipses(std::uint64_t seed, int count, double* out6) {
  return guarded([&] {
    auto es = random_ellipses(seed, count);
    for (int i = 0; i < count; ++i) {
      const double v[6] = {es[i].x0, es[i].y0, es[i].a, es[i].b, es[i].angle, es[i].density};
      std::memcpy(out6 + 6 * i, v, sizeof v);
    }
  });
}

int or_shepp_logan(double* out6) {
  return guarded([&] {
    auto es = shepp_logan_ellipses();
    for (std::size_t i = 0; i < es.size(); ++i) {
      const double v[6] = {es[i].x0, es[i].y0, es[i].a, es[i].b, es[i].angle, es[i].density};
      std::memcpy(out6 + 6 * i, v, sizeof v);
    }
  });
}

int or_rasterize(const double* ell6, int count, const or_grid* g, double* values) {
  return guarded([&] {
    std::vector<Ellipse> es(static_cast<std::size_t>(count));
    for (int i = 0; i < count; ++i) {
      const double* v = ell6 + 6 * i;
      es[i] = Ellipse{v[0], v[1], v[2], v[3], v[4], v[5]};
    }
    put(rasterize(es, to_grid(g)), values);
  });
}

int or_forward_project(void* m, const double* f, std::int64_t n, double* p) {
  return guarded([&] {
    const Matrix& a = *static_cast<Matrix*>(m);
    put(forward_project(a, vec(f, n)), p);
  });
}

int or_forward_project_csr(void* c, const double* f, double* p) {
  return guarded([&] {
    const Csr& a = *static_cast<Csr*>(c);
    put(forward_project_csr(a, vec(f, a.cols)), p);
  });
}

int or_add_noise(double* p, std::int64_t m, double sigma, std::uint64_t seed) {
  return guarded([&] {
    Vector v = vec(p, m);
    add_noise(v, sigma, seed);
    put(v, p);
  });
}

// Rng stream for fixtures (reference tests/support/oracles.hpp:29-50).
int or_rng_uniform(std::uint64_t seed, std::int64_t n, double lo, double hi, double* out) {
  return guarded([&] {
    Rng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
  });
}

}  // extern "C"
