// C++ facade of symsplit_b200 with the reference's API shape
// (/root/reference/proj/include/symsplit/{matrix,centro,geometry,solvers}.hpp):
// the same function names, argument meaning and exception types
// (symsplit::Error, symsplit::SymmetryError), over the C ABI in
// symsplit_b200.h. Header-only; link against libsymsplit_b200.so.
//
// Differences from the reference, all deliberate:
//  * Eigen types are replaced by Eigen-free equivalents: Vector is
//    std::vector<double>; Matrix is a device-resident sparse matrix handle
//    (construct from compressed-column arrays, triplets or a dense
//    column-major array);
//  * Method::sart (the default here; the reference defaults to dense_minnorm),
//    Method::cgls and Method::dense_minnorm all run on the device;
//    SolveOptions gains `dtype` (fp64 = reference arithmetic, fp32 = the
//    bandwidth-halving variant; SART only);
//  * every call runs on the GPU of the Context it was created on.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "symsplit_b200.h"

namespace symsplit {

using Index = std::int64_t;
using Vector = std::vector<double>;

// reference matrix.hpp:22-25
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

enum class SymmetryStatus { ok = 0, odd_row_count = 1, odd_col_count = 2 };

// reference centro.hpp:16-22
struct SymmetryReport {
  bool holds = false;
  double max_violation = 0.0;
  Index worst_row = 1;
  Index worst_col = 1;
  SymmetryStatus status = SymmetryStatus::ok;
};

// reference centro.hpp:73-78
class SymmetryError : public Error {
 public:
  SymmetryError(const std::string& what, SymmetryReport r) : Error(what), report(r) {}
  SymmetryReport report;
};

// reference io.hpp:14-20 (path/line are part of the message here)
class IoError : public Error {
 public:
  using Error::Error;
};

namespace detail {
inline SymmetryReport to_report(const ss_symmetry_report& r) {
  return SymmetryReport{r.holds != 0, r.max_violation, r.worst_row, r.worst_col,
                        static_cast<SymmetryStatus>(r.status)};
}
inline void check(int rc, const ss_symmetry_report* rep = nullptr) {
  if (rc == SS_OK) return;
  const std::string msg = ss_last_error();
  if (rc == SS_ERR_SYMMETRY) {
    throw SymmetryError(msg, rep ? to_report(*rep) : SymmetryReport{});
  }
  if (rc == SS_ERR_IO) throw IoError(msg);
  throw Error(msg);
}
}  // namespace detail

// One CUDA stream + workspace on one device.
class Context {
 public:
  explicit Context(int device = 0) {
    ss_ctx_t h = nullptr;
    detail::check(ss_ctx_create(device, &h));
    h_.reset(h, [](ss_ctx_t c) { ss_ctx_destroy(c); });
  }
  ss_ctx_t get() const { return h_.get(); }
  static Context& default_context() {
    static Context ctx(0);
    return ctx;
  }

 private:
  std::shared_ptr<ss_context> h_;
};

// reference DenseStorage (Eigen::MatrixXd): column-major, 0-based (i, j)
struct DenseStorage {
  Index r = 0, c = 0;
  Vector data;  // column-major
  DenseStorage() = default;
  DenseStorage(Index rows, Index cols)
      : r(rows), c(cols), data(static_cast<std::size_t>(rows * cols), 0.0) {}
  Index rows() const { return r; }
  Index cols() const { return c; }
  double& operator()(Index i, Index j) { return data[static_cast<std::size_t>(j * r + i)]; }
  double operator()(Index i, Index j) const { return data[static_cast<std::size_t>(j * r + i)]; }
};

// reference matrix.hpp:34-87 (device sparse storage only)
class Matrix {
 public:
  Matrix() = default;
  explicit Matrix(ss_matrix_t h) : h_(h, [](ss_matrix_t m) { ss_matrix_destroy(m); }) {}

  static Matrix from_csc(Index rows, Index cols, const std::vector<int32_t>& outer,
                         const std::vector<int32_t>& inner, const Vector& values,
                         const Context& ctx = Context::default_context()) {
    ss_matrix_t h = nullptr;
    detail::check(ss_matrix_from_csc(ctx.get(), rows, cols, static_cast<int64_t>(values.size()),
                                     outer.data(), inner.data(), values.data(), &h));
    return Matrix(h);
  }
  struct Triplet {
    int32_t row, col;
    double value;
  };
  // Matrix::from_triplets (matrix.cpp:12-18): repeats summed in order
  static Matrix from_triplets(Index rows, Index cols, const std::vector<Triplet>& ts,
                              const Context& ctx = Context::default_context()) {
    std::vector<int32_t> r(ts.size()), c(ts.size());
    Vector v(ts.size());
    for (std::size_t k = 0; k < ts.size(); ++k) {
      r[k] = ts[k].row;
      c[k] = ts[k].col;
      v[k] = ts[k].value;
    }
    ss_matrix_t h = nullptr;
    detail::check(ss_matrix_from_triplets(ctx.get(), rows, cols, static_cast<int64_t>(ts.size()),
                                          r.data(), c.data(), v.data(), &h));
    return Matrix(h);
  }
  // Dense column-major data; nonzeros are stored.
  static Matrix dense(Index rows, Index cols, const Vector& colmajor,
                      const Context& ctx = Context::default_context()) {
    std::vector<Triplet> ts;
    for (Index j = 0; j < cols; ++j) {
      for (Index i = 0; i < rows; ++i) {
        const double v = colmajor[static_cast<std::size_t>(j * rows + i)];
        if (v != 0.0) ts.push_back({static_cast<int32_t>(i), static_cast<int32_t>(j), v});
      }
    }
    return from_triplets(rows, cols, ts, ctx);
  }

  Index rows() const { return shape().first; }
  Index cols() const { return shape().second; }
  std::pair<Index, Index> shape() const {
    int64_t r = 0, c = 0, s = 0;
    detail::check(ss_matrix_shape(h_.get(), &r, &c, &s));
    return {r, c};
  }
  std::int64_t stored() const {
    int64_t r = 0, c = 0, s = 0;
    detail::check(ss_matrix_shape(h_.get(), &r, &c, &s));
    return s;
  }
  std::int64_t nonzeros() const {
    int64_t n = 0;
    detail::check(ss_matrix_nonzeros(h_.get(), &n));
    return n;
  }
  double fill_ratio() const {
    double f = 0.0;
    detail::check(ss_matrix_fill_ratio(h_.get(), &f));
    return f;
  }
  Vector apply(const Vector& x) const {
    if (static_cast<Index>(x.size()) != cols()) throw Error("matrix-vector size mismatch");
    Vector y(static_cast<std::size_t>(rows()));
    detail::check(ss_matrix_apply(h_.get(), x.data(), y.data()));
    return y;
  }
  Vector apply_transpose(const Vector& y) const {
    if (static_cast<Index>(y.size()) != rows()) throw Error("matrix-vector size mismatch");
    Vector x(static_cast<std::size_t>(cols()));
    detail::check(ss_matrix_apply_transpose(h_.get(), y.data(), x.data()));
    return x;
  }
  bool is_sparse() const { return true; }  // device storage is always compressed
  // reference matrix.cpp:44-50
  double coeff(Index i, Index j) const {
    double v = 0.0;
    detail::check(ss_matrix_coeff(h_.get(), i, j, &v));
    return v;
  }
  // reference matrix.hpp:76-87: every stored entry as f(row, col, value) in
  // compressed-column order (the order Eigen's InnerIterator visits)
  template <class F>
  void for_each(F&& f) const {
    std::vector<int32_t> outer, inner;
    Vector values;
    to_csc(outer, inner, values);
    for (Index j = 0; j + 1 < static_cast<Index>(outer.size()); ++j) {
      for (int32_t k = outer[static_cast<std::size_t>(j)];
           k < outer[static_cast<std::size_t>(j) + 1]; ++k) {
        f(static_cast<Index>(inner[static_cast<std::size_t>(k)]), j,
          values[static_cast<std::size_t>(k)]);
      }
    }
  }
  // reference matrix.cpp:52-55 (DenseStorage: column-major rows x cols)
  DenseStorage to_dense() const;
  // CSC download (reference Eigen compressed storage): outer, inner, values
  void to_csc(std::vector<int32_t>& outer, std::vector<int32_t>& inner, Vector& values) const {
    outer.resize(static_cast<std::size_t>(cols() + 1));
    inner.resize(static_cast<std::size_t>(stored()));
    values.resize(static_cast<std::size_t>(stored()));
    detail::check(ss_matrix_download_csc(h_.get(), outer.data(), inner.data(), values.data()));
  }
  ss_matrix_t get() const { return h_.get(); }

 private:
  std::shared_ptr<ss_matrix> h_;
};

inline DenseStorage Matrix::to_dense() const {
  const auto [m, n] = shape();
  DenseStorage d(m, n);
  for_each([&](Index i, Index j, double v) { d(i, j) = v; });
  return d;
}

// reference centro.hpp:24-51
struct CentroSystem {
  Matrix a;
  Vector p;
  double symmetry_tol = 1e-12;
};

struct SplitSystem {
  Matrix a1;
  Vector p1;
  Matrix a2;
  Vector p2;
  double parent_fill = 0.0;
  double fill1 = 0.0;
  double fill2 = 0.0;
};

struct SolutionPair {
  Vector f1;
  Vector f2;
};

enum class Method { dense_minnorm, cgls, sart };
enum class Mode { direct, split };

// reference solvers.hpp:19-27
struct SolveOptions {
  Method method = Method::sart;
  int max_iters = 200;
  double tol = 1e-10;
  double relaxation = 1.0;
  bool deterministic = true;
  int parallelism = 0;
  std::int64_t dense_cap = 50'000'000;
  int dtype = SS_F64;  // B200 addition: SS_F64 or SS_F32
};

// reference solvers.hpp:29-45
struct SolveReport {
  Vector f;
  double residual_norm = 0.0;
  double solution_norm = 0.0;
  int iterations = 0;
  double wall_time_seconds = 0.0;
  Method method = Method::sart;
  Mode mode = Mode::direct;
  std::vector<double> residual_history;
  double split_seconds = 0.0;
  double recombine_seconds = 0.0;
  double branch1_seconds = 0.0;
  double branch2_seconds = 0.0;
};

namespace detail {
inline ss_solve_options to_c(const SolveOptions& o) {
  const int m = o.method == Method::cgls ? SS_METHOD_CGLS
                                         : (o.method == Method::dense_minnorm ? SS_METHOD_DENSE
                                                                              : SS_METHOD_SART);
  return ss_solve_options{o.max_iters, o.tol, o.relaxation, o.parallelism, o.dtype, m,
                          o.dense_cap};
}
inline SolveReport from_c(Vector f, const ss_solve_report& r, Mode mode) {
  SolveReport rep;
  rep.f = std::move(f);
  rep.residual_norm = r.residual_norm;
  rep.solution_norm = r.solution_norm;
  rep.iterations = r.iterations;
  rep.wall_time_seconds = r.wall_time_seconds;
  rep.mode = mode;
  rep.split_seconds = r.split_seconds;
  rep.recombine_seconds = r.recombine_seconds;
  rep.branch1_seconds = r.branch1_seconds;
  rep.branch2_seconds = r.branch2_seconds;
  return rep;
}
}  // namespace detail

// ------------------------------------------------------------------ centro
inline SymmetryReport verify_symmetry(const Matrix& a, double tol) {
  ss_symmetry_report r{};
  detail::check(ss_verify_symmetry(a.get(), tol, &r));
  return detail::to_report(r);
}

inline std::pair<Vector, Vector> split_rhs(const Vector& p,
                                           const Context& ctx = Context::default_context()) {
  Vector p1(p.size() / 2), p2(p.size() / 2);
  detail::check(ss_split_rhs(ctx.get(), p.data(), static_cast<int64_t>(p.size()), p1.data(),
                             p2.data()));
  return {std::move(p1), std::move(p2)};
}

inline SplitSystem split_system(const CentroSystem& sys) {
  const std::size_t mh = sys.p.size() / 2;
  SplitSystem out;
  out.p1.resize(mh);
  out.p2.resize(mh);
  ss_matrix_t a1 = nullptr, a2 = nullptr;
  double fills[3] = {0, 0, 0};
  ss_symmetry_report rep{};
  detail::check(ss_split_system(sys.a.get(), sys.p.data(), static_cast<int64_t>(sys.p.size()),
                                sys.symmetry_tol, &a1, &a2, out.p1.data(), out.p2.data(), fills,
                                &rep),
                &rep);
  out.a1 = Matrix(a1);
  out.a2 = Matrix(a2);
  out.parent_fill = fills[0];
  out.fill1 = fills[1];
  out.fill2 = fills[2];
  return out;
}

inline SolutionPair decompose_solution(const Vector& f,
                                       const Context& ctx = Context::default_context()) {
  SolutionPair s{Vector(f.size() / 2), Vector(f.size() / 2)};
  detail::check(ss_decompose_solution(ctx.get(), f.data(), static_cast<int64_t>(f.size()),
                                      s.f1.data(), s.f2.data()));
  return s;
}

inline Vector recombine_solution(const SolutionPair& pair,
                                 const Context& ctx = Context::default_context()) {
  if (pair.f1.size() != pair.f2.size()) {
    throw Error("recombine_solution: component lengths differ");
  }
  Vector f(2 * pair.f1.size());
  detail::check(ss_recombine_solution(ctx.get(), pair.f1.data(), pair.f2.data(),
                                      static_cast<int64_t>(pair.f1.size()), f.data()));
  return f;
}

// ------------------------------------------------------------------ solvers
inline SolveReport sart_solve(const Matrix& a, const Vector& p, const SolveOptions& opts) {
  const ss_solve_options o = detail::to_c(opts);
  Vector f(static_cast<std::size_t>(a.cols()));
  Vector hist(static_cast<std::size_t>(opts.max_iters > 0 ? opts.max_iters + 1 : 1));
  ss_solve_report r{};
  detail::check(ss_sart_solve(a.get(), p.data(), static_cast<int64_t>(p.size()), &o, f.data(),
                              static_cast<int64_t>(f.size()), &r, hist.data()));
  SolveReport rep = detail::from_c(std::move(f), r, Mode::direct);
  rep.residual_history.assign(hist.begin(), hist.begin() + r.history_len);
  return rep;
}

// reference solvers.cpp:99-146
inline SolveReport cgls_solve(const Matrix& a, const Vector& p, const SolveOptions& opts) {
  SolveOptions o = opts;
  o.method = Method::cgls;
  const ss_solve_options c = detail::to_c(o);
  Vector f(static_cast<std::size_t>(a.cols()));
  Vector hist(static_cast<std::size_t>(opts.max_iters > 0 ? opts.max_iters + 1 : 1));
  ss_solve_report r{};
  detail::check(ss_cgls_solve(a.get(), p.data(), static_cast<int64_t>(p.size()), &c, f.data(),
                              static_cast<int64_t>(f.size()), &r, hist.data()));
  SolveReport rep = detail::from_c(std::move(f), r, Mode::direct);
  rep.method = Method::cgls;
  rep.residual_history.assign(hist.begin(), hist.begin() + r.history_len);
  return rep;
}

// reference pseudo_solve_dense (solvers.cpp:81-97)
inline Vector pseudo_solve_dense(const Matrix& a, const Vector& p,
                                 std::int64_t dense_cap = 50'000'000) {
  Vector f(static_cast<std::size_t>(a.cols()));
  detail::check(ss_pseudo_solve_dense(a.get(), p.data(), static_cast<int64_t>(p.size()),
                                      dense_cap, f.data(), static_cast<int64_t>(f.size())));
  return f;
}

inline SolveReport solve_direct(const CentroSystem& sys, const SolveOptions& opts) {
  if (opts.method == Method::cgls) return cgls_solve(sys.a, sys.p, opts);
  if (opts.method == Method::dense_minnorm) {
    const ss_solve_options c = detail::to_c(opts);
    Vector f(static_cast<std::size_t>(sys.a.cols()));
    ss_solve_report r{};
    detail::check(ss_solve_direct(sys.a.get(), sys.p.data(), static_cast<int64_t>(sys.p.size()),
                                  &c, f.data(), static_cast<int64_t>(f.size()), &r));
    SolveReport rep = detail::from_c(std::move(f), r, Mode::direct);
    rep.method = Method::dense_minnorm;
    return rep;
  }
  return sart_solve(sys.a, sys.p, opts);
}

inline SolveReport solve_split(const CentroSystem& sys, const SolveOptions& opts) {
  const ss_solve_options o = detail::to_c(opts);
  Vector f(static_cast<std::size_t>(sys.a.cols()));
  ss_solve_report r{};
  const int rc = ss_solve_split(sys.a.get(), sys.p.data(), static_cast<int64_t>(sys.p.size()),
                                sys.symmetry_tol, &o, f.data(), static_cast<int64_t>(f.size()),
                                &r);
  if (rc == SS_ERR_SYMMETRY) {
    // the SymmetryError carries its report (reference centro.cpp:144-156)
    const std::string msg = ss_last_error();
    ss_symmetry_report sr{};
    ss_verify_symmetry(sys.a.get(), sys.symmetry_tol, &sr);
    throw SymmetryError(msg, detail::to_report(sr));
  }
  detail::check(rc);
  SolveReport rep = detail::from_c(std::move(f), r, Mode::split);
  rep.method = opts.method;
  return rep;
}

// ------------------------------------------------------------------ geometry
inline constexpr double kPi = 3.14159265358979323846;
inline constexpr double degrees_to_radians(double deg) { return deg * kPi / 180.0; }

// reference geometry.hpp:22-37 (GridSpec): same fields, defaults and helpers
struct GridSpec {
  int n_x = 32;
  int n_y = 32;
  double voxel_size = 0.1 / 32;
  double center_x = 0.0;
  double y_bottom = 0.25;

  int cell_count() const { return n_x * n_y; }
  double width() const { return n_x * voxel_size; }
  double height() const { return n_y * voxel_size; }
  double x_left() const { return center_x - 0.5 * width(); }
  double x_right() const { return center_x + 0.5 * width(); }
  double y_top() const { return y_bottom + height(); }
  // reference geometry.cpp:59-66
  std::pair<double, double> cell_center(int c, int r) const {
    if (c < 1 || c > n_x || r < 1 || r > n_y) throw Error("cell_center: cell index out of range");
    return {center_x + (c - 0.5 - 0.5 * n_x) * voxel_size,
            y_bottom + (n_y - r + 0.5) * voxel_size};
  }
  // reference geometry.cpp:68-74
  void validate() const {
    if (n_x < 2 || n_x % 2 != 0) throw Error("grid: n_x must be even and positive (mirror pairing)");
    if (n_y < 1) throw Error("grid: n_y must be positive");
    if (!(voxel_size > 0)) throw Error("grid: voxel_size must be positive");
  }
  ss_grid_spec c() const { return ss_grid_spec{n_x, n_y, voxel_size, center_x, y_bottom}; }
};

// reference geometry.hpp:57-68 (ScanGeometry): same fields and defaults
struct ScanGeometry {
  int k = 24;
  double gamma = degrees_to_radians(30.0);  // radians
  double h_e = 1.0;
  double h_m = 0.25;
  double l_m = 0.43;
  int n_p = 1024;
  double a_e = 7e-4;
  double obj_size = 0.1;

  // the C ABI's geometry record (its grid_nx / grid_ny are not read where a
  // GridSpec is passed alongside)
  ss_scan_config c(int grid_nx = 32, int grid_ny = 32) const {
    return ss_scan_config{k, gamma, h_e, h_m, l_m, n_p, a_e, obj_size, grid_nx, grid_ny};
  }
  // reference geometry.cpp:94-105 (the same checks, messages and order)
  void validate() const {
    std::vector<double> a(static_cast<std::size_t>(k > 0 ? k : 0) + 1);
    const ss_scan_config cc = c();
    detail::check(ss_emitter_angles(&cc, a.data()));
  }
};

// reference geometry.hpp:137-141 (ScanConfig)
struct ScanConfig {
  ScanGeometry geom;
  int grid_nx = 32;
  int grid_ny = 32;

  ss_scan_config c() const { return geom.c(grid_nx, grid_ny); }
  static ScanConfig from_c(const ss_scan_config& s) {
    ScanConfig o;
    o.geom = ScanGeometry{s.k, s.gamma, s.h_e, s.h_m, s.l_m, s.n_p, s.a_e, s.obj_size};
    o.grid_nx = s.grid_nx;
    o.grid_ny = s.grid_ny;
    return o;
  }
};

// reference geometry.cpp:352-401
inline ScanConfig parse_scan_config(const std::string& text) {
  ss_scan_config c{};
  detail::check(ss_parse_scan_config(text.c_str(), &c));
  return ScanConfig::from_c(c);
}

// reference geometry.cpp:403-411
inline GridSpec make_grid(const ScanConfig& c) {
  const ss_scan_config cc = c.c();
  ss_grid_spec g{};
  detail::check(ss_make_grid(&cc, &g));
  return GridSpec{g.n_x, g.n_y, g.voxel_size, g.center_x, g.y_bottom};
}

// reference geometry.cpp:76-92 (1-based)
inline int snake_index(int c, int r, const GridSpec& g) {
  const ss_grid_spec gc = g.c();
  int j = 0;
  detail::check(ss_snake_index(c, r, &gc, &j));
  return j;
}
inline std::pair<int, int> snake_inverse(int j, const GridSpec& g) {
  const ss_grid_spec gc = g.c();
  int c = 0, r = 0;
  detail::check(ss_snake_inverse(j, &gc, &c, &r));
  return {c, r};
}

// reference geometry.hpp:74-88 (Point, Ray, RaySet)
struct Point {
  double x = 0.0, y = 0.0;
};
struct Ray {
  Point source, detector;
};
struct RaySet {
  std::vector<Ray> rays;
  int positions = 0;
  int samples_per_position = 0;
  double sample_pitch = 0.0;
  Index count() const { return static_cast<Index>(rays.size()); }
};

// reference geometry.cpp:107-117
inline std::vector<double> emitter_angles(const ScanGeometry& geom) {
  std::vector<double> a(static_cast<std::size_t>(geom.k > 0 ? geom.k : 0));
  const ss_scan_config c = geom.c();
  detail::check(ss_emitter_angles(&c, a.data()));
  return a;
}

// reference geometry.cpp:119-130
inline std::vector<Point> emitter_positions(const ScanGeometry& geom, double center_x = 0.0) {
  std::vector<double> xy(2 * static_cast<std::size_t>(geom.k > 0 ? geom.k : 0));
  const ss_scan_config c = geom.c();
  detail::check(ss_emitter_positions(&c, center_x, xy.data()));
  std::vector<Point> out(xy.size() / 2);
  for (std::size_t i = 0; i < out.size(); ++i) out[i] = Point{xy[2 * i], xy[2 * i + 1]};
  return out;
}

// reference geometry.cpp:132-173: traced half then the reversed mirror half
inline RaySet enumerate_rays(const ScanGeometry& geom, const GridSpec& grid) {
  const ss_scan_config c = geom.c();
  const ss_grid_spec g = grid.c();
  int64_t n = 0;
  int samples = 0;
  double pitch = 0.0;
  detail::check(ss_enumerate_rays_grid(&c, &g, nullptr, &n, &samples, &pitch));
  std::vector<double> r4(4 * static_cast<std::size_t>(n));
  detail::check(ss_enumerate_rays_grid(&c, &g, r4.data(), &n, &samples, &pitch));
  RaySet out;
  out.rays.resize(static_cast<std::size_t>(n));
  for (std::size_t i = 0; i < out.rays.size(); ++i) {
    out.rays[i] = Ray{{r4[4 * i], r4[4 * i + 1]}, {r4[4 * i + 2], r4[4 * i + 3]}};
  }
  out.positions = geom.k;
  out.samples_per_position = samples;
  out.sample_pitch = pitch;
  return out;
}

// reference geometry.cpp:175-225 (1-based snake columns, path order), device tracer
inline std::vector<std::pair<int, double>> ray_weights(
    const Ray& ray, const GridSpec& grid, const Context& ctx = Context::default_context()) {
  const double r4[4] = {ray.source.x, ray.source.y, ray.detector.x, ray.detector.y};
  const ss_grid_spec g = grid.c();
  int64_t n = 0;
  detail::check(ss_ray_weights(ctx.get(), r4, &g, 0, nullptr, nullptr, &n));
  std::vector<int> cols(static_cast<std::size_t>(n));
  Vector lens(static_cast<std::size_t>(n));
  detail::check(ss_ray_weights(ctx.get(), r4, &g, n, cols.data(), lens.data(), &n));
  std::vector<std::pair<int, double>> out(cols.size());
  for (std::size_t q = 0; q < cols.size(); ++q) out[q] = {cols[q], lens[q]};
  return out;
}

// reference geometry.hpp:118 / geometry.cpp:227-275: A on the GPU (traced
// half + mirror rows), p = 0, symmetry_tol = 0. `parallelism` is accepted for
// parity; the device build is identical for any value.
inline CentroSystem build_system(const ScanGeometry& geom, const GridSpec& grid,
                                 int parallelism = 0,
                                 const Context& ctx = Context::default_context()) {
  const ss_scan_config c = geom.c();
  const ss_grid_spec g = grid.c();
  ss_matrix_t h = nullptr;
  detail::check(ss_build_system_grid(ctx.get(), &c, &g, parallelism, &h));
  CentroSystem sys{Matrix(h), {}, 0.0};
  sys.p.assign(static_cast<std::size_t>(sys.a.rows()), 0.0);
  return sys;
}

// convenience: the grid of a whole scan configuration (make_grid(cfg))
inline CentroSystem build_system(const ScanConfig& cfg, int parallelism = 0,
                                 const Context& ctx = Context::default_context()) {
  return build_system(cfg.geom, make_grid(cfg), parallelism, ctx);
}

// ------------------------------------------------------------------ file formats
// reference io.hpp:22-36
inline Matrix read_matrix_market(const std::string& path,
                                 const Context& ctx = Context::default_context()) {
  ss_matrix_t h = nullptr;
  detail::check(ss_read_matrix_market(ctx.get(), path.c_str(), &h));
  return Matrix(h);
}

inline void write_matrix_market(const Matrix& a, const std::string& path) {
  detail::check(ss_write_matrix_market(a.get(), path.c_str()));
}

inline Vector read_vector_csv(const std::string& path) {
  int64_t n = 0;
  detail::check(ss_read_vector_csv(path.c_str(), nullptr, 0, &n));
  Vector v(static_cast<std::size_t>(n));
  detail::check(ss_read_vector_csv(path.c_str(), v.data(), n, &n));
  return v;
}

inline void write_vector_csv(const Vector& v, const std::string& path) {
  detail::check(ss_write_vector_csv(path.c_str(), v.data(), static_cast<int64_t>(v.size())));
}

// ------------------------------------------------------------------ phantom
// reference phantom.hpp:16-27 (Ellipse); contains() is host-side libm as in
// phantom.cpp:8-16 (the device rasterizer uses host-computed sin/cos too)
struct Ellipse {
  double x0 = 0.0;
  double y0 = 0.0;
  double a = 1.0;
  double b = 1.0;
  double angle = 0.0;
  double density = 0.0;
  bool contains(double x, double y) const {
    const double dx = x - x0, dy = y - y0;
    const double ca = std::cos(angle), sa = std::sin(angle);
    const double u = (dx * ca + dy * sa) / a;
    const double v = (-dx * sa + dy * ca) / b;
    return u * u + v * v <= 1.0;
  }
};

// reference phantom.cpp:18-32
inline std::vector<Ellipse> shepp_logan_ellipses() {
  const auto deg = [](double d) { return degrees_to_radians(d); };
  return {{0.0, 0.0, 0.69, 0.92, deg(0.0), 2.0},
          {0.0, -0.0184, 0.6624, 0.874, deg(0.0), -0.98},
          {0.22, 0.0, 0.11, 0.31, deg(-18.0), -0.02},
          {-0.22, 0.0, 0.16, 0.41, deg(18.0), -0.02},
          {0.0, 0.35, 0.21, 0.25, deg(0.0), 0.01},
          {0.0, 0.1, 0.046, 0.046, deg(0.0), 0.01},
          {0.0, -0.1, 0.046, 0.046, deg(0.0), 0.01},
          {-0.08, -0.605, 0.046, 0.023, deg(0.0), 0.01},
          {0.0, -0.606, 0.023, 0.023, deg(0.0), 0.01},
          {0.06, -0.605, 0.023, 0.046, deg(0.0), 0.01}};
}

// reference phantom.hpp:31-36
struct PhantomImage {
  GridSpec grid;
  Vector values;  // length grid.cell_count(), snake order
  double min_value = 0.0;
  double max_value = 0.0;
};

// reference phantom.cpp:34-58, rasterized on the device
inline PhantomImage rasterize(const std::vector<Ellipse>& ellipses, const GridSpec& grid,
                              const Context& ctx = Context::default_context()) {
  grid.validate();
  std::vector<double> e6;
  e6.reserve(6 * ellipses.size());
  for (const Ellipse& e : ellipses) e6.insert(e6.end(), {e.x0, e.y0, e.a, e.b, e.angle, e.density});
  PhantomImage img;
  img.grid = grid;
  img.values.assign(static_cast<std::size_t>(grid.cell_count()), 0.0);
  const ss_grid_spec g = grid.c();
  detail::check(ss_rasterize(ctx.get(), e6.data(), static_cast<int>(ellipses.size()), &g,
                             img.values.data()));
  if (!img.values.empty()) {
    img.min_value = *std::min_element(img.values.begin(), img.values.end());
    img.max_value = *std::max_element(img.values.begin(), img.values.end());
  }
  return img;
}

inline Vector forward_project(const Matrix& a, const Vector& f, double noise_sigma = 0.0,
                              std::uint64_t seed = 0) {
  if (static_cast<Index>(f.size()) != a.cols()) {
    throw Error("forward_project: image length does not match columns");
  }
  Vector p(static_cast<std::size_t>(a.rows()));
  detail::check(ss_forward_project(a.get(), f.data(), p.data()));
  if (noise_sigma != 0.0) {
    detail::check(ss_add_noise(p.data(), static_cast<int64_t>(p.size()), noise_sigma, seed));
  }
  return p;
}

}  // namespace symsplit
