// TEST INFRASTRUCTURE ONLY — never linked into, loaded by, or called from the
// product path (paper_1902_10559_b200/). Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may use it.
//
// CPU restatement of the reference `symsplit` hot path
// (/root/reference/proj/src/{matrix,centro,geometry,solvers,phantom}.cpp),
// written without Eigen because Eigen3 is absent from this image and from the
// GPU box (reference proj/CMakeLists.txt:18 requires it; nothing vendors it).
// Eigen's arithmetic on the path is restated from its published behaviour
// (Eigen 3.3/3.4, un-vendored, version unpinned: "find_package(Eigen3 3.3)"):
//   * SparseMatrix<double> = compressed ColMajor, int StorageIndex;
//   * setFromTriplets: RowMajor temporary in triplet order, collapseDuplicates
//     sums repeats left-associatively in insertion order keeping the first slot,
//     transposed copy orders rows ascending inside every column;
//   * ColMajor sparse * dense: y = 0; for j ascending, for stored i ascending:
//     y[i] += v * x[j];
//   * transpose() * y: per column tmp = 0; tmp += v * y[i]; out[j] = tmp;
//   * VectorXd::norm(): sqrt of an SSE2 (2-lane, 2-packet unrolled) redux.
// Host code of the reference builds with the default x86-64 target: no FMA
// contraction, hence this file is compiled with -ffp-contract=off.
//
// Pinned against every known-answer test of the reference for this path
// (tests/test_oracle_*.py, fixtures in tests/golden/reference_pins.json).
#pragma once

#include <cstdint>
#include <functional>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace oracle {

using Index = std::int64_t;
using Vector = std::vector<double>;

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline constexpr Index mirror(Index i, Index n) { return n - 1 - i; }

// Eigen::Triplet<double> with the default int StorageIndex.
struct Triplet {
  int row;
  int col;
  double value;
};

// Compressed sparse column (reference Matrix sparse storage, matrix.hpp:18).
struct Csc {
  Index rows = 0, cols = 0;
  std::vector<int> outer;   // cols + 1
  std::vector<int> inner;   // row index, ascending inside a column
  std::vector<double> values;
  Index nnz() const { return static_cast<Index>(values.size()); }
};

// Compressed sparse row (Eigen::SparseMatrix<double, RowMajor>).
struct Csr {
  Index rows = 0, cols = 0;
  std::vector<int> ptr;     // rows + 1
  std::vector<int> idx;     // column index, ascending inside a row
  std::vector<double> values;
  Index nnz() const { return static_cast<Index>(values.size()); }
};

Csc csc_from_triplets(Index rows, Index cols, const std::vector<Triplet>& ts);
Csr csc_to_csr(const Csc& a);
Csc csr_to_csc(const Csr& a);

// reference proj/include/symsplit/matrix.hpp:34-87
class Matrix {
 public:
  Matrix() = default;
  static Matrix dense(Index rows, Index cols, Vector colmajor);
  static Matrix sparse(Csc s);
  static Matrix from_triplets(Index rows, Index cols,
                              const std::vector<Triplet>& ts);

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  bool is_sparse() const { return sparse_; }
  std::int64_t nonzeros() const;
  double fill_ratio() const;
  double coeff(Index i, Index j) const;
  const Csc& csc() const { return csc_; }
  const Vector& dense_data() const { return dense_; }  // column-major
  Vector to_dense() const;

  Vector apply(const Vector& x) const;
  Vector apply_transpose(const Vector& y) const;

  template <class F>
  void for_each(F&& f) const {
    if (sparse_) {
      for (Index j = 0; j < csc_.cols; ++j) {
        for (int k = csc_.outer[j]; k < csc_.outer[j + 1]; ++k) {
          f(static_cast<Index>(csc_.inner[k]), j, csc_.values[k]);
        }
      }
    } else {
      for (Index j = 0; j < cols_; ++j) {
        for (Index i = 0; i < rows_; ++i) f(i, j, dense_[j * rows_ + i]);
      }
    }
  }

 private:
  void check_finite() const;
  bool sparse_ = false;
  Index rows_ = 0, cols_ = 0;
  Vector dense_;
  Csc csc_;
};

// Eigen VectorXd::squaredNorm()/norm() with SSE2 packets (see header note).
double squared_norm(const Vector& v);
double norm(const Vector& v);
bool all_finite(const Vector& v);

// ---------------------------------------------------------------- centro
enum class SymmetryStatus { ok = 0, odd_row_count = 1, odd_col_count = 2 };

struct SymmetryReport {
  bool holds = false;
  double max_violation = 0.0;
  Index worst_row = 1;
  Index worst_col = 1;
  SymmetryStatus status = SymmetryStatus::ok;
};

struct SymmetryError : Error {
  SymmetryError(const std::string& w, SymmetryReport r) : Error(w), report(r) {}
  SymmetryReport report;
};

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
  double parent_fill = 0.0, fill1 = 0.0, fill2 = 0.0;
};

struct SolutionPair {
  Vector f1, f2;
};

SymmetryReport verify_symmetry(const Matrix& a, double tol);
Matrix symmetrize(const Matrix& a);
std::pair<Vector, Vector> split_rhs(const Vector& p);
std::pair<Matrix, Matrix> split_matrix(const Matrix& a);
SplitSystem split_system(const CentroSystem& sys);
SolutionPair decompose_solution(const Vector& f);
Vector recombine_solution(const SolutionPair& pair);
Matrix reconstruct_matrix(const Matrix& a1, const Matrix& a2);

// Fast fold used to cross-check the GPU fold: output row bi merges full-A rows
// bi and M-1-bi (TL, BL, TR, BR term order). Produces the
// same bits as split_matrix on sparse input (asserted by the tests).
void fold_rows_csr(const Csr& a, Csr& a1, Csr& a2);

// ---------------------------------------------------------------- geometry
inline constexpr double kPi = 3.14159265358979323846;
inline constexpr double degrees_to_radians(double deg) { return deg * kPi / 180.0; }

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
  std::pair<double, double> cell_center(int c, int r) const;
  void validate() const;
};

int snake_index(int c, int r, const GridSpec& g);
std::pair<int, int> snake_inverse(int j, const GridSpec& g);

struct ScanGeometry {
  int k = 24;
  double gamma = degrees_to_radians(30.0);
  double h_e = 1.0;
  double h_m = 0.25;
  double l_m = 0.43;
  int n_p = 1024;
  double a_e = 7e-4;
  double obj_size = 0.1;
  void validate() const;
};

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

struct ScanConfig {
  ScanGeometry geom;
  int grid_nx = 32;
  int grid_ny = 32;
};

std::vector<double> emitter_angles(const ScanGeometry& g);
std::vector<Point> emitter_positions(const ScanGeometry& g, double center_x);
RaySet enumerate_rays(const ScanGeometry& g, const GridSpec& grid);
std::vector<std::pair<int, double>> ray_weights(const Ray& ray, const GridSpec& grid);
CentroSystem build_system(const ScanGeometry& g, const GridSpec& grid, int parallelism = 0);
// Traced half of A as CSR (rows 0..M/2-1, columns ascending, repeats summed in
// traversal order) — the fast path the GPU tracer mirrors.
Csr build_traced_csr(const ScanGeometry& g, const GridSpec& grid, int parallelism = 0);
// Full A (M x N) as CSR from the traced half by the mirror rule.
Csr full_csr_from_traced(const Csr& traced, Index m, Index n);
ScanConfig parse_scan_config(const std::string& text);
GridSpec make_grid(const ScanConfig& c);

// ---------------------------------------------------------------- phantom
struct Ellipse {
  double x0 = 0.0, y0 = 0.0, a = 1.0, b = 1.0, angle = 0.0, density = 0.0;
  bool contains(double x, double y) const;
};
std::vector<Ellipse> shepp_logan_ellipses();
// BASELINE synthetic phantom: `count` ellipses drawn from Rng(seed) in the
// order x0, y0 in U[-0.7,0.7]; a, b in U[0.05,0.5]; angle in U[0,pi);
// density in U[0,1].
std::vector<Ellipse> random_ellipses(std::uint64_t seed, int count);
Vector rasterize(const std::vector<Ellipse>& es, const GridSpec& grid);
Vector forward_project(const Matrix& a, const Vector& f);
Vector forward_project_csr(const Csr& a, const Vector& f);
void add_noise(Vector& p, double sigma, std::uint64_t seed);

// reference proj/tests/support/oracles.hpp:29-50
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : e_(seed) {}
  double uniform() { return static_cast<double>(e_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  int integer(int lo, int hi) {
    const auto span = static_cast<std::uint64_t>(hi - lo + 1);
    return lo + static_cast<int>(e_() % span);
  }
  double normal();

 private:
  std::mt19937_64 e_;
};

// ---------------------------------------------------------------- solvers
enum class Method { sart, cgls };

struct SolveOptions {
  Method method = Method::sart;
  int max_iters = 200;
  double tol = 1e-10;
  double relaxation = 1.0;
  int parallelism = 0;
};

struct SolveReport {
  Vector f;
  double residual_norm = 0.0;
  double solution_norm = 0.0;
  int iterations = 0;
  double wall_time_seconds = 0.0;
  std::vector<double> residual_history;
  double split_seconds = 0.0, recombine_seconds = 0.0;
  double branch1_seconds = 0.0, branch2_seconds = 0.0;
};

SolveReport sart_solve(const Matrix& a, const Vector& p, const SolveOptions& o);
SolveReport cgls_solve(const Matrix& a, const Vector& p, const SolveOptions& o);
SolveReport run_method(const Matrix& a, const Vector& p, const SolveOptions& o);
SolveReport solve_direct_sart(const CentroSystem& sys, const SolveOptions& o);
SolveReport solve_split_sart(const CentroSystem& sys, const SolveOptions& o);
// Same loop on an already folded pair (the part the reference times as
// branch wall time); used by the CPU baseline.
SolveReport solve_split_prepared(const SplitSystem& ss, const SolveOptions& o,
                                 bool parallel);

}  // namespace oracle
