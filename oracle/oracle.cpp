// TEST INFRASTRUCTURE ONLY (see oracle.hpp). Each function cites the
// reference file:line it restates; paths are relative to /root/reference/proj.
#include "oracle.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <exception>
#include <limits>
#include <sstream>
#include <thread>

namespace oracle {

namespace {
using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}
}  // namespace

// ------------------------------------------------------------------ sparse
// Eigen internal::set_from_triplets (called by src/matrix.cpp:16,
// src/centro.cpp:125-126 / reference lines 211-212 of centro.cpp).
Csc csc_from_triplets(Index rows, Index cols, const std::vector<Triplet>& ts) {
  const std::size_t n = ts.size();
  // pass 1: count per row of the RowMajor temporary
  std::vector<std::int64_t> rstart(static_cast<std::size_t>(rows) + 1, 0);
  for (const Triplet& t : ts) {
    if (t.row < 0 || t.row >= rows || t.col < 0 || t.col >= cols) {
      throw Error("triplet index out of range");
    }
    ++rstart[static_cast<std::size_t>(t.row) + 1];
  }
  for (Index r = 0; r < rows; ++r) rstart[r + 1] += rstart[r];
  // pass 2: insertBackUncompressed in triplet order
  std::vector<int> tcol(n);
  std::vector<double> tval(n);
  {
    std::vector<std::int64_t> pos(rstart.begin(), rstart.end() - 1);
    for (const Triplet& t : ts) {
      const std::int64_t k = pos[t.row]++;
      tcol[k] = t.col;
      tval[k] = t.value;
    }
  }
  // pass 3: collapseDuplicates (first slot kept, value = acc + new)
  std::vector<std::int64_t> wi(static_cast<std::size_t>(cols), -1);
  std::vector<std::int64_t> rptr(static_cast<std::size_t>(rows) + 1, 0);
  std::int64_t count = 0;
  for (Index r = 0; r < rows; ++r) {
    const std::int64_t start = count;
    for (std::int64_t k = rstart[r]; k < rstart[r + 1]; ++k) {
      const int c = tcol[k];
      if (wi[c] >= start) {
        tval[wi[c]] = tval[wi[c]] + tval[k];
      } else {
        tval[count] = tval[k];
        tcol[count] = c;
        wi[c] = count;
        ++count;
      }
    }
    rptr[r + 1] = count;
  }
  // pass 4: transposed copy -> CSC with rows ascending in every column
  Csc out;
  out.rows = rows;
  out.cols = cols;
  out.outer.assign(static_cast<std::size_t>(cols) + 1, 0);
  for (std::int64_t k = 0; k < count; ++k) ++out.outer[tcol[k] + 1];
  for (Index c = 0; c < cols; ++c) out.outer[c + 1] += out.outer[c];
  out.inner.resize(count);
  out.values.resize(count);
  std::vector<int> pos(out.outer.begin(), out.outer.end() - 1);
  for (Index r = 0; r < rows; ++r) {
    for (std::int64_t k = rptr[r]; k < rptr[r + 1]; ++k) {
      const int p = pos[tcol[k]]++;
      out.inner[p] = static_cast<int>(r);
      out.values[p] = tval[k];
    }
  }
  return out;
}

Csr csc_to_csr(const Csc& a) {
  Csr out;
  out.rows = a.rows;
  out.cols = a.cols;
  out.ptr.assign(static_cast<std::size_t>(a.rows) + 1, 0);
  for (int r : a.inner) ++out.ptr[r + 1];
  for (Index r = 0; r < a.rows; ++r) out.ptr[r + 1] += out.ptr[r];
  out.idx.resize(a.inner.size());
  out.values.resize(a.values.size());
  std::vector<int> pos(out.ptr.begin(), out.ptr.end() - 1);
  for (Index c = 0; c < a.cols; ++c) {
    for (int k = a.outer[c]; k < a.outer[c + 1]; ++k) {
      const int p = pos[a.inner[k]]++;
      out.idx[p] = static_cast<int>(c);
      out.values[p] = a.values[k];
    }
  }
  return out;
}

Csc csr_to_csc(const Csr& a) {
  Csc out;
  out.rows = a.rows;
  out.cols = a.cols;
  out.outer.assign(static_cast<std::size_t>(a.cols) + 1, 0);
  for (int c : a.idx) ++out.outer[c + 1];
  for (Index c = 0; c < a.cols; ++c) out.outer[c + 1] += out.outer[c];
  out.inner.resize(a.idx.size());
  out.values.resize(a.values.size());
  std::vector<int> pos(out.outer.begin(), out.outer.end() - 1);
  for (Index r = 0; r < a.rows; ++r) {
    for (int k = a.ptr[r]; k < a.ptr[r + 1]; ++k) {
      const int p = pos[a.idx[k]]++;
      out.inner[p] = static_cast<int>(r);
      out.values[p] = a.values[k];
    }
  }
  return out;
}

// ------------------------------------------------------------------ Matrix
// src/matrix.cpp:5-84
Matrix Matrix::dense(Index rows, Index cols, Vector colmajor) {
  if (rows < 0 || cols < 0) throw Error("matrix shape must be non-negative");
  if (static_cast<Index>(colmajor.size()) != rows * cols) {
    throw Error("dense data size mismatch");
  }
  Matrix m;
  m.sparse_ = false;
  m.rows_ = rows;
  m.cols_ = cols;
  m.dense_ = std::move(colmajor);
  m.check_finite();
  return m;
}

Matrix Matrix::sparse(Csc s) {
  Matrix m;
  m.sparse_ = true;
  m.rows_ = s.rows;
  m.cols_ = s.cols;
  m.csc_ = std::move(s);
  m.check_finite();
  return m;
}

Matrix Matrix::from_triplets(Index rows, Index cols,
                             const std::vector<Triplet>& ts) {
  if (rows < 0 || cols < 0) throw Error("matrix shape must be non-negative");
  return sparse(csc_from_triplets(rows, cols, ts));
}

std::int64_t Matrix::nonzeros() const {
  std::int64_t n = 0;
  for_each([&](Index, Index, double v) {
    if (v != 0.0) ++n;
  });
  return n;
}

double Matrix::fill_ratio() const {
  const double size = static_cast<double>(rows_) * static_cast<double>(cols_);
  return size > 0 ? static_cast<double>(nonzeros()) / size : 0.0;
}

double Matrix::coeff(Index i, Index j) const {
  if (i < 0 || i >= rows_ || j < 0 || j >= cols_) {
    throw Error("matrix index out of range");
  }
  if (!sparse_) return dense_[j * rows_ + i];
  const auto b = csc_.inner.begin() + csc_.outer[j];
  const auto e = csc_.inner.begin() + csc_.outer[j + 1];
  const auto it = std::lower_bound(b, e, static_cast<int>(i));
  if (it != e && *it == i) return csc_.values[it - csc_.inner.begin()];
  return 0.0;
}

Vector Matrix::to_dense() const {
  if (!sparse_) return dense_;
  Vector d(static_cast<std::size_t>(rows_ * cols_), 0.0);
  for_each([&](Index i, Index j, double v) { d[j * rows_ + i] = v; });
  return d;
}

Vector Matrix::apply(const Vector& x) const {
  if (static_cast<Index>(x.size()) != cols_) {
    throw Error("matrix-vector size mismatch");
  }
  Vector y(static_cast<std::size_t>(rows_), 0.0);
  if (sparse_) {
    for (Index j = 0; j < cols_; ++j) {
      const double xj = x[j];
      for (int k = csc_.outer[j]; k < csc_.outer[j + 1]; ++k) {
        y[csc_.inner[k]] += csc_.values[k] * xj;
      }
    }
  } else {
    for (Index j = 0; j < cols_; ++j) {
      for (Index i = 0; i < rows_; ++i) y[i] += dense_[j * rows_ + i] * x[j];
    }
  }
  return y;
}

Vector Matrix::apply_transpose(const Vector& y) const {
  if (static_cast<Index>(y.size()) != rows_) {
    throw Error("matrix-vector size mismatch");
  }
  Vector out(static_cast<std::size_t>(cols_), 0.0);
  for (Index j = 0; j < cols_; ++j) {
    double tmp = 0.0;
    if (sparse_) {
      for (int k = csc_.outer[j]; k < csc_.outer[j + 1]; ++k) {
        tmp += csc_.values[k] * y[csc_.inner[k]];
      }
    } else {
      for (Index i = 0; i < rows_; ++i) tmp += dense_[j * rows_ + i] * y[i];
    }
    out[j] = 0.0 + tmp;
  }
  return out;
}

void Matrix::check_finite() const {
  bool ok = true;
  for_each([&](Index, Index, double v) {
    if (!std::isfinite(v)) ok = false;
  });
  if (!ok) throw Error("matrix contains non-finite values");
}

double squared_norm(const Vector& v) {
  const std::size_t size = v.size();
  if (size == 0) return 0.0;
  const std::size_t ps = 2;
  const std::size_t aligned2 = (size / (2 * ps)) * (2 * ps);
  const std::size_t aligned = (size / ps) * ps;
  if (aligned == 0) {
    double res = v[0] * v[0];
    for (std::size_t i = 1; i < size; ++i) res = res + v[i] * v[i];
    return res;
  }
  double p0[2] = {v[0] * v[0], v[1] * v[1]};
  if (aligned > ps) {
    double p1[2] = {v[2] * v[2], v[3] * v[3]};
    for (std::size_t i = 2 * ps; i < aligned2; i += 2 * ps) {
      p0[0] = p0[0] + v[i] * v[i];
      p0[1] = p0[1] + v[i + 1] * v[i + 1];
      p1[0] = p1[0] + v[i + 2] * v[i + 2];
      p1[1] = p1[1] + v[i + 3] * v[i + 3];
    }
    p0[0] = p0[0] + p1[0];
    p0[1] = p0[1] + p1[1];
    if (aligned > aligned2) {
      p0[0] = p0[0] + v[aligned2] * v[aligned2];
      p0[1] = p0[1] + v[aligned2 + 1] * v[aligned2 + 1];
    }
  }
  double res = p0[0] + p0[1];
  for (std::size_t i = aligned; i < size; ++i) res = res + v[i] * v[i];
  return res;
}

double norm(const Vector& v) { return std::sqrt(squared_norm(v)); }

bool all_finite(const Vector& v) {
  for (double x : v) {
    if (!std::isfinite(x)) return false;
  }
  return true;
}

// ------------------------------------------------------------------ centro
namespace {
void require_symmetric(const Matrix& a, double tol, const char* op) {
  // src/centro.cpp:27-42
  const SymmetryReport rep = verify_symmetry(a, tol);
  if (!rep.holds) {
    std::ostringstream msg;
    msg << op << ": matrix is not centrosymmetric";
    if (rep.status == SymmetryStatus::odd_row_count) {
      msg << " (odd row count)";
    } else if (rep.status == SymmetryStatus::odd_col_count) {
      msg << " (odd column count)";
    } else {
      msg << " (max violation " << rep.max_violation << " at (" << rep.worst_row
          << "," << rep.worst_col << "), tol " << tol << ")";
    }
    throw SymmetryError(msg.str(), rep);
  }
}
}  // namespace

// src/centro.cpp:46-66
SymmetryReport verify_symmetry(const Matrix& a, double tol) {
  if (tol < 0) throw Error("verify_symmetry: tol must be non-negative");
  SymmetryReport rep;
  const Index m = a.rows(), n = a.cols();
  if (m % 2 != 0) {
    rep.status = SymmetryStatus::odd_row_count;
  } else if (n % 2 != 0) {
    rep.status = SymmetryStatus::odd_col_count;
  }
  rep.max_violation = 0.0;
  a.for_each([&](Index i, Index j, double v) {
    const double d = std::abs(v - a.coeff(mirror(i, m), mirror(j, n)));
    if (d > rep.max_violation) {
      rep.max_violation = d;
      rep.worst_row = i + 1;
      rep.worst_col = j + 1;
    }
  });
  rep.holds = rep.status == SymmetryStatus::ok && rep.max_violation <= tol;
  return rep;
}

// src/centro.cpp:68-87 (dense branch only is needed by the pins)
Matrix symmetrize(const Matrix& a) {
  const Index m = a.rows(), n = a.cols();
  if (a.is_sparse()) {
    std::vector<Triplet> ts;
    a.for_each([&](Index i, Index j, double v) {
      ts.push_back({static_cast<int>(i), static_cast<int>(j), 0.5 * v});
      ts.push_back({static_cast<int>(mirror(i, m)), static_cast<int>(mirror(j, n)),
                    0.5 * v});
    });
    return Matrix::from_triplets(m, n, ts);
  }
  const Vector& d = a.dense_data();
  Vector out(static_cast<std::size_t>(m * n));
  for (Index j = 0; j < n; ++j) {
    for (Index i = 0; i < m; ++i) {
      out[j * m + i] = 0.5 * d[j * m + i] + 0.5 * d[mirror(j, n) * m + mirror(i, m)];
    }
  }
  return Matrix::dense(m, n, std::move(out));
}

// src/centro.cpp:89-99
std::pair<Vector, Vector> split_rhs(const Vector& p) {
  const Index m = static_cast<Index>(p.size());
  if (m % 2 != 0) throw Error("split_rhs: vector length must be even");
  const Index mh = m / 2;
  Vector p1(mh), p2(mh);
  for (Index i = 0; i < mh; ++i) {
    p1[i] = p[i] - p[mirror(i, m)];
    p2[i] = p[i] + p[mirror(i, m)];
  }
  return {std::move(p1), std::move(p2)};
}

namespace {
Csc prune_nonzero(const Csc& s) {
  // Eigen SparseMatrix::prune(keep) with keep = (v != 0.0): order preserved.
  Csc out;
  out.rows = s.rows;
  out.cols = s.cols;
  out.outer.assign(static_cast<std::size_t>(s.cols) + 1, 0);
  out.inner.reserve(s.inner.size());
  out.values.reserve(s.values.size());
  for (Index j = 0; j < s.cols; ++j) {
    for (int k = s.outer[j]; k < s.outer[j + 1]; ++k) {
      if (s.values[k] != 0.0) {
        out.inner.push_back(s.inner[k]);
        out.values.push_back(s.values[k]);
      }
    }
    out.outer[j + 1] = static_cast<int>(out.values.size());
  }
  return out;
}
}  // namespace

// src/centro.cpp:103-140
std::pair<Matrix, Matrix> split_matrix(const Matrix& a) {
  const Index m = a.rows(), n = a.cols();
  if (m % 2 != 0 || n % 2 != 0) {
    throw Error("split_matrix: dimensions must be even");
  }
  const Index mh = m / 2, nh = n / 2;
  if (a.is_sparse()) {
    std::vector<Triplet> t1, t2;
    t1.reserve(static_cast<std::size_t>(a.csc().nnz()));
    t2.reserve(static_cast<std::size_t>(a.csc().nnz()));
    a.for_each([&](Index i, Index j, double v) {
      const Index bi = i < mh ? i : mirror(i, m);
      const Index bj = j < nh ? j : mirror(j, n);
      const double h = 0.5 * v;
      const bool first_term = (i < mh) == (j < nh);
      t1.push_back({static_cast<int>(bi), static_cast<int>(bj), first_term ? h : -h});
      t2.push_back({static_cast<int>(bi), static_cast<int>(bj), h});
    });
    Csc s1 = csc_from_triplets(mh, nh, t1);
    Csc s2 = csc_from_triplets(mh, nh, t2);
    return {Matrix::sparse(prune_nonzero(s1)), Matrix::sparse(prune_nonzero(s2))};
  }
  const Vector& d = a.dense_data();
  Vector a1(static_cast<std::size_t>(mh * nh)), a2(static_cast<std::size_t>(mh * nh));
  for (Index j = 0; j < nh; ++j) {
    for (Index i = 0; i < mh; ++i) {
      a1[j * mh + i] = d[j * m + i] - d[j * m + mirror(i, m)];
      a2[j * mh + i] = d[j * m + i] + d[j * m + mirror(i, m)];
    }
  }
  return {Matrix::dense(mh, nh, std::move(a1)), Matrix::dense(mh, nh, std::move(a2))};
}

// src/centro.cpp:144-156
SplitSystem split_system(const CentroSystem& sys) {
  if (static_cast<Index>(sys.p.size()) != sys.a.rows()) {
    throw Error("split_system: right-hand side length does not match rows");
  }
  require_symmetric(sys.a, sys.symmetry_tol, "split_system");
  auto [a1, a2] = split_matrix(sys.a);
  auto [p1, p2] = split_rhs(sys.p);
  SplitSystem out{std::move(a1), std::move(p1), std::move(a2), std::move(p2)};
  out.parent_fill = sys.a.fill_ratio();
  out.fill1 = out.a1.fill_ratio();
  out.fill2 = out.a2.fill_ratio();
  return out;
}

// src/centro.cpp:158-168
SolutionPair decompose_solution(const Vector& f) {
  const Index n = static_cast<Index>(f.size());
  if (n % 2 != 0) throw Error("decompose_solution: vector length must be even");
  const Index nh = n / 2;
  SolutionPair pair{Vector(nh), Vector(nh)};
  for (Index j = 0; j < nh; ++j) {
    pair.f1[j] = f[j] - f[mirror(j, n)];
    pair.f2[j] = f[j] + f[mirror(j, n)];
  }
  return pair;
}

// src/centro.cpp:170-185
Vector recombine_solution(const SolutionPair& pair) {
  if (pair.f1.size() != pair.f2.size()) {
    throw Error("recombine_solution: component lengths differ");
  }
  if (!all_finite(pair.f1) || !all_finite(pair.f2)) {
    throw Error("recombine_solution: non-finite component");
  }
  const Index nh = static_cast<Index>(pair.f1.size());
  const Index n = 2 * nh;
  Vector f(n);
  for (Index j = 0; j < nh; ++j) {
    f[j] = 0.5 * (pair.f2[j] + pair.f1[j]);
    f[mirror(j, n)] = 0.5 * (pair.f2[j] - pair.f1[j]);
  }
  return f;
}

// src/centro.cpp:187-231 (test-fixture helper: make_centro_matrix)
Matrix reconstruct_matrix(const Matrix& a1, const Matrix& a2) {
  if (a1.rows() != a2.rows() || a1.cols() != a2.cols()) {
    throw Error("reconstruct_matrix: halves have different shapes");
  }
  const Index mh = a1.rows(), nh = a1.cols();
  const Index m = 2 * mh, n = 2 * nh;
  if (a1.is_sparse() || a2.is_sparse()) {
    std::vector<Triplet> ts;
    const auto scatter = [&](Index i, Index j, double tl, double bl) {
      ts.push_back({(int)i, (int)j, tl});
      ts.push_back({(int)mirror(i, m), (int)mirror(j, n), tl});
      ts.push_back({(int)mirror(i, m), (int)j, bl});
      ts.push_back({(int)i, (int)mirror(j, n), bl});
    };
    a1.for_each([&](Index i, Index j, double d) { scatter(i, j, 0.5 * d, -0.5 * d); });
    a2.for_each([&](Index i, Index j, double s) { scatter(i, j, 0.5 * s, 0.5 * s); });
    return Matrix::sparse(prune_nonzero(csc_from_triplets(m, n, ts)));
  }
  const Vector& d1 = a1.dense_data();
  const Vector& d2 = a2.dense_data();
  Vector out(static_cast<std::size_t>(m * n));
  for (Index j = 0; j < nh; ++j) {
    for (Index i = 0; i < mh; ++i) {
      const double tl = 0.5 * (d2[j * mh + i] + d1[j * mh + i]);
      const double bl = 0.5 * (d2[j * mh + i] - d1[j * mh + i]);
      out[j * m + i] = tl;
      out[mirror(j, n) * m + mirror(i, m)] = tl;
      out[j * m + mirror(i, m)] = bl;
      out[mirror(j, n) * m + i] = bl;
    }
  }
  return Matrix::dense(m, n, std::move(out));
}

// Fast fold: the bucket (bi, bj) receives, in triplet
// order, TL = A(bi,bj), BL = A(M-1-bi,bj), TR = A(bi,N-1-bj),
// BR = A(M-1-bi,N-1-bj); each enters as 0.5*v (sign -,- for BL/TR in A1),
// summed left to right starting from the first present term; exact zeros
// are pruned.
void fold_rows_csr(const Csr& a, Csr& a1, Csr& a2) {
  const Index m = a.rows, n = a.cols;
  if (m % 2 != 0 || n % 2 != 0) throw Error("split_matrix: dimensions must be even");
  const Index mh = m / 2, nh = n / 2;
  for (Csr* o : {&a1, &a2}) {
    o->rows = mh;
    o->cols = nh;
    o->ptr.assign(static_cast<std::size_t>(mh) + 1, 0);
    o->idx.clear();
    o->values.clear();
  }
  for (Index bi = 0; bi < mh; ++bi) {
    const Index top = bi, bot = mirror(bi, m);
    // four cursors: TL ascending over top's cols < nh; BL ascending over
    // bot's cols < nh; TR over top's cols >= nh walked backwards (bj = n-1-c
    // ascending); BR likewise over bot.
    int tl = a.ptr[top], tl_end = a.ptr[top];
    while (tl_end < a.ptr[top + 1] && a.idx[tl_end] < nh) ++tl_end;
    int tr = a.ptr[top + 1] - 1;
    const int tr_end = tl_end - 1;
    int bl = a.ptr[bot], bl_end = a.ptr[bot];
    while (bl_end < a.ptr[bot + 1] && a.idx[bl_end] < nh) ++bl_end;
    int br = a.ptr[bot + 1] - 1;
    const int br_end = bl_end - 1;
    for (;;) {
      Index bj = nh;
      if (tl < tl_end) bj = std::min<Index>(bj, a.idx[tl]);
      if (bl < bl_end) bj = std::min<Index>(bj, a.idx[bl]);
      if (tr > tr_end) bj = std::min<Index>(bj, n - 1 - a.idx[tr]);
      if (br > br_end) bj = std::min<Index>(bj, n - 1 - a.idx[br]);
      if (bj == nh) break;
      bool have = false;
      double s1 = 0.0, s2 = 0.0;
      const auto add = [&](double h, bool neg) {
        if (!have) {
          s1 = neg ? -h : h;
          s2 = h;
          have = true;
        } else {
          s1 = s1 + (neg ? -h : h);
          s2 = s2 + h;
        }
      };
      if (tl < tl_end && a.idx[tl] == bj) add(0.5 * a.values[tl++], false);
      if (bl < bl_end && a.idx[bl] == bj) add(0.5 * a.values[bl++], true);
      if (tr > tr_end && n - 1 - a.idx[tr] == bj) add(0.5 * a.values[tr--], true);
      if (br > br_end && n - 1 - a.idx[br] == bj) add(0.5 * a.values[br--], false);
      if (s1 != 0.0) {
        a1.idx.push_back(static_cast<int>(bj));
        a1.values.push_back(s1);
      }
      if (s2 != 0.0) {
        a2.idx.push_back(static_cast<int>(bj));
        a2.values.push_back(s2);
      }
    }
    a1.ptr[bi + 1] = static_cast<int>(a1.values.size());
    a2.ptr[bi + 1] = static_cast<int>(a2.values.size());
  }
}

// ------------------------------------------------------------------ geometry
namespace {
struct ClipRange {
  double t_in = 0.0;
  double t_out = 1.0;
};

// src/geometry.cpp:19-36
std::optional<ClipRange> clip_to_grid(const Ray& ray, const GridSpec& grid) {
  const double dx = ray.detector.x - ray.source.x;
  const double dy = ray.detector.y - ray.source.y;
  ClipRange range;
  const auto clip_axis = [&](double p0, double d, double lo, double hi) {
    if (d == 0.0) return p0 > lo && p0 < hi;
    double ta = (lo - p0) / d;
    double tb = (hi - p0) / d;
    if (ta > tb) std::swap(ta, tb);
    range.t_in = std::max(range.t_in, ta);
    range.t_out = std::min(range.t_out, tb);
    return true;
  };
  if (!clip_axis(ray.source.x, dx, grid.x_left(), grid.x_right())) return {};
  if (!clip_axis(ray.source.y, dy, grid.y_bottom, grid.y_top())) return {};
  if (!(range.t_out > range.t_in)) return {};
  return range;
}

// src/geometry.cpp:40-46
double x_boundary(const GridSpec& g, int k) {
  return g.center_x + (k - g.n_x / 2) * g.voxel_size;
}
double y_boundary(const GridSpec& g, int k) { return g.y_bottom + k * g.voxel_size; }

// src/geometry.cpp:48-55
int thread_budget(int requested, Index work) {
  int budget = requested;
  if (budget <= 0) {
    const unsigned hw = std::thread::hardware_concurrency();
    budget = hw > 0 ? static_cast<int>(hw) : 1;
  }
  return static_cast<int>(std::min<Index>(budget, std::max<Index>(work, 1)));
}

template <class F>
void parallel_chunks(Index items, int parallelism, F&& fn) {
  const int workers = thread_budget(parallelism, items);
  if (workers <= 1) {
    fn(0, items);
    return;
  }
  std::vector<std::thread> pool;
  const Index chunk = (items + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    const Index b = w * chunk, e = std::min(items, b + chunk);
    if (b >= e) break;
    pool.emplace_back(fn, b, e);
  }
  for (auto& t : pool) t.join();
}
}  // namespace

// src/geometry.cpp:59-74
std::pair<double, double> GridSpec::cell_center(int c, int r) const {
  if (c < 1 || c > n_x || r < 1 || r > n_y) {
    throw Error("cell_center: cell index out of range");
  }
  const double x = center_x + (c - 0.5 - 0.5 * n_x) * voxel_size;
  const double y = y_bottom + (n_y - r + 0.5) * voxel_size;
  return {x, y};
}

void GridSpec::validate() const {
  if (n_x < 2 || n_x % 2 != 0) {
    throw Error("grid: n_x must be even and positive (mirror pairing)");
  }
  if (n_y < 1) throw Error("grid: n_y must be positive");
  if (!(voxel_size > 0)) throw Error("grid: voxel_size must be positive");
}

// src/geometry.cpp:76-92
int snake_index(int c, int r, const GridSpec& g) {
  if (c < 1 || c > g.n_x || r < 1 || r > g.n_y) {
    throw Error("snake_index: cell index out of range");
  }
  const int base = (c - 1) * g.n_y;
  return c % 2 == 1 ? base + r : base + (g.n_y - r + 1);
}

std::pair<int, int> snake_inverse(int j, const GridSpec& g) {
  if (j < 1 || j > g.cell_count()) throw Error("snake_inverse: index out of range");
  const int c = (j - 1) / g.n_y + 1;
  const int off = (j - 1) % g.n_y + 1;
  const int r = c % 2 == 1 ? off : g.n_y - off + 1;
  return {c, r};
}

// src/geometry.cpp:94-105
void ScanGeometry::validate() const {
  if (k < 2 || k % 2 != 0) {
    throw Error("geometry: k must be even and >= 2 (mirror pairing)");
  }
  if (!(gamma > 0) || !(gamma < kPi / 2)) {
    throw Error("geometry: gamma must lie in (0, pi/2)");
  }
  if (!(h_e > 0) || !(h_m > 0) || !(l_m > 0) || !(obj_size > 0)) {
    throw Error("geometry: lengths must be positive");
  }
  if (n_p < 1) throw Error("geometry: n_p must be >= 1");
}

// src/geometry.cpp:107-117
std::vector<double> emitter_angles(const ScanGeometry& g) {
  g.validate();
  const int k = g.k;
  std::vector<double> angles(k);
  const double step = 2.0 * g.gamma / (k - 1);
  for (int i = 0; i < k / 2; ++i) {
    angles[i] = -g.gamma + i * step;
    angles[k - 1 - i] = -angles[i];
  }
  return angles;
}

// src/geometry.cpp:119-130
std::vector<Point> emitter_positions(const ScanGeometry& g, double cx) {
  const auto angles = emitter_angles(g);
  std::vector<Point> s(angles.size());
  for (int i = 0; i < g.k / 2; ++i) {
    s[i] = Point{cx + g.h_e * std::sin(angles[i]), g.h_m + g.h_e * std::cos(angles[i])};
    s[g.k - 1 - i] = Point{2.0 * cx - s[i].x, s[i].y};
  }
  return s;
}

// src/geometry.cpp:132-173
RaySet enumerate_rays(const ScanGeometry& g, const GridSpec& grid) {
  g.validate();
  grid.validate();
  const double cx = grid.center_x;
  const auto sources = emitter_positions(g, cx);
  const double native = g.l_m / g.n_p;
  const double pitch = std::max(native, 0.5 * grid.voxel_size);
  const int samples = std::max(1, static_cast<int>(std::floor(g.l_m / pitch)));
  const auto reflect = [cx](const Ray& r) {
    return Ray{Point{2.0 * cx - r.source.x, r.source.y},
               Point{2.0 * cx - r.detector.x, r.detector.y}};
  };
  std::vector<Ray> kept, mirrored;
  for (int pos = 0; pos < g.k / 2; ++pos) {
    for (int q = 0; q < samples; ++q) {
      const Ray ray{sources[pos], Point{cx + (q + 0.5 - 0.5 * samples) * pitch, 0.0}};
      if (!clip_to_grid(ray, grid)) continue;
      kept.push_back(ray);
      mirrored.push_back(reflect(ray));
    }
  }
  if (kept.empty()) {
    throw Error("enumerate_rays: no ray intersects the reconstruction region");
  }
  std::reverse(mirrored.begin(), mirrored.end());
  RaySet out;
  out.rays = std::move(kept);
  out.rays.insert(out.rays.end(), mirrored.begin(), mirrored.end());
  out.positions = g.k;
  out.samples_per_position = samples;
  out.sample_pitch = pitch;
  return out;
}

// src/geometry.cpp:175-225
std::vector<std::pair<int, double>> ray_weights(const Ray& ray, const GridSpec& grid) {
  grid.validate();
  const double dx = ray.detector.x - ray.source.x;
  const double dy = ray.detector.y - ray.source.y;
  const double seg_len = std::hypot(dx, dy);
  if (seg_len == 0.0) throw Error("ray_weights: degenerate ray");
  const auto range = clip_to_grid(ray, grid);
  if (!range) return {};
  std::vector<double> ts;
  ts.reserve(static_cast<std::size_t>(grid.n_x + grid.n_y + 2));
  ts.push_back(range->t_in);
  const auto collect = [&](double p0, double d, int count, auto boundary_at) {
    if (d == 0.0) return;
    for (int k = 0; k <= count; ++k) {
      const double t = (boundary_at(k) - p0) / d;
      if (t > range->t_in && t < range->t_out) ts.push_back(t);
    }
  };
  collect(ray.source.x, dx, grid.n_x, [&](int k) { return x_boundary(grid, k); });
  collect(ray.source.y, dy, grid.n_y, [&](int k) { return y_boundary(grid, k); });
  ts.push_back(range->t_out);
  std::sort(ts.begin(), ts.end());
  std::vector<std::pair<int, double>> w;
  w.reserve(ts.size());
  for (std::size_t s = 0; s + 1 < ts.size(); ++s) {
    const double ta = ts[s], tb = ts[s + 1];
    if (!(tb > ta)) continue;
    const double tm = 0.5 * (ta + tb);
    const double xm = ray.source.x + tm * dx;
    const double ym = ray.source.y + tm * dy;
    const int c = std::clamp(
        static_cast<int>(std::floor((xm - grid.x_left()) / grid.voxel_size)), 0,
        grid.n_x - 1);
    const int fb = std::clamp(
        static_cast<int>(std::floor((ym - grid.y_bottom) / grid.voxel_size)), 0,
        grid.n_y - 1);
    const int j = snake_index(c + 1, grid.n_y - fb, grid);
    const double len = (tb - ta) * seg_len;
    if (!w.empty() && w.back().first == j) {
      w.back().second += len;
    } else {
      w.emplace_back(j, len);
    }
  }
  return w;
}

namespace {
std::vector<std::vector<std::pair<int, double>>> trace_half(const RaySet& rays,
                                                            const GridSpec& grid,
                                                            int parallelism) {
  const Index mh = rays.count() / 2;
  std::vector<std::vector<std::pair<int, double>>> traced(static_cast<std::size_t>(mh));
  parallel_chunks(mh, parallelism, [&](Index b, Index e) {
    for (Index i = b; i < e; ++i) traced[i] = ray_weights(rays.rays[i], grid);
  });
  return traced;
}
}  // namespace

// src/geometry.cpp:227-275
CentroSystem build_system(const ScanGeometry& g, const GridSpec& grid, int parallelism) {
  const RaySet rays = enumerate_rays(g, grid);
  const Index m = rays.count(), mh = m / 2, n = grid.cell_count();
  const auto traced = trace_half(rays, grid, parallelism);
  std::size_t nnz = 0;
  for (const auto& row : traced) nnz += row.size();
  std::vector<Triplet> ts;
  ts.reserve(2 * nnz);
  for (Index i = 0; i < mh; ++i) {
    for (const auto& [j, len] : traced[i]) {
      const Index col = j - 1;
      ts.push_back({static_cast<int>(i), static_cast<int>(col), len});
      ts.push_back({static_cast<int>(mirror(i, m)), static_cast<int>(mirror(col, n)), len});
    }
  }
  CentroSystem sys;
  sys.a = Matrix::from_triplets(m, n, ts);
  sys.p = Vector(static_cast<std::size_t>(m), 0.0);
  sys.symmetry_tol = 0.0;
  return sys;
}

Csr build_traced_csr(const ScanGeometry& g, const GridSpec& grid, int parallelism) {
  const RaySet rays = enumerate_rays(g, grid);
  const Index m = rays.count(), mh = m / 2, n = grid.cell_count();
  auto traced = trace_half(rays, grid, parallelism);
  Csr out;
  out.rows = mh;
  out.cols = n;
  out.ptr.assign(static_cast<std::size_t>(mh) + 1, 0);
  // Per row: stable sort by column, repeated columns summed in traversal
  // order (what setFromTriplets does with them).
  std::vector<std::vector<std::pair<int, double>>> rows(static_cast<std::size_t>(mh));
  parallel_chunks(mh, parallelism, [&](Index b, Index e) {
    for (Index i = b; i < e; ++i) {
      auto& t = traced[i];
      std::stable_sort(t.begin(), t.end(),
                       [](const auto& x, const auto& y) { return x.first < y.first; });
      auto& r = rows[i];
      for (const auto& [j, len] : t) {
        if (!r.empty() && r.back().first == j - 1) {
          r.back().second = r.back().second + len;
        } else {
          r.emplace_back(j - 1, len);
        }
      }
    }
  });
  for (Index i = 0; i < mh; ++i) out.ptr[i + 1] = out.ptr[i] + static_cast<int>(rows[i].size());
  out.idx.resize(out.ptr[mh]);
  out.values.resize(out.ptr[mh]);
  for (Index i = 0; i < mh; ++i) {
    int k = out.ptr[i];
    for (const auto& [c, v] : rows[i]) {
      out.idx[k] = c;
      out.values[k] = v;
      ++k;
    }
  }
  return out;
}

Csr full_csr_from_traced(const Csr& t, Index m, Index n) {
  const Index mh = m / 2;
  if (t.rows != mh) throw Error("traced rows mismatch");
  Csr out;
  out.rows = m;
  out.cols = n;
  out.ptr.assign(static_cast<std::size_t>(m) + 1, 0);
  const Index nnz_half = t.nnz();
  out.idx.resize(static_cast<std::size_t>(2 * nnz_half));
  out.values.resize(static_cast<std::size_t>(2 * nnz_half));
  for (Index i = 0; i < mh; ++i) out.ptr[i + 1] = t.ptr[i + 1];
  for (Index r = mh; r < m; ++r) {
    const Index src = mirror(r, m);
    out.ptr[r + 1] = out.ptr[r] + (t.ptr[src + 1] - t.ptr[src]);
  }
  std::copy(t.idx.begin(), t.idx.end(), out.idx.begin());
  std::copy(t.values.begin(), t.values.end(), out.values.begin());
  for (Index r = mh; r < m; ++r) {
    const Index src = mirror(r, m);
    int k = out.ptr[r];
    for (int s = t.ptr[src + 1] - 1; s >= t.ptr[src]; --s) {
      out.idx[k] = static_cast<int>(mirror(t.idx[s], n));
      out.values[k] = t.values[s];
      ++k;
    }
  }
  return out;
}

// src/geometry.cpp:352-411
ScanConfig parse_scan_config(const std::string& text) {
  ScanConfig config;
  std::istringstream in(text);
  std::string line;
  long line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line.erase(hash);
    for (char& ch : line) {
      if (ch == '=' || ch == '\t' || ch == '\r') ch = ' ';
    }
    std::istringstream fields(line);
    std::string key;
    if (!(fields >> key)) continue;
    double value = 0.0;
    if (!(fields >> value)) {
      throw Error("config line " + std::to_string(line_no) +
                  ": missing numeric value for key '" + key + "'");
    }
    std::string extra;
    if (fields >> extra) {
      throw Error("config line " + std::to_string(line_no) + ": trailing content '" +
                  extra + "'");
    }
    if (key == "k") config.geom.k = static_cast<int>(value);
    else if (key == "gamma_deg") config.geom.gamma = degrees_to_radians(value);
    else if (key == "h_e") config.geom.h_e = value;
    else if (key == "h_m") config.geom.h_m = value;
    else if (key == "l_m") config.geom.l_m = value;
    else if (key == "n_p") config.geom.n_p = static_cast<int>(value);
    else if (key == "grid_nx") config.grid_nx = static_cast<int>(value);
    else if (key == "grid_ny") config.grid_ny = static_cast<int>(value);
    else if (key == "obj_size") config.geom.obj_size = value;
    else
      throw Error("config line " + std::to_string(line_no) + ": unknown key '" + key + "'");
  }
  return config;
}

GridSpec make_grid(const ScanConfig& c) {
  GridSpec g;
  g.n_x = c.grid_nx;
  g.n_y = c.grid_ny;
  g.voxel_size = c.geom.obj_size / c.grid_nx;
  g.center_x = 0.0;
  g.y_bottom = c.geom.h_m;
  return g;
}

// ------------------------------------------------------------------ phantom
// src/phantom.cpp:8-16
bool Ellipse::contains(double x, double y) const {
  const double dx = x - x0;
  const double dy = y - y0;
  const double ca = std::cos(angle);
  const double sa = std::sin(angle);
  const double u = (dx * ca + dy * sa) / a;
  const double v = (-dx * sa + dy * ca) / b;
  return u * u + v * v <= 1.0;
}

// src/phantom.cpp:18-32
std::vector<Ellipse> shepp_logan_ellipses() {
  const auto deg = [](double d) { return degrees_to_radians(d); };
  return {
      {0.0, 0.0, 0.69, 0.92, deg(0.0), 2.0},
      {0.0, -0.0184, 0.6624, 0.874, deg(0.0), -0.98},
      {0.22, 0.0, 0.11, 0.31, deg(-18.0), -0.02},
      {-0.22, 0.0, 0.16, 0.41, deg(18.0), -0.02},
      {0.0, 0.35, 0.21, 0.25, deg(0.0), 0.01},
      {0.0, 0.1, 0.046, 0.046, deg(0.0), 0.01},
      {0.0, -0.1, 0.046, 0.046, deg(0.0), 0.01},
      {-0.08, -0.605, 0.046, 0.023, deg(0.0), 0.01},
      {0.0, -0.606, 0.023, 0.023, deg(0.0), 0.01},
      {0.06, -0.605, 0.023, 0.046, deg(0.0), 0.01},
  };
}

std::vector<Ellipse> random_ellipses(std::uint64_t seed, int count) {
  Rng rng(seed);
  std::vector<Ellipse> es(static_cast<std::size_t>(count));
  for (auto& e : es) {
    e.x0 = rng.uniform(-0.7, 0.7);
    e.y0 = rng.uniform(-0.7, 0.7);
    e.a = rng.uniform(0.05, 0.5);
    e.b = rng.uniform(0.05, 0.5);
    e.angle = rng.uniform(0.0, kPi);
    e.density = rng.uniform(0.0, 1.0);
  }
  return es;
}

// src/phantom.cpp:34-58
Vector rasterize(const std::vector<Ellipse>& es, const GridSpec& grid) {
  grid.validate();
  Vector values(static_cast<std::size_t>(grid.cell_count()), 0.0);
  const double half_w = 0.5 * grid.width();
  const double half_h = 0.5 * grid.height();
  const double y_mid = grid.y_bottom + half_h;
  for (int c = 1; c <= grid.n_x; ++c) {
    for (int r = 1; r <= grid.n_y; ++r) {
      const auto [x, y] = grid.cell_center(c, r);
      const double u = (x - grid.center_x) / half_w;
      const double v = (y - y_mid) / half_h;
      double value = 0.0;
      for (const Ellipse& e : es) {
        if (e.contains(u, v)) value += e.density;
      }
      values[snake_index(c, r, grid) - 1] = value;
    }
  }
  return values;
}

namespace {
// src/phantom.cpp:75-104
double folded_row_sum_sparse(const Csr& a, const Vector& f, Index i) {
  const Index n = a.cols;
  const Index begin = a.ptr[i], end = a.ptr[i + 1];
  double acc = 0.0;
  Index l = begin, r = end - 1;
  while (l <= r && l < end) {
    const Index cl = a.idx[l];
    const Index cr_m = mirror(a.idx[r], n);
    if (l == r) {
      acc += a.values[l] * f[cl];
      break;
    }
    if (cl < cr_m) {
      acc += a.values[l] * f[cl];
      ++l;
    } else if (cl > cr_m) {
      acc += a.values[r] * f[a.idx[r]];
      --r;
    } else {
      acc += a.values[l] * f[cl] + a.values[r] * f[a.idx[r]];
      ++l;
      --r;
    }
  }
  return acc;
}
}  // namespace

Vector forward_project_csr(const Csr& a, const Vector& f) {
  if (static_cast<Index>(f.size()) != a.cols) {
    throw Error("forward_project: image length does not match columns");
  }
  if (!all_finite(f)) throw Error("forward_project: non-finite image");
  Vector p(static_cast<std::size_t>(a.rows));
  for (Index i = 0; i < a.rows; ++i) p[i] = folded_row_sum_sparse(a, f, i);
  return p;
}

// src/phantom.cpp:108-127 (dense branch folded_row_sum_dense :65-73)
Vector forward_project(const Matrix& a, const Vector& f) {
  if (static_cast<Index>(f.size()) != a.cols()) {
    throw Error("forward_project: image length does not match columns");
  }
  if (!all_finite(f)) throw Error("forward_project: non-finite image");
  if (a.is_sparse()) return forward_project_csr(csc_to_csr(a.csc()), f);
  const Index m = a.rows(), n = a.cols();
  const Vector& d = a.dense_data();
  Vector p(static_cast<std::size_t>(m));
  for (Index i = 0; i < m; ++i) {
    double acc = 0.0;
    for (Index j = 0; j < n / 2; ++j) {
      acc += d[j * m + i] * f[j] + d[mirror(j, n) * m + i] * f[mirror(j, n)];
    }
    if (n % 2 != 0) acc += d[(n / 2) * m + i] * f[n / 2];
    p[i] = acc;
  }
  return p;
}

// src/phantom.cpp:129-149
void add_noise(Vector& p, double sigma, std::uint64_t seed) {
  if (sigma < 0) throw Error("forward_project: negative noise sigma");
  if (sigma == 0) return;
  std::mt19937_64 engine(seed);
  const auto uniform = [&engine]() {
    return (static_cast<double>(engine() >> 11) + 0.5) * 0x1.0p-53;
  };
  const Index size = static_cast<Index>(p.size());
  for (Index i = 0; i < size; i += 2) {
    const double u1 = uniform();
    const double u2 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * kPi * u2;
    p[i] += sigma * radius * std::cos(angle);
    if (i + 1 < size) p[i + 1] += sigma * radius * std::sin(angle);
  }
}

double Rng::normal() {
  const double u1 = (static_cast<double>(e_() >> 11) + 0.5) * 0x1.0p-53;
  const double u2 = (static_cast<double>(e_() >> 11) + 0.5) * 0x1.0p-53;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
}

// ------------------------------------------------------------------ solvers
namespace {
// src/solvers.cpp:28-36
void check_system(const Matrix& a, const Vector& p, const char* op) {
  if (static_cast<Index>(p.size()) != a.rows()) {
    std::ostringstream msg;
    msg << op << ": rhs length " << p.size() << " does not match rows " << a.rows();
    throw Error(msg.str());
  }
  if (!all_finite(p)) throw Error(std::string(op) + ": non-finite rhs");
}

int effective_parallelism(int requested) {
  if (requested > 0) return requested;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}
}  // namespace

// src/solvers.cpp:148-199
SolveReport sart_solve(const Matrix& a, const Vector& p, const SolveOptions& opts) {
  check_system(a, p, "sart_solve");
  if (opts.relaxation <= 0 || opts.relaxation > 2) {
    throw Error("sart_solve: relaxation must be in (0, 2]");
  }
  if (opts.max_iters < 1) throw Error("sart_solve: max_iters must be >= 1");
  const Index m = a.rows(), n = a.cols();
  Vector row_sums(static_cast<std::size_t>(m), 0.0), col_sums(static_cast<std::size_t>(n), 0.0);
  a.for_each([&](Index i, Index j, double v) {
    row_sums[i] += std::abs(v);
    col_sums[j] += std::abs(v);
  });
  double rmax = m > 0 ? row_sums[0] : 0.0;
  for (double s : row_sums) rmax = std::max(rmax, s);
  if (rmax == 0.0) throw Error("sart_solve: matrix has no nonzero rows");
  Vector row_inv(m), col_inv(n);
  for (Index i = 0; i < m; ++i) row_inv[i] = row_sums[i] > 0 ? 1.0 / row_sums[i] : 0.0;
  for (Index j = 0; j < n; ++j) col_inv[j] = col_sums[j] > 0 ? 1.0 / col_sums[j] : 0.0;

  SolveReport rep;
  const auto t0 = Clock::now();
  Vector x(static_cast<std::size_t>(n), 0.0);
  const double p_norm = norm(p);
  int it = 0;
  Vector r(m), weighted(m);
  while (it < opts.max_iters) {
    const Vector ax = a.apply(x);
    for (Index i = 0; i < m; ++i) r[i] = p[i] - ax[i];
    const double res = norm(r);
    rep.residual_history.push_back(res);
    if (res <= opts.tol * p_norm) break;
    for (Index i = 0; i < m; ++i) weighted[i] = row_inv[i] * r[i];
    const Vector bp = a.apply_transpose(weighted);
    for (Index j = 0; j < n; ++j) x[j] += opts.relaxation * (bp[j] * col_inv[j]);
    if (!all_finite(x)) {
      throw Error("sart_solve: diverged (non-finite iterate at iteration " +
                  std::to_string(it + 1) + ")");
    }
    ++it;
  }
  rep.f = std::move(x);
  rep.iterations = it;
  rep.wall_time_seconds = seconds_since(t0);
  const Vector af = a.apply(rep.f);
  Vector rr(m);
  for (Index i = 0; i < m; ++i) rr[i] = af[i] - p[i];
  rep.residual_norm = norm(rr);
  rep.solution_norm = norm(rep.f);
  return rep;
}

// src/solvers.cpp:99-146
SolveReport cgls_solve(const Matrix& a, const Vector& p, const SolveOptions& opts) {
  check_system(a, p, "cgls_solve");
  if (opts.tol <= 0) throw Error("cgls_solve: tol must be positive");
  if (opts.max_iters < 1) throw Error("cgls_solve: max_iters must be >= 1");
  SolveReport rep;
  const auto t0 = Clock::now();
  const Index m = a.rows(), n = a.cols();
  Vector x(static_cast<std::size_t>(n), 0.0);
  Vector r = p;
  Vector s = a.apply_transpose(r);
  Vector d = s;
  double gamma = squared_norm(s);
  const double stop = opts.tol * std::sqrt(gamma);
  int it = 0;
  while (it < opts.max_iters && std::sqrt(gamma) > stop) {
    const Vector q = a.apply(d);
    const double qq = squared_norm(q);
    if (qq == 0.0) break;
    const double alpha = gamma / qq;
    if (!std::isfinite(alpha)) {
      throw Error("cgls_solve: diverged (non-finite step at iteration " + std::to_string(it + 1) +
                  ")");
    }
    for (Index j = 0; j < n; ++j) x[j] += alpha * d[j];
    for (Index i = 0; i < m; ++i) r[i] -= alpha * q[i];
    s = a.apply_transpose(r);
    const double gamma_new = squared_norm(s);
    if (!std::isfinite(gamma_new)) {
      throw Error("cgls_solve: diverged (non-finite residual at iteration " +
                  std::to_string(it + 1) + ")");
    }
    const double beta = gamma_new / gamma;
    for (Index j = 0; j < n; ++j) d[j] = s[j] + beta * d[j];
    gamma = gamma_new;
    ++it;
    rep.residual_history.push_back(norm(r));
  }
  rep.f = std::move(x);
  rep.iterations = it;
  rep.wall_time_seconds = seconds_since(t0);
  const Vector af = a.apply(rep.f);
  Vector rr(static_cast<std::size_t>(m));
  for (Index i = 0; i < m; ++i) rr[i] = af[i] - p[i];
  rep.residual_norm = norm(rr);
  rep.solution_norm = norm(rep.f);
  return rep;
}

// src/solvers.cpp:38-57 (iterative methods)
SolveReport run_method(const Matrix& a, const Vector& p, const SolveOptions& o) {
  return o.method == Method::cgls ? cgls_solve(a, p, o) : sart_solve(a, p, o);
}

// src/solvers.cpp:201-205
SolveReport solve_direct_sart(const CentroSystem& sys, const SolveOptions& o) {
  return run_method(sys.a, sys.p, o);
}

SolveReport solve_split_prepared(const SplitSystem& ss, const SolveOptions& opts,
                                 bool parallel) {
  SolveReport branch[2];
  std::exception_ptr errors[2] = {nullptr, nullptr};
  const auto run_branch = [&](int which) noexcept {
    try {
      const Matrix& a = which == 0 ? ss.a1 : ss.a2;
      const Vector& p = which == 0 ? ss.p1 : ss.p2;
      branch[which] = run_method(a, p, opts);
    } catch (...) {
      errors[which] = std::current_exception();
    }
  };
  if (parallel) {
    std::thread worker(run_branch, 0);
    run_branch(1);
    worker.join();
  } else {
    run_branch(0);
    run_branch(1);
  }
  if (errors[0] || errors[1]) {
    std::ostringstream msg;
    msg << "solve_split: branch failure:";
    for (int which = 0; which < 2; ++which) {
      if (!errors[which]) continue;
      try {
        std::rethrow_exception(errors[which]);
      } catch (const std::exception& e) {
        msg << " [system " << which + 1 << "] " << e.what();
      }
    }
    throw Error(msg.str());
  }
  const auto t_rec0 = Clock::now();
  Vector f = recombine_solution({branch[0].f, branch[1].f});
  SolveReport rep;
  rep.recombine_seconds = seconds_since(t_rec0);
  rep.f = std::move(f);
  rep.iterations = std::max(branch[0].iterations, branch[1].iterations);
  rep.branch1_seconds = branch[0].wall_time_seconds;
  rep.branch2_seconds = branch[1].wall_time_seconds;
  const double bt = parallel ? std::max(rep.branch1_seconds, rep.branch2_seconds)
                             : rep.branch1_seconds + rep.branch2_seconds;
  rep.wall_time_seconds = bt + rep.recombine_seconds;
  return rep;
}

// src/solvers.cpp:207-269
SolveReport solve_split_sart(const CentroSystem& sys, const SolveOptions& opts) {
  const auto t0 = Clock::now();
  SplitSystem ss = split_system(sys);
  const double split_seconds = seconds_since(t0);
  const bool parallel = effective_parallelism(opts.parallelism) >= 2;
  SolveReport rep = solve_split_prepared(ss, opts, parallel);
  rep.split_seconds = split_seconds;
  rep.wall_time_seconds += split_seconds;
  const Vector af = sys.a.apply(rep.f);
  Vector rr(af.size());
  for (std::size_t i = 0; i < af.size(); ++i) rr[i] = af[i] - sys.p[i];
  rep.residual_norm = norm(rr);
  rep.solution_norm = norm(rep.f);
  return rep;
}

}  // namespace oracle
