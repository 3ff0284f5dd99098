// Host side of the build path: scan configuration, ray enumeration and the
// per-ray constants the GPU tracer consumes. Everything that needs libm
// (sin/cos/hypot/log) stays here so its bits match the reference's glibc
// build; the O(nnz) work happens on the device (ops.cu).
// Compiled with -ffp-contract=off (the reference host build has no FMA).
#include <algorithm>
#include <cmath>
#include <random>
#include <sstream>

#include "internal.hpp"

namespace ssb {

namespace {
constexpr double kPi = 3.14159265358979323846;

// Parametric clip of the segment [0,1] against the grid box
// (reference proj/src/geometry.cpp:19-36). Returns false for a miss.
bool clip_segment(double sx, double sy, double ex, double ey, const Grid& g, double& t_in,
                  double& t_out) {
  const double dx = ex - sx, dy = ey - sy;
  t_in = 0.0;
  t_out = 1.0;
  const auto axis = [&](double p0, double d, double lo, double hi) {
    if (d == 0.0) return p0 > lo && p0 < hi;
    double a = (lo - p0) / d, b = (hi - p0) / d;
    if (a > b) std::swap(a, b);
    t_in = std::max(t_in, a);
    t_out = std::min(t_out, b);
    return true;
  };
  if (!axis(sx, dx, g.x_left(), g.x_right())) return false;
  if (!axis(sy, dy, g.y_bottom, g.y_top())) return false;
  return t_out > t_in;
}
}  // namespace

// reference geometry.cpp:68-74
void Grid::validate() const {
  if (n_x < 2 || n_x % 2 != 0) fail("grid: n_x must be even and positive (mirror pairing)");
  if (n_y < 1) fail("grid: n_y must be positive");
  if (!(voxel_size > 0)) fail("grid: voxel_size must be positive");
}

// reference geometry.cpp:94-105
void validate_geometry(const ss_scan_config& c) {
  if (c.k < 2 || c.k % 2 != 0) fail("geometry: k must be even and >= 2 (mirror pairing)");
  if (!(c.gamma > 0) || !(c.gamma < kPi / 2)) fail("geometry: gamma must lie in (0, pi/2)");
  if (!(c.h_e > 0) || !(c.h_m > 0) || !(c.l_m > 0) || !(c.obj_size > 0)) {
    fail("geometry: lengths must be positive");
  }
  if (c.n_p < 1) fail("geometry: n_p must be >= 1");
}

// reference geometry.cpp:403-411
Grid make_grid(const ss_scan_config& c) {
  Grid g;
  g.n_x = c.grid_nx;
  g.n_y = c.grid_ny;
  g.voxel_size = c.obj_size / c.grid_nx;
  g.center_x = 0.0;
  g.y_bottom = c.h_m;
  return g;
}

// reference geometry.cpp:76-92 (1-based)
int snake_index(int c, int r, const Grid& g) {
  if (c < 1 || c > g.n_x || r < 1 || r > g.n_y) fail("snake_index: cell index out of range");
  const int base = (c - 1) * g.n_y;
  return (c & 1) ? base + r : base + (g.n_y - r + 1);
}

std::pair<int, int> snake_inverse(int j, const Grid& g) {
  if (j < 1 || j > g.cell_count()) fail("snake_inverse: index out of range");
  const int c = (j - 1) / g.n_y + 1;
  const int off = (j - 1) % g.n_y + 1;
  return {c, (c & 1) ? off : g.n_y - off + 1};
}

// Rays in reference order (geometry.cpp:107-173): emitter angle i and its
// sign-flipped partner, sources by libm sin/cos, detector samples at
// pitch max(l_m/n_p, vs/2); missing rays dropped in mirror pairs; the
// mirrored list reversed so ray M-1-i reflects ray i. Only the traced half
// (i < M/2) is kept in SoA form, with the exact clip range and hypot length
// the device walk needs.
// reference geometry.cpp:107-117: most negative first, upper half exact sign flips
std::vector<double> emitter_angles(const ss_scan_config& c) {
  validate_geometry(c);
  const int k = c.k;
  std::vector<double> ang(k);
  const double step = 2.0 * c.gamma / (k - 1);
  for (int i = 0; i < k / 2; ++i) {
    ang[i] = -c.gamma + i * step;
    ang[k - 1 - i] = -ang[i];
  }
  return ang;
}

// reference geometry.cpp:119-130: sources on the circle of radius h_e about
// (cx, h_m); the upper half reflected about x = cx (bitwise mirror pairs)
void emitter_positions(const ss_scan_config& c, double cx, std::vector<double>& srcx,
                       std::vector<double>& srcy) {
  const std::vector<double> ang = emitter_angles(c);
  const int k = c.k;
  srcx.assign(k, 0.0);
  srcy.assign(k, 0.0);
  for (int i = 0; i < k / 2; ++i) {
    srcx[i] = cx + c.h_e * std::sin(ang[i]);
    srcy[i] = c.h_m + c.h_e * std::cos(ang[i]);
    srcx[k - 1 - i] = 2.0 * cx - srcx[i];
    srcy[k - 1 - i] = srcy[i];
  }
}

bool clip_ray(double sx, double sy, double ex, double ey, const Grid& g, double& t_in,
              double& t_out) {
  return clip_segment(sx, sy, ex, ey, g, t_in, t_out);
}

RayTable enumerate_rays(const ss_scan_config& c, const Grid& g, bool keep_all) {
  validate_geometry(c);
  g.validate();
  const int k = c.k;
  const double cx = g.center_x;
  std::vector<double> srcx, srcy;
  emitter_positions(c, cx, srcx, srcy);
  const double native = c.l_m / c.n_p;
  const double pitch = std::max(native, 0.5 * g.voxel_size);
  const int samples = std::max(1, static_cast<int>(std::floor(c.l_m / pitch)));

  RayTable t;
  t.samples = samples;
  t.pitch = pitch;
  for (int pos = 0; pos < k / 2; ++pos) {
    for (int q = 0; q < samples; ++q) {
      const double ex = cx + (q + 0.5 - 0.5 * samples) * pitch;
      double tin, tout;
      if (!clip_segment(srcx[pos], srcy[pos], ex, 0.0, g, tin, tout)) continue;
      const double dx = ex - srcx[pos], dy = 0.0 - srcy[pos];
      const double seg = std::hypot(dx, dy);
      if (seg == 0.0) fail("ray_weights: degenerate ray");
      t.sx.push_back(srcx[pos]);
      t.sy.push_back(srcy[pos]);
      t.dx.push_back(dx);
      t.dy.push_back(dy);
      t.seg_len.push_back(seg);
      t.t_in.push_back(tin);
      t.t_out.push_back(tout);
    }
  }
  if (t.sx.empty()) fail("enumerate_rays: no ray intersects the reconstruction region");
  const std::int64_t mh = static_cast<std::int64_t>(t.sx.size());
  t.m = 2 * mh;
  if (keep_all) {
    t.all4.resize(static_cast<std::size_t>(4 * t.m));
    // Detector points exactly as enumerated (sx + dx could round).
    std::int64_t i = 0;
    for (int pos = 0; pos < k / 2; ++pos) {
      for (int q = 0; q < samples; ++q) {
        const double ex = cx + (q + 0.5 - 0.5 * samples) * pitch;
        double tin, tout;
        if (!clip_segment(srcx[pos], srcy[pos], ex, 0.0, g, tin, tout)) continue;
        double* a = &t.all4[4 * i];
        a[0] = srcx[pos];
        a[1] = srcy[pos];
        a[2] = ex;
        a[3] = 0.0;
        double* b = &t.all4[4 * (t.m - 1 - i)];
        b[0] = 2.0 * cx - srcx[pos];
        b[1] = srcy[pos];
        b[2] = 2.0 * cx - ex;
        b[3] = 0.0;
        ++i;
      }
    }
  }
  return t;
}

// reference geometry.cpp:352-401
ss_scan_config parse_scan_config(const std::string& text) {
  ss_scan_config c;
  c.k = 24;
  c.gamma = 30.0 * kPi / 180.0;
  c.h_e = 1.0;
  c.h_m = 0.25;
  c.l_m = 0.43;
  c.n_p = 1024;
  c.a_e = 7e-4;
  c.obj_size = 0.1;
  c.grid_nx = 32;
  c.grid_ny = 32;
  std::istringstream in(text);
  std::string line;
  long no = 0;
  while (std::getline(in, line)) {
    ++no;
    if (auto h = line.find('#'); h != std::string::npos) line.erase(h);
    std::replace_if(line.begin(), line.end(),
                    [](char ch) { return ch == '=' || ch == '\t' || ch == '\r'; }, ' ');
    std::istringstream fields(line);
    std::string key, extra;
    if (!(fields >> key)) continue;
    double v = 0.0;
    const std::string where = "config line " + std::to_string(no) + ": ";
    if (!(fields >> v)) fail(where + "missing numeric value for key '" + key + "'");
    if (fields >> extra) fail(where + "trailing content '" + extra + "'");
    if (key == "k") c.k = static_cast<int>(v);
    else if (key == "gamma_deg") c.gamma = v * kPi / 180.0;
    else if (key == "h_e") c.h_e = v;
    else if (key == "h_m") c.h_m = v;
    else if (key == "l_m") c.l_m = v;
    else if (key == "n_p") c.n_p = static_cast<int>(v);
    else if (key == "grid_nx") c.grid_nx = static_cast<int>(v);
    else if (key == "grid_ny") c.grid_ny = static_cast<int>(v);
    else if (key == "obj_size") c.obj_size = v;
    else fail(where + "unknown key '" + key + "'");
  }
  return c;
}

// BASELINE phantom: Rng = mt19937_64 with uniform =
// (e() >> 11) * 2^-53 (reference tests/support/oracles.hpp:29-38).
void random_ellipses(std::uint64_t seed, int count, double* out6) {
  std::mt19937_64 e(seed);
  const auto u = [&e](double lo, double hi) {
    return lo + (hi - lo) * (static_cast<double>(e() >> 11) * 0x1.0p-53);
  };
  for (int i = 0; i < count; ++i) {
    double* o = out6 + 6 * i;
    o[0] = u(-0.7, 0.7);
    o[1] = u(-0.7, 0.7);
    o[2] = u(0.05, 0.5);
    o[3] = u(0.05, 0.5);
    o[4] = u(0.0, kPi);
    o[5] = u(0.0, 1.0);
  }
}

// Seeded Gaussian noise on p (reference phantom.cpp:129-149): Box-Muller on
// pairs (i, i+1), uniform = ((e() >> 11) + 0.5) * 2^-53.
void add_noise(double* p, std::int64_t m, double sigma, std::uint64_t seed) {
  if (sigma < 0) fail("forward_project: negative noise sigma");
  if (sigma == 0) return;
  std::mt19937_64 e(seed);
  const auto u = [&e]() { return (static_cast<double>(e() >> 11) + 0.5) * 0x1.0p-53; };
  for (std::int64_t i = 0; i < m; i += 2) {
    const double u1 = u(), u2 = u();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * kPi * u2;
    p[i] += sigma * rad * std::cos(th);
    if (i + 1 < m) p[i + 1] += sigma * rad * std::sin(th);
  }
}

}  // namespace ssb
