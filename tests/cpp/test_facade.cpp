// C++ facade (include/symsplit_b200.hpp) exercised like the reference's own
// doctest unit tests (proj/tests/unit/test_centro.cpp, test_solvers.cpp),
// checked against the oracle (test infrastructure). Prints "ALL PASSED".
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/symsplit_b200.hpp"
#include "../../oracle/oracle.hpp"

static int failures = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    if (!(c)) {                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);          \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

int main() {
  using namespace symsplit;
  // Example 1 (oracles.hpp:165-178), column-major
  const Vector ex1 = {1, 2, 7, 1, 3, 4, 3, 9, 5, 6, 8, 7, 7, 8, 6, 5, 9, 3, 4, 3, 1, 7, 2, 1};
  const Vector rhs = {5, 6, 8, 7};
  {  // test_centro.cpp:66-85, :126-133
    const SplitSystem s = split_system({Matrix::dense(4, 6, ex1), rhs, 0.0});
    std::vector<int32_t> o, i;
    Vector v;
    s.a1.to_csc(o, i, v);
    CHECK(s.a1.nonzeros() == 5 && v.size() == 5);
    CHECK(s.p1[0] == -2.0 && s.p1[1] == -2.0 && s.p2[0] == 12.0 && s.p2[1] == 14.0);
    const Vector e2 = {2, 9, 12, 7, 12, 14};  // a2 column-major
    s.a2.to_csc(o, i, v);
    CHECK(v.size() == 6);
    for (std::size_t k = 0; k < v.size(); ++k) CHECK(v[k] == e2[k]);
  }
  {  // test_centro.cpp:114-124
    Vector bad = ex1;
    bad[0] = 9;
    bool thrown = false;
    try {
      split_system({Matrix::dense(4, 6, bad), rhs, 1e-12});
    } catch (const SymmetryError& e) {
      thrown = e.report.max_violation == 8.0 && e.report.worst_row == 1;
    }
    CHECK(thrown);
  }
  {  // test_centro.cpp:215-228
    const Vector f = recombine_solution({{14, 10, -29}, {84, 80, -93}});
    const Vector want = {49, 45, -61, -32, 35, 35};
    for (int k = 0; k < 6; ++k) CHECK(f[k] == want[k]);
  }
  {  // test_solvers.cpp:153-171
    Vector eye(25, 0.0), p = {0.5, 0.25, 0.75, 0.125, 1.0};
    for (int k = 0; k < 5; ++k) eye[k * 5 + k] = 1.0;
    SolveOptions o;
    o.tol = 1e-12;
    const SolveReport r = sart_solve(Matrix::dense(5, 5, eye), p, o);
    CHECK(r.iterations == 1);
    for (int k = 0; k < 5; ++k) CHECK(std::abs(r.f[k] - p[k]) <= 1e-12);
    bool thrown = false;
    try {
      sart_solve(Matrix::from_triplets(4, 4, {}), Vector(4, 1.0), SolveOptions{});
    } catch (const Error& e) {
      thrown = std::string(e.what()).find("no nonzero rows") != std::string::npos;
    }
    CHECK(thrown);
  }
  {  // BASELINE config 1 through the facade vs the oracle
    // the reference CLI's call shape (tools/main.cpp:160-162, :278, :406-407)
    ScanConfig cfg;
    cfg.geom.k = 10;
    cfg.geom.gamma = degrees_to_radians(18.0);
    cfg.geom.h_e = 2.0;
    cfg.geom.h_m = 1e-4;
    cfg.geom.l_m = 1.0;
    cfg.geom.n_p = 128;
    cfg.geom.obj_size = 1.0;
    cfg.grid_nx = cfg.grid_ny = 64;
    const int parallelism = 0;
    const GridSpec grid = make_grid(cfg);
    CentroSystem sys = build_system(cfg.geom, grid, parallelism);
    CHECK(sys.a.rows() == 1280 && sys.a.stored() == 98032 && sys.symmetry_tol == 0.0);
    std::vector<double> ell(48);
    ss_random_ellipses(1000, 8, ell.data());
    std::vector<Ellipse> es;
    for (int q = 0; q < 8; ++q) {
      es.push_back({ell[6 * q], ell[6 * q + 1], ell[6 * q + 2], ell[6 * q + 3], ell[6 * q + 4],
                    ell[6 * q + 5]});
    }
    const PhantomImage truth = rasterize(es, grid);
    CHECK(truth.values.size() == 4096 && truth.max_value >= truth.min_value);
    sys.p = forward_project(sys.a, truth.values);
    SolveOptions o;
    o.max_iters = 50;
    o.tol = 0.0;
    const SolveReport got = solve_split(sys, o);

    oracle::ScanConfig oc;
    oc.geom.k = 10;
    oc.geom.gamma = oracle::degrees_to_radians(18.0);
    oc.geom.h_e = 2.0;
    oc.geom.h_m = 1e-4;
    oc.geom.l_m = 1.0;
    oc.geom.n_p = 128;
    oc.geom.obj_size = 1.0;
    oc.grid_nx = oc.grid_ny = 64;
    oracle::CentroSystem os = oracle::build_system(oc.geom, oracle::make_grid(oc));
    os.p = sys.p;
    {  // Matrix::coeff / for_each / to_dense (matrix.hpp:53-81) on the built A
      std::vector<int32_t> outer, inner;
      Vector vals;
      sys.a.to_csc(outer, inner, vals);
      const auto& oa = os.a;
      std::size_t k = 0;
      bool order_ok = true;
      sys.a.for_each([&](Index i, Index j, double v) {
        order_ok = order_ok && k < vals.size() && inner[k] == i && vals[k] == v &&
                   outer[static_cast<std::size_t>(j)] <= static_cast<int32_t>(k) &&
                   static_cast<int32_t>(k) < outer[static_cast<std::size_t>(j) + 1];
        ++k;
      });
      CHECK(order_ok && k == vals.size());
      // coeff at stored entries and at a zero, bit for bit with the oracle
      bool coeff_ok = true;
      for (std::size_t q = 0; q < vals.size(); q += 997) {
        Index j = 0;
        while (outer[static_cast<std::size_t>(j) + 1] <= static_cast<int32_t>(q)) ++j;
        coeff_ok = coeff_ok && sys.a.coeff(inner[q], j) == vals[q] &&
                   oa.coeff(inner[q], j) == vals[q];
      }
      CHECK(coeff_ok);
      CHECK(sys.a.coeff(0, 4095) == oa.coeff(0, 4095));
      bool thrown = false;
      try {
        sys.a.coeff(1280, 0);
      } catch (const Error& e) {
        thrown = std::string(e.what()) == "matrix index out of range";
      }
      CHECK(thrown);
      const DenseStorage d = sys.a.to_dense();
      double dsum = 0.0, vsum = 0.0;
      for (double v : d.data) dsum += v;
      for (double v : vals) vsum += v;
      CHECK(d.rows() == 1280 && d.cols() == 4096 && std::abs(dsum - vsum) <= 1e-9 * vsum);
      CHECK(d(inner[0], 0) == vals[0]);
      // enumerate_rays / GridSpec helpers with the reference's numbers
      const RaySet rays = enumerate_rays(cfg.geom, grid);
      CHECK(rays.count() == 1280 && rays.positions == 10 && rays.samples_per_position == 128);
      const auto cc = grid.cell_center(1, 1);
      const auto occ = oracle::make_grid(oc).cell_center(1, 1);
      CHECK(cc.first == occ.first && cc.second == occ.second);
    }
    oracle::SolveOptions oo;
    oo.max_iters = 50;
    oo.tol = 0.0;
    const oracle::SolveReport want = oracle::solve_split_sart(os, oo);
    double num = 0, den = 0;
    for (std::size_t k = 0; k < want.f.size(); ++k) {
      num += (got.f[k] - want.f[k]) * (got.f[k] - want.f[k]);
      den += want.f[k] * want.f[k];
    }
    CHECK(std::sqrt(num / den) <= 1e-10);
    CHECK(got.iterations == 50 && got.mode == Mode::split);
  }
  {  // geometry entry points (geometry.cpp:107-225) against the oracle, bit for bit
    const ScanGeometry c = parse_scan_config("k 10\ngamma_deg 18\nh_e 2.0\nh_m 1e-4\n").geom;
    oracle::ScanGeometry og;
    og.k = 10;
    og.gamma = oracle::degrees_to_radians(18.0);
    og.h_e = 2.0;
    og.h_m = 1e-4;
    const std::vector<double> a = emitter_angles(c);
    const std::vector<double> oa = oracle::emitter_angles(og);
    CHECK(a.size() == oa.size() && std::equal(a.begin(), a.end(), oa.begin()));
    const std::vector<Point> pos = emitter_positions(c, 0.0);
    const auto opos = oracle::emitter_positions(og, 0.0);
    bool same = pos.size() == opos.size();
    for (std::size_t i = 0; same && i < pos.size(); ++i) {
      same = pos[i].x == opos[i].x && pos[i].y == opos[i].y;
    }
    CHECK(same);
    bool bad = false;  // ScanGeometry::validate (geometry.cpp:94-105)
    try {
      ScanGeometry odd;
      odd.k = 3;
      odd.validate();
    } catch (const Error& e) {
      bad = std::string(e.what()) == "geometry: k must be even and >= 2 (mirror pairing)";
    }
    CHECK(bad);
    GridSpec g{4, 5, 0.1, 0.0, 1.0};
    const double xc = (2 - 0.5 - 0.5 * 4) * 0.1;
    const auto w = ray_weights(Ray{{xc, 3.0}, {xc, 0.0}}, g);
    CHECK(w.size() == 5);
    for (const auto& e : w) CHECK(std::abs(e.second - 0.1) <= 1e-12);
  }
  if (failures == 0) std::printf("ALL PASSED\n");
  return failures == 0 ? 0 : 1;
}
