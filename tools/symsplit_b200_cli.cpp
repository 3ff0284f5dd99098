// symsplit_b200 — command-line front end over the C++ facade, with the
// reference CLI's `build` and `solve` subcommands (proj/tools/main.cpp:157-259),
// flags and exit codes (0 ok, 1 check failure, 2 usage, 3 io). Everything
// numeric runs on the GPU through libsymsplit_b200.so.
//
//   symsplit_b200 build --config scan.cfg [--out-matrix a.mtx]
//                       [--phantom shepp-logan --out-rhs p.csv] [--json]
//   symsplit_b200 solve --matrix a.mtx --rhs p.csv [--mode direct|split]
//                       [--method sart|cgls] [--tol T] [--max-iters K]
//                       [--relaxation L] [--sym-tol S] [--dtype f64|f32]
//                       [--out f.csv] [--truth t.csv] [--parallel N] [--json]
//
// The reference's default --method is `dense` (Eigen complete orthogonal
// decomposition); here the default is `sart`, the B200 product path (`dense`
// runs the device SVD pseudo-inverse, capped at 5e7 entries like the reference).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <string>

#include "symsplit_b200.hpp"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitCheckFailure = 1;
constexpr int kExitUsage = 2;
constexpr int kExitIo = 3;

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::map<std::string, std::string> opt;
  bool json = false;
  std::string get(const std::string& k, const std::string& d = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? d : it->second;
  }
  bool has(const std::string& k) const { return opt.count(k) != 0; }
};

Args parse(int argc, char** argv, int first) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string k = argv[i];
    if (k == "--json") {
      a.json = true;
      continue;
    }
    if (k.rfind("--", 0) != 0) throw Usage("unexpected argument: " + k);
    if (i + 1 >= argc) throw Usage("missing value for " + k);
    a.opt[k.substr(2)] = argv[++i];
  }
  return a;
}

double num(const Args& a, const std::string& k, double d) {
  if (!a.has(k)) return d;
  try {
    return std::stod(a.get(k));
  } catch (const std::exception&) {
    throw Usage("--" + k + ": not a number");
  }
}

std::string read_text(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw symsplit::IoError("cannot open config file: " + path);
  std::ostringstream s;
  s << in.rdbuf();
  return s.str();
}

double rel_error(const symsplit::Vector& got, const symsplit::Vector& want) {
  double num2 = 0, den2 = 0;
  for (std::size_t i = 0; i < want.size(); ++i) {
    num2 += (got[i] - want[i]) * (got[i] - want[i]);
    den2 += want[i] * want[i];
  }
  return den2 > 0 ? std::sqrt(num2 / den2) : std::sqrt(num2);
}

const char* method_name(symsplit::Method m) {
  return m == symsplit::Method::cgls ? "cgls" : (m == symsplit::Method::sart ? "sart" : "dense");
}

// reference tools/main.cpp:157-201
int run_build(const Args& a) {
  if (!a.has("config")) throw Usage("build: --config is required");
  symsplit::ScanConfig cfg;
  try {
    cfg = symsplit::parse_scan_config(read_text(a.get("config")));
  } catch (const symsplit::IoError&) {
    throw;
  } catch (const symsplit::Error& e) {
    throw symsplit::IoError(std::string(e.what()) + " in " + a.get("config"));
  }
  const char* env = std::getenv("SYMSPLIT_PARALLEL");
  const int par = static_cast<int>(num(a, "parallel", env ? std::atof(env) : 0.0));
  // the reference's call shape (tools/main.cpp:160-171)
  const symsplit::GridSpec grid = symsplit::make_grid(cfg);
  symsplit::CentroSystem sys = symsplit::build_system(cfg.geom, grid, par);
  const std::string phantom = a.get("phantom");
  if (!phantom.empty()) {
    if (phantom != "shepp-logan") throw Usage("--phantom: unknown phantom: " + phantom);
    const symsplit::PhantomImage image = symsplit::rasterize(symsplit::shepp_logan_ellipses(), grid);
    sys.p = symsplit::forward_project(sys.a, image.values);
  }
  if (a.has("out-matrix")) symsplit::write_matrix_market(sys.a, a.get("out-matrix"));
  if (a.has("out-rhs")) {
    if (phantom.empty()) throw Usage("--out-rhs: requires --phantom");
    symsplit::write_vector_csv(sys.p, a.get("out-rhs"));
  }
  const symsplit::SplitSystem split = symsplit::split_system(sys);
  const auto sym = symsplit::verify_symmetry(sys.a, 0.0);
  if (a.json) {
    std::printf("{\"rows\": %lld, \"cols\": %lld, \"nnz\": %lld, \"fill\": %.17g, "
                "\"fill1\": %.17g, \"fill2\": %.17g, \"symmetric\": %s}\n",
                static_cast<long long>(sys.a.rows()), static_cast<long long>(sys.a.cols()),
                static_cast<long long>(sys.a.nonzeros()), split.parent_fill, split.fill1,
                split.fill2, sym.holds ? "true" : "false");
  } else {
    std::printf("rows=%lld cols=%lld nnz=%lld\n", static_cast<long long>(sys.a.rows()),
                static_cast<long long>(sys.a.cols()), static_cast<long long>(sys.a.nonzeros()));
    std::printf("fill=%.6f fill1=%.6f fill2=%.6f symmetric=%s\n", split.parent_fill, split.fill1,
                split.fill2, sym.holds ? "yes" : "no");
  }
  return sym.holds ? kExitOk : kExitCheckFailure;
}

// reference tools/main.cpp:206-259
int run_solve(const Args& a) {
  if (!a.has("matrix") || !a.has("rhs")) throw Usage("solve: --matrix and --rhs are required");
  symsplit::CentroSystem sys;
  sys.p = symsplit::read_vector_csv(a.get("rhs"));
  sys.a = symsplit::read_matrix_market(a.get("matrix"));
  sys.symmetry_tol = num(a, "sym-tol", 1e-12);
  if (static_cast<std::int64_t>(sys.p.size()) != sys.a.rows()) {
    throw symsplit::Error("rhs length does not match the matrix rows");
  }
  symsplit::SolveOptions o;
  const std::string method = a.get("method", "sart");
  if (method == "sart") o.method = symsplit::Method::sart;
  else if (method == "cgls") o.method = symsplit::Method::cgls;
  else if (method == "dense" || method == "dense_minnorm") o.method = symsplit::Method::dense_minnorm;
  else throw symsplit::Error("unknown method name: " + method);
  o.tol = num(a, "tol", 1e-10);
  o.max_iters = static_cast<int>(num(a, "max-iters", 2000));
  o.relaxation = num(a, "relaxation", 1.0);
  // reference --parallel / SYMSPLIT_PARALLEL worker budget; the device path is
  // deterministic for every value, so it only reaches the host-side builders
  const char* env = std::getenv("SYMSPLIT_PARALLEL");
  o.parallelism = static_cast<int>(num(a, "parallel", env ? std::atof(env) : 0.0));
  const std::string dtype = a.get("dtype", "f64");
  if (dtype != "f64" && dtype != "f32") throw Usage("--dtype: must be f64 or f32");
  o.dtype = dtype == "f32" ? SS_F32 : SS_F64;
  const std::string mode = a.get("mode", "direct");
  symsplit::SolveReport rep;
  if (mode == "direct") {
    rep = symsplit::solve_direct(sys, o);
  } else if (mode == "split") {
    try {
      rep = symsplit::solve_split(sys, o);
    } catch (const symsplit::SymmetryError& e) {
      std::ostringstream msg;
      msg << "split mode needs a centrosymmetric matrix: max violation "
          << e.report.max_violation << " at (" << e.report.worst_row << ","
          << e.report.worst_col << ") exceeds tol " << sys.symmetry_tol;
      throw symsplit::Error(msg.str());
    }
  } else {
    throw Usage("--mode: must be direct or split");
  }
  if (a.has("out")) symsplit::write_vector_csv(rep.f, a.get("out"));
  double err = -1.0;
  if (a.has("truth")) err = rel_error(rep.f, symsplit::read_vector_csv(a.get("truth")));
  if (a.json) {
    std::printf("{\"method\": \"%s\", \"mode\": \"%s\", \"residual_norm\": %.17g, "
                "\"solution_norm\": %.17g, \"iterations\": %d, \"wall_time_seconds\": %.17g",
                method_name(rep.method), mode.c_str(), rep.residual_norm, rep.solution_norm,
                rep.iterations, rep.wall_time_seconds);
    if (mode == "split") {
      std::printf(", \"split_seconds\": %.17g, \"recombine_seconds\": %.17g, "
                  "\"branch_seconds\": [%.17g, %.17g]",
                  rep.split_seconds, rep.recombine_seconds, rep.branch1_seconds,
                  rep.branch2_seconds);
    }
    if (err >= 0) std::printf(", \"rel_error\": %.17g", err);
    std::printf("}\n");
  } else {
    std::printf("method=%s mode=%s iterations=%d residual=%.6e |f|=%.6e time=%.4fs\n",
                method_name(rep.method), mode.c_str(), rep.iterations, rep.residual_norm,
                rep.solution_norm, rep.wall_time_seconds);
    if (err >= 0) std::printf("rel_error=%.6e\n", err);
  }
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: symsplit_b200 {build|solve} [options]\n");
    return kExitUsage;
  }
  const std::string cmd = argv[1];
  try {
    const Args a = parse(argc, argv, 2);
    if (cmd == "build") return run_build(a);
    if (cmd == "solve") return run_solve(a);
    throw Usage("unknown subcommand: " + cmd);
  } catch (const Usage& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitUsage;
  } catch (const symsplit::IoError& e) {
    std::fprintf(stderr, "io error: %s\n", e.what());
    return kExitIo;
  } catch (const symsplit::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitCheckFailure;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "unexpected error: %s\n", e.what());
    return kExitCheckFailure;
  }
}
