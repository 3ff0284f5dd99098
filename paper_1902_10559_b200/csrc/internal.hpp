// Internal types of the symsplit_b200 library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <memory>
#include <vector>

#include "../../include/symsplit_b200.h"

namespace ssb {

// Status-carrying exception; the C ABI maps it to SS_ERR_* + message.
struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(const std::string& msg, int code = SS_ERR_INVALID) {
  throw Failure(code, msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw Failure(SS_ERR_OOM, std::string(what) + ": out of device memory");
  }
  throw Failure(SS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define SSB_CUDA(x) ::ssb::cuda_check((x), #x)

constexpr std::size_t kSlackBytes = 128;

// Stream on which device buffers are allocated and freed (stream-ordered
// pool allocator). Every C-ABI entry point sets it to its context's stream,
// so allocation, use and release are ordered on one stream and the pool
// hands memory back without device-wide synchronisation.
cudaStream_t& alloc_stream();

// Owning device buffer from the stream-ordered pool (cudaMallocAsync; 256-byte
// aligned, which the 128-bit loads of the SpMV kernels rely on).
template <class T>
class DBuf {
 public:
  DBuf() = default;
  explicit DBuf(std::size_t n) { alloc(n); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) { o.p_ = nullptr; o.n_ = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      s_ = o.s_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(std::size_t n) {
    release();
    if (n == 0) n = 1;  // keep a valid pointer for empty arrays
    void* q = nullptr;
    s_ = alloc_stream();
    // 128 bytes of slack: vector loads may round the last access up.
    SSB_CUDA(cudaMallocAsync(&q, n * sizeof(T) + kSlackBytes, s_));
    p_ = static_cast<T*>(q);
    n_ = n;
  }
  void release() {
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  explicit operator bool() const { return p_ != nullptr; }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
  cudaStream_t s_ = nullptr;
};

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  std::size_t l2_bytes = 0;
  std::int64_t launches = 0;
  DBuf<char> scratch;  // CUB temporary storage, grown on demand
  // NCCL (row-sharded plans); opaque to avoid the header here
  void* comm = nullptr;
  int nranks = 1, rank = 0;
  void* solver = nullptr;   // cuSOLVER handle (dense min-norm path), created on first use
  void* solver2 = nullptr;  // second handle + stream: the concurrent folded branch
  cudaStream_t side = nullptr;

  void* temp(std::size_t bytes) {
    if (scratch.size() < bytes) scratch.alloc(bytes + bytes / 4);
    return scratch.get();
  }
  void launched(int n = 1) { launches += n; }
  // blocking copy ordered on this context's stream (never on the legacy stream)
  void copy(void* dst, const void* src, std::size_t bytes) {
    if (bytes) SSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, stream));
    sync();
  }
  void sync() { SSB_CUDA(cudaStreamSynchronize(stream)); }
  void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) cuda_check(e, what);
    ++launches;
  }
};

// Second stream of a context: the concurrent folded branch of solve_split
// (dense and CGLS methods), created on first use and destroyed with the context.
inline cudaStream_t side_stream(Context* ctx) {
  if (!ctx->side) SSB_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
  return ctx->side;
}

// Phase timing for diagnostics (SSB_TRACE=1 prints to stderr).
struct PhaseTrace {
  Context* ctx;
  bool on;
  std::chrono::steady_clock::time_point t;
  explicit PhaseTrace(Context* c)
      : ctx(c), on(std::getenv("SSB_TRACE") != nullptr), t(std::chrono::steady_clock::now()) {}
  void mark(const char* what) {
    if (!on) return;
    ctx->sync();
    const auto n = std::chrono::steady_clock::now();
    cudaMemPool_t pool;
    unsigned long long reserved = 0;
    if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) {
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    }
    std::fprintf(stderr, "[ssb]     %-24s %9.3f ms  (pool %llu MB)\n", what,
                 std::chrono::duration<double, std::milli>(n - t).count(), reserved >> 20);
    t = n;
  }
};

// Device sparse matrix: CSR master (fp64, int32 — Eigen's int StorageIndex),
// CSC and fp32 copies built on demand. Rows/cols are 0-based.
struct Matrix {
  Context* ctx = nullptr;
  std::int64_t rows = 0, cols = 0, nnz = 0;
  DBuf<int> rowptr, colidx;
  DBuf<double> val;
  bool has_csc = false;
  DBuf<int> colptr, rowidx;
  DBuf<double> cval;
  bool has_f32 = false;
  DBuf<float> val32, cval32;
  DBuf<int> csc_perm;  // CSR position of each CSC entry (kept on request)
  // solve_split's derived data of this (immutable) matrix -- its fold A1/A2
  // and the paired SART plan over them -- kept for the next call (capi.cu)
  std::shared_ptr<struct SolveCache> solve_cache;

  void ensure_csc(bool keep_perm = false);
  // CSC of a matrix with ref's exact CSR pattern: ref's ordering, own values
  void csc_like(const Matrix& ref);
  void ensure_f32();
};

// ---------------------------------------------------------------- host geometry
struct Grid {
  int n_x = 32, n_y = 32;
  double voxel_size = 0.1 / 32, center_x = 0.0, y_bottom = 0.25;
  int cell_count() const { return n_x * n_y; }
  double width() const { return n_x * voxel_size; }
  double height() const { return n_y * voxel_size; }
  double x_left() const { return center_x - 0.5 * width(); }
  double x_right() const { return center_x + 0.5 * width(); }
  double y_top() const { return y_bottom + height(); }
  void validate() const;
};

struct RayTable {  // traced half, structure of arrays (host)
  std::int64_t m = 0;  // total rays M (both halves)
  int samples = 0;
  double pitch = 0.0;
  std::vector<double> sx, sy, dx, dy, seg_len, t_in, t_out;  // M/2 each
  std::vector<double> all4;                                  // optional (sx,sy,dx,dy) x M
};

void validate_geometry(const ss_scan_config& c);
Grid make_grid(const ss_scan_config& c);
RayTable enumerate_rays(const ss_scan_config& c, const Grid& g, bool keep_all);
std::vector<double> emitter_angles(const ss_scan_config& c);
void emitter_positions(const ss_scan_config& c, double center_x, std::vector<double>& x,
                       std::vector<double>& y);
bool clip_ray(double sx, double sy, double ex, double ey, const Grid& g, double& t_in,
              double& t_out);
// reference ray_weights (geometry.cpp:175-225) for one ray, walked on the
// device with the build's tracer: (1-based snake column, length) in path order
void ray_weights_dev(Context* ctx, double sx, double sy, double ex, double ey, const Grid& g,
                     std::vector<int>& cols, std::vector<double>& lens);
ss_scan_config parse_scan_config(const std::string& text);
int snake_index(int c, int r, const Grid& g);
std::pair<int, int> snake_inverse(int j, const Grid& g);
void random_ellipses(std::uint64_t seed, int count, double* out6);
void add_noise(double* p, std::int64_t m, double sigma, std::uint64_t seed);

// ---------------------------------------------------------------- device ops (ops.cu)
Matrix* matrix_from_csr_device(Context* ctx, std::int64_t rows, std::int64_t cols,
                               std::int64_t nnz, DBuf<int>&& rowptr, DBuf<int>&& colidx,
                               DBuf<double>&& val);
Matrix* matrix_from_sorted_triplets(Context* ctx, std::int64_t rows, std::int64_t cols,
                                    std::int64_t count, unsigned long long* keys,
                                    double* vals);
Matrix* matrix_from_triplets_host(Context* ctx, std::int64_t rows, std::int64_t cols,
                                  std::int64_t count, const int* r, const int* c,
                                  const double* v);
Matrix* matrix_from_csc_host(Context* ctx, std::int64_t rows, std::int64_t cols,
                             std::int64_t nnz, const int* outer, const int* inner,
                             const double* v);
Matrix* build_system(Context* ctx, const ss_scan_config& cfg);
Matrix* build_system(Context* ctx, const ss_scan_config& cfg, const Grid& g);
void check_finite(Matrix& a);
std::int64_t nonzeros(Matrix& a);
ss_symmetry_report verify_symmetry(Matrix& a, double tol);
void fold(Matrix& a, Matrix*& a1, Matrix*& a2);
// fold with the symmetry check fused in; !holds -> a1 = a2 = nullptr
ss_symmetry_report fold_checked(Matrix& a, double tol, Matrix*& a1, Matrix*& a2);
bool same_pattern(Matrix& a, Matrix& b);
void scan_counts(Context* ctx, const int* counts_np1, int* ptr, std::int64_t n);
// dense minimum-norm solve of a (reference pseudo_solve_dense), p and f on the device
void pseudo_solve_dense_dev(Matrix& a, const double* p, double* f, std::int64_t dense_cap);
// both folded branches concurrently (main + side stream, two host threads);
// per-branch wall seconds; a failing branch leaves its message and code
void pseudo_solve_dense_pair(Matrix* a[2], const double* p[2], double* f[2],
                             std::int64_t dense_cap, double seconds[2], std::string errs[2],
                             int codes[2]);
void release_solver(Context* ctx);
void union_pattern(Matrix& a, Matrix& b, Matrix*& ua, Matrix*& ub);
void split_rhs_dev(Context* ctx, const double* p, double* p1, double* p2, std::int64_t mh);
void recombine_dev(Context* ctx, const double* f1, const double* f2, double* f,
                   std::int64_t nh, std::int64_t nrhs);
void decompose_dev(Context* ctx, const double* f, double* f1, double* f2, std::int64_t nh);
void abs_sums(Matrix& a, double* row_sums, double* col_sums);
void apply_dev(Matrix& a, const double* x, double* y);            // y = A x
void apply_transpose_dev(Matrix& a, const double* y, double* x);  // x = A^T y
void residual_dev(Matrix& a, const double* x, const double* p, double* r);  // r = A x - p
double norm2_dev(Context* ctx, const double* v, std::int64_t n);  // deterministic sum of squares
double max_dev(Context* ctx, const double* v, std::int64_t n);
bool all_finite_dev(Context* ctx, const double* v, std::int64_t n);
void rasterize_dev(Context* ctx, const double* ell6, int count, const Grid& g, double* out);
void forward_project_dev(Matrix& a, const double* f, double* p);
// CGLS (cgls.cu): f_dev receives x in fp64; report gets iterations/history/time
void cgls_device_pair(Matrix* a[2], const double* p[2], const ss_solve_options& o, double* f[2],
                      ss_solve_report rep[2], std::string errs[2], int codes[2]);
// both folded systems in one CGLS loop over the paired tiled streams (sart.cu)
void cgls_device_paired(Matrix* a1, Matrix* a2, const double* p[2], const ss_solve_options& o,
                        double* f[2], ss_solve_report rep[2], std::string errs[2], int codes[2]);
void cgls_device(Matrix& a, const double* p_dev, const ss_solve_options& o, double* f_dev,
                 ss_solve_report* rep, double* hist_host);

template <class T>
void cast_dev(Context* ctx, const double* src, T* dst, std::int64_t n);

}  // namespace ssb
