// Dense minimum-norm solve (reference pseudo_solve_dense, proj/src/solvers.cpp:81-97,
// SURVEY §8f rank 4): the reference densifies the system and solves it with
// Eigen's complete orthogonal decomposition at threshold max(m,n)*eps; its own
// tests pin that against the SVD pseudo-inverse (tests/support/oracles.hpp:101-113).
// Here: densify on the device (column-major, arranged tall), one cuSOLVER gesvd
// (a library factorisation, like a cuBLAS GEMM — this is not the SART path), and
// the pseudo-inverse apply x = V diag(1/s_i, s_i > max(m,n)*eps*s_0) U^T p with
// fixed-order matvec kernels. cuSOLVER is resolved with dlopen at first use, so a
// process that already loaded one (PyTorch's) keeps it.
#include <cusolverDn.h>
#include <dlfcn.h>

#include <algorithm>
#include <cfloat>
#include <mutex>
#include <sstream>
#include <string>

#include "internal.hpp"

namespace ssb {

namespace {

struct CusolverApi {
  cusolverStatus_t (*Create)(cusolverDnHandle_t*) = nullptr;
  cusolverStatus_t (*Destroy)(cusolverDnHandle_t) = nullptr;
  cusolverStatus_t (*SetStream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
  cusolverStatus_t (*GesvdBufferSize)(cusolverDnHandle_t, int, int, int*) = nullptr;
  cusolverStatus_t (*Gesvd)(cusolverDnHandle_t, signed char, signed char, int, int, double*, int,
                            double*, double*, int, double*, int, double*, int, double*,
                            int*) = nullptr;
};

const CusolverApi& cusolver() {
  static CusolverApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      const char* e = dlerror();
      err = e ? e : "dlopen failed";
      return;
    }
    api.Create = reinterpret_cast<decltype(api.Create)>(dlsym(h, "cusolverDnCreate"));
    api.Destroy = reinterpret_cast<decltype(api.Destroy)>(dlsym(h, "cusolverDnDestroy"));
    api.SetStream = reinterpret_cast<decltype(api.SetStream)>(dlsym(h, "cusolverDnSetStream"));
    api.GesvdBufferSize = reinterpret_cast<decltype(api.GesvdBufferSize)>(
        dlsym(h, "cusolverDnDgesvd_bufferSize"));
    api.Gesvd = reinterpret_cast<decltype(api.Gesvd)>(dlsym(h, "cusolverDnDgesvd"));
  });
  if (!api.Create || !api.Destroy || !api.SetStream || !api.GesvdBufferSize || !api.Gesvd) {
    fail("cuSOLVER unavailable: " + (err.empty() ? std::string("missing symbols") : err),
         SS_ERR_CUDA);
  }
  return api;
}

void solver_check(cusolverStatus_t s, const char* what) {
  if (s != CUSOLVER_STATUS_SUCCESS) {
    fail(std::string(what) + ": cuSOLVER status " + std::to_string(static_cast<int>(s)),
         SS_ERR_CUDA);
  }
}

cusolverDnHandle_t solver_handle(Context* ctx) {
  const CusolverApi& api = cusolver();
  if (!ctx->solver) {
    cusolverDnHandle_t h = nullptr;
    solver_check(api.Create(&h), "cusolverDnCreate");
    ctx->solver = h;
  }
  auto h = static_cast<cusolverDnHandle_t>(ctx->solver);
  solver_check(api.SetStream(h, ctx->stream), "cusolverDnSetStream");
  return h;
}

constexpr int kT = 256;

int grid_n(Context* ctx, long long n) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((n + kT - 1) / kT,
                                                                     ctx->sm_count * 8LL)));
}

// B (r x c, column-major, r = max(m,n)) = A when m >= n, A^T otherwise
__global__ void densify_kernel(const int* __restrict__ ptr, const int* __restrict__ col,
                               const double* __restrict__ val, long long m, bool tall,
                               long long ld, double* __restrict__ b) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
      const long long j = col[k];
      b[tall ? i + j * ld : j + i * ld] = val[k];  // compressed storage: one entry per (i, j)
    }
  }
}

// y[j] = sum_i M[i + j*ld] v[i], i ascending (one warp per output)
__global__ void matvec_t_kernel(const double* __restrict__ mat, long long rows, long long cols,
                                long long ld, const double* __restrict__ v, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (long long j = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; j < cols;
       j += ((long long)gridDim.x * blockDim.x) >> 5) {
    double s = 0.0;
    for (long long i = lane; i < rows; i += 32) s += mat[i + j * ld] * v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[j] = s;
  }
}

// y[i] = sum_j M[i + j*ld] v[j], j ascending (one thread per output, coalesced)
__global__ void matvec_kernel(const double* __restrict__ mat, long long rows, long long cols,
                              long long ld, const double* __restrict__ v, double* __restrict__ y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows;
       i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (long long j = 0; j < cols; ++j) s += mat[i + j * ld] * v[j];
    y[i] = s;
  }
}

// y_i /= s_i for s_i > cutoff = max(m,n)*eps*s_0, else 0 (the pseudo-inverse)
__global__ void pinv_scale_kernel(const double* __restrict__ s, long long k, double factor,
                                  double* __restrict__ y) {
  const double cutoff = k > 0 ? factor * s[0] : 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < k;
       i += (long long)gridDim.x * blockDim.x) {
    y[i] = s[i] > cutoff ? y[i] / s[i] : 0.0;
  }
}

}  // namespace

void pseudo_solve_dense_dev(Matrix& a, const double* p, double* f, std::int64_t dense_cap) {
  Context* ctx = a.ctx;
  const std::int64_t m = a.rows, n = a.cols;
  if (m * n > dense_cap) {
    std::ostringstream msg;
    msg << "pseudo_solve_dense: " << m << "x" << n << " exceeds the dense cap of " << dense_cap
        << " entries";
    fail(msg.str());
  }
  if (n > 0) SSB_CUDA(cudaMemsetAsync(f, 0, n * sizeof(double), ctx->stream));
  if (m == 0 || n == 0) {
    ctx->sync();
    return;
  }
  if (std::max(m, n) > 0x7fffffff / std::max<std::int64_t>(1, std::min(m, n))) {
    fail("pseudo_solve_dense: matrix too large for the dense factorisation");
  }
  const bool tall = m >= n;
  const int r = static_cast<int>(std::max(m, n)), c = static_cast<int>(std::min(m, n));
  DBuf<double> b(static_cast<std::size_t>(r) * c), s(c), u(static_cast<std::size_t>(r) * c),
      vt(static_cast<std::size_t>(c) * c), y(c), rwork(c);
  DBuf<int> info(1);
  SSB_CUDA(cudaMemsetAsync(b.get(), 0, sizeof(double) * r * c, ctx->stream));
  densify_kernel<<<grid_n(ctx, m), kT, 0, ctx->stream>>>(a.rowptr.get(), a.colidx.get(),
                                                        a.val.get(), m, tall, tall ? m : n,
                                                        b.get());
  ctx->check_launch("densify_kernel");
  const CusolverApi& api = cusolver();
  cusolverDnHandle_t h = solver_handle(ctx);
  int lwork = 0;
  solver_check(api.GesvdBufferSize(h, r, c, &lwork), "cusolverDnDgesvd_bufferSize");
  DBuf<double> work(std::max(lwork, 1));
  // thin SVD B = U diag(s) VT (gesvd requires rows >= cols: B is arranged tall)
  solver_check(api.Gesvd(h, 'S', 'S', r, c, b.get(), r, s.get(), u.get(), r, vt.get(), c,
                         work.get(), lwork, rwork.get(), info.get()),
               "cusolverDnDgesvd");
  int inf = 0;
  ctx->copy(&inf, info.get(), sizeof(int));
  if (inf != 0) fail("pseudo_solve_dense: SVD did not converge (info " + std::to_string(inf) + ")");
  const double factor = static_cast<double>(std::max(m, n)) * DBL_EPSILON;
  if (tall) {  // A = U S VT: x = VT^T S+ U^T p
    matvec_t_kernel<<<grid_n(ctx, 32LL * c), kT, 0, ctx->stream>>>(u.get(), r, c, r, p, y.get());
    pinv_scale_kernel<<<grid_n(ctx, c), kT, 0, ctx->stream>>>(s.get(), c, factor, y.get());
    matvec_t_kernel<<<grid_n(ctx, 32LL * c), kT, 0, ctx->stream>>>(vt.get(), c, c, c, y.get(), f);
  } else {     // A^T = U S VT, A = VT^T S U^T: x = U S+ VT p
    matvec_kernel<<<grid_n(ctx, c), kT, 0, ctx->stream>>>(vt.get(), c, c, c, p, y.get());
    pinv_scale_kernel<<<grid_n(ctx, c), kT, 0, ctx->stream>>>(s.get(), c, factor, y.get());
    matvec_kernel<<<grid_n(ctx, r), kT, 0, ctx->stream>>>(u.get(), r, c, r, y.get(), f);
  }
  ctx->check_launch("pseudo-inverse apply");
  ctx->sync();
}

void release_solver(Context* ctx) {
  if (ctx->solver) {
    cusolver().Destroy(static_cast<cusolverDnHandle_t>(ctx->solver));
    ctx->solver = nullptr;
  }
}

}  // namespace ssb
