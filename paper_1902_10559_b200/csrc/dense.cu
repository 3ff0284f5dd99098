// Dense minimum-norm solve (reference pseudo_solve_dense, proj/src/solvers.cpp:81-97,
// SURVEY §8f rank 4): the reference densifies the system and solves it with
// Eigen's complete orthogonal decomposition at threshold max(m,n)*eps; its own
// tests pin that against the SVD pseudo-inverse (tests/support/oracles.hpp:101-113).
// Here: densify on the device (column-major, arranged tall), cuSOLVER geqrf +
// an SVD of the square factor R (library factorisations, like a cuBLAS GEMM —
// this is not the SART path), and
// the pseudo-inverse apply x = V diag(1/s_i, s_i > max(m,n)*eps*s_0) U^T p with
// fixed-order matvec kernels. cuSOLVER is resolved with dlopen at first use, so a
// process that already loaded one (PyTorch's) keeps it.
#include <cusolverDn.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cfloat>
#include <cstdlib>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>

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
  cusolverStatus_t (*GeqrfBufferSize)(cusolverDnHandle_t, int, int, double*, int, int*) = nullptr;
  cusolverStatus_t (*Geqrf)(cusolverDnHandle_t, int, int, double*, int, double*, double*, int,
                            int*) = nullptr;
  cusolverStatus_t (*OrmqrBufferSize)(cusolverDnHandle_t, cublasSideMode_t, cublasOperation_t,
                                      int, int, int, const double*, int, const double*,
                                      const double*, int, int*) = nullptr;
  cusolverStatus_t (*Ormqr)(cusolverDnHandle_t, cublasSideMode_t, cublasOperation_t, int, int,
                            int, const double*, int, const double*, double*, int, double*, int,
                            int*) = nullptr;
  cusolverStatus_t (*CreateGesvdjInfo)(gesvdjInfo_t*) = nullptr;
  cusolverStatus_t (*DestroyGesvdjInfo)(gesvdjInfo_t) = nullptr;
  cusolverStatus_t (*GesvdjBufferSize)(cusolverDnHandle_t, cusolverEigMode_t, int, int, int,
                                       const double*, int, const double*, const double*, int,
                                       const double*, int, int*, gesvdjInfo_t) = nullptr;
  cusolverStatus_t (*Gesvdj)(cusolverDnHandle_t, cusolverEigMode_t, int, int, int, double*, int,
                             double*, double*, int, double*, int, double*, int, int*,
                             gesvdjInfo_t) = nullptr;
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
    api.GeqrfBufferSize = reinterpret_cast<decltype(api.GeqrfBufferSize)>(
        dlsym(h, "cusolverDnDgeqrf_bufferSize"));
    api.Geqrf = reinterpret_cast<decltype(api.Geqrf)>(dlsym(h, "cusolverDnDgeqrf"));
    api.OrmqrBufferSize = reinterpret_cast<decltype(api.OrmqrBufferSize)>(
        dlsym(h, "cusolverDnDormqr_bufferSize"));
    api.Ormqr = reinterpret_cast<decltype(api.Ormqr)>(dlsym(h, "cusolverDnDormqr"));
    api.CreateGesvdjInfo = reinterpret_cast<decltype(api.CreateGesvdjInfo)>(
        dlsym(h, "cusolverDnCreateGesvdjInfo"));
    api.DestroyGesvdjInfo = reinterpret_cast<decltype(api.DestroyGesvdjInfo)>(
        dlsym(h, "cusolverDnDestroyGesvdjInfo"));
    api.GesvdjBufferSize = reinterpret_cast<decltype(api.GesvdjBufferSize)>(
        dlsym(h, "cusolverDnDgesvdj_bufferSize"));
    api.Gesvdj = reinterpret_cast<decltype(api.Gesvdj)>(dlsym(h, "cusolverDnDgesvdj"));
  });
  if (!api.Create || !api.Destroy || !api.SetStream || !api.GesvdBufferSize || !api.Gesvd ||
      !api.GeqrfBufferSize || !api.Geqrf || !api.OrmqrBufferSize || !api.Ormqr ||
      !api.CreateGesvdjInfo || !api.DestroyGesvdjInfo || !api.GesvdjBufferSize || !api.Gesvdj) {
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

// R (c x c) = upper triangle of the geqrf output (r x c, column-major)
__global__ void upper_kernel(const double* __restrict__ qr, long long r, long long c,
                             double* __restrict__ rr) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < c * c;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t % c, j = t / c;
    rr[t] = i <= j ? qr[i + j * r] : 0.0;
  }
}

// y_i /= s_i for s_i > cutoff = max(m,n)*eps*max(s), else 0 (the pseudo-inverse);
// one block (k <= 7071 under the reference's dense cap)
__global__ void pinv_scale_kernel(const double* __restrict__ s, long long k, double factor,
                                  double* __restrict__ y) {
  __shared__ double smax[kT];
  double mx = 0.0;
  for (long long i = threadIdx.x; i < k; i += blockDim.x) mx = fmax(mx, s[i]);
  smax[threadIdx.x] = mx;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + o]);
    __syncthreads();
  }
  const double cutoff = factor * smax[0];
  for (long long i = threadIdx.x; i < k; i += blockDim.x) {
    y[i] = s[i] > cutoff ? y[i] / s[i] : 0.0;
  }
}

}  // namespace

namespace {

// one solve lane: a stream, its cuSOLVER handle and its launch count (two lanes
// run the folded branches of solve_split concurrently, like the reference's
// two threads)
struct Lane {
  Context* ctx;
  cudaStream_t st;
  cusolverDnHandle_t h;
  std::int64_t launches = 0;
  void launched(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) cuda_check(e, what);
    ++launches;
  }
  void sync() { SSB_CUDA(cudaStreamSynchronize(st)); }
};

void dense_core(Matrix& a, const double* p, double* f, std::int64_t dense_cap, Lane& L) {
  Context* ctx = a.ctx;
  const std::int64_t m = a.rows, n = a.cols;
  if (m * n > dense_cap) {
    std::ostringstream msg;
    msg << "pseudo_solve_dense: " << m << "x" << n << " exceeds the dense cap of " << dense_cap
        << " entries";
    fail(msg.str());
  }
  if (n > 0) SSB_CUDA(cudaMemsetAsync(f, 0, n * sizeof(double), L.st));
  if (m == 0 || n == 0) {
    L.sync();
    return;
  }
  if (std::max(m, n) > 0x7fffffff / std::max<std::int64_t>(1, std::min(m, n))) {
    fail("pseudo_solve_dense: matrix too large for the dense factorisation");
  }
  const bool tall = m >= n;
  const int r = static_cast<int>(std::max(m, n)), c = static_cast<int>(std::min(m, n));
  const bool qr = r > c;  // tall B: QR first, then the SVD of the c x c factor R
  DBuf<double> b(static_cast<std::size_t>(r) * c), s(c), ur(static_cast<std::size_t>(c) * c),
      vt(static_cast<std::size_t>(c) * c), rr(qr ? static_cast<std::size_t>(c) * c : 1),
      tau(c), w(r), y(c), rwork(c);
  DBuf<int> info(1);
  SSB_CUDA(cudaMemsetAsync(b.get(), 0, sizeof(double) * r * c, L.st));
  densify_kernel<<<grid_n(ctx, m), kT, 0, L.st>>>(a.rowptr.get(), a.colidx.get(),
                                                        a.val.get(), m, tall, tall ? m : n,
                                                        b.get());
  L.launched("densify_kernel");
  const CusolverApi& api = cusolver();
  cusolverDnHandle_t h = L.h;
  int lw_qr = 0, lw_ormt = 0, lw_ormn = 0, lw_svd = 0;
  if (qr) {
    solver_check(api.GeqrfBufferSize(h, r, c, b.get(), r, &lw_qr), "cusolverDnDgeqrf_bufferSize");
    solver_check(api.OrmqrBufferSize(h, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, r, 1, c, b.get(), r,
                                     tau.get(), w.get(), r, &lw_ormt),
                 "cusolverDnDormqr_bufferSize");
    solver_check(api.OrmqrBufferSize(h, CUBLAS_SIDE_LEFT, CUBLAS_OP_N, r, 1, c, b.get(), r,
                                     tau.get(), w.get(), r, &lw_ormn),
                 "cusolverDnDormqr_bufferSize");
  }
  solver_check(api.GesvdBufferSize(h, c, c, &lw_svd), "cusolverDnDgesvd_bufferSize");
  const int lwork = std::max({lw_qr, lw_ormt, lw_ormn, lw_svd, 1});
  DBuf<double> work(lwork);
  const auto check_info = [&](const char* what) {
    int inf = 0;
    SSB_CUDA(cudaMemcpyAsync(&inf, info.get(), sizeof(int), cudaMemcpyDeviceToHost, L.st));
    L.sync();
    if (inf != 0) fail(std::string("pseudo_solve_dense: ") + what + " failed (info " +
                       std::to_string(inf) + ")");
  };
  double* fac = b.get();  // the c x c matrix whose SVD is taken
  if (qr) {
    solver_check(api.Geqrf(h, r, c, b.get(), r, tau.get(), work.get(), lwork, info.get()),
                 "cusolverDnDgeqrf");
    check_info("QR");
    upper_kernel<<<grid_n(ctx, static_cast<long long>(c) * c), kT, 0, L.st>>>(
        b.get(), r, c, rr.get());
    L.launched("upper_kernel");
    fac = rr.get();
  }
  // SVD of the c x c factor: fac = Ur diag(s) V^T (B = Q Ur diag(s) V^T). Jacobi
  // (gesvdj, V returned) by default; SSB_SVD=qr selects the bidiagonal gesvd (V^T).
  const char* sv = std::getenv("SSB_SVD");
  const bool jacobi = !(sv && std::string(sv) == "qr");
  if (jacobi) {
    gesvdjInfo_t prm = nullptr;
    solver_check(api.CreateGesvdjInfo(&prm), "cusolverDnCreateGesvdjInfo");
    int lwj = 0;
    const cusolverStatus_t st = api.GesvdjBufferSize(h, CUSOLVER_EIG_MODE_VECTOR, 1, c, c, fac, c,
                                                     s.get(), ur.get(), c, vt.get(), c, &lwj, prm);
    if (st != CUSOLVER_STATUS_SUCCESS) api.DestroyGesvdjInfo(prm);
    solver_check(st, "cusolverDnDgesvdj_bufferSize");
    DBuf<double> wj(std::max(lwj, 1));
    const cusolverStatus_t st2 = api.Gesvdj(h, CUSOLVER_EIG_MODE_VECTOR, 1, c, c, fac, c, s.get(),
                                            ur.get(), c, vt.get(), c, wj.get(), lwj, info.get(),
                                            prm);
    api.DestroyGesvdjInfo(prm);
    solver_check(st2, "cusolverDnDgesvdj");
  } else {
    solver_check(api.Gesvd(h, 'S', 'S', c, c, fac, c, s.get(), ur.get(), c, vt.get(), c,
                           work.get(), lwork, rwork.get(), info.get()),
                 "cusolverDnDgesvd");
  }
  check_info("SVD");
  // apply V (or V^T): with gesvdj `vt` holds V, with gesvd it holds V^T
  const auto apply_v = [&](const double* in, double* out) {  // out = V in
    if (jacobi) matvec_kernel<<<grid_n(ctx, c), kT, 0, L.st>>>(vt.get(), c, c, c, in, out);
    else matvec_t_kernel<<<grid_n(ctx, 32LL * c), kT, 0, L.st>>>(vt.get(), c, c, c, in, out);
  };
  const auto apply_vt = [&](const double* in, double* out) {  // out = V^T in
    if (jacobi) matvec_t_kernel<<<grid_n(ctx, 32LL * c), kT, 0, L.st>>>(vt.get(), c, c, c, in, out);
    else matvec_kernel<<<grid_n(ctx, c), kT, 0, L.st>>>(vt.get(), c, c, c, in, out);
  };
  const double factor = static_cast<double>(std::max(m, n)) * DBL_EPSILON;
  if (tall) {  // A = Q Ur S VT: x = VT^T S+ Ur^T (Q^T p)[:c]
    SSB_CUDA(cudaMemcpyAsync(w.get(), p, sizeof(double) * r, cudaMemcpyDeviceToDevice,
                             L.st));
    if (qr) {
      solver_check(api.Ormqr(h, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, r, 1, c, b.get(), r, tau.get(),
                             w.get(), r, work.get(), lwork, info.get()),
                   "cusolverDnDormqr");
      check_info("Q^T p");
    }
    matvec_t_kernel<<<grid_n(ctx, 32LL * c), kT, 0, L.st>>>(ur.get(), c, c, c, w.get(),
                                                                  y.get());
    pinv_scale_kernel<<<1, kT, 0, L.st>>>(s.get(), c, factor, y.get());
    apply_v(y.get(), f);
  } else {     // A^T = Q Ur S VT, A = VT^T S Ur^T Q^T: x = Q [Ur S+ VT p; 0]
    apply_vt(p, y.get());
    pinv_scale_kernel<<<1, kT, 0, L.st>>>(s.get(), c, factor, y.get());
    SSB_CUDA(cudaMemsetAsync(w.get(), 0, sizeof(double) * r, L.st));
    matvec_kernel<<<grid_n(ctx, c), kT, 0, L.st>>>(ur.get(), c, c, c, y.get(), w.get());
    if (qr) {
      solver_check(api.Ormqr(h, CUBLAS_SIDE_LEFT, CUBLAS_OP_N, r, 1, c, b.get(), r, tau.get(),
                             w.get(), r, work.get(), lwork, info.get()),
                   "cusolverDnDormqr");
      check_info("Q z");
    }
    SSB_CUDA(cudaMemcpyAsync(f, w.get(), sizeof(double) * r, cudaMemcpyDeviceToDevice,
                             L.st));
  }
  L.launched("pseudo-inverse apply");
  L.sync();
}

}  // namespace

void pseudo_solve_dense_dev(Matrix& a, const double* p, double* f, std::int64_t dense_cap) {
  Context* ctx = a.ctx;
  Lane L{ctx, ctx->stream, solver_handle(ctx)};
  try {
    dense_core(a, p, f, dense_cap, L);
  } catch (...) {
    ctx->launches += L.launches;
    throw;
  }
  ctx->launches += L.launches;
}

void pseudo_solve_dense_pair(Matrix* a[2], const double* p[2], double* f[2],
                             std::int64_t dense_cap, double seconds[2], std::string errs[2],
                             int codes[2]) {
  Context* ctx = a[0]->ctx;
  cudaStream_t side = side_stream(ctx);
  if (!ctx->solver2) {
    cusolverDnHandle_t h2 = nullptr;
    solver_check(cusolver().Create(&h2), "cusolverDnCreate");
    ctx->solver2 = h2;
  }
  solver_check(cusolver().SetStream(static_cast<cusolverDnHandle_t>(ctx->solver2), side),
               "cusolverDnSetStream");
  ctx->sync();  // inputs and outputs were produced / allocated on the main stream
  Lane lanes[2] = {{ctx, ctx->stream, solver_handle(ctx)},
                   {ctx, side, static_cast<cusolverDnHandle_t>(ctx->solver2)}};
  const auto run = [&](int s) {
    const auto t0 = std::chrono::steady_clock::now();
    try {
      dense_core(*a[s], p[s], f[s], dense_cap, lanes[s]);
    } catch (const Failure& e) {
      errs[s] = e.what();
      codes[s] = e.code;
    } catch (const std::exception& e) {
      errs[s] = e.what();
      codes[s] = SS_ERR_INVALID;
    }
    seconds[s] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  std::thread worker([&] {
    cudaSetDevice(ctx->device);
    alloc_stream() = side;  // this thread's buffers are ordered on the side stream
    run(1);
  });
  run(0);
  worker.join();
  ctx->launches += lanes[0].launches + lanes[1].launches;
}


void release_solver(Context* ctx) {
  for (void** h : {&ctx->solver, &ctx->solver2}) {
    if (*h) {
      cusolver().Destroy(static_cast<cusolverDnHandle_t>(*h));
      *h = nullptr;
    }
  }
  if (ctx->side) {
    cudaStreamDestroy(ctx->side);
    ctx->side = nullptr;
  }
}

}  // namespace ssb
