// CGLS on the device (reference cgls_solve, proj/src/solvers.cpp:99-146), the
// iterative method the reference's `bench`/`recon` use on sparse systems
// (tools/main.cpp:326-335, :416-419). SURVEY §8f ranks it "next" after the
// input side: it shares the CSR/CSC SpMV structure of SART.
//
// Per iteration (all on the context stream, captured once into a CUDA graph):
//   K1 q = A d, sum q^2 ; last block: qq == 0 -> break, alpha = gamma/qq
//   K2 x += alpha d, r -= alpha q, sum r^2 (history |r|)
//   K3 s = A^T r, sum s^2 ; last block: beta = gamma'/gamma, gamma = gamma',
//      stop when sqrt(gamma) <= tol * sqrt(gamma0)
//   K4 d = s + beta d
// Scalars and the loop-exit flag live on the device (no host round trip per
// iteration); every reduction is a fixed-order two-level tree.
#include <cmath>
#include <memory>
#include <string>

#include "internal.hpp"

namespace ssb {

namespace {

constexpr int kT = 256;
constexpr int kVS = 8;  // lanes per compressed vector

template <class T>
struct CglsK {
  const int *rp, *ci, *cp, *ri;
  const T *rv, *cv;
  T *x, *r, *s, *d, *q;
  long long m, n;
  double* part;     // per-block partial sums [gridDim]
  double* sc;       // gamma, alpha, beta, stop, rnorm2
  int* st;          // done, iterations, err_step_at, err_res_at
  unsigned* ticket;
  double* hist;
  double tol;
};

__device__ __forceinline__ bool last_block_cg(unsigned* ticket) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) __threadfence();
  return last;
}

__device__ double block_sum(double v) {
  __shared__ double sh[kT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < kT / 32; ++w) t += sh[w];
  }
  __syncthreads();
  return t;
}

// fixed-order sum of the per-block partials, by the last block
__device__ double sum_partials(const double* part, int nblk) {
  __shared__ double sh[kT];
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += part[b];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  return sh[0];
}

// phase 0: q = A d (rows); phase 1: s = A^T r (columns) inside the loop;
// phase 2: s = A^T r before the loop (r = p), sets gamma0 and the stop level.
template <class T>
__global__ void __launch_bounds__(kT) cgls_matvec_kernel(CglsK<T> k, int phase, int it) {
  if (phase != 2 && *(volatile int*)&k.st[0]) return;
  const bool rows = phase == 0;
  const int* ptr = rows ? k.rp : k.cp;
  const int* idx = rows ? k.ci : k.ri;
  const T* val = rows ? k.rv : k.cv;
  const T* vec = rows ? k.d : k.r;
  T* out = rows ? k.q : k.s;
  const long long nv = rows ? k.m : k.n;
  const int lane = threadIdx.x & (kVS - 1);
  const unsigned mask = ((1u << kVS) - 1u) << ((threadIdx.x & 31) & ~(kVS - 1));
  const long long g0 = (blockIdx.x * (long long)kT + threadIdx.x) / kVS;
  const long long ng = (long long)gridDim.x * kT / kVS;
  double sq = 0.0;
  for (long long g = g0; g < nv; g += ng) {
    T acc = T(0);
    for (int e = ptr[g] + lane; e < ptr[g + 1]; e += kVS) acc += val[e] * vec[idx[e]];
#pragma unroll
    for (int o = kVS / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(mask, acc, o, kVS);
    if (lane == 0) {
      out[g] = acc;
      sq += static_cast<double>(acc) * static_cast<double>(acc);
    }
  }
  const double b = block_sum(sq);
  if (threadIdx.x == 0) k.part[blockIdx.x] = b;
  if (!last_block_cg(k.ticket)) return;
  const double tot = sum_partials(k.part, gridDim.x);
  if (threadIdx.x == 0) {
    *k.ticket = 0;
    if (phase == 0) {  // solvers.cpp:124-129
      if (tot == 0.0) {
        k.st[0] = 1;  // d in the null space: break
      } else {
        const double alpha = k.sc[0] / tot;
        k.sc[1] = alpha;
        if (!isfinite(alpha)) {
          k.st[2] = it + 1;
          k.st[0] = 1;
        }
      }
    } else if (phase == 1) {  // solvers.cpp:132-141
      if (!isfinite(tot)) {
        k.st[3] = it + 1;
        k.st[0] = 1;
      } else {
        k.sc[2] = tot / k.sc[0];
        k.sc[0] = tot;
        k.st[1] = it + 1;
        k.hist[it] = sqrt(k.sc[4]);
        if (!(sqrt(tot) > k.sc[3])) k.st[0] = 1;  // loop condition of the next pass
      }
    } else {  // solvers.cpp:115-120
      k.sc[0] = tot;
      k.sc[3] = k.tol * sqrt(tot);
      k.st[1] = 0;
      if (!(sqrt(tot) > k.sc[3])) k.st[0] = 1;
    }
  }
}

// x += alpha d ; r -= alpha q ; sum r^2 (solvers.cpp:130-131, :142)
template <class T>
__global__ void __launch_bounds__(kT) cgls_axpy_kernel(CglsK<T> k) {
  if (*(volatile int*)&k.st[0]) return;
  const T alpha = static_cast<T>(k.sc[1]);
  const long long tid = blockIdx.x * (long long)kT + threadIdx.x;
  const long long stride = (long long)gridDim.x * kT;
  for (long long j = tid; j < k.n; j += stride) k.x[j] = k.x[j] + alpha * k.d[j];
  double sq = 0.0;
  for (long long i = tid; i < k.m; i += stride) {
    const T ri = k.r[i] - alpha * k.q[i];
    k.r[i] = ri;
    sq += static_cast<double>(ri) * static_cast<double>(ri);
  }
  const double b = block_sum(sq);
  if (threadIdx.x == 0) k.part[blockIdx.x] = b;
  if (!last_block_cg(k.ticket)) return;
  const double tot = sum_partials(k.part, gridDim.x);
  if (threadIdx.x == 0) {
    *k.ticket = 0;
    k.sc[4] = tot;
  }
}

// d = s + beta d (solvers.cpp:139); d = s before the loop (beta = 0)
template <class T>
__global__ void cgls_dupdate_kernel(CglsK<T> k, int init) {
  if (!init && *(volatile int*)&k.st[0]) return;
  const T beta = init ? T(0) : static_cast<T>(k.sc[2]);
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k.n;
       j += (long long)gridDim.x * blockDim.x) {
    k.d[j] = init ? k.s[j] : k.s[j] + beta * k.d[j];
  }
}

template <class T>
__global__ void cgls_cast_kernel(const double* src, T* dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    dst[i] = static_cast<T>(src[i]);
  }
}

template <class T>
__global__ void cgls_out_kernel(const T* src, double* dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    dst[i] = static_cast<double>(src[i]);
  }
}

template <class T>
void run_cgls(Matrix& a, const double* p_dev, const ss_solve_options& o, double* f_dev,
              ss_solve_report* rep, double* hist_host) {
  Context* ctx = a.ctx;
  a.ensure_csc();
  if (sizeof(T) == 4) a.ensure_f32();
  const long long m = a.rows, n = a.cols;
  DBuf<T> x(n), r(m), s(n), d(n), q(m);
  int occ = 0;
  SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cgls_matvec_kernel<T>, kT, 0));
  const int blocks = std::max(1, std::min<int>(occ * ctx->sm_count,
                                               static_cast<int>((std::max(m, n) * kVS + kT - 1) / kT)));
  DBuf<double> part(blocks), sc(5), hist(o.max_iters + 1);
  DBuf<int> st(4);
  DBuf<unsigned> ticket(1);
  CglsK<T> k{a.rowptr.get(), a.colidx.get(), a.colptr.get(), a.rowidx.get(),
             sizeof(T) == 4 ? reinterpret_cast<const T*>(a.val32.get())
                            : reinterpret_cast<const T*>(a.val.get()),
             sizeof(T) == 4 ? reinterpret_cast<const T*>(a.cval32.get())
                            : reinterpret_cast<const T*>(a.cval.get()),
             x.get(), r.get(), s.get(), d.get(), q.get(), m, n, part.get(), sc.get(), st.get(),
             ticket.get(), hist.get(), o.tol};
  const int gv = std::max(1, static_cast<int>(std::min<long long>((std::max(m, n) + kT - 1) / kT,
                                                                    ctx->sm_count * 8LL)));
  cudaEvent_t e0, e1;
  SSB_CUDA(cudaEventCreate(&e0));
  SSB_CUDA(cudaEventCreate(&e1));
  // graph: init + max_iters iterations
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  SSB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  SSB_CUDA(cudaMemsetAsync(x.get(), 0, n * sizeof(T), ctx->stream));
  SSB_CUDA(cudaMemsetAsync(st.get(), 0, 4 * sizeof(int), ctx->stream));
  SSB_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned), ctx->stream));
  cgls_cast_kernel<T><<<gv, kT, 0, ctx->stream>>>(p_dev, r.get(), m);
  cgls_matvec_kernel<T><<<blocks, kT, 0, ctx->stream>>>(k, 2, 0);
  cgls_dupdate_kernel<T><<<gv, kT, 0, ctx->stream>>>(k, 1);
  for (int it = 0; it < o.max_iters; ++it) {
    cgls_matvec_kernel<T><<<blocks, kT, 0, ctx->stream>>>(k, 0, it);
    cgls_axpy_kernel<T><<<blocks, kT, 0, ctx->stream>>>(k);
    cgls_matvec_kernel<T><<<blocks, kT, 0, ctx->stream>>>(k, 1, it);
    cgls_dupdate_kernel<T><<<gv, kT, 0, ctx->stream>>>(k, 0);
  }
  SSB_CUDA(cudaStreamEndCapture(ctx->stream, &g));
  SSB_CUDA(cudaGraphInstantiate(&ge, g, 0));
  cudaGraphDestroy(g);
  SSB_CUDA(cudaEventRecord(e0, ctx->stream));
  SSB_CUDA(cudaGraphLaunch(ge, ctx->stream));
  SSB_CUDA(cudaEventRecord(e1, ctx->stream));
  ctx->launches += 3 + 4LL * o.max_iters;
  SSB_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  SSB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaGraphExecDestroy(ge);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  int hs[4];
  ctx->copy(hs, st.get(), sizeof hs);
  if (hs[2]) {
    throw Failure(SS_ERR_DIVERGED, "cgls_solve: diverged (non-finite step at iteration " +
                                       std::to_string(hs[2]) + ")");
  }
  if (hs[3]) {
    throw Failure(SS_ERR_DIVERGED, "cgls_solve: diverged (non-finite residual at iteration " +
                                       std::to_string(hs[3]) + ")");
  }
  cgls_out_kernel<T><<<gv, kT, 0, ctx->stream>>>(x.get(), f_dev, n);
  ctx->check_launch("cgls_out_kernel");
  if (hist_host && hs[1] > 0) ctx->copy(hist_host, hist.get(), hs[1] * sizeof(double));
  ctx->sync();
  rep->iterations = hs[1];
  rep->history_len = hs[1];
  rep->wall_time_seconds = ms * 1e-3;
}

}  // namespace

// reference cgls_solve (solvers.cpp:99-146) on the device; f_dev receives x
// (fp64), the report gets iterations, history length and device loop time.
void cgls_device(Matrix& a, const double* p_dev, const ss_solve_options& o, double* f_dev,
                 ss_solve_report* rep, double* hist_host) {
  if (o.tol <= 0) fail("cgls_solve: tol must be positive");
  if (o.max_iters < 1) fail("cgls_solve: max_iters must be >= 1");
  if (o.dtype == SS_F32) run_cgls<float>(a, p_dev, o, f_dev, rep, hist_host);
  else run_cgls<double>(a, p_dev, o, f_dev, rep, hist_host);
}

}  // namespace ssb
