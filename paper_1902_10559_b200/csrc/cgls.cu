// CGLS on the device (reference cgls_solve, proj/src/solvers.cpp:99-146), the
// iterative method the reference's `bench`/`recon` use on sparse systems
// (tools/main.cpp:326-335, :416-419). SURVEY §8f ranks it "next" after the
// input side: it shares the CSR/CSC SpMV structure of SART.
//
// Per iteration (all on the context stream, the body of a CUDA-graph
// conditional WHILE node, so the loop ends on the device as soon as the
// reference's break / stop test fires -- no host round trip, no idle launches):
//   K1 q = A d, sum q^2 ; last block: qq == 0 -> break, alpha = gamma/qq
//   K2 x += alpha d, r -= alpha q, sum r^2 (history |r|)
//   K3 s = A^T r, sum s^2 ; last block: beta = gamma'/gamma, gamma = gamma',
//      stop when sqrt(gamma) <= tol * sqrt(gamma0)
//   K4 d = s + beta d
//   K5 (one thread) ++iteration; loop again while not done and < max_iters
// Scalars, the iteration counter and the loop-exit flag live on the device;
// every reduction is a fixed-order two-level tree.
#include <cmath>
#include <memory>
#include <string>
#include <thread>

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
  int* st;          // done, iterations, err_step_at, err_res_at, loop counter
  unsigned* ticket;
  double* hist;
  double tol;
  int max_iters;
  cudaGraphConditionalHandle cond;  // the WHILE node's condition
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
__global__ void __launch_bounds__(kT) cgls_matvec_kernel(CglsK<T> k, int phase) {
  if (phase != 2 && *(volatile int*)&k.st[0]) return;
  const int it = *(volatile int*)&k.st[4];
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

// end of one loop pass: count it and set the WHILE condition
template <class T>
__global__ void cgls_next_kernel(CglsK<T> k) {
  const int done = *(volatile int*)&k.st[0];
  const int nit = k.st[4] + 1;
  k.st[4] = nit;
  cudaGraphSetConditional(k.cond, !done && nit < k.max_iters ? 1u : 0u);
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

// one CGLS solve on stream `st` (the context stream, or the side stream of a
// concurrent folded branch); the matrix's CSC / fp32 copies must exist
template <class T>
void run_cgls(Matrix& a, const double* p_dev, const ss_solve_options& o, double* f_dev,
              ss_solve_report* rep, double* hist_host, cudaStream_t st,
              std::int64_t& launches) {
  Context* ctx = a.ctx;
  const long long m = a.rows, n = a.cols;
  DBuf<T> x(n), r(m), s(n), d(n), q(m);
  int occ = 0;
  SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cgls_matvec_kernel<T>, kT, 0));
  const int blocks = std::max(1, std::min<int>(occ * ctx->sm_count,
                                               static_cast<int>((std::max(m, n) * kVS + kT - 1) / kT)));
  DBuf<double> part(blocks), sc(5), hist(o.max_iters + 1);
  DBuf<int> state(5);
  DBuf<unsigned> ticket(1);
  CglsK<T> k{a.rowptr.get(), a.colidx.get(), a.colptr.get(), a.rowidx.get(),
             sizeof(T) == 4 ? reinterpret_cast<const T*>(a.val32.get())
                            : reinterpret_cast<const T*>(a.val.get()),
             sizeof(T) == 4 ? reinterpret_cast<const T*>(a.cval32.get())
                            : reinterpret_cast<const T*>(a.cval.get()),
             x.get(), r.get(), s.get(), d.get(), q.get(), m, n, part.get(), sc.get(), state.get(),
             ticket.get(), hist.get(), o.tol, o.max_iters, 0};
  const int gv = std::max(1, static_cast<int>(std::min<long long>((std::max(m, n) + kT - 1) / kT,
                                                                    ctx->sm_count * 8LL)));
  cudaEvent_t e0, e1;
  SSB_CUDA(cudaEventCreate(&e0));
  SSB_CUDA(cudaEventCreate(&e1));
  // graph: init nodes, then a WHILE node whose body is one CGLS pass
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  SSB_CUDA(cudaGraphCreate(&g, 0));
  SSB_CUDA(cudaGraphConditionalHandleCreate(&k.cond, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp{};
  try {
    SSB_CUDA(cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    SSB_CUDA(cudaMemsetAsync(x.get(), 0, n * sizeof(T), st));
    SSB_CUDA(cudaMemsetAsync(state.get(), 0, 5 * sizeof(int), st));
    SSB_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned), st));
    cgls_cast_kernel<T><<<gv, kT, 0, st>>>(p_dev, r.get(), m);
    cgls_matvec_kernel<T><<<blocks, kT, 0, st>>>(k, 2);
    cgls_dupdate_kernel<T><<<gv, kT, 0, st>>>(k, 1);
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    std::size_t nd = 0;
    SSB_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd));
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = k.cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    SSB_CUDA(cudaGraphAddNode(&cnode, g, deps, nd, &cp));
    SSB_CUDA(cudaStreamUpdateCaptureDependencies(st, &cnode, 1,
                                                 cudaStreamSetCaptureDependencies));
    SSB_CUDA(cudaStreamEndCapture(st, &g));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    SSB_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    cgls_matvec_kernel<T><<<blocks, kT, 0, st>>>(k, 0);
    cgls_axpy_kernel<T><<<blocks, kT, 0, st>>>(k);
    cgls_matvec_kernel<T><<<blocks, kT, 0, st>>>(k, 1);
    cgls_dupdate_kernel<T><<<gv, kT, 0, st>>>(k, 0);
    cgls_next_kernel<T><<<1, 1, 0, st>>>(k);
    SSB_CUDA(cudaStreamEndCapture(st, &body));
    SSB_CUDA(cudaGraphInstantiate(&ge, g, 0));
  } catch (...) {
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess &&
        cs != cudaStreamCaptureStatusNone) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(st, &junk);
    }
    cudaGraphDestroy(g);
    throw;
  }
  cudaGraphDestroy(g);
  SSB_CUDA(cudaEventRecord(e0, st));
  SSB_CUDA(cudaGraphLaunch(ge, st));
  SSB_CUDA(cudaEventRecord(e1, st));
  launches += 3;  // + 5 per executed pass, added from the device counter below
  SSB_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  SSB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaGraphExecDestroy(ge);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const auto to_host = [&](void* dst, const void* src, std::size_t bytes) {
    SSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    SSB_CUDA(cudaStreamSynchronize(st));
  };
  int hs[5];
  to_host(hs, state.get(), sizeof hs);
  launches += 5LL * hs[4];
  if (hs[2]) {
    throw Failure(SS_ERR_DIVERGED, "cgls_solve: diverged (non-finite step at iteration " +
                                       std::to_string(hs[2]) + ")");
  }
  if (hs[3]) {
    throw Failure(SS_ERR_DIVERGED, "cgls_solve: diverged (non-finite residual at iteration " +
                                       std::to_string(hs[3]) + ")");
  }
  cgls_out_kernel<T><<<gv, kT, 0, st>>>(x.get(), f_dev, n);
  cuda_check(cudaGetLastError(), "cgls_out_kernel");
  ++launches;
  if (hist_host && hs[1] > 0) to_host(hist_host, hist.get(), hs[1] * sizeof(double));
  SSB_CUDA(cudaStreamSynchronize(st));
  rep->iterations = hs[1];
  rep->history_len = hs[1];
  rep->wall_time_seconds = ms * 1e-3;
}

}  // namespace

namespace {
void check_cgls_options(const ss_solve_options& o) {
  if (o.tol <= 0) fail("cgls_solve: tol must be positive");
  if (o.max_iters < 1) fail("cgls_solve: max_iters must be >= 1");
}

void prepare(Matrix& a, const ss_solve_options& o) {
  a.ensure_csc();
  if (o.dtype == SS_F32) a.ensure_f32();
}

void run_on(Matrix& a, const double* p_dev, const ss_solve_options& o, double* f_dev,
            ss_solve_report* rep, double* hist_host, cudaStream_t st, std::int64_t& launches) {
  if (o.dtype == SS_F32) run_cgls<float>(a, p_dev, o, f_dev, rep, hist_host, st, launches);
  else run_cgls<double>(a, p_dev, o, f_dev, rep, hist_host, st, launches);
}
}  // namespace

// reference cgls_solve (solvers.cpp:99-146) on the device; f_dev receives x
// (fp64), the report gets iterations, history length and device loop time.
void cgls_device(Matrix& a, const double* p_dev, const ss_solve_options& o, double* f_dev,
                 ss_solve_report* rep, double* hist_host) {
  check_cgls_options(o);
  prepare(a, o);
  std::int64_t launches = 0;
  try {
    run_on(a, p_dev, o, f_dev, rep, hist_host, a.ctx->stream, launches);
  } catch (...) {
    a.ctx->launches += launches;
    throw;
  }
  a.ctx->launches += launches;
}

// both folded branches concurrently: branch 0 on the context stream (this
// thread), branch 1 on the side stream (a worker thread), like the reference's
// two solve_split threads; failures are reported per branch
void cgls_device_pair(Matrix* a[2], const double* p[2], const ss_solve_options& o, double* f[2],
                      ss_solve_report rep[2], std::string errs[2], int codes[2]) {
  check_cgls_options(o);
  Context* ctx = a[0]->ctx;
  prepare(*a[0], o);
  prepare(*a[1], o);
  cudaStream_t side = side_stream(ctx);
  ctx->sync();
  std::int64_t launches[2] = {0, 0};
  const auto run = [&](int s, cudaStream_t st) {
    try {
      run_on(*a[s], p[s], o, f[s], &rep[s], nullptr, st, launches[s]);
    } catch (const Failure& e) {
      errs[s] = e.what();
      codes[s] = e.code;
    } catch (const std::exception& e) {
      errs[s] = e.what();
      codes[s] = SS_ERR_INVALID;
    }
  };
  std::thread worker([&] {
    cudaSetDevice(ctx->device);
    alloc_stream() = side;
    run(1, side);
  });
  run(0, ctx->stream);
  worker.join();
  ctx->launches += launches[0] + launches[1];
}

}  // namespace ssb
