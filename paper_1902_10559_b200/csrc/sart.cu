// Hot path: the SART iteration of reference sart_solve
// (proj/src/solvers.cpp:178-191) on sm_100a, both folded systems per launch.
//
//   K1 sart_fwd  (CSR, VS lanes per row, 128-bit loads of 4 indices + 4 values):
//        r_i = p_i - (A x)_i ;  w_i = row_inv_i * r_i ;  block partial of sum r_i^2
//        last block: ||r|| -> history[it]; stop flag when ||r|| <= tol*||p||
//   K2 sart_back (CSC, VS lanes per column):
//        x_j += lambda * ((A^T w)_j * col_inv_j)    (skipped once stopped)
//
// Each iteration streams every matrix byte once as CSR and once as CSC (the
// north-star byte model); vectors are gathered through L1/L2. Norms use a
// fixed-order two-level reduction (no float atomics): results are bitwise
// reproducible run to run and independent of `parallelism`.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>

#include "plan.hpp"

namespace ssb {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

template <class T>
struct SysK {
  const int* rp;   // CSR row pointer
  const int* ci;   // CSR column index
  const T* rv;     // CSR values
  const int* cp;   // CSC column pointer
  const int* ri;   // CSC row index
  const T* cv;     // CSC values
  const T* p;
  const T* rinv;
  const T* cinv;
  T* x;
  T* w;
};

template <class T>
struct SartK {
  SysK<T> s[2];
  int nsys;
  int nrhs;
  long long rows0, rows_total;  // system 0 rows are [0, rows0)
  long long cols0, cols_total;
  double* partial;              // [nsys*nrhs][gridDim.x of K1]
  const double* pnorm;          // [nsys*nrhs]
  double tol;
  double relax;
  double* history;              // [nsys*nrhs][hstride]
  int hstride;
  int* state;                   // [nsys*nrhs][4]
  unsigned* ticket;
  // row-sharded: K2 writes the partial back-projection to bp_out[0..cols)
  // and K1's ||r_g||^2 lands in bp_out[cols] (one all-reduce per iteration)
  T* bp_out;
};

// ------------------------------------------------------------ loads
__device__ __forceinline__ void load4(const float* p, float (&v)[4]) {
  const float4 t = __ldg(reinterpret_cast<const float4*>(p));
  v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
}
__device__ __forceinline__ void load4(const double* p, double (&v)[4]) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

__device__ __forceinline__ double upd(double x, double relax, double u, double ci) {
  return __dadd_rn(x, __dmul_rn(relax, __dmul_rn(u, ci)));  // x += lambda*(u*ci)
}
__device__ __forceinline__ float upd(float x, double relax, float u, float ci) {
  return __fadd_rn(x, __fmul_rn(static_cast<float>(relax), __fmul_rn(u, ci)));
}

// Dot product of one compressed vector [beg,end) with a gathered dense
// vector, by VS cooperating lanes: scalar head up to the 16-byte boundary,
// 4-wide vector body (int4 indices + 4 values per lane per step, two steps
// in flight), scalar tail, then a VS-lane butterfly.
template <class T, int VS>
__device__ __forceinline__ T seg_dot(const int* __restrict__ idx, const T* __restrict__ val,
                                     const T* __restrict__ vec, int beg, int end, int lane,
                                     unsigned mask) {
  T acc = T(0);
  int a = (beg + 3) & ~3;
  if (a > end) a = end;
  if (beg + lane < a) acc += val[beg + lane] * __ldg(vec + idx[beg + lane]);
  const int nvec = (end - a) >> 2;
  const int b = a + (nvec << 2);
  int q = lane;
  for (; q + VS < nvec; q += 2 * VS) {
    const int k0 = a + (q << 2), k1 = k0 + (VS << 2);
    const int4 c0 = __ldg(reinterpret_cast<const int4*>(idx + k0));
    const int4 c1 = __ldg(reinterpret_cast<const int4*>(idx + k1));
    T v0[4], v1[4];
    load4(val + k0, v0);
    load4(val + k1, v1);
    const T x00 = __ldg(vec + c0.x), x01 = __ldg(vec + c0.y), x02 = __ldg(vec + c0.z),
            x03 = __ldg(vec + c0.w);
    const T x10 = __ldg(vec + c1.x), x11 = __ldg(vec + c1.y), x12 = __ldg(vec + c1.z),
            x13 = __ldg(vec + c1.w);
    acc += v0[0] * x00 + v0[1] * x01 + v0[2] * x02 + v0[3] * x03;
    acc += v1[0] * x10 + v1[1] * x11 + v1[2] * x12 + v1[3] * x13;
  }
  if (q < nvec) {
    const int k0 = a + (q << 2);
    const int4 c0 = __ldg(reinterpret_cast<const int4*>(idx + k0));
    T v0[4];
    load4(val + k0, v0);
    acc += v0[0] * __ldg(vec + c0.x) + v0[1] * __ldg(vec + c0.y) + v0[2] * __ldg(vec + c0.z) +
           v0[3] * __ldg(vec + c0.w);
  }
  if (b + lane < end) acc += val[b + lane] * __ldg(vec + idx[b + lane]);
#pragma unroll
  for (int off = VS / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(mask, acc, off, VS);
  return acc;
}

template <int VS>
__device__ __forceinline__ unsigned group_mask() {
  if (VS == 32) return 0xffffffffu;
  const unsigned lane = threadIdx.x & 31;
  return ((1u << VS) - 1u) << (lane & ~(VS - 1u));
}

__device__ __forceinline__ bool sys_on(const int* state, int idx) {
  const volatile int* s = state + 4 * idx;
  return s[0] == 0 && s[2] == 0;
}

// Fixed-order reduction of per-block partials by the last block of K1, then
// the reference's check-before-update stopping rule (solvers.cpp:180-182).
__device__ void finish_norms(double* partial, int nblk, int nsr, const double* pnorm, double tol,
                             double* history, int hstride, int* state, int it) {
  __shared__ double sh[kThreads];
  for (int q = 0; q < nsr; ++q) {
    if (!sys_on(state, q)) continue;
    double s = 0.0;
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += partial[q * nblk + b];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const double res = sqrt(sh[0]);
      history[q * hstride + it] = res;
      if (res <= tol * pnorm[q]) {
        state[4 * q + 0] = 1;
        state[4 * q + 1] = it;
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ bool last_block(unsigned* ticket) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// ------------------------------------------------------------ single RHS kernels
template <class T, int VS>
__global__ void __launch_bounds__(kThreads) sart_fwd_kernel(SartK<T> k, int it) {
  __shared__ double red[2][kWarps];
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const long long group = (blockIdx.x * (long long)kThreads + threadIdx.x) / VS;
  const long long ngroups = (long long)gridDim.x * kThreads / VS;
  const bool on0 = sys_on(k.state, 0);
  const bool on1 = k.nsys > 1 && sys_on(k.state, 1);
  double acc0 = 0.0, acc1 = 0.0;
  for (long long g = group; g < k.rows_total; g += ngroups) {
    const int s = g >= k.rows0 ? 1 : 0;
    if (!(s ? on1 : on0)) continue;
    const SysK<T>& S = k.s[s];
    const int i = static_cast<int>(g - (s ? k.rows0 : 0));
    const T dot = seg_dot<T, VS>(S.ci, S.rv, S.x, S.rp[i], S.rp[i + 1], lane, mask);
    if (lane == 0) {
      const T r = S.p[i] - dot;
      S.w[i] = S.rinv[i] * r;
      const double rd = static_cast<double>(r);
      if (s) acc1 += rd * rd; else acc0 += rd * rd;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc0 += __shfl_xor_sync(0xffffffffu, acc0, o);
    acc1 += __shfl_xor_sync(0xffffffffu, acc1, o);
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][warp] = acc0;
    red[1][warp] = acc1;
  }
  __syncthreads();
  if (threadIdx.x < k.nsys) {
    double t = 0.0;
    for (int q = 0; q < kWarps; ++q) t += red[threadIdx.x][q];
    k.partial[threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
  if (k.bp_out) return;  // sharded plans reduce ||r||^2 across ranks instead
  if (last_block(k.ticket)) {
    finish_norms(k.partial, gridDim.x, k.nsys, k.pnorm, k.tol, k.history, k.hstride,
                 k.state, it);
    if (threadIdx.x == 0) *k.ticket = 0;
  }
}

template <class T, int VS>
__global__ void __launch_bounds__(kThreads) sart_back_kernel(SartK<T> k, int it) {
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const long long group = (blockIdx.x * (long long)kThreads + threadIdx.x) / VS;
  const long long ngroups = (long long)gridDim.x * kThreads / VS;
  const bool on0 = sys_on(k.state, 0);
  const bool on1 = k.nsys > 1 && sys_on(k.state, 1);
  for (long long g = group; g < k.cols_total; g += ngroups) {
    const int s = g >= k.cols0 ? 1 : 0;
    if (!(s ? on1 : on0)) continue;
    const SysK<T>& S = k.s[s];
    const int j = static_cast<int>(g - (s ? k.cols0 : 0));
    const T u = seg_dot<T, VS>(S.ri, S.cv, S.w, S.cp[j], S.cp[j + 1], lane, mask);
    if (lane == 0) {
      if (k.bp_out) {
        k.bp_out[j] = u;
      } else {
        const T xn = upd(S.x[j], k.relax, u, S.cinv[j]);
        S.x[j] = xn;
        if (!isfinite(static_cast<double>(xn))) atomicCAS(&k.state[4 * s + 2], 0, it + 1);
      }
    }
  }
}

// ------------------------------------------------------------ multi-RHS kernels
// Slices share A; X/W/P are [n][S] so one warp's 32 lanes read 32 consecutive
// slices of a gathered row (coalesced 128 B for fp32) while the matrix entry
// is loaded once per warp and broadcast: matrix bytes amortise over S.
template <class T, int SPL>
__global__ void __launch_bounds__(kThreads) sart_fwd_multi_kernel(SartK<T> k, int it) {
  extern __shared__ double mred[];  // [kWarps][nsys*S]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int S = k.nrhs;
  const long long gw = (blockIdx.x * (long long)kThreads + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kThreads) >> 5;
  double r2a[SPL], r2b[SPL];
  bool ona[SPL], onb[SPL];
#pragma unroll
  for (int q = 0; q < SPL; ++q) {
    const int sl = lane + 32 * q;
    r2a[q] = r2b[q] = 0.0;
    ona[q] = sl < S && sys_on(k.state, sl);
    onb[q] = sl < S && k.nsys > 1 && sys_on(k.state, S + sl);
  }
  for (long long g = gw; g < k.rows_total; g += nw) {
    const int s = g >= k.rows0 ? 1 : 0;
    const SysK<T>& Sy = k.s[s];
    const int i = static_cast<int>(g - (s ? k.rows0 : 0));
    T acc[SPL];
#pragma unroll
    for (int q = 0; q < SPL; ++q) acc[q] = T(0);
    const int beg = Sy.rp[i], end = Sy.rp[i + 1];
    for (int base = beg; base < end; base += 32) {
      const int kk = base + lane;
      const int c = kk < end ? __ldg(Sy.ci + kk) : 0;
      const T v = kk < end ? __ldg(Sy.rv + kk) : T(0);
      const int cnt = min(32, end - base);
      for (int e = 0; e < cnt; ++e) {
        const int ce = __shfl_sync(0xffffffffu, c, e);
        const T ve = __shfl_sync(0xffffffffu, v, e);
        const T* xr = Sy.x + static_cast<long long>(ce) * S;
#pragma unroll
        for (int q = 0; q < SPL; ++q) {
          const int sl = lane + 32 * q;
          if (sl < S) acc[q] += ve * __ldg(xr + sl);
        }
      }
    }
    const T ri = Sy.rinv[i];
#pragma unroll
    for (int q = 0; q < SPL; ++q) {
      const int sl = lane + 32 * q;
      if (s ? onb[q] : ona[q]) {
        const long long o = static_cast<long long>(i) * S + sl;
        const T r = Sy.p[o] - acc[q];
        Sy.w[o] = ri * r;
        const double r2 = static_cast<double>(r) * static_cast<double>(r);
        if (s) r2b[q] += r2; else r2a[q] += r2;
      }
    }
  }
  const int nsr = k.nsys * S;
#pragma unroll
  for (int q = 0; q < SPL; ++q) {
    const int sl = lane + 32 * q;
    if (sl < S) {
      mred[warp * nsr + sl] = r2a[q];
      if (k.nsys > 1) mred[warp * nsr + S + sl] = r2b[q];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nsr; t += kThreads) {
    double a = 0.0;
    for (int q = 0; q < kWarps; ++q) a += mred[q * nsr + t];
    k.partial[static_cast<long long>(t) * gridDim.x + blockIdx.x] = a;
  }
  if (last_block(k.ticket)) {
    finish_norms(k.partial, gridDim.x, nsr, k.pnorm, k.tol, k.history, k.hstride,
                 k.state, it);
    if (threadIdx.x == 0) *k.ticket = 0;
  }
}

template <class T, int SPL>
__global__ void __launch_bounds__(kThreads) sart_back_multi_kernel(SartK<T> k, int it) {
  const int lane = threadIdx.x & 31;
  const int S = k.nrhs;
  const long long gw = (blockIdx.x * (long long)kThreads + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kThreads) >> 5;
  bool ona[SPL], onb[SPL];
#pragma unroll
  for (int q = 0; q < SPL; ++q) {
    const int sl = lane + 32 * q;
    ona[q] = sl < S && sys_on(k.state, sl);
    onb[q] = sl < S && k.nsys > 1 && sys_on(k.state, S + sl);
  }
  for (long long g = gw; g < k.cols_total; g += nw) {
    const int s = g >= k.cols0 ? 1 : 0;
    const SysK<T>& Sy = k.s[s];
    const int j = static_cast<int>(g - (s ? k.cols0 : 0));
    T acc[SPL];
#pragma unroll
    for (int q = 0; q < SPL; ++q) acc[q] = T(0);
    const int beg = Sy.cp[j], end = Sy.cp[j + 1];
    for (int base = beg; base < end; base += 32) {
      const int kk = base + lane;
      const int r = kk < end ? __ldg(Sy.ri + kk) : 0;
      const T v = kk < end ? __ldg(Sy.cv + kk) : T(0);
      const int cnt = min(32, end - base);
      for (int e = 0; e < cnt; ++e) {
        const int re = __shfl_sync(0xffffffffu, r, e);
        const T ve = __shfl_sync(0xffffffffu, v, e);
        const T* wr = Sy.w + static_cast<long long>(re) * S;
#pragma unroll
        for (int q = 0; q < SPL; ++q) {
          const int sl = lane + 32 * q;
          if (sl < S) acc[q] += ve * __ldg(wr + sl);
        }
      }
    }
    const T ci = Sy.cinv[j];
#pragma unroll
    for (int q = 0; q < SPL; ++q) {
      const int sl = lane + 32 * q;
      if (s ? onb[q] : ona[q]) {
        const long long o = static_cast<long long>(j) * S + sl;
        const T xn = upd(Sy.x[o], k.relax, acc[q], ci);
        Sy.x[o] = xn;
        if (!isfinite(static_cast<double>(xn))) atomicCAS(&k.state[4 * (s * S + sl) + 2], 0, it + 1);
      }
    }
  }
}

// ------------------------------------------------------------ sharded update
// After the all-reduce of [A_g^T w_g | ||r_g||^2] every rank applies the same
// update (SURVEY §8e level 3) with the reference's check-before-update order.
template <class T>
__global__ void sart_sharded_update_kernel(T* x, const T* bp, const T* cinv, long long cols,
                                           const double* pnorm, double tol, double relax,
                                           double* history, int* state, int it) {
  if (!sys_on(state, 0)) return;
  const double res = sqrt(static_cast<double>(bp[cols]));
  if (blockIdx.x == 0 && threadIdx.x == 0) history[it] = res;
  if (res <= tol * pnorm[0]) return;  // break before the update
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < cols;
       j += (long long)gridDim.x * blockDim.x) {
    const T xn = upd(x[j], relax, bp[j], cinv[j]);
    x[j] = xn;
    if (!isfinite(static_cast<double>(xn))) atomicCAS(&state[2], 0, it + 1);
  }
}

template <class T>
__global__ void sharded_stop_kernel(const T* bp, long long cols, const double* pnorm, double tol,
                                    int* state, int it) {
  if (state[0] == 0 && state[2] == 0 && sqrt(static_cast<double>(bp[cols])) <= tol * pnorm[0]) {
    state[0] = 1;
    state[1] = it;
  }
}

// Fixed-order sum of the forward kernel's per-block ||r_g||^2 partials into
// the all-reduce slot bp[cols].
template <class T>
__global__ void sharded_r2_kernel(const double* partial, int nblk, T* slot) {
  __shared__ double sh[kThreads];
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += partial[b];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *slot = static_cast<T>(sh[0]);
}

template <class T>
__global__ void inv_kernel(const double* sums, T* inv, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    inv[i] = static_cast<T>(sums[i] > 0 ? 1.0 / sums[i] : 0.0);
  }
}

template <class T>
__global__ void to_f64_kernel(const T* src, double* dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    dst[i] = static_cast<double>(src[i]);
  }
}

// slice-major host layout <-> [n][S] device layout
template <class T>
__global__ void transpose_in_kernel(const double* src, T* dst, long long n, int S) {
  const long long total = n * S;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < total;
       k += (long long)gridDim.x * blockDim.x) {
    const long long s = k / n, i = k % n;
    dst[i * S + s] = static_cast<T>(src[k]);
  }
}

template <class T>
__global__ void transpose_out_kernel(const T* src, double* dst, long long n, int S) {
  const long long total = n * S;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < total;
       k += (long long)gridDim.x * blockDim.x) {
    const long long s = k / n, i = k % n;
    dst[k] = static_cast<double>(src[i * S + s]);
  }
}

// ||p_s||^2 per slice (fixed order), for the stopping rule.
template <class T>
__global__ void pnorm_kernel(const T* p, long long n, int S, double* out) {
  __shared__ double sh[kThreads];
  const int s = blockIdx.x;
  double a = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = static_cast<double>(p[i * S + s]);
    a += v * v;
  }
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[s] = sqrt(sh[0]);
}

__global__ void square_kernel(double* v, int n) {
  if (threadIdx.x < n) v[threadIdx.x] = v[threadIdx.x] * v[threadIdx.x];
}

__global__ void sqrt_kernel(double* v, int n) {
  if (threadIdx.x < n) v[threadIdx.x] = sqrt(v[threadIdx.x]);
}

int pick_vs(double avg) {
  if (avg >= 256) return 32;
  if (avg >= 96) return 16;
  if (avg >= 40) return 8;
  return 4;
}

template <class T>
SartK<T> make_args(Plan& P) {
  SartK<T> k{};
  for (int s = 0; s < P.nsys; ++s) {
    Matrix* a = P.a[s];
    SysK<T>& S = k.s[s];
    S.rp = a->rowptr.get();
    S.ci = a->colidx.get();
    S.cp = a->colptr.get();
    S.ri = a->rowidx.get();
    if constexpr (sizeof(T) == 4) {
      S.rv = a->val32.get();
      S.cv = a->cval32.get();
    } else {
      S.rv = a->val.get();
      S.cv = a->cval.get();
    }
    S.p = reinterpret_cast<const T*>(P.p[s].get());
    S.rinv = reinterpret_cast<const T*>(P.rinv[s].get());
    S.cinv = reinterpret_cast<const T*>(P.cinv[s].get());
    S.x = reinterpret_cast<T*>(P.x[s].get());
    S.w = reinterpret_cast<T*>(P.w[s].get());
  }
  if (P.nsys == 1) k.s[1] = k.s[0];
  k.nsys = P.nsys;
  k.nrhs = P.nrhs;
  k.rows0 = P.rows[0];
  k.rows_total = P.rows[0] + (P.nsys > 1 ? P.rows[1] : 0);
  k.cols0 = P.cols[0];
  k.cols_total = P.cols[0] + (P.nsys > 1 ? P.cols[1] : 0);
  k.partial = P.partial.get();
  k.pnorm = P.pnorm.get();
  k.tol = P.opts.tol;
  k.relax = P.opts.relaxation;
  k.history = P.history.get();
  k.hstride = P.opts.max_iters + 1;
  k.state = P.state.get();
  k.ticket = P.ticket.get();
  if (P.sharded) {
    k.bp_out = reinterpret_cast<T*>(P.bp.get());
  }
  return k;
}

template <class T, int VS>
void launch_fwd1(Plan& P, const SartK<T>& k, int it) {
  sart_fwd_kernel<T, VS><<<P.fwd_blocks, kThreads, 0, P.ctx->stream>>>(k, it);
}
template <class T, int VS>
void launch_back1(Plan& P, const SartK<T>& k, int it) {
  sart_back_kernel<T, VS><<<P.back_blocks, kThreads, 0, P.ctx->stream>>>(k, it);
}

template <class T>
void launch_fwd(Plan& P, const SartK<T>& k, int it) {
  if (P.nrhs > 1) {
    const int spl = (P.nrhs + 31) / 32;
    const std::size_t sh = sizeof(double) * kWarps * P.nsys * P.nrhs;
    switch (spl) {
      case 1: sart_fwd_multi_kernel<T, 1><<<P.fwd_blocks, kThreads, sh, P.ctx->stream>>>(k, it); break;
      case 2: sart_fwd_multi_kernel<T, 2><<<P.fwd_blocks, kThreads, sh, P.ctx->stream>>>(k, it); break;
      case 3:
      case 4: sart_fwd_multi_kernel<T, 4><<<P.fwd_blocks, kThreads, sh, P.ctx->stream>>>(k, it); break;
      default: sart_fwd_multi_kernel<T, 8><<<P.fwd_blocks, kThreads, sh, P.ctx->stream>>>(k, it); break;
    }
    return;
  }
  switch (P.vs_fwd) {
    case 4: launch_fwd1<T, 4>(P, k, it); break;
    case 8: launch_fwd1<T, 8>(P, k, it); break;
    case 16: launch_fwd1<T, 16>(P, k, it); break;
    default: launch_fwd1<T, 32>(P, k, it); break;
  }
}

template <class T>
void launch_back(Plan& P, const SartK<T>& k, int it) {
  if (P.nrhs > 1) {
    const int spl = (P.nrhs + 31) / 32;
    switch (spl) {
      case 1: sart_back_multi_kernel<T, 1><<<P.back_blocks, kThreads, 0, P.ctx->stream>>>(k, it); break;
      case 2: sart_back_multi_kernel<T, 2><<<P.back_blocks, kThreads, 0, P.ctx->stream>>>(k, it); break;
      case 3:
      case 4: sart_back_multi_kernel<T, 4><<<P.back_blocks, kThreads, 0, P.ctx->stream>>>(k, it); break;
      default: sart_back_multi_kernel<T, 8><<<P.back_blocks, kThreads, 0, P.ctx->stream>>>(k, it); break;
    }
    return;
  }
  switch (P.vs_back) {
    case 4: launch_back1<T, 4>(P, k, it); break;
    case 8: launch_back1<T, 8>(P, k, it); break;
    case 16: launch_back1<T, 16>(P, k, it); break;
    default: launch_back1<T, 32>(P, k, it); break;
  }
}

template <class T>
int occupancy_blocks(Plan& P, bool fwd) {
  int per_sm = 0;
  cudaError_t e;
  if (P.nrhs > 1) {
    const std::size_t sh = fwd ? sizeof(double) * kWarps * P.nsys * P.nrhs : 0;
    e = fwd ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sart_fwd_multi_kernel<T, 8>,
                                                            kThreads, sh)
            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sart_back_multi_kernel<T, 8>,
                                                            kThreads, 0);
  } else {
    e = fwd ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sart_fwd_kernel<T, 32>,
                                                            kThreads, 0)
            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sart_back_kernel<T, 8>,
                                                            kThreads, 0);
  }
  SSB_CUDA(e);
  return std::max(1, per_sm) * P.ctx->sm_count;
}

template <class T>
void do_iterations(Plan& P, int first, int count) {
  const SartK<T> k = make_args<T>(P);
  for (int it = first; it < first + count; ++it) {
    if (P.sharded) {
      // K1 over local rows, fixed-order ||r_g||^2, K2 partial back-projection,
      // all-reduce [bp | r2], identical update on every rank.
      T* bp = reinterpret_cast<T*>(P.bp.get());
      const long long cols = P.cols[0];
      launch_fwd<T>(P, k, it);
      P.ctx->check_launch("sart_fwd(sharded)");
      sharded_r2_kernel<T><<<1, kThreads, 0, P.ctx->stream>>>(P.partial.get(), P.fwd_blocks,
                                                             bp + cols);
      P.ctx->check_launch("sharded_r2_kernel");
      launch_back<T>(P, k, it);
      P.ctx->check_launch("sart_back(sharded)");
      ncclResult_t nr = ncclAllReduce(bp, bp, static_cast<std::size_t>(cols + 1),
                                      sizeof(T) == 4 ? ncclFloat32 : ncclFloat64, ncclSum,
                                      static_cast<ncclComm_t>(P.ctx->comm), P.ctx->stream);
      if (nr != ncclSuccess) {
        fail(std::string("ncclAllReduce: ") + ncclGetErrorString(nr), SS_ERR_NCCL);
      }
      sart_sharded_update_kernel<T><<<P.back_blocks, kThreads, 0, P.ctx->stream>>>(
          reinterpret_cast<T*>(P.x[0].get()), bp, reinterpret_cast<const T*>(P.cinv[0].get()),
          cols, P.pnorm.get(), P.opts.tol, P.opts.relaxation, P.history.get(), P.state.get(), it);
      P.ctx->check_launch("sart_sharded_update_kernel");
      sharded_stop_kernel<T><<<1, 1, 0, P.ctx->stream>>>(bp, cols, P.pnorm.get(), P.opts.tol,
                                                        P.state.get(), it);
      P.ctx->check_launch("sharded_stop_kernel");
      continue;
    }
    launch_fwd<T>(P, k, it);
    P.ctx->check_launch("sart_fwd_kernel");
    launch_back<T>(P, k, it);
    P.ctx->check_launch("sart_back_kernel");
  }
}

int grid1(Context* ctx, long long n) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((n + 255) / 256,
                                                                     ctx->sm_count * 16LL)));
}

}  // namespace

// ====================================================================== Plan
Plan::~Plan() {
  if (graph) cudaGraphExecDestroy(graph);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  delete own;
}

void Plan::enqueue_reset() {
  for (int s = 0; s < nsys; ++s) {
    SSB_CUDA(cudaMemsetAsync(x[s].get(), 0, cols[s] * nrhs * tsize(), ctx->stream));
  }
  SSB_CUDA(cudaMemsetAsync(state.get(), 0, state.size() * sizeof(int), ctx->stream));
  SSB_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned), ctx->stream));
}

void Plan::enqueue_iterations(int first, int count) {
  if (dtype == SS_F32) do_iterations<float>(*this, first, count);
  else do_iterations<double>(*this, first, count);
}

void Plan::build_graph() {
  if (graph || sharded) return;  // NCCL calls stay out of the captured graph
  cudaGraph_t g = nullptr;
  SSB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  const std::int64_t before = ctx->launches;
  try {
    enqueue_reset();
    enqueue_iterations(0, opts.max_iters);
  } catch (...) {
    cudaStreamEndCapture(ctx->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  ctx->launches = before;  // captured, not launched
  SSB_CUDA(cudaStreamEndCapture(ctx->stream, &g));
  SSB_CUDA(cudaGraphInstantiate(&graph, g, 0));
  cudaGraphDestroy(g);
}

void Plan::launch() {
  SSB_CUDA(cudaEventRecord(ev0, ctx->stream));
  if (graph) {
    SSB_CUDA(cudaGraphLaunch(graph, ctx->stream));
    ctx->launches += static_cast<std::int64_t>(2) * opts.max_iters;
  } else {
    enqueue_reset();
    enqueue_iterations(0, opts.max_iters);
  }
  SSB_CUDA(cudaEventRecord(ev1, ctx->stream));
  launched = true;
}

void Plan::finish(ss_solve_report* rep) {
  if (!launched) fail("plan: finish without launch");
  SSB_CUDA(cudaEventSynchronize(ev1));
  SSB_CUDA(cudaEventElapsedTime(&last_ms, ev0, ev1));
  std::vector<int> st(state.size());
  SSB_CUDA(cudaMemcpy(st.data(), state.get(), st.size() * sizeof(int), cudaMemcpyDeviceToHost));
  int iters = 0;
  for (int q = 0; q < nsys * nrhs; ++q) {
    if (st[4 * q + 2] != 0) {
      throw Failure(SS_ERR_DIVERGED,
                    "sart_solve: diverged (non-finite iterate at iteration " +
                        std::to_string(st[4 * q + 2]) + ")");
    }
    iters = std::max(iters, st[4 * q] ? st[4 * q + 1] : opts.max_iters);
  }
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->iterations = iters;
    rep->wall_time_seconds = last_ms * 1e-3;
    rep->branch1_seconds = rep->wall_time_seconds;
    rep->branch2_seconds = nsys > 1 ? rep->wall_time_seconds : 0.0;
    rep->history_len = (st[0] ? st[1] + 1 : opts.max_iters);
  }
}

void Plan::finish_rhs(int which) {
  double* pn = pnorm.get() + which * nrhs;
  if (dtype == SS_F32) {
    pnorm_kernel<float><<<nrhs, kThreads, 0, ctx->stream>>>(
        reinterpret_cast<const float*>(p[which].get()), rows[which], nrhs, pn);
  } else {
    pnorm_kernel<double><<<nrhs, kThreads, 0, ctx->stream>>>(
        reinterpret_cast<const double*>(p[which].get()), rows[which], nrhs, pn);
  }
  ctx->check_launch("pnorm_kernel");
  if (sharded) {
    // ||p||^2 = sum over ranks of the local ||p_g||^2
    square_kernel<<<1, 32, 0, ctx->stream>>>(pn, nrhs);
    ctx->check_launch("square_kernel");
    const ncclResult_t r = ncclAllReduce(pn, pn, nrhs, ncclFloat64, ncclSum,
                                         static_cast<ncclComm_t>(ctx->comm), ctx->stream);
    if (r != ncclSuccess) fail(std::string("ncclAllReduce: ") + ncclGetErrorString(r), SS_ERR_NCCL);
    sqrt_kernel<<<1, 32, 0, ctx->stream>>>(pn, nrhs);
    ctx->check_launch("sqrt_kernel");
  }
  ctx->sync();
}

void Plan::set_rhs_device_f64(int which, const double* src) {
  if (which < 0 || which >= nsys) fail("plan: system index out of range");
  const std::int64_t n = rows[which] * nrhs;
  const int g = grid1(ctx, n);
  if (dtype == SS_F32) {
    transpose_in_kernel<float><<<g, 256, 0, ctx->stream>>>(
        src, reinterpret_cast<float*>(p[which].get()), rows[which], nrhs);
  } else {
    transpose_in_kernel<double><<<g, 256, 0, ctx->stream>>>(
        src, reinterpret_cast<double*>(p[which].get()), rows[which], nrhs);
  }
  ctx->check_launch("transpose_in_kernel");
  finish_rhs(which);
}

void Plan::set_rhs_host(int which, const double* p_host) {
  if (which < 0 || which >= nsys) fail("plan: system index out of range");
  const std::int64_t n = rows[which] * nrhs;
  DBuf<double> tmp(n);
  SSB_CUDA(cudaMemcpyAsync(tmp.get(), p_host, n * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
  set_rhs_device_f64(which, tmp.get());
}

void Plan::set_rhs_device(int which, const void* p_dev) {
  if (which < 0 || which >= nsys) fail("plan: system index out of range");
  SSB_CUDA(cudaMemcpyAsync(p[which].get(), p_dev, rows[which] * nrhs * tsize(),
                           cudaMemcpyDeviceToDevice, ctx->stream));
  finish_rhs(which);
}

int Plan::diverged_at(int which) const {
  int st[4] = {0, 0, 0, 0};
  SSB_CUDA(cudaMemcpy(st, state.get() + 4 * which * nrhs, sizeof st, cudaMemcpyDeviceToHost));
  return st[2];
}

void Plan::recombine_device(double* f_dev) {
  if (nsys != 2 || nrhs != 1) fail("plan: recombine needs the folded pair");
  const std::int64_t nh = cols[0];
  DBuf<double> f1(nh), f2(nh);
  const int g = grid1(ctx, nh);
  if (dtype == SS_F32) {
    to_f64_kernel<float><<<g, 256, 0, ctx->stream>>>(reinterpret_cast<const float*>(x[0].get()),
                                                    f1.get(), nh);
    to_f64_kernel<float><<<g, 256, 0, ctx->stream>>>(reinterpret_cast<const float*>(x[1].get()),
                                                    f2.get(), nh);
  } else {
    to_f64_kernel<double><<<g, 256, 0, ctx->stream>>>(reinterpret_cast<const double*>(x[0].get()),
                                                     f1.get(), nh);
    to_f64_kernel<double><<<g, 256, 0, ctx->stream>>>(reinterpret_cast<const double*>(x[1].get()),
                                                     f2.get(), nh);
  }
  ctx->check_launch("to_f64_kernel");
  if (!all_finite_dev(ctx, f1.get(), nh) || !all_finite_dev(ctx, f2.get(), nh)) {
    fail("recombine_solution: non-finite component");
  }
  recombine_dev(ctx, f1.get(), f2.get(), f_dev, nh, 1);
}

void Plan::get_solution(int which, double* f) {
  if (which < 0 || which >= nsys) fail("plan: system index out of range");
  const std::int64_t n = cols[which] * nrhs;
  DBuf<double> tmp(n);
  const int g = grid1(ctx, n);
  if (dtype == SS_F32) {
    transpose_out_kernel<float><<<g, 256, 0, ctx->stream>>>(
        reinterpret_cast<const float*>(x[which].get()), tmp.get(), cols[which], nrhs);
  } else {
    transpose_out_kernel<double><<<g, 256, 0, ctx->stream>>>(
        reinterpret_cast<const double*>(x[which].get()), tmp.get(), cols[which], nrhs);
  }
  ctx->check_launch("transpose_out_kernel");
  SSB_CUDA(cudaMemcpyAsync(f, tmp.get(), n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
}

void Plan::get_history(int which, int slice, double* h, int* len) {
  if (which < 0 || which >= nsys || slice < 0 || slice >= nrhs) fail("plan: index out of range");
  const int q = which * nrhs + slice;
  int st[4];
  SSB_CUDA(cudaMemcpy(st, state.get() + 4 * q, sizeof st, cudaMemcpyDeviceToHost));
  const int n = st[0] ? st[1] + 1 : opts.max_iters;
  if (h) {
    SSB_CUDA(cudaMemcpy(h, history.get() + static_cast<std::int64_t>(q) * (opts.max_iters + 1),
                        n * sizeof(double), cudaMemcpyDeviceToHost));
  }
  *len = n;
}

void Plan::recombine(double* f) {
  if (nsys != 2) fail("plan: recombine needs the folded pair");
  const std::int64_t nh = cols[0];
  DBuf<double> f1(nh * nrhs), f2(nh * nrhs), out(2 * nh * nrhs);
  const int g = grid1(ctx, nh * nrhs);
  if (dtype == SS_F32) {
    to_f64_kernel<float><<<g, 256, 0, ctx->stream>>>(reinterpret_cast<const float*>(x[0].get()),
                                                    f1.get(), nh * nrhs);
    to_f64_kernel<float><<<g, 256, 0, ctx->stream>>>(reinterpret_cast<const float*>(x[1].get()),
                                                    f2.get(), nh * nrhs);
  } else {
    to_f64_kernel<double><<<g, 256, 0, ctx->stream>>>(
        reinterpret_cast<const double*>(x[0].get()), f1.get(), nh * nrhs);
    to_f64_kernel<double><<<g, 256, 0, ctx->stream>>>(
        reinterpret_cast<const double*>(x[1].get()), f2.get(), nh * nrhs);
  }
  ctx->check_launch("to_f64_kernel");
  recombine_dev(ctx, f1.get(), f2.get(), out.get(), nh, nrhs);
  SSB_CUDA(cudaMemcpyAsync(f, out.get(), 2 * nh * nrhs * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  ctx->sync();
}

void Plan::profile(int iters, float* fwd_ms, float* back_ms) {
  cudaEvent_t e[3];
  for (auto& q : e) SSB_CUDA(cudaEventCreate(&q));
  float tf = 0.f, tb = 0.f;
  enqueue_reset();
  for (int it = 0; it < iters; ++it) {
    const int i = it % std::max(1, opts.max_iters);
    SSB_CUDA(cudaEventRecord(e[0], ctx->stream));
    if (dtype == SS_F32) {
      const SartK<float> k = make_args<float>(*this);
      launch_fwd<float>(*this, k, i);
      ctx->check_launch("sart_fwd_kernel");
      SSB_CUDA(cudaEventRecord(e[1], ctx->stream));
      launch_back<float>(*this, k, i);
    } else {
      const SartK<double> k = make_args<double>(*this);
      launch_fwd<double>(*this, k, i);
      ctx->check_launch("sart_fwd_kernel");
      SSB_CUDA(cudaEventRecord(e[1], ctx->stream));
      launch_back<double>(*this, k, i);
    }
    ctx->check_launch("sart_back_kernel");
    SSB_CUDA(cudaEventRecord(e[2], ctx->stream));
    SSB_CUDA(cudaEventSynchronize(e[2]));
    float a = 0.f, b = 0.f;
    SSB_CUDA(cudaEventElapsedTime(&a, e[0], e[1]));
    SSB_CUDA(cudaEventElapsedTime(&b, e[1], e[2]));
    tf += a;
    tb += b;
  }
  for (auto& q : e) cudaEventDestroy(q);
  *fwd_ms = tf;
  *back_ms = tb;
}

void Plan::stats(std::int64_t* mbytes, std::int64_t* vbytes, int* kernels) const {
  std::int64_t mb = 0, vb = 0;
  const std::int64_t b = static_cast<std::int64_t>(tsize());
  for (int s = 0; s < nsys; ++s) {
    const std::int64_t nnz = a[s]->nnz;
    mb += 2 * nnz * (b + 4) + 4 * ((rows[s] + 1) + (cols[s] + 1));
    vb += (3 * rows[s] + 4 * cols[s]) * b * nrhs;
  }
  if (mbytes) *mbytes = mb;
  if (vbytes) *vbytes = vb;
  if (kernels) *kernels = 2;
}

namespace {
void alloc_common(Plan& P) {
  const std::size_t tb = P.tsize();
  for (int s = 0; s < P.nsys; ++s) {
    P.x[s].alloc(P.cols[s] * P.nrhs * tb);
    P.w[s].alloc(P.rows[s] * P.nrhs * tb);
    P.p[s].alloc(P.rows[s] * P.nrhs * tb);
    P.rinv[s].alloc(P.rows[s] * tb);
    P.cinv[s].alloc(P.cols[s] * tb);
    SSB_CUDA(cudaMemsetAsync(P.p[s].get(), 0, P.rows[s] * P.nrhs * tb, P.ctx->stream));
  }
  const int nsr = P.nsys * P.nrhs;
  P.partial.alloc(static_cast<std::size_t>(nsr) * P.fwd_blocks);
  P.pnorm.alloc(nsr);
  SSB_CUDA(cudaMemsetAsync(P.pnorm.get(), 0, nsr * sizeof(double), P.ctx->stream));
  P.history.alloc(static_cast<std::size_t>(nsr) * (P.opts.max_iters + 1));
  P.state.alloc(4 * nsr);
  P.ticket.alloc(1);
  SSB_CUDA(cudaMemsetAsync(P.state.get(), 0, 4 * nsr * sizeof(int), P.ctx->stream));
  SSB_CUDA(cudaMemsetAsync(P.ticket.get(), 0, sizeof(unsigned), P.ctx->stream));
  SSB_CUDA(cudaEventCreate(&P.ev0));
  SSB_CUDA(cudaEventCreate(&P.ev1));
}

// Normalisers (solvers.cpp:156-168): absolute row/column sums in fp64 in
// the reference order, inverses with the zero guard, cast to the plan type.
void normalisers(Plan& P, int s, double* max_row_sum) {
  Matrix* a = P.a[s];
  DBuf<double> rs(P.rows[s]), cs(P.cols[s]);
  abs_sums(*a, rs.get(), cs.get());
  *max_row_sum = max_dev(P.ctx, rs.get(), P.rows[s]);
  const int gr = grid1(P.ctx, P.rows[s]), gc = grid1(P.ctx, P.cols[s]);
  if (P.dtype == SS_F32) {
    inv_kernel<float><<<gr, 256, 0, P.ctx->stream>>>(rs.get(),
                                                     reinterpret_cast<float*>(P.rinv[s].get()),
                                                     P.rows[s]);
    inv_kernel<float><<<gc, 256, 0, P.ctx->stream>>>(cs.get(),
                                                     reinterpret_cast<float*>(P.cinv[s].get()),
                                                     P.cols[s]);
  } else {
    inv_kernel<double><<<gr, 256, 0, P.ctx->stream>>>(rs.get(),
                                                      reinterpret_cast<double*>(P.rinv[s].get()),
                                                      P.rows[s]);
    inv_kernel<double><<<gc, 256, 0, P.ctx->stream>>>(cs.get(),
                                                      reinterpret_cast<double*>(P.cinv[s].get()),
                                                      P.cols[s]);
  }
  P.ctx->check_launch("inv_kernel");
  P.ctx->sync();
}
}  // namespace

Plan* make_plan(Context* ctx, Matrix* a1, Matrix* a2, const ss_solve_options& o, int nrhs) {
  if (o.relaxation <= 0 || o.relaxation > 2) fail("sart_solve: relaxation must be in (0, 2]");
  if (o.max_iters < 1) fail("sart_solve: max_iters must be >= 1");
  if (o.dtype != SS_F64 && o.dtype != SS_F32) fail("plan: unknown dtype");
  if (nrhs < 1 || nrhs > 256) fail("plan: nrhs must be in [1, 256]");
  if (a2 && (a2->rows != a1->rows || a2->cols != a1->cols)) {
    fail("plan: folded systems must have equal shapes");
  }
  auto P = std::make_unique<Plan>();
  P->ctx = ctx;
  P->opts = o;
  P->nrhs = nrhs;
  P->dtype = o.dtype;
  P->nsys = a2 ? 2 : 1;
  P->a[0] = a1;
  P->a[1] = a2;
  double nnz_total = 0, rows_total = 0, cols_total = 0;
  for (int s = 0; s < P->nsys; ++s) {
    Matrix* a = P->a[s];
    a->ensure_csc();
    if (o.dtype == SS_F32) a->ensure_f32();
    P->rows[s] = a->rows;
    P->cols[s] = a->cols;
    nnz_total += a->nnz;
    rows_total += a->rows;
    cols_total += a->cols;
  }
  P->vs_fwd = pick_vs(rows_total > 0 ? nnz_total / rows_total : 0);
  P->vs_back = pick_vs(cols_total > 0 ? nnz_total / cols_total : 0);
  if (o.dtype == SS_F32) {
    P->fwd_blocks = occupancy_blocks<float>(*P, true);
    P->back_blocks = occupancy_blocks<float>(*P, false);
  } else {
    P->fwd_blocks = occupancy_blocks<double>(*P, true);
    P->back_blocks = occupancy_blocks<double>(*P, false);
  }
  // never more blocks than row/column groups to work on
  const long long fwd_groups = static_cast<long long>(rows_total) *
                               (nrhs > 1 ? 32 : P->vs_fwd);
  const long long back_groups = static_cast<long long>(cols_total) *
                                (nrhs > 1 ? 32 : P->vs_back);
  P->fwd_blocks = static_cast<int>(std::max<long long>(
      1, std::min<long long>(P->fwd_blocks, (fwd_groups + kThreads - 1) / kThreads)));
  P->back_blocks = static_cast<int>(std::max<long long>(
      1, std::min<long long>(P->back_blocks, (back_groups + kThreads - 1) / kThreads)));
  alloc_common(*P);
  for (int s = 0; s < P->nsys; ++s) {
    double mx = 0;
    normalisers(*P, s, &mx);
    P->empty_rows[s] = !(mx > 0.0);
  }
  if (P->nsys == 1 && P->empty_rows[0]) fail("sart_solve: matrix has no nonzero rows");
  P->build_graph();
  return P.release();
}

void partition_rows(const int* rowptr, std::int64_t rows, int parts, std::int64_t* bounds) {
  if (parts < 1) fail("partition_rows: parts must be >= 1");
  const double total = static_cast<double>(rowptr[rows]) + static_cast<double>(rows);
  bounds[0] = 0;
  std::int64_t r = 0;
  for (int q = 1; q < parts; ++q) {
    // rows weighted by nnz + 1 (row pointer / vector traffic)
    const double target = total * q / parts;
    while (r < rows && static_cast<double>(rowptr[r]) + static_cast<double>(r) < target) ++r;
    bounds[q] = std::max(bounds[q - 1], r);
  }
  bounds[parts] = rows;
}

// Row-sharded plan: keeps rows [rb, re) of the folded system `a` (all its
// columns). Column normalisers come from the full matrix (every rank holds
// the same column sums), row normalisers from the local rows.
Plan* make_sharded_plan(Context* ctx, Matrix* a, std::int64_t rb, std::int64_t re,
                        const ss_solve_options& o) {
  if (!ctx->comm) fail("plan: context has no NCCL communicator");
  if (rb < 0 || re > a->rows || rb > re) fail("plan: row range out of bounds");
  if (o.relaxation <= 0 || o.relaxation > 2) fail("sart_solve: relaxation must be in (0, 2]");
  if (o.max_iters < 1) fail("sart_solve: max_iters must be >= 1");
  a->ensure_csc();
  // host-side slice of the CSR row block, then a local matrix on device
  std::vector<int> ptr(a->rows + 1);
  SSB_CUDA(cudaMemcpy(ptr.data(), a->rowptr.get(), ptr.size() * sizeof(int),
                      cudaMemcpyDeviceToHost));
  const std::int64_t k0 = ptr[rb], k1 = ptr[re], nloc = k1 - k0, rloc = re - rb;
  std::vector<int> lptr(rloc + 1), lcol(nloc), lrow(nloc);
  std::vector<double> lval(nloc);
  for (std::int64_t r = 0; r <= rloc; ++r) lptr[r] = static_cast<int>(ptr[rb + r] - k0);
  SSB_CUDA(cudaMemcpy(lcol.data(), a->colidx.get() + k0, nloc * sizeof(int), cudaMemcpyDeviceToHost));
  SSB_CUDA(cudaMemcpy(lval.data(), a->val.get() + k0, nloc * sizeof(double), cudaMemcpyDeviceToHost));
  for (std::int64_t r = 0; r < rloc; ++r) {
    for (int k = lptr[r]; k < lptr[r + 1]; ++k) lrow[k] = static_cast<int>(r);
  }
  auto P = std::make_unique<Plan>();
  P->own = matrix_from_triplets_host(ctx, rloc, a->cols, nloc, lrow.data(), lcol.data(),
                                     lval.data());
  P->own->ensure_csc();
  if (o.dtype == SS_F32) P->own->ensure_f32();
  P->ctx = ctx;
  P->opts = o;
  P->nrhs = 1;
  P->dtype = o.dtype;
  P->nsys = 1;
  P->sharded = true;
  P->row_begin = rb;
  P->row_end = re;
  P->a[0] = P->own;
  P->rows[0] = rloc;
  P->cols[0] = a->cols;
  P->vs_fwd = pick_vs(rloc > 0 ? double(nloc) / rloc : 0);
  P->vs_back = pick_vs(a->cols > 0 ? double(nloc) / a->cols : 0);
  if (o.dtype == SS_F32) {
    P->fwd_blocks = occupancy_blocks<float>(*P, true);
    P->back_blocks = occupancy_blocks<float>(*P, false);
  } else {
    P->fwd_blocks = occupancy_blocks<double>(*P, true);
    P->back_blocks = occupancy_blocks<double>(*P, false);
  }
  alloc_common(*P);
  P->bp.alloc((a->cols + 1) * P->tsize());
  // normalisers: rows from the local block, columns from the full matrix
  DBuf<double> rs_full(a->rows), cs_full(a->cols);
  abs_sums(*a, rs_full.get(), cs_full.get());
  const int gr = grid1(ctx, rloc), gc = grid1(ctx, a->cols);
  if (o.dtype == SS_F32) {
    inv_kernel<float><<<gr, 256, 0, ctx->stream>>>(rs_full.get() + rb,
                                                   reinterpret_cast<float*>(P->rinv[0].get()), rloc);
    inv_kernel<float><<<gc, 256, 0, ctx->stream>>>(cs_full.get(),
                                                   reinterpret_cast<float*>(P->cinv[0].get()),
                                                   a->cols);
  } else {
    inv_kernel<double><<<gr, 256, 0, ctx->stream>>>(rs_full.get() + rb,
                                                    reinterpret_cast<double*>(P->rinv[0].get()), rloc);
    inv_kernel<double><<<gc, 256, 0, ctx->stream>>>(cs_full.get(),
                                                    reinterpret_cast<double*>(P->cinv[0].get()),
                                                    a->cols);
  }
  ctx->check_launch("inv_kernel");
  if (!(max_dev(ctx, rs_full.get(), a->rows) > 0.0)) fail("sart_solve: matrix has no nonzero rows");
  ctx->sync();
  return P.release();
}

}  // namespace ssb
