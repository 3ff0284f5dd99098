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

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "nccl_dyn.hpp"
#include "plan.hpp"

namespace ssb {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef SSB_DIRECT_MIN_BLOCKS
#define SSB_DIRECT_MIN_BLOCKS 4
#endif
constexpr int kDirectMinBlocks = SSB_DIRECT_MIN_BLOCKS;  // 32 registers: full occupancy

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
  // multi-RHS column band of this K1 pass: row i's entries [bb[i], be[i])
  // (nullptr: the whole row, rp[i]..rp[i+1])
  const int* bb;
  const int* be;
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
  int sys_blocks[2];            // CTA-uniform dispatch: first CTA of system 1 (fwd, back)
  T* xx;                        // paired plans: iterates interleaved [cols][2]
  T* ww;                        //               weighted residuals [rows][2]
  const T* rv2;                 //               CSR values interleaved [nnz][2]
  const T* cv2;                 //               CSC values interleaved [nnz][2]
  const T* pe;                  //               per row {p1, p2, rinv1, rinv2}
  const T* cc;                  //               per column {cinv1, cinv2}
  const int* tpf;               //               tiled: padded row pointer / indices
  const int* tif;
  const int* tpb;               //               tiled: padded column pointer / indices
  const int* tib;
  const unsigned short* tof;    //               u16 tiled: offsets / tile bases / first tile (K1)
  const int* tbf;
  const int* tff;
  const unsigned short* tob;    //               u16 tiled (K2)
  const int* tbb;
  const int* tfb;
  // mirror-coded pair streams (TL 4/5, see seg_dot2m): per tile {int32 base,
  // sign words}; rv2 / cv2 then hold one value per entry. Buckets whose two
  // values are not +-equal live in a per-vector exception list.
  const unsigned* thf;
  const unsigned* thb;
  const int* epf;  // exceptions, K1: per row pointer, column, {a1, a2}
  const int* eif;
  const T* evf;
  const int* epb;  // exceptions, K2: per column pointer, row, {a1, a2}
  const int* eib;
  const T* evb;
  // row-sharded: K2 writes the partial back-projection to bp_out[0..cols);
  // K1's ||r_g||^2 goes to an fp64 slot behind it (one grouped all-reduce)
  T* bp_out;
  // graph WHILE-loop mode: the iteration index lives on the device; the last
  // block of K1 advances it and decides whether the loop body runs again
  int* iter;
  cudaGraphConditionalHandle cond;
  int max_iters;
};

// iteration index of this launch: K1 reads the counter K1's last block then
// advances, so K2 of the same pass sees it + 1. iter[1] != 0 once the loop is
// over (max_iters reached or every system stopped): the remaining unrolled
// passes of the WHILE body return at once.
template <class T>
__device__ __forceinline__ int pass_index(const SartK<T>& k, int it, bool fwd) {
  if (!k.iter) return it;
  const int c = *(volatile const int*)k.iter;
  return fwd ? c : c - 1;
}

// iter[1]: 0 while the loop runs; 1 once K1's last block ended it (the K2 of
// that same pass still runs: it applies the final update of every system still
// on -- sart_solve updates x on every one of its max_iters iterations); 2 once
// a later K1 of the unrolled body found the loop over, so the K2 after it
// returns too.
template <class T>
__device__ __forceinline__ bool loop_over(const SartK<T>& k, bool fwd) {
  if (!k.iter) return false;
  const int o = *(volatile const int*)(k.iter + 1);
  if (fwd) {
    if (o != 0 && blockIdx.x == 0 && threadIdx.x == 0) k.iter[1] = 2;
    return o != 0;
  }
  return o == 2;
}

// last block of K1 in WHILE-loop mode: advance the pass counter and run
// another pass while iterations remain and some system / slice is still on
template <class T>
__device__ __forceinline__ void loop_next(const SartK<T>& k, int it) {
  if (!k.iter || threadIdx.x != 0) return;
  const int nit = it + 1;
  k.iter[0] = nit;
  bool any = false;
  for (int q = 0; q < k.nsys * k.nrhs && !any; ++q) {
    const volatile int* st = k.state + 4 * q;  // not stopped, not diverged
    any = st[0] == 0 && st[2] == 0;
  }
  const bool more = nit < k.max_iters && any;
  k.iter[1] = more ? 0 : 1;
  cudaGraphSetConditional(k.cond, more ? 1u : 0u);
}

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
// vector by VS cooperating lanes. The scalar head (up to the 16-byte
// boundary) and tail are loaded first; the 4-wide body issues UF steps of
// (int4 indices + 4 values) per lane before any dependent gather, so
// UF*VS*32 bytes of matrix stream are in flight per group; then a VS-lane
// butterfly.
template <class T, int VS, int UF>
__device__ __forceinline__ T seg_dot(const int* __restrict__ idx, const T* __restrict__ val,
                                     const T* __restrict__ vec, int beg, int end, int lane,
                                     unsigned mask) {
  T acc = T(0);
  int a = (beg + 3) & ~3;
  if (a > end) a = end;
  const int nvec = (end - a) >> 2;
  const int b = a + (nvec << 2);
  const bool hon = beg + lane < a, ton = b + lane < end;
  T hv = T(0), tv = T(0);
  int hc = 0, tc = 0;
  if (hon) {
    hv = __ldg(val + beg + lane);
    hc = __ldg(idx + beg + lane);
  }
  if (ton) {
    tv = __ldg(val + b + lane);
    tc = __ldg(idx + b + lane);
  }
  int q = lane;
  for (; q + (UF - 1) * VS < nvec; q += UF * VS) {
    int4 c[UF];
    T v[UF][4];
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const int k0 = a + ((q + u * VS) << 2);
      c[u] = __ldg(reinterpret_cast<const int4*>(idx + k0));
      load4(val + k0, v[u]);
    }
    T g[UF][4];
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      g[u][0] = __ldg(vec + c[u].x);
      g[u][1] = __ldg(vec + c[u].y);
      g[u][2] = __ldg(vec + c[u].z);
      g[u][3] = __ldg(vec + c[u].w);
    }
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      acc += v[u][0] * g[u][0] + v[u][1] * g[u][1] + v[u][2] * g[u][2] + v[u][3] * g[u][3];
    }
  }
  for (; q < nvec; q += VS) {
    const int k0 = a + (q << 2);
    const int4 c0 = __ldg(reinterpret_cast<const int4*>(idx + k0));
    T v0[4];
    load4(val + k0, v0);
    acc += v0[0] * __ldg(vec + c0.x) + v0[1] * __ldg(vec + c0.y) + v0[2] * __ldg(vec + c0.z) +
           v0[3] * __ldg(vec + c0.w);
  }
  if (hon) acc += hv * __ldg(vec + hc);
  if (ton) acc += tv * __ldg(vec + tc);
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

// One system's run flag from one 16-byte L2 load (sys_on's two dependent
// volatile loads in one): for kernels that read the state once at their start,
// after the grid dependency. Every thread of every CTA reads the same line, so
// the number of dependent round trips is what the start of a pass waits for.
__device__ __forceinline__ bool sys_on_cg(const int* state, int idx) {
  const int4 s = __ldcg(reinterpret_cast<const int4*>(state) + idx);
  return s.x == 0 && s.z == 0;
}

// Both systems' run flags of a paired plan for a whole CTA: threads 0 / 1 load
// one system's state words each (one 16-byte L2 load) and broadcast through
// shared memory. Every thread evaluating sys_on sent 4,736 warps x up to 4
// dependent loads at one L2 line at the start of each pass (measured in the
// resident kernel: 4.7 us per pass).
__device__ __forceinline__ void cta_run_flags(const int* state, bool& on0, bool& on1) {
  __shared__ int run_sh[2];
  if (threadIdx.x < 2) {
    const int4 s = __ldcg(reinterpret_cast<const int4*>(state) + threadIdx.x);
    run_sh[threadIdx.x] = (s.x == 0 && s.z == 0) ? 1 : 0;
  }
  __syncthreads();
  on0 = run_sh[0] != 0;
  on1 = run_sh[1] != 0;
}

// Fixed-order reduction of per-block partials by the last block of K1, then
// the reference's check-before-update stopping rule (solvers.cpp:180-182).
__device__ void finish_norms(double* partial, int nblk, int nsr, const double* pnorm, double tol,
                             double* history, int hstride, int* state, int it) {
  // one warp per system / slice, all in parallel and without block barriers
  // (this runs on the critical path between K1 and K2): lane l sums partials
  // l, l+32, ... in order, then a fixed xor tree
  const int nw = static_cast<int>(blockDim.x) >> 5, lane = threadIdx.x & 31;
  for (int q = threadIdx.x >> 5; q < nsr; q += nw) {
    if (!sys_on(state, q)) continue;
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += partial[static_cast<long long>(q) * nblk + b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const double res = sqrt(s);
      history[q * hstride + it] = res;
      if (res <= tol * pnorm[q]) {
        state[4 * q + 0] = 1;
        state[4 * q + 1] = it;
      }
    }
  }
  __syncthreads();
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
// Grid-stride over the compressed vectors of one system, VS lanes each. The
// system is CTA-uniform and a template parameter (CTAs [0, split) serve
// system 0), so array pointers come straight from the parameter bank. The
// next vector's pointer pair and epilogue operands are fetched before the
// current dot product so their latency hides behind it.
template <class T>
struct VecCursor {
  int i, beg, end;
  T e1, e2;
};

template <class T, bool FWD, int SYS>
__device__ __forceinline__ void fetch_vec(const SartK<T>& k, int i, int lane, VecCursor<T>& c) {
  const SysK<T>& S = k.s[SYS];
  const int* ptr = FWD ? S.rp : S.cp;
  c.i = i;
  c.beg = __ldg(ptr + i);
  c.end = __ldg(ptr + i + 1);
  c.e1 = T(0);
  c.e2 = T(0);
  if (lane == 0) {
    if (FWD) {
      c.e1 = S.p[i];
      c.e2 = S.rinv[i];
    } else {
      c.e1 = k.bp_out ? T(0) : S.x[i];
      c.e2 = S.cinv[i];
    }
  }
}

template <class T, int VS, int UF, int SYS>
__device__ __forceinline__ double fwd_rows(const SartK<T>& k, long long group, long long ngroups,
                                           int lane, unsigned mask) {
  const SysK<T>& S = k.s[SYS];
  const long long n = SYS ? k.rows_total - k.rows0 : k.rows0;
  double acc = 0.0;
  VecCursor<T> cur, nxt;
  if (group < n) fetch_vec<T, true, SYS>(k, static_cast<int>(group), lane, cur);
  for (long long g = group; g < n; g += ngroups) {
    if (g + ngroups < n) fetch_vec<T, true, SYS>(k, static_cast<int>(g + ngroups), lane, nxt);
    const T dot = seg_dot<T, VS, UF>(S.ci, S.rv, S.x, cur.beg, cur.end, lane, mask);
    if (lane == 0) {
      const T r = cur.e1 - dot;
      S.w[cur.i] = cur.e2 * r;
      acc += static_cast<double>(r) * static_cast<double>(r);
    }
    cur = nxt;
  }
  return acc;
}

template <class T, int VS, int UF, int SYS>
__device__ __forceinline__ void back_cols(const SartK<T>& k, long long group, long long ngroups,
                                          int lane, unsigned mask, int it) {
  const SysK<T>& S = k.s[SYS];
  const long long n = SYS ? k.cols_total - k.cols0 : k.cols0;
  VecCursor<T> cur, nxt;
  if (group < n) fetch_vec<T, false, SYS>(k, static_cast<int>(group), lane, cur);
  for (long long g = group; g < n; g += ngroups) {
    if (g + ngroups < n) fetch_vec<T, false, SYS>(k, static_cast<int>(g + ngroups), lane, nxt);
    const T u = seg_dot<T, VS, UF>(S.ri, S.cv, S.w, cur.beg, cur.end, lane, mask);
    if (lane == 0) {
      if (k.bp_out) {
        k.bp_out[cur.i] = u;
      } else {
        const T xn = upd(cur.e1, k.relax, u, cur.e2);
        S.x[cur.i] = xn;
        if (!isfinite(static_cast<double>(xn))) atomicCAS(&k.state[4 * SYS + 2], 0, it + 1);
      }
    }
    cur = nxt;
  }
}

template <class T, int VS, int UF>
__global__ void __launch_bounds__(kThreads, kDirectMinBlocks) sart_fwd_kernel(SartK<T> k, int it) {
  it = pass_index(k, it, true);
  if (loop_over(k, true)) return;
  __shared__ double red[2][kWarps];
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const int split = k.sys_blocks[0];
  const int sys = static_cast<int>(blockIdx.x) >= split ? 1 : 0;
  const int bx = sys ? blockIdx.x - split : blockIdx.x;
  const int nb = sys ? gridDim.x - split : min(split, static_cast<int>(gridDim.x));
  const long long group = (bx * (long long)kThreads + threadIdx.x) / VS;
  const long long ngroups = (long long)nb * kThreads / VS;
  double acc = 0.0;
  if (sys_on(k.state, sys)) {
    acc = sys ? fwd_rows<T, VS, UF, 1>(k, group, ngroups, lane, mask)
              : fwd_rows<T, VS, UF, 0>(k, group, ngroups, lane, mask);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[0][warp] = acc;
  __syncthreads();
  if (threadIdx.x < k.nsys) {
    double t = 0.0;
    if (threadIdx.x == sys) {
      for (int q = 0; q < kWarps; ++q) t += red[0][q];
    }
    k.partial[threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
  if (k.bp_out) return;  // sharded plans reduce ||r||^2 across ranks instead
  if (last_block(k.ticket)) {
    finish_norms(k.partial, gridDim.x, k.nsys, k.pnorm, k.tol, k.history, k.hstride,
                 k.state, it);
    loop_next(k, it);
    if (threadIdx.x == 0) *k.ticket = 0;
  }
}

template <class T, int VS, int UF>
__global__ void __launch_bounds__(kThreads, kDirectMinBlocks) sart_back_kernel(SartK<T> k, int it) {
  it = pass_index(k, it, false);
  if (loop_over(k, false)) return;
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const int split = k.sys_blocks[1];
  const int sys = static_cast<int>(blockIdx.x) >= split ? 1 : 0;
  const int bx = sys ? blockIdx.x - split : blockIdx.x;
  const int nb = sys ? gridDim.x - split : min(split, static_cast<int>(gridDim.x));
  const long long group = (bx * (long long)kThreads + threadIdx.x) / VS;
  const long long ngroups = (long long)nb * kThreads / VS;
  if (!sys_on(k.state, sys)) return;
  if (sys) back_cols<T, VS, UF, 1>(k, group, ngroups, lane, mask, it);
  else back_cols<T, VS, UF, 0>(k, group, ngroups, lane, mask, it);
}

// ------------------------------------------------------------ paired kernels
// The fold puts A1 = TL - BL and A2 = TL + BL on the same buckets; a plan over
// the folded pair streams ONE index array and two value arrays (the union
// pattern, cancelled A1 entries as explicit zeros, which leaves every sum
// unchanged) and gathers x1/x2 (w1/w2) together: 4 + 2b bytes per bucket
// instead of 2(4 + b), and one pointer/epilogue chain per row for both systems.
template <class T> struct Vec2;
template <> struct Vec2<float> { using type = float2; };
template <> struct Vec2<double> { using type = double2; };

// 4 consecutive entries of the interleaved value stream: v[2q] (system 0),
// v[2q+1] (system 1).
// Matrix-stream loads: read-only path, or (CS) the evict-first streaming
// hint (ld.global.cs) so a stream larger than L2 does not displace the
// gathered x / w. Plans enable it for fp32 streams of 1-16x the L2 (+2.5% on
// config 3; it costs 3.5% on fp64, 13% on the L2-resident config 2 and 2.6%
// on config 5's 11.6 GB stream). The remainder loop keeps the read-only
// path for its offsets (measured faster).
template <bool CS, class V>
__device__ __forceinline__ V lds(const V* p) {
  if constexpr (CS) return __ldcs(p);
  else return __ldg(p);
}

template <bool CS = false>
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
  const float4 a = lds<CS>(reinterpret_cast<const float4*>(p));
  const float4 b = lds<CS>(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <bool CS = false>
__device__ __forceinline__ void load8(const double* p, double (&v)[8]) {
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const double2 a = lds<CS>(reinterpret_cast<const double2*>(p) + h);
    v[2 * h] = a.x;
    v[2 * h + 1] = a.y;
  }
}

template <class T, int VS, int UF>
__device__ __forceinline__ void seg_dot2(const int* __restrict__ idx, const T* __restrict__ v2,
                                         const typename Vec2<T>::type* __restrict__ xv, int beg,
                                         int end, int lane, unsigned mask, T& acc_a, T& acc_b) {
  using T2 = typename Vec2<T>::type;
  T sa = T(0), sb = T(0);
  int a = (beg + 3) & ~3;
  if (a > end) a = end;
  const int nvec = (end - a) >> 2;
  const int b = a + (nvec << 2);
  const bool hon = beg + lane < a, ton = b + lane < end;
  T2 hv, tv;
  hv.x = hv.y = tv.x = tv.y = T(0);
  int hc = 0, tc = 0;
  if (hon) {
    hc = __ldg(idx + beg + lane);
    hv = __ldg(reinterpret_cast<const T2*>(v2) + beg + lane);
  }
  if (ton) {
    tc = __ldg(idx + b + lane);
    tv = __ldg(reinterpret_cast<const T2*>(v2) + b + lane);
  }
  int q = lane;
  for (; q + (UF - 1) * VS < nvec; q += UF * VS) {
    int4 c[UF];
    T v[UF][8];
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const int k0 = a + ((q + u * VS) << 2);
      c[u] = __ldg(reinterpret_cast<const int4*>(idx + k0));
      load8(v2 + 2 * k0, v[u]);
    }
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const T2 g0 = __ldg(xv + c[u].x), g1 = __ldg(xv + c[u].y), g2 = __ldg(xv + c[u].z),
               g3 = __ldg(xv + c[u].w);
      sa += v[u][0] * g0.x + v[u][2] * g1.x + v[u][4] * g2.x + v[u][6] * g3.x;
      sb += v[u][1] * g0.y + v[u][3] * g1.y + v[u][5] * g2.y + v[u][7] * g3.y;
    }
  }
  for (; q < nvec; q += VS) {
    const int k0 = a + (q << 2);
    const int4 c0 = __ldg(reinterpret_cast<const int4*>(idx + k0));
    T v[8];
    load8(v2 + 2 * k0, v);
    const T2 g0 = __ldg(xv + c0.x), g1 = __ldg(xv + c0.y), g2 = __ldg(xv + c0.z),
             g3 = __ldg(xv + c0.w);
    sa += v[0] * g0.x + v[2] * g1.x + v[4] * g2.x + v[6] * g3.x;
    sb += v[1] * g0.y + v[3] * g1.y + v[5] * g2.y + v[7] * g3.y;
  }
  if (hon) {
    const T2 g = __ldg(xv + hc);
    sa += hv.x * g.x;
    sb += hv.y * g.y;
  }
  if (ton) {
    const T2 g = __ldg(xv + tc);
    sa += tv.x * g.x;
    sb += tv.y * g.y;
  }
#pragma unroll
  for (int off = VS / 2; off > 0; off >>= 1) {
    sa += __shfl_xor_sync(mask, sa, off, VS);
    sb += __shfl_xor_sync(mask, sb, off, VS);
  }
  acc_a = sa;
  acc_b = sb;
}

// Tiled layout (built by tile_stream_kernel): every vector starts on a quad
// boundary and holds a multiple of 4 entries (zero-valued padding), and
// within each tile of R <= VS quads the quad of lane l carries the original
// entries l, l+R, l+2R, l+3R. Component j of the UF steps therefore gathers
// consecutive entries across the lanes of one instruction -- neighbouring
// voxels (rays) in the snake numbering -- so one gather touches a few L1
// lines instead of one per lane. No scalar head/tail: fewer registers.
template <class T, int VS, int UF>
__device__ __forceinline__ void seg_dot2t(const int* __restrict__ idx, const T* __restrict__ v2,
                                          const typename Vec2<T>::type* __restrict__ xv, int beg,
                                          int end, int lane, unsigned mask, T& acc_a, T& acc_b) {
  using T2 = typename Vec2<T>::type;
  T sa = T(0), sb = T(0);
  const int nvec = (end - beg) >> 2;
  int q = lane;
  for (; q + (UF - 1) * VS < nvec; q += UF * VS) {
    int4 c[UF];
    T v[UF][8];
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const int k0 = beg + ((q + u * VS) << 2);
      c[u] = __ldg(reinterpret_cast<const int4*>(idx + k0));
      load8(v2 + 2 * k0, v[u]);
    }
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const T2 g0 = __ldg(xv + c[u].x), g1 = __ldg(xv + c[u].y), g2 = __ldg(xv + c[u].z),
               g3 = __ldg(xv + c[u].w);
      sa += v[u][0] * g0.x + v[u][2] * g1.x + v[u][4] * g2.x + v[u][6] * g3.x;
      sb += v[u][1] * g0.y + v[u][3] * g1.y + v[u][5] * g2.y + v[u][7] * g3.y;
    }
  }
  for (; q < nvec; q += VS) {
    const int k0 = beg + (q << 2);
    const int4 c0 = __ldg(reinterpret_cast<const int4*>(idx + k0));
    T v[8];
    load8(v2 + 2 * k0, v);
    const T2 g0 = __ldg(xv + c0.x), g1 = __ldg(xv + c0.y), g2 = __ldg(xv + c0.z),
             g3 = __ldg(xv + c0.w);
    sa += v[0] * g0.x + v[2] * g1.x + v[4] * g2.x + v[6] * g3.x;
    sb += v[1] * g0.y + v[3] * g1.y + v[5] * g2.y + v[7] * g3.y;
  }
#pragma unroll
  for (int off = VS / 2; off > 0; off >>= 1) {
    sa += __shfl_xor_sync(mask, sa, off, VS);
    sb += __shfl_xor_sync(mask, sb, off, VS);
  }
  acc_a = sa;
  acc_b = sb;
}

// The tiled layout with 16-bit indices: each tile (the VS quads one step of
// a VS-lane group covers) stores an int32 base (its smallest index) and every
// entry a uint16 offset from it -- 2 bytes per entry instead of 4 on the
// stream. Used when every tile of the plan spans < 65536 indices.
__device__ __forceinline__ int4 decode16(uint2 o, int b) {
  return make_int4(b + static_cast<int>(o.x & 0xffffu), b + static_cast<int>(o.x >> 16),
                   b + static_cast<int>(o.y & 0xffffu), b + static_cast<int>(o.y >> 16));
}

template <class T, int VS, int UF, bool CS = false>
__device__ __forceinline__ void seg_dot2c(const unsigned short* __restrict__ off,
                                          const int* __restrict__ tbase, int tf,
                                          const T* __restrict__ v2,
                                          const typename Vec2<T>::type* __restrict__ xv, int beg,
                                          int end, int lane, unsigned mask, T& acc_a, T& acc_b) {
  using T2 = typename Vec2<T>::type;
  T sa = T(0), sb = T(0);
  const int nvec = (end - beg) >> 2;
  int q = lane;
  for (; q + (UF - 1) * VS < nvec; q += UF * VS) {
    uint2 o[UF];
    int b[UF];
    T v[UF][8];
    const int t0 = tf + (q - lane) / VS;
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const int k0 = beg + ((q + u * VS) << 2);
      o[u] = lds<CS>(reinterpret_cast<const uint2*>(off + k0));
      b[u] = __ldg(tbase + t0 + u);
      load8<CS>(v2 + 2 * k0, v[u]);
    }
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const int4 c = decode16(o[u], b[u]);
      const T2 g0 = __ldg(xv + c.x), g1 = __ldg(xv + c.y), g2 = __ldg(xv + c.z),
               g3 = __ldg(xv + c.w);
      sa += v[u][0] * g0.x + v[u][2] * g1.x + v[u][4] * g2.x + v[u][6] * g3.x;
      sb += v[u][1] * g0.y + v[u][3] * g1.y + v[u][5] * g2.y + v[u][7] * g3.y;
    }
  }
  for (; q < nvec; q += VS) {
    const int k0 = beg + (q << 2);
    const int4 c = decode16(__ldg(reinterpret_cast<const uint2*>(off + k0)),
                            __ldg(tbase + tf + (q - lane) / VS));
    T v[8];
    load8<CS>(v2 + 2 * k0, v);
    const T2 g0 = __ldg(xv + c.x), g1 = __ldg(xv + c.y), g2 = __ldg(xv + c.z),
             g3 = __ldg(xv + c.w);
    sa += v[0] * g0.x + v[2] * g1.x + v[4] * g2.x + v[6] * g3.x;
    sb += v[1] * g0.y + v[3] * g1.y + v[5] * g2.y + v[7] * g3.y;
  }
#pragma unroll
  for (int off2 = VS / 2; off2 > 0; off2 >>= 1) {
    sa += __shfl_xor_sync(mask, sa, off2, VS);
    sb += __shfl_xor_sync(mask, sb, off2, VS);
  }
  acc_a = sa;
  acc_b = sb;
}

// Mirror-coded pair stream. Every bucket of the fold holds a1 = +-a2 unless
// its row meets both a voxel and that voxel's point mirror (the 4-term
// buckets of split_matrix, centro.cpp:103-130): TL only gives a1 = a2 = TL,
// TR only gives a1 = -TR, a2 = TR. So the stream stores a2 once per entry plus
// one sign bit for a1 -- exact in any precision, since negation is -- and the
// few remaining buckets move to a per-vector exception list {index, a1, a2}
// (their slot in the stream holds 0). fp32: 6 instead of 10 bytes per entry.
// The sign bits of a tile sit in its header next to the base: lane l's four
// entries are bits 4l..4l+3 (header = uint2 {base, bits} for VS <= 8, uint4
// {base, bits 0-31, bits 32-63, -} for VS = 16, 8 words for VS = 32).
template <int VS>
__device__ __forceinline__ void load_hdr(const unsigned* __restrict__ h, int t, int lane,
                                         int& base, unsigned& nib) {
  if constexpr (VS <= 8) {
    const uint2 w = __ldg(reinterpret_cast<const uint2*>(h) + t);
    base = static_cast<int>(w.x);
    nib = w.y >> (4 * lane);
  } else if constexpr (VS == 16) {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(h) + t);
    base = static_cast<int>(w.x);
    nib = (lane < 8 ? w.y : w.z) >> (4 * (lane & 7));
  } else {
    base = static_cast<int>(__ldg(h + 8 * t));
    nib = __ldg(h + 8 * t + 1 + (lane >> 3)) >> (4 * (lane & 7));
  }
}

__device__ __forceinline__ float flip(float v, unsigned nib, int j) {
  return __int_as_float(__float_as_int(v) ^ static_cast<int>((nib << (31 - j)) & 0x80000000u));
}
__device__ __forceinline__ double flip(double v, unsigned nib, int j) {
  return __hiloint2double(__double2hiint(v) ^ static_cast<int>((nib << (31 - j)) & 0x80000000u),
                          __double2loint(v));
}

template <bool CS>
__device__ __forceinline__ void load4s(const float* p, float (&v)[4]) {
  const float4 t = lds<CS>(reinterpret_cast<const float4*>(p));
  v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
}
template <bool CS>
__device__ __forceinline__ void load4s(const double* p, double (&v)[4]) {
  const double2 a = lds<CS>(reinterpret_cast<const double2*>(p));
  const double2 b = lds<CS>(reinterpret_cast<const double2*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

// With U16 = false (tiles spanning >= 65536 indices, e.g. config 5's K2) the
// entries keep int32 indices (tidx) and the header's base word is unused.
// gathered-vector load: read-only path, or (NC = false) a plain load for a
// vector that other CTAs rewrite during the same (persistent) kernel
template <bool NC, class V>
__device__ __forceinline__ V ldx(const V* p) {
  if constexpr (NC) return __ldg(p);
  else return *p;
}

template <class T, int VS, int UF, bool CS = false, bool U16 = true, bool NC = true>
__device__ __forceinline__ void seg_dot2m(const unsigned short* __restrict__ off,
                                          const int* __restrict__ tidx,
                                          const unsigned* __restrict__ hdr, int tf,
                                          const T* __restrict__ v1,
                                          const typename Vec2<T>::type* __restrict__ xv, int beg,
                                          int end, int eb, int ee, const int* __restrict__ eidx,
                                          const T* __restrict__ ev2, int lane, unsigned mask,
                                          T& acc_a, T& acc_b) {
  using T2 = typename Vec2<T>::type;
  T sa = T(0), sb = T(0);
  const int nvec = (end - beg) >> 2;
  int q = lane;
  for (; q + (UF - 1) * VS < nvec; q += UF * VS) {
    uint2 o[UF];
    int4 ci[UF];
    int b[UF];
    unsigned s[UF];
    T v[UF][4];
    const int t0 = tf + (q - lane) / VS;
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const int k0 = beg + ((q + u * VS) << 2);
      if constexpr (U16) o[u] = lds<CS>(reinterpret_cast<const uint2*>(off + k0));
      else ci[u] = lds<CS>(reinterpret_cast<const int4*>(tidx + k0));
      load_hdr<VS>(hdr, t0 + u, lane, b[u], s[u]);
      load4s<CS>(v1 + k0, v[u]);
    }
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      int4 c;
      if constexpr (U16) c = decode16(o[u], b[u]);
      else c = ci[u];
      const T2 g0 = ldx<NC>(xv + c.x), g1 = ldx<NC>(xv + c.y), g2 = ldx<NC>(xv + c.z),
               g3 = ldx<NC>(xv + c.w);
      sa += flip(v[u][0], s[u], 0) * g0.x + flip(v[u][1], s[u], 1) * g1.x +
            flip(v[u][2], s[u], 2) * g2.x + flip(v[u][3], s[u], 3) * g3.x;
      sb += v[u][0] * g0.y + v[u][1] * g1.y + v[u][2] * g2.y + v[u][3] * g3.y;
    }
  }
  for (; q < nvec; q += VS) {
    const int k0 = beg + (q << 2);
    int b;
    unsigned s;
    load_hdr<VS>(hdr, tf + (q - lane) / VS, lane, b, s);
    int4 c;
    if constexpr (U16) c = decode16(__ldg(reinterpret_cast<const uint2*>(off + k0)), b);
    else c = __ldg(reinterpret_cast<const int4*>(tidx + k0));
    T v[4];
    load4s<CS>(v1 + k0, v);
    const T2 g0 = ldx<NC>(xv + c.x), g1 = ldx<NC>(xv + c.y), g2 = ldx<NC>(xv + c.z),
             g3 = ldx<NC>(xv + c.w);
    sa += flip(v[0], s, 0) * g0.x + flip(v[1], s, 1) * g1.x + flip(v[2], s, 2) * g2.x +
          flip(v[3], s, 3) * g3.x;
    sb += v[0] * g0.y + v[1] * g1.y + v[2] * g2.y + v[3] * g3.y;
  }
  for (int e = eb + lane; e < ee; e += VS) {  // exception buckets (rare)
    const int c = __ldg(eidx + e);
    const T2 a = __ldg(reinterpret_cast<const T2*>(ev2) + e);
    const T2 g = ldx<NC>(xv + c);
    sa += a.x * g.x;
    sb += a.y * g.y;
  }
#pragma unroll
  for (int off2 = VS / 2; off2 > 0; off2 >>= 1) {
    sa += __shfl_xor_sync(mask, sa, off2, VS);
    sb += __shfl_xor_sync(mask, sb, off2, VS);
  }
  acc_a = sa;
  acc_b = sb;
}

template <class T, int VS, int UF, int TL>
__global__ void __launch_bounds__(kThreads, kDirectMinBlocks) sart_fwd_pair_kernel(SartK<T> k, int it) {
  using T2 = typename Vec2<T>::type;
  __shared__ double red[2][kWarps];
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const long long group = (blockIdx.x * (long long)kThreads + threadIdx.x) / VS;
  const long long ngroups = (long long)gridDim.x * kThreads / VS;
  const int n = static_cast<int>(k.rows0);
  const int* __restrict__ ptr = TL != 0 ? k.tpf : k.s[0].rp;  // tiled: padded pointer
  int g = static_cast<int>(group);
  const int gend = n, gstep = static_cast<int>(ngroups);
  // the stream layout is constant: the first row's bounds load while the
  // previous pass drains (PDL), only its results wait for the dependency
  int beg = 0, end = 0, tf = 0, eb = 0, ee = 0;
  if (g < gend) {
    beg = __ldg(ptr + g);
    end = __ldg(ptr + g + 1);
    if (TL >= 2) tf = __ldg(k.tff + g);
    if (TL >= 4 && k.epf) {
      eb = __ldg(k.epf + g);
      ee = __ldg(k.epf + g + 1);
    }
  }
  cudaGridDependencySynchronize();
  it = pass_index(k, it, true);
  if (loop_over(k, true)) return;
  // both systems' state words as two independent 16-byte L2 loads: one round
  // trip instead of up to four dependent ones (the per-CTA broadcast of K2
  // costs this kernel registers: spills in the fp64 and 16-lane variants)
  const int4 st0 = __ldcg(reinterpret_cast<const int4*>(k.state));
  const int4 st1 = __ldcg(reinterpret_cast<const int4*>(k.state) + 1);
  const bool on0 = st0.x == 0 && st0.z == 0, on1 = st1.x == 0 && st1.z == 0;
  double r2a = 0.0, r2b = 0.0;
  if (on0 || on1) {
    for (; g < gend; g += gstep) {
      const int gn = g + gstep;
      int nbeg = 0, nend = 0, ntf = 0, neb = 0, nee = 0;
      if (gn < gend) {  // next row's bounds, ahead of this row's dot product
        nbeg = __ldg(ptr + gn);
        nend = __ldg(ptr + gn + 1);
        if (TL >= 2) ntf = __ldg(k.tff + gn);
        if (TL >= 4 && k.epf) {
          neb = __ldg(k.epf + gn);
          nee = __ldg(k.epf + gn + 1);
        }
      }
      T e[4] = {T(0), T(0), T(0), T(0)};  // {p1, p2, rinv1, rinv2}, issued before the dot
      if (lane == 0) load4(k.pe + 4 * static_cast<long long>(g), e);
      T da, db;
      if (TL >= 4) {
        seg_dot2m<T, VS, UF, TL == 5, TL != 6>(k.tof, k.tif, k.thf, tf, k.rv2,
                                                reinterpret_cast<const T2*>(k.xx), beg, end, eb,
                                                ee, k.eif, k.evf, lane, mask, da, db);
      } else if (TL >= 2) {
        seg_dot2c<T, VS, UF, TL == 3>(k.tof, k.tbf, tf, k.rv2, reinterpret_cast<const T2*>(k.xx),
                                      beg, end, lane, mask, da, db);
      } else if (TL == 1) {
        seg_dot2t<T, VS, UF>(k.tif, k.rv2, reinterpret_cast<const T2*>(k.xx), beg, end, lane,
                             mask, da, db);
      } else {
        seg_dot2<T, VS, UF>(k.s[0].ci, k.rv2, reinterpret_cast<const T2*>(k.xx), beg, end, lane,
                            mask, da, db);
      }
      if (lane == 0) {
        const T ra = e[0] - da, rb = e[1] - db;
        T2 wo;
        wo.x = on0 ? e[2] * ra : T(0);
        wo.y = on1 ? e[3] * rb : T(0);
        reinterpret_cast<T2*>(k.ww)[g] = wo;
        if (on0) r2a += static_cast<double>(ra) * static_cast<double>(ra);
        if (on1) r2b += static_cast<double>(rb) * static_cast<double>(rb);
      }
      beg = nbeg;
      end = nend;
      tf = ntf;
      eb = neb;
      ee = nee;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r2a += __shfl_xor_sync(0xffffffffu, r2a, o);
    r2b += __shfl_xor_sync(0xffffffffu, r2b, o);
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][warp] = r2a;
    red[1][warp] = r2b;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double t = 0.0;
    for (int q = 0; q < kWarps; ++q) t += red[threadIdx.x][q];
    k.partial[threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
  if (last_block(k.ticket)) {
    finish_norms(k.partial, gridDim.x, 2, k.pnorm, k.tol, k.history, k.hstride, k.state, it);
    loop_next(k, it);
    if (threadIdx.x == 0) *k.ticket = 0;
  }
}

template <class T, int VS, int UF, int TL>
__global__ void __launch_bounds__(kThreads, kDirectMinBlocks) sart_back_pair_kernel(SartK<T> k, int it) {
  cudaGridDependencySynchronize();  // PDL: launched while the previous pass drains
  it = pass_index(k, it, false);
  if (loop_over(k, false)) return;
  using T2 = typename Vec2<T>::type;
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const long long group = (blockIdx.x * (long long)kThreads + threadIdx.x) / VS;
  const long long ngroups = (long long)gridDim.x * kThreads / VS;
  // run flags: one load per CTA and a broadcast (fp32: K2 51.1 -> 47.4 us on
  // config 3), or two independent 16-byte loads per thread (fp64, where the
  // CTA barrier of the broadcast measured slower: 85.5 vs 87.1 us)
  bool on0, on1;
  if constexpr (sizeof(T) == 4) {
    cta_run_flags(k.state, on0, on1);
  } else {
    const int4 st0 = __ldcg(reinterpret_cast<const int4*>(k.state));
    const int4 st1 = __ldcg(reinterpret_cast<const int4*>(k.state) + 1);
    on0 = st0.x == 0 && st0.z == 0;
    on1 = st1.x == 0 && st1.z == 0;
  }
  if (!on0 && !on1) return;
  const int n = static_cast<int>(k.cols0);
  const int* __restrict__ ptr = TL != 0 ? k.tpb : k.s[0].cp;
  int g = static_cast<int>(group);
  const int gend = n, gstep = static_cast<int>(ngroups);
  int beg = 0, end = 0, tf = 0, eb = 0, ee = 0;
  if (g < gend) {
    beg = __ldg(ptr + g);
    end = __ldg(ptr + g + 1);
    if (TL >= 2) tf = __ldg(k.tfb + g);
    if (TL >= 4 && k.epb) {
      eb = __ldg(k.epb + g);
      ee = __ldg(k.epb + g + 1);
    }
  }
  for (; g < gend; g += gstep) {
    const int gn = g + gstep;
    int nbeg = 0, nend = 0, ntf = 0, neb = 0, nee = 0;
    if (gn < gend) {
      nbeg = __ldg(ptr + gn);
      nend = __ldg(ptr + gn + 1);
      if (TL >= 2) ntf = __ldg(k.tfb + gn);
      if (TL >= 4 && k.epb) {
        neb = __ldg(k.epb + gn);
        nee = __ldg(k.epb + gn + 1);
      }
    }
    T2 xo, ci;
    xo.x = xo.y = ci.x = ci.y = T(0);
    if (lane == 0) {  // {x1, x2} and {cinv1, cinv2}, issued before the dot
      xo = reinterpret_cast<const T2*>(k.xx)[g];
      ci = __ldg(reinterpret_cast<const T2*>(k.cc) + g);
    }
    T ua, ub;
    if (TL >= 4) {
      seg_dot2m<T, VS, UF, TL == 5, TL != 6>(k.tob, k.tib, k.thb, tf, k.cv2,
                                              reinterpret_cast<const T2*>(k.ww), beg, end, eb, ee,
                                              k.eib, k.evb, lane, mask, ua, ub);
    } else if (TL >= 2) {
      seg_dot2c<T, VS, UF, TL == 3>(k.tob, k.tbb, tf, k.cv2, reinterpret_cast<const T2*>(k.ww),
                                    beg, end, lane, mask, ua, ub);
    } else if (TL == 1) {
      seg_dot2t<T, VS, UF>(k.tib, k.cv2, reinterpret_cast<const T2*>(k.ww), beg, end, lane, mask,
                           ua, ub);
    } else {
      seg_dot2<T, VS, UF>(k.s[0].ri, k.cv2, reinterpret_cast<const T2*>(k.ww), beg, end, lane,
                          mask, ua, ub);
    }
    if (lane == 0) {
      if (on0) xo.x = upd(xo.x, k.relax, ua, ci.x);
      if (on1) xo.y = upd(xo.y, k.relax, ub, ci.y);
      reinterpret_cast<T2*>(k.xx)[g] = xo;
      if (on0 && !isfinite(static_cast<double>(xo.x))) atomicCAS(&k.state[2], 0, it + 1);
      if (on1 && !isfinite(static_cast<double>(xo.y))) atomicCAS(&k.state[4 + 2], 0, it + 1);
    }
    beg = nbeg;
    end = nend;
    tf = ntf;
    eb = neb;
    ee = nee;
  }
}

// ------------------------------------------------------------ persistent paired loop
// Small folded pairs (configs 1-2: L2-resident, ~10 us per pass of two
// launches) are launch- and tail-latency bound. The persistent kernel runs the
// whole loop in one cooperative launch: per pass the K1 phase (rows) and the
// K2 phase (columns) of the pair kernels, separated by grid barriers. Every
// CTA sums the per-CTA ||r||^2 partials in the same fixed order as
// finish_norms, so all CTAs take the same stop decision (the reference's
// check-before-update rule, solvers.cpp:180-182) without a further barrier;
// CTA 0 records the history. Gathered vectors are read with plain loads (they
// change inside the kernel); the gpu-scope fences of the barrier order them.
constexpr long long kBarrierSpinCycles = 4000000000LL;  // ~2 s: a lost CTA traps

// Grid barrier of the persistent loops (all CTAs co-resident): every CTA adds 1 and CTA 0
// adds 2^31 - (n - 1), so bit 31 of the word flips exactly when all n CTAs
// have arrived and the low bits are back at 0 (no reset, no last-arriver hop,
// no generation word). `phase` is the bit-31 value that ends the caller's
// next barrier: thread 0 reads it from the word before its first arrival
// (the bit cannot flip before this CTA arrives) and flips it per barrier.
// One release-ordered reduction after the CTA's bar.sync (publishes every
// thread's stores), acquire polling by thread 0, then bar.sync: the other
// threads' weak loads are ordered after the acquire through the CTA barrier.
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_sync_flip(unsigned* bar, unsigned& phase) {
  __syncthreads();
  if (threadIdx.x == 0) {
    phase ^= 0x80000000u;
    const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u;
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(inc) : "memory");
    const long long t0 = clock64();
    while ((ld_acquire_gpu(bar) & 0x80000000u) != phase) {
      if (clock64() - t0 > kBarrierSpinCycles) __trap();
    }
  }
  __syncthreads();
}

// the two systems' run flags read by one thread per CTA and broadcast (every
// thread reading the state words made one L2 line a hot spot: ~4.7 us per pass
// with 148 x 32 warps)
__device__ __forceinline__ void load_run_flags(const int* state, int* flags) {
  if (threadIdx.x < 2) flags[threadIdx.x] = sys_on(state, threadIdx.x) ? 1 : 0;
  __syncthreads();
}

template <class T, int VSF, int VSB, int UF, int TL>
__global__ void __launch_bounds__(kThreads, 2)
    sart_persistent_pair_kernel(SartK<T> k, int first, int count, unsigned* bar) {
  using T2 = typename Vec2<T>::type;
  constexpr bool U16 = TL != 6;
  __shared__ double red[2][kWarps];
  __shared__ double sh[kThreads];
  __shared__ int go[2];
  __shared__ int run[2];
  const int nrow = static_cast<int>(k.rows0), ncol = static_cast<int>(k.cols0);
  unsigned phase = threadIdx.x == 0 ? ld_acquire_gpu(bar) & 0x80000000u : 0u;
  for (int it = first; it < first + count; ++it) {
    load_run_flags(k.state, run);
    const bool on0 = run[0] != 0, on1 = run[1] != 0;
    if (!on0 && !on1) break;  // every CTA reads the same settled state
    // ---- K1 phase: r = p - A x, w = row_inv r, per-CTA ||r||^2 partials
    {
      const int lane = threadIdx.x & (VSF - 1);
      const unsigned mask = group_mask<VSF>();
      const int gstep = static_cast<int>((long long)gridDim.x * kThreads / VSF);
      double r2a = 0.0, r2b = 0.0;
      for (int g = static_cast<int>((blockIdx.x * (long long)kThreads + threadIdx.x) / VSF);
           g < nrow; g += gstep) {
        const int beg = __ldg(k.tpf + g), end = __ldg(k.tpf + g + 1), tf = __ldg(k.tff + g);
        int eb = 0, ee = 0;
        if (k.epf) {
          eb = __ldg(k.epf + g);
          ee = __ldg(k.epf + g + 1);
        }
        T e[4] = {T(0), T(0), T(0), T(0)};
        if (lane == 0) load4(k.pe + 4 * static_cast<long long>(g), e);
        T da, db;
        seg_dot2m<T, VSF, UF, false, U16, false>(k.tof, k.tif, k.thf, tf, k.rv2,
                                                reinterpret_cast<const T2*>(k.xx), beg, end, eb,
                                                ee, k.eif, k.evf, lane, mask, da, db);
        if (lane == 0) {
          const T ra = e[0] - da, rb = e[1] - db;
          T2 wo;
          wo.x = on0 ? e[2] * ra : T(0);
          wo.y = on1 ? e[3] * rb : T(0);
          reinterpret_cast<T2*>(k.ww)[g] = wo;
          if (on0) r2a += static_cast<double>(ra) * static_cast<double>(ra);
          if (on1) r2b += static_cast<double>(rb) * static_cast<double>(rb);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        r2a += __shfl_xor_sync(0xffffffffu, r2a, o);
        r2b += __shfl_xor_sync(0xffffffffu, r2b, o);
      }
      const int warp = threadIdx.x >> 5;
      if ((threadIdx.x & 31) == 0) {
        red[0][warp] = r2a;
        red[1][warp] = r2b;
      }
      __syncthreads();
      if (threadIdx.x < 2) {
        double t = 0.0;
        for (int q = 0; q < kWarps; ++q) t += red[threadIdx.x][q];
        k.partial[threadIdx.x * gridDim.x + blockIdx.x] = t;
      }
    }
    grid_sync_flip(bar, phase);
    // ---- ||r|| and the stop test, identically in every CTA (finish_norms order)
    for (int q = 0; q < 2; ++q) {
      const bool on = q ? on1 : on0;
      if (!on) {
        if (threadIdx.x == 0) go[q] = 0;
        continue;
      }
      double t = 0.0;
      const volatile double* part = k.partial + q * gridDim.x;
      for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += kThreads) t += part[b];
      sh[threadIdx.x] = t;
      __syncthreads();
      for (int o = kThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        const double res = sqrt(sh[0]);
        const bool stop = res <= k.tol * k.pnorm[q];
        go[q] = stop ? 0 : 1;
        if (blockIdx.x == 0) {
          k.history[q * k.hstride + it] = res;
          if (stop) {
            k.state[4 * q + 0] = 1;
            k.state[4 * q + 1] = it;
          }
        }
      }
      __syncthreads();
    }
    const bool u0 = go[0] != 0, u1 = go[1] != 0;
    if (!u0 && !u1) break;  // both stopped (CTA 0 recorded it)
    // ---- K2 phase: x += lambda col_inv (A^T w)
    {
      const int lane = threadIdx.x & (VSB - 1);
      const unsigned mask = group_mask<VSB>();
      const int gstep = static_cast<int>((long long)gridDim.x * kThreads / VSB);
      for (int g = static_cast<int>((blockIdx.x * (long long)kThreads + threadIdx.x) / VSB);
           g < ncol; g += gstep) {
        const int beg = __ldg(k.tpb + g), end = __ldg(k.tpb + g + 1), tf = __ldg(k.tfb + g);
        int eb = 0, ee = 0;
        if (k.epb) {
          eb = __ldg(k.epb + g);
          ee = __ldg(k.epb + g + 1);
        }
        T2 xo, ci;
        xo.x = xo.y = ci.x = ci.y = T(0);
        if (lane == 0) {
          xo = reinterpret_cast<const T2*>(k.xx)[g];
          ci = __ldg(reinterpret_cast<const T2*>(k.cc) + g);
        }
        T ua, ub;
        seg_dot2m<T, VSB, UF, false, U16, false>(k.tob, k.tib, k.thb, tf, k.cv2,
                                                reinterpret_cast<const T2*>(k.ww), beg, end, eb,
                                                ee, k.eib, k.evb, lane, mask, ua, ub);
        if (lane == 0) {
          if (u0) xo.x = upd(xo.x, k.relax, ua, ci.x);
          if (u1) xo.y = upd(xo.y, k.relax, ub, ci.y);
          reinterpret_cast<T2*>(k.xx)[g] = xo;
          if (u0 && !isfinite(static_cast<double>(xo.x))) atomicCAS(&k.state[2], 0, it + 1);
          if (u1 && !isfinite(static_cast<double>(xo.y))) atomicCAS(&k.state[4 + 2], 0, it + 1);
        }
      }
    }
    grid_sync_flip(bar, phase);
  }
}

// ------------------------------------------------------------ cluster-persistent paired loop
// The smallest folded pairs (config 1: 640 x 2048 per system, ~1 MB of paired
// streams) are bound by per-pass latency, not bytes: the grid-persistent
// kernel re-reads its stream from L2 every pass and synchronises through a
// global atomic barrier (~10 us per pass). Here the whole grid is ONE
// thread-block cluster (16 CTAs of 512 threads where the device allows it,
// else 8), and nothing crosses the cluster through global memory inside the
// loop:
//  * each CTA owns an even share of the rows (K1) and of the columns (K2) --
//    one vector per lane group -- and copies its share of the mirror-coded
//    streams (offsets, values, tile headers, exception lists, bounds, per-row
//    {p, rinv}, per-column cinv) into shared memory once per solve;
//  * every CTA keeps full replicas of x and w in shared memory: K1 gathers x
//    and K2 gathers w from shared memory only;
//  * each new w row / x column and each CTA's ||r||^2 pair is pushed into every
//    CTA's replica with st.async, whose bytes complete on the receiver's
//    mbarrier (expected bytes per pass: all rows + one pair per CTA / all
//    columns). A pass waits on its own mbarrier only: no cluster-wide barrier,
//    no release fence on the producer side, no L1 invalidation (measured on
//    B200: a barrier.cluster after global stores costs ~1,700 cycles,
//    tools/cluster_probe.cu);
//  * every CTA sums the ||r||^2 pairs in rank order and takes the same stop
//    decision (solvers.cpp:180-182); CTA 0 records the history and the stop in
//    global state; a CTA that saw a non-finite update sends -1 as its partial,
//    which turns that system off everywhere (its iteration is recorded in the
//    state word as in the other kernels).
// Ordering: a CTA sends pass i+1's w only after receiving every column of pass
// i, which each CTA sends after its own reads of w -- so replicas are never
// overwritten while read (and symmetrically for x). Row and column dot
// products keep the pair kernels' tile order: bitwise the same iterates as the
// two-launch loop for the same lane-group widths. Config 1 fp64: 96K -> 178K
// it/s.
constexpr int kClusterThreads = 512;
constexpr int kMaxCluster = 16;
constexpr int kClusterSmemMax = 200 * 1024;  // staged streams per CTA (dynamic smem)

__device__ __forceinline__ void cluster_barrier() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// block of CTA b: vectors [b*per, min((b+1)*per, n)) and the stream ranges
// they cover (entries, tiles, exceptions)
struct CBlock {
  int v0, v1, e0, e1, t0, t1, x0, x1;
};

__device__ __forceinline__ CBlock cblock(const int* tp, const int* tfst, const int* ep, int n,
                                         int per, int b) {
  CBlock c;
  c.v0 = min(b * per, n);
  c.v1 = min(c.v0 + per, n);
  c.e0 = tp[c.v0];
  c.e1 = tp[c.v1];
  c.t0 = tfst[c.v0];
  c.t1 = tfst[c.v1];
  c.x0 = ep ? ep[c.v0] : 0;
  c.x1 = ep ? ep[c.v1] : 0;
  return c;
}

// byte sizes of a block's staged arrays (16-byte aligned sections)
template <class T>
__host__ __device__ __forceinline__ long long cstage_bytes(const CBlock& c, int hw, int per_vec) {
  const auto al = [](long long x) { return (x + 15) & ~15ll; };
  const long long nv = c.v1 - c.v0, ne = c.e1 - c.e0, nt = c.t1 - c.t0, nx = c.x1 - c.x0;
  return al(ne * sizeof(T)) + al(nx * 2 * sizeof(T)) + al(nv * per_vec * sizeof(T)) +
         al(nt * hw * 4ll) + 3 * al((nv + 1) * 4) + al(nx * 4) + al(ne * 2);
}

// staged arrays of one direction in shared memory (indices relative to the block)
template <class T>
struct CStage {
  const T* val;
  const T* exv;
  const T* pv;  // per-vector operands: {p1, p2, rinv1, rinv2} (K1) / {cinv1, cinv2} (K2)
  const unsigned* hdr;
  const int* tp;
  const int* tf;
  const int* ep;
  const int* exi;
  const unsigned short* off;
};

template <class V>
__device__ __forceinline__ void ccopy(V* dst, const V* src, long long n) {
  for (long long i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// copy one block's stream share into shared memory at `base`; returns the bytes used
template <class T>
__device__ long long cstage_load(char* base, const CBlock& c, int hw, int per_vec,
                                 const unsigned short* off, const T* val, const unsigned* hdr,
                                 const int* tp, const int* tfst, const int* ep, const int* exi,
                                 const T* exv, const T* pv, CStage<T>& st) {
  const auto al = [](long long x) { return (x + 15) & ~15ll; };
  const long long nv = c.v1 - c.v0, ne = c.e1 - c.e0, nt = c.t1 - c.t0, nx = c.x1 - c.x0;
  char* p = base;
  T* sval = reinterpret_cast<T*>(p);
  p += al(ne * sizeof(T));
  T* sexv = reinterpret_cast<T*>(p);
  p += al(nx * 2 * sizeof(T));
  T* spv = reinterpret_cast<T*>(p);
  p += al(nv * per_vec * sizeof(T));
  unsigned* shdr = reinterpret_cast<unsigned*>(p);
  p += al(nt * hw * 4ll);
  int* stp = reinterpret_cast<int*>(p);
  p += al((nv + 1) * 4);
  int* stf = reinterpret_cast<int*>(p);
  p += al((nv + 1) * 4);
  int* sep = reinterpret_cast<int*>(p);
  p += al((nv + 1) * 4);
  int* sexi = reinterpret_cast<int*>(p);
  p += al(nx * 4);
  unsigned short* soff = reinterpret_cast<unsigned short*>(p);
  p += al(ne * 2);
  // values: whole quads (entries start on multiples of 4)
  if constexpr (sizeof(T) == 4) {
    ccopy(reinterpret_cast<float4*>(sval), reinterpret_cast<const float4*>(val + c.e0), ne / 4);
  } else {
    ccopy(reinterpret_cast<double2*>(sval), reinterpret_cast<const double2*>(val + c.e0), ne / 2);
  }
  ccopy(reinterpret_cast<uint2*>(soff), reinterpret_cast<const uint2*>(off + c.e0), ne / 4);
  ccopy(reinterpret_cast<uint2*>(shdr), reinterpret_cast<const uint2*>(hdr + 1ll * c.t0 * hw),
        nt * hw / 2);
  ccopy(sexv, exv + 2ll * c.x0, 2 * nx);
  ccopy(sexi, exi + c.x0, nx);
  ccopy(spv, pv + 1ll * per_vec * c.v0, nv * per_vec);
  for (long long i = threadIdx.x; i <= nv; i += blockDim.x) {
    stp[i] = tp[c.v0 + i] - c.e0;
    stf[i] = tfst[c.v0 + i] - c.t0;
    sep[i] = ep ? ep[c.v0 + i] - c.x0 : 0;
  }
  st.val = sval;
  st.exv = sexv;
  st.pv = spv;
  st.hdr = shdr;
  st.tp = stp;
  st.tf = stf;
  st.ep = sep;
  st.exi = sexi;
  st.off = soff;
  return p - base;
}

// seg_dot2m over a staged (shared-memory) stream; x / w gathered from global
// with plain loads (rewritten by other CTAs between passes)
template <class T, int VS, int UF>
__device__ __forceinline__ void seg_dot2m_s(const CStage<T>& st, int tf,
                                            const typename Vec2<T>::type* xv, int beg, int end,
                                            int eb, int ee, int lane, unsigned mask, T& acc_a,
                                            T& acc_b) {
  using T2 = typename Vec2<T>::type;
  T sa = T(0), sb = T(0);
  const int nvec = (end - beg) >> 2;
  const auto hdr = [&](int t, int& base, unsigned& nib) {
    if constexpr (VS <= 8) {
      const uint2 w = reinterpret_cast<const uint2*>(st.hdr)[t];
      base = static_cast<int>(w.x);
      nib = w.y >> (4 * lane);
    } else if constexpr (VS == 16) {
      const uint4 w = reinterpret_cast<const uint4*>(st.hdr)[t];
      base = static_cast<int>(w.x);
      nib = (lane < 8 ? w.y : w.z) >> (4 * (lane & 7));
    } else {
      base = static_cast<int>(st.hdr[8 * t]);
      nib = st.hdr[8 * t + 1 + (lane >> 3)] >> (4 * (lane & 7));
    }
  };
  const auto vals = [&](int k0, T (&v)[4]) {
    if constexpr (sizeof(T) == 4) {
      const float4 t = *reinterpret_cast<const float4*>(st.val + k0);
      v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else {
      const double2 a = *reinterpret_cast<const double2*>(st.val + k0);
      const double2 b = *(reinterpret_cast<const double2*>(st.val + k0) + 1);
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
  };
  int q = lane;
  for (; q + (UF - 1) * VS < nvec; q += UF * VS) {
    int4 c[UF];
    unsigned s[UF];
    T v[UF][4];
    const int t0 = tf + (q - lane) / VS;
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const int k0 = beg + ((q + u * VS) << 2);
      int b;
      hdr(t0 + u, b, s[u]);
      c[u] = decode16(*reinterpret_cast<const uint2*>(st.off + k0), b);
      vals(k0, v[u]);
    }
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const T2 g0 = xv[c[u].x], g1 = xv[c[u].y], g2 = xv[c[u].z], g3 = xv[c[u].w];
      sa += flip(v[u][0], s[u], 0) * g0.x + flip(v[u][1], s[u], 1) * g1.x +
            flip(v[u][2], s[u], 2) * g2.x + flip(v[u][3], s[u], 3) * g3.x;
      sb += v[u][0] * g0.y + v[u][1] * g1.y + v[u][2] * g2.y + v[u][3] * g3.y;
    }
  }
  for (; q < nvec; q += VS) {
    const int k0 = beg + (q << 2);
    int b;
    unsigned s;
    hdr(tf + (q - lane) / VS, b, s);
    const int4 c = decode16(*reinterpret_cast<const uint2*>(st.off + k0), b);
    T v[4];
    vals(k0, v);
    const T2 g0 = xv[c.x], g1 = xv[c.y], g2 = xv[c.z], g3 = xv[c.w];
    sa += flip(v[0], s, 0) * g0.x + flip(v[1], s, 1) * g1.x + flip(v[2], s, 2) * g2.x +
          flip(v[3], s, 3) * g3.x;
    sb += v[0] * g0.y + v[1] * g1.y + v[2] * g2.y + v[3] * g3.y;
  }
  for (int e = eb + lane; e < ee; e += VS) {  // exception buckets (rare)
    const int c = st.exi[e];
    const T2 a = reinterpret_cast<const T2*>(st.exv)[e];
    const T2 g = xv[c];
    sa += a.x * g.x;
    sb += a.y * g.y;
  }
#pragma unroll
  for (int off2 = VS / 2; off2 > 0; off2 >>= 1) {
    sa += __shfl_xor_sync(mask, sa, off2, VS);
    sb += __shfl_xor_sync(mask, sb, off2, VS);
  }
  acc_a = sa;
  acc_b = sb;
}

// copy n interleaved pairs global -> shared (one round of L2 latency: every
// thread's loads are in flight together)
template <class T2>
__device__ __forceinline__ void crefresh(T2* dst, const T2* src, int n, int t = threadIdx.x,
                                         int nt = kClusterThreads) {
  for (int i = t; i < n; i += nt) dst[i] = __ldcg(src + i);  // L2 only: nothing left in L1
}

// sum of v over the 32 lanes of a warp in a fixed butterfly order
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- point-to-point exchange inside the cluster: st.async into the peer's
// shared memory, completion counted in bytes on the peer's mbarrier (no
// cluster-wide barrier, no release fence on the producer, no L1 invalidation
// on the consumer)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned cl_map(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(unsigned mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
               : "memory");
}
// wait for the phase of parity `par` (bounded: a lost peer traps, ~2 s)
__device__ __forceinline__ void mbar_wait(unsigned mb, unsigned par) {
  unsigned done = 0;
  const long long t0 = clock64();
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(mb), "r"(par)
        : "memory");
    if (done) return;
    if (clock64() - t0 > kBarrierSpinCycles) __trap();
  }
}
__device__ __forceinline__ void st_async(unsigned ra, double2 v, unsigned rmb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               ::"r"(ra), "d"(v.x), "d"(v.y), "r"(rmb) : "memory");
}
__device__ __forceinline__ void st_async(unsigned ra, float2 v, unsigned rmb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
               ::"r"(ra), "f"(v.x), "f"(v.y), "r"(rmb) : "memory");
}

template <class T, int VSF, int VSB, int UF>
__global__ void __launch_bounds__(kClusterThreads, 1)
    sart_cluster_pair_kernel(SartK<T> k, int first, int count) {
  using T2 = typename Vec2<T>::type;
  constexpr int NW = kClusterThreads / 32;
  constexpr int HWF = VSF <= 8 ? 2 : (VSF == 16 ? 4 : 8);
  constexpr int HWB = VSB <= 8 ? 2 : (VSB == 16 ? 4 : 8);
  static_assert(NW <= 32, "one partial per lane of warp 0");
  extern __shared__ __align__(16) char cl_smem[];
  __shared__ double red[2][NW];
  __shared__ __align__(16) double2 part[kMaxCluster];  // {||r1||^2, ||r2||^2} of each CTA
  __shared__ __align__(8) unsigned long long mbar[2];  // [0]: w + partials, [1]: x
  __shared__ int ldiv[2];  // this CTA saw a non-finite update of system q
  __shared__ int go[2];
  const int nrow = static_cast<int>(k.rows0), ncol = static_cast<int>(k.cols0);
  const unsigned nct = gridDim.x;
  const int warp = threadIdx.x >> 5, wl = threadIdx.x & 31;
  // ---- stage this CTA's stream share (once per solve) and the x / w replicas
  // row / column blocks spread evenly over the cluster (<= one vector per lane group)
  const CBlock bf = cblock(k.tpf, k.tff, k.epf, nrow, (nrow + nct - 1) / nct, blockIdx.x);
  const CBlock bb = cblock(k.tpb, k.tfb, k.epb, ncol, (ncol + nct - 1) / nct, blockIdx.x);
  // replicas first: the same shared-memory offsets in every CTA (st.async targets)
  T2* sx = reinterpret_cast<T2*>(cl_smem);  // replica of the iterate {x1, x2}
  T2* sw = sx + ncol;                       // replica of {w1, w2}
  CStage<T> sf, sb;
  long long used = (2ll * (ncol + nrow) * sizeof(T) + 15) & ~15ll;
  used += cstage_load<T>(cl_smem + used, bf, HWF, 4, k.tof, k.rv2, k.thf, k.tpf, k.tff, k.epf,
                         k.eif, k.evf, k.pe, sf);
  cstage_load<T>(cl_smem + used, bb, HWB, 2, k.tob, k.cv2, k.thb, k.tpb, k.tfb, k.epb, k.eib,
                 k.evb, k.cc, sb);
  crefresh(sx, reinterpret_cast<const T2*>(k.xx), ncol);
  const unsigned mb_w = smem_u32(&mbar[0]), mb_x = smem_u32(&mbar[1]);
  const unsigned bytes_w = static_cast<unsigned>(nrow * sizeof(T2) + nct * sizeof(double2));
  const unsigned bytes_x = static_cast<unsigned>(ncol * sizeof(T2));
  if (threadIdx.x == 0) {
    mbar_init(mb_w, 1);
    mbar_init(mb_x, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 2) ldiv[threadIdx.x] = 0;
  bool run0 = sys_on(k.state, 0), run1 = sys_on(k.state, 1);
  const double thr0 = k.tol * k.pnorm[0], thr1 = k.tol * k.pnorm[1];
  __syncthreads();
  cluster_barrier();  // every CTA's mbarriers exist before any st.async lands
  unsigned par = 0;
  for (int it = first; it < first + count; ++it) {
    if (!run0 && !run1) break;  // the same decision in every CTA
    if (threadIdx.x == 0) mbar_expect(mb_w, bytes_w);
    // ---- K1 phase over this CTA's rows: r = p - A x, w = row_inv r; each
    // row's w goes to every CTA's replica
    {
      const int lane = threadIdx.x & (VSF - 1);
      const unsigned mask = group_mask<VSF>();
      const int li = threadIdx.x / VSF;
      double r2a = 0.0, r2b = 0.0;
      if (li < bf.v1 - bf.v0) {
        T da, db;
        seg_dot2m_s<T, VSF, UF>(sf, sf.tf[li], sx, sf.tp[li], sf.tp[li + 1], sf.ep[li],
                                sf.ep[li + 1], lane, mask, da, db);
        if (lane == 0) {
          const T* e = sf.pv + 4 * li;
          const T ra = e[0] - da, rb = e[1] - db;
          T2 wo;
          wo.x = run0 ? e[2] * ra : T(0);
          wo.y = run1 ? e[3] * rb : T(0);
          const unsigned la = smem_u32(sw + bf.v0 + li);
          for (unsigned r = 0; r < nct; ++r) st_async(cl_map(la, r), wo, cl_map(mb_w, r));
          if (run0) r2a = static_cast<double>(ra) * static_cast<double>(ra);
          if (run1) r2b = static_cast<double>(rb) * static_cast<double>(rb);
        }
      }
      r2a = warp_sum(r2a);
      r2b = warp_sum(r2b);
      if (wl == 0) {
        red[0][warp] = r2a;
        red[1][warp] = r2b;
      }
      __syncthreads();
      if (warp == 0) {  // this CTA's partial pair -> every CTA (-1: it saw a divergence)
        double2 t;
        t.x = warp_sum(wl < NW ? red[0][wl] : 0.0);
        t.y = warp_sum(wl < NW ? red[1][wl] : 0.0);
        if (ldiv[0]) t.x = -1.0;
        if (ldiv[1]) t.y = -1.0;
        if (wl < static_cast<int>(nct)) {
          st_async(cl_map(smem_u32(&part[blockIdx.x]), wl), t, cl_map(mb_w, wl));
        }
      }
    }
    mbar_wait(mb_w, par);
    // ---- ||r|| and the stop test (warp q: system q), the same in every CTA
    if (warp < 2) {
      const bool on = warp ? run1 : run0;
      const double v = wl < static_cast<int>(nct) ? (warp ? part[wl].y : part[wl].x) : 0.0;
      const bool div = __any_sync(0xffffffffu, v < 0.0);
      const double t = warp_sum(v);
      if (wl == 0) {
        int gq = 0;
        if (on && !div) {
          const double res = sqrt(t);
          const bool stop = res <= (warp ? thr1 : thr0);
          gq = stop ? 0 : 1;
          if (blockIdx.x == 0) {
            k.history[warp * k.hstride + it] = res;
            if (stop) {
              k.state[4 * warp + 0] = 1;
              k.state[4 * warp + 1] = it;
            }
          }
        }
        go[warp] = gq;
      }
    } else if (threadIdx.x == 64) {
      mbar_expect(mb_x, bytes_x);
    }
    __syncthreads();
    run0 = go[0] != 0;
    run1 = go[1] != 0;
    if (!run0 && !run1) break;  // both stopped (CTA 0 recorded it)
    // ---- K2 phase over this CTA's columns: x += lambda col_inv (A^T w); each
    // column's x goes to every CTA's replica and to global memory
    {
      const int lane = threadIdx.x & (VSB - 1);
      const unsigned mask = group_mask<VSB>();
      const int li = threadIdx.x / VSB;
      if (li < bb.v1 - bb.v0) {
        const int g = bb.v0 + li;
        T ua, ub;
        seg_dot2m_s<T, VSB, UF>(sb, sb.tf[li], sw, sb.tp[li], sb.tp[li + 1], sb.ep[li],
                                sb.ep[li + 1], lane, mask, ua, ub);
        if (lane == 0) {
          T2 xo = sx[g];
          const T* ci = sb.pv + 2 * li;
          if (run0) xo.x = upd(xo.x, k.relax, ua, ci[0]);
          if (run1) xo.y = upd(xo.y, k.relax, ub, ci[1]);
          reinterpret_cast<T2*>(k.xx)[g] = xo;
          if (run0 && !isfinite(static_cast<double>(xo.x))) {
            atomicCAS(&k.state[2], 0, it + 1);
            ldiv[0] = 1;
          }
          if (run1 && !isfinite(static_cast<double>(xo.y))) {
            atomicCAS(&k.state[4 + 2], 0, it + 1);
            ldiv[1] = 1;
          }
          const unsigned la = smem_u32(sx + g);
          for (unsigned r = 0; r < nct; ++r) st_async(cl_map(la, r), xo, cl_map(mb_x, r));
        }
      }
    }
    mbar_wait(mb_x, par);
    par ^= 1u;
    __syncthreads();  // ldiv of this pass visible to warp 0 of the next
  }
}

// ------------------------------------------------------------ stream-resident persistent loop
// Folded pairs whose mirror-coded streams fit the GPU's shared memory
// (config 2 fp32: 23 MB over 148 SMs = 160 KB per CTA; fp64: K1's stream only,
// SB = false, K2 then streams from L2 as in the grid kernel) but not one cluster:
// the grid is one CTA per SM, every CTA owns a contiguous block of rows (K1)
// and of columns (K2) and copies its share of both streams (offsets, values,
// tile headers, exception lists, bounds, {p, rinv}, cinv) into shared memory
// once per launch. A pass then reads no matrix byte from L2 or HBM: only the
// gathers of x / w (L2) and the two grid barriers remain. Rows and columns
// keep the pair kernels' tile order (seg_dot2m_s): bitwise the iterates of the
// two-launch loop with the same lane-group widths; every CTA sums the per-CTA
// ||r||^2 partials in the same fixed order and takes the same stop decision.
constexpr int kResThreads = 1024;
constexpr int kResSmemMax = 216 * 1024;  // staged streams per CTA (dynamic smem)
#ifdef SSB_RES_TIMING
__device__ unsigned long long res_ticks[8];
#define RES_T(i) if (blockIdx.x == 0 && threadIdx.x == 0) { const long long t_ = clock64(); res_ticks[i] += t_ - tl_; tl_ = t_; }
#else
#define RES_T(i)
#endif

template <class T, int VSF, int VSB, int UF, bool SB>
__global__ void __launch_bounds__(kResThreads, 1)
    sart_resident_pair_kernel(SartK<T> k, int first, int count, unsigned* bar) {
  using T2 = typename Vec2<T>::type;
  constexpr int NW = kResThreads / 32;
  constexpr int HWF = VSF <= 8 ? 2 : (VSF == 16 ? 4 : 8);
  constexpr int HWB = VSB <= 8 ? 2 : (VSB == 16 ? 4 : 8);
  extern __shared__ __align__(16) char rs_smem[];
  __shared__ double red[2][NW];
  __shared__ int go[2];
  __shared__ int run[2];
  const int nrow = static_cast<int>(k.rows0), ncol = static_cast<int>(k.cols0);
  const int nct = static_cast<int>(gridDim.x);
  const int warp = threadIdx.x >> 5, wl = threadIdx.x & 31;
  const CBlock bf = cblock(k.tpf, k.tff, k.epf, nrow, (nrow + nct - 1) / nct, blockIdx.x);
  const CBlock bb = cblock(k.tpb, k.tfb, k.epb, ncol, (ncol + nct - 1) / nct, blockIdx.x);
  CStage<T> sf, sb;
  const long long used = cstage_load<T>(rs_smem, bf, HWF, 4, k.tof, k.rv2, k.thf, k.tpf, k.tff,
                                        k.epf, k.eif, k.evf, k.pe, sf);
  if constexpr (SB) {  // (SB = false: only K1's stream fits; K2 streams from L2)
    cstage_load<T>(rs_smem + used, bb, HWB, 2, k.tob, k.cv2, k.thb, k.tpb, k.tfb, k.epb, k.eib,
                   k.evb, k.cc, sb);
  }
  __syncthreads();
  const T2* xg = reinterpret_cast<const T2*>(k.xx);
  const T2* wg = reinterpret_cast<const T2*>(k.ww);
  unsigned phase = threadIdx.x == 0 ? ld_acquire_gpu(bar) & 0x80000000u : 0u;
#ifdef SSB_RES_TIMING
  long long tl_ = clock64();
#endif
  for (int it = first; it < first + count; ++it) {
    load_run_flags(k.state, run);
    const bool on0 = run[0] != 0, on1 = run[1] != 0;
    if (!on0 && !on1) break;  // every CTA reads the same settled state
    RES_T(0)
    // ---- K1 phase over this CTA's rows: r = p - A x, w = row_inv r
    {
      const int lane = threadIdx.x & (VSF - 1);
      const unsigned mask = group_mask<VSF>();
      double r2a = 0.0, r2b = 0.0;
      for (int li = threadIdx.x / VSF; li < bf.v1 - bf.v0; li += kResThreads / VSF) {
        T da, db;
        seg_dot2m_s<T, VSF, UF>(sf, sf.tf[li], xg, sf.tp[li], sf.tp[li + 1], sf.ep[li],
                                sf.ep[li + 1], lane, mask, da, db);
        if (lane == 0) {
          const T* e = sf.pv + 4 * li;
          const T ra = e[0] - da, rb = e[1] - db;
          T2 wo;
          wo.x = on0 ? e[2] * ra : T(0);
          wo.y = on1 ? e[3] * rb : T(0);
          reinterpret_cast<T2*>(k.ww)[bf.v0 + li] = wo;
          if (on0) r2a += static_cast<double>(ra) * static_cast<double>(ra);
          if (on1) r2b += static_cast<double>(rb) * static_cast<double>(rb);
        }
      }
      r2a = warp_sum(r2a);
      r2b = warp_sum(r2b);
      if (wl == 0) {
        red[0][warp] = r2a;
        red[1][warp] = r2b;
      }
      __syncthreads();
      if (warp < 2) {
        const double t = warp_sum(wl < NW ? red[warp][wl] : 0.0);
        if (wl == 0) k.partial[warp * nct + blockIdx.x] = t;
      }
    }
    RES_T(1)
    grid_sync_flip(bar, phase);
    RES_T(2)
    // ---- ||r|| and the stop test (warp q: system q), identically in every CTA
    if (warp < 2) {
      const bool on = warp ? on1 : on0;
      double t = 0.0;
      for (int b = wl; b < nct; b += 32) t += __ldcg(k.partial + warp * nct + b);
      t = warp_sum(t);
      if (wl == 0) {
        int gq = 0;
        if (on) {
          const double res = sqrt(t);
          const bool stop = res <= k.tol * k.pnorm[warp];
          gq = stop ? 0 : 1;
          if (blockIdx.x == 0) {
            k.history[warp * k.hstride + it] = res;
            if (stop) {
              k.state[4 * warp + 0] = 1;
              k.state[4 * warp + 1] = it;
            }
          }
        }
        go[warp] = gq;
      }
    }
    __syncthreads();
    const bool u0 = go[0] != 0, u1 = go[1] != 0;
    if (!u0 && !u1) break;  // both stopped (CTA 0 recorded it)
    RES_T(3)
    // ---- K2 phase over this CTA's columns: x += lambda col_inv (A^T w)
    {
      const int lane = threadIdx.x & (VSB - 1);
      const unsigned mask = group_mask<VSB>();
      for (int li = threadIdx.x / VSB; li < bb.v1 - bb.v0; li += kResThreads / VSB) {
        const int g = bb.v0 + li;
        T2 xo;
        xo.x = xo.y = T(0);
        if (lane == 0) xo = xg[g];
        T ua, ub;
        T2 ci;
        ci.x = ci.y = T(0);
        if constexpr (SB) {
          seg_dot2m_s<T, VSB, UF>(sb, sb.tf[li], wg, sb.tp[li], sb.tp[li + 1], sb.ep[li],
                                  sb.ep[li + 1], lane, mask, ua, ub);
          if (lane == 0) {
            ci.x = sb.pv[2 * li];
            ci.y = sb.pv[2 * li + 1];
          }
        } else {
          const int beg = __ldg(k.tpb + g), end = __ldg(k.tpb + g + 1), tf = __ldg(k.tfb + g);
          int eb = 0, ee = 0;
          if (k.epb) {
            eb = __ldg(k.epb + g);
            ee = __ldg(k.epb + g + 1);
          }
          if (lane == 0) ci = __ldg(reinterpret_cast<const T2*>(k.cc) + g);
          seg_dot2m<T, VSB, UF, false, true, false>(k.tob, k.tib, k.thb, tf, k.cv2, wg, beg, end,
                                                    eb, ee, k.eib, k.evb, lane, mask, ua, ub);
        }
        if (lane == 0) {
          if (u0) xo.x = upd(xo.x, k.relax, ua, ci.x);
          if (u1) xo.y = upd(xo.y, k.relax, ub, ci.y);
          reinterpret_cast<T2*>(k.xx)[g] = xo;
          if (u0 && !isfinite(static_cast<double>(xo.x))) atomicCAS(&k.state[2], 0, it + 1);
          if (u1 && !isfinite(static_cast<double>(xo.y))) atomicCAS(&k.state[4 + 2], 0, it + 1);
        }
      }
    }
    RES_T(4)
    grid_sync_flip(bar, phase);
    RES_T(5)
  }
}

// ------------------------------------------------------------ single-system tiled kernels
// One system (sart_solve, the per-rank system of a 2-GPU run, a row shard) on
// the same tiled stream layout as the folded pair: quads padded, entries
// permuted within 4*VS-entry tiles, 16-bit offsets + tile bases when they fit.
template <class T, int VS, int UF, bool U16>
__device__ __forceinline__ T seg_dot1(const int* __restrict__ idx,
                                      const unsigned short* __restrict__ off,
                                      const int* __restrict__ tbase, int tf,
                                      const T* __restrict__ val, const T* __restrict__ vec, int beg,
                                      int end, int lane, unsigned mask) {
  T acc = T(0);
  const int nvec = (end - beg) >> 2;
  int q = lane;
  for (; q + (UF - 1) * VS < nvec; q += UF * VS) {
    int4 c[UF];
    T v[UF][4];
    const int t0 = tf + (q - lane) / VS;
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      const int k0 = beg + ((q + u * VS) << 2);
      if (U16) {
        c[u] = decode16(__ldg(reinterpret_cast<const uint2*>(off + k0)), __ldg(tbase + t0 + u));
      } else {
        c[u] = __ldg(reinterpret_cast<const int4*>(idx + k0));
      }
      load4(val + k0, v[u]);
    }
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      acc += v[u][0] * __ldg(vec + c[u].x) + v[u][1] * __ldg(vec + c[u].y) +
             v[u][2] * __ldg(vec + c[u].z) + v[u][3] * __ldg(vec + c[u].w);
    }
  }
  for (; q < nvec; q += VS) {
    const int k0 = beg + (q << 2);
    const int4 c = U16 ? decode16(__ldg(reinterpret_cast<const uint2*>(off + k0)),
                                  __ldg(tbase + tf + (q - lane) / VS))
                       : __ldg(reinterpret_cast<const int4*>(idx + k0));
    T v[4];
    load4(val + k0, v);
    acc += v[0] * __ldg(vec + c.x) + v[1] * __ldg(vec + c.y) + v[2] * __ldg(vec + c.z) +
           v[3] * __ldg(vec + c.w);
  }
#pragma unroll
  for (int o = VS / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(mask, acc, o, VS);
  return acc;
}

template <class T, int VS, int UF, bool U16>
__global__ void __launch_bounds__(kThreads, kDirectMinBlocks) sart_fwd_tiled_kernel(SartK<T> k, int it) {
  cudaGridDependencySynchronize();  // PDL: launched while the previous pass drains
  it = pass_index(k, it, true);
  if (loop_over(k, true)) return;
  __shared__ double red[kWarps];
  const SysK<T>& S = k.s[0];
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const int n = static_cast<int>(k.rows0);
  const int gstep = static_cast<int>((long long)gridDim.x * kThreads / VS);
  int g = static_cast<int>((blockIdx.x * (long long)kThreads + threadIdx.x) / VS);
  double r2 = 0.0;
  if (sys_on_cg(k.state, 0)) {
    int beg = 0, end = 0, tf = 0;
    if (g < n) {
      beg = __ldg(k.tpf + g);
      end = __ldg(k.tpf + g + 1);
      if (U16) tf = __ldg(k.tff + g);
    }
    for (; g < n; g += gstep) {
      const int gn = g + gstep;
      int nbeg = 0, nend = 0, ntf = 0;
      if (gn < n) {
        nbeg = __ldg(k.tpf + gn);
        nend = __ldg(k.tpf + gn + 1);
        if (U16) ntf = __ldg(k.tff + gn);
      }
      T pv = T(0), ri = T(0);
      if (lane == 0) {
        pv = S.p[g];
        ri = S.rinv[g];
      }
      const T dot = seg_dot1<T, VS, UF, U16>(k.tif, k.tof, k.tbf, tf, k.rv2, S.x, beg, end,
                                             lane, mask);
      if (lane == 0) {
        const T r = pv - dot;
        S.w[g] = ri * r;
        r2 += static_cast<double>(r) * static_cast<double>(r);
      }
      beg = nbeg;
      end = nend;
      tf = ntf;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < kWarps; ++q) t += red[q];
    k.partial[blockIdx.x] = t;
  }
  if (k.bp_out) return;  // sharded plans reduce ||r||^2 across ranks instead
  if (last_block(k.ticket)) {
    finish_norms(k.partial, gridDim.x, 1, k.pnorm, k.tol, k.history, k.hstride, k.state, it);
    loop_next(k, it);
    if (threadIdx.x == 0) *k.ticket = 0;
  }
}

template <class T, int VS, int UF, bool U16>
__global__ void __launch_bounds__(kThreads, kDirectMinBlocks) sart_back_tiled_kernel(SartK<T> k, int it) {
  cudaGridDependencySynchronize();  // PDL: launched while the previous pass drains
  it = pass_index(k, it, false);
  if (loop_over(k, false)) return;
  const SysK<T>& S = k.s[0];
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const int n = static_cast<int>(k.cols0);
  const int gstep = static_cast<int>((long long)gridDim.x * kThreads / VS);
  int g = static_cast<int>((blockIdx.x * (long long)kThreads + threadIdx.x) / VS);
  if (!sys_on_cg(k.state, 0)) return;
  int beg = 0, end = 0, tf = 0;
  if (g < n) {
    beg = __ldg(k.tpb + g);
    end = __ldg(k.tpb + g + 1);
    if (U16) tf = __ldg(k.tfb + g);
  }
  for (; g < n; g += gstep) {
    const int gn = g + gstep;
    int nbeg = 0, nend = 0, ntf = 0;
    if (gn < n) {
      nbeg = __ldg(k.tpb + gn);
      nend = __ldg(k.tpb + gn + 1);
      if (U16) ntf = __ldg(k.tfb + gn);
    }
    T xo = T(0), ci = T(0);
    if (lane == 0 && !k.bp_out) {
      xo = S.x[g];
      ci = S.cinv[g];
    }
    const T u = seg_dot1<T, VS, UF, U16>(k.tib, k.tob, k.tbb, tf, k.cv2, S.w, beg, end, lane,
                                         mask);
    if (lane == 0) {
      if (k.bp_out) {
        k.bp_out[g] = u;
      } else {
        const T xn = upd(xo, k.relax, u, ci);
        S.x[g] = xn;
        if (!isfinite(static_cast<double>(xn))) atomicCAS(&k.state[2], 0, it + 1);
      }
    }
    beg = nbeg;
    end = nend;
    tf = ntf;
  }
}

// dst[stride*i + slot] = src[i] (building interleaved paired streams)
template <class T, class S>
__global__ void interleave_kernel(const S* src, T* dst, long long n, int stride, int slot) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    dst[stride * i + slot] = static_cast<T>(src[i]);
  }
}

// x1, x2 of a paired plan out of the interleaved iterate (end of every solve)
template <class T>
__global__ void deinterleave_kernel(const T* xx, T* x1, T* x2, long long n) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    x1[j] = xx[2 * j];
    x2[j] = xx[2 * j + 1];
  }
}

// Tiled paired stream of one compressed matrix (see seg_dot2t): one warp per
// vector writes its padded, tile-permuted indices and interleaved values.
// Padding repeats the vector's last index (an L1-hot gather) with value 0.
template <class T, class S>
__global__ void tile_stream_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                                   const S* __restrict__ v0, const S* __restrict__ v1,
                                   long long nvec, const int* __restrict__ tptr,
                                   int* __restrict__ tidx, T* __restrict__ tv2, int tile) {
  const int lane = threadIdx.x & 31;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long s = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
       s < nvec; s += nw) {
    const int beg = ptr[s], len = ptr[s + 1] - beg;
    const int ob = tptr[s], lp = tptr[s + 1] - ob;
    const int pad = len > 0 ? idx[beg + len - 1] : 0;
    for (int p = lane; p < lp; p += 32) {
      const int t0 = (p / tile) * tile;
      const int r = min(tile, lp - t0) >> 2;  // quads in this tile
      const int w = p - t0;
      const int o = t0 + (w & 3) * r + (w >> 2);
      int c = pad;
      T a = T(0), b = T(0);
      if (o < len) {
        c = idx[beg + o];
        a = static_cast<T>(v0[beg + o]);  // fp64 master values rounded once to the plan type
        if (v1) b = static_cast<T>(v1[beg + o]);
      }
      tidx[ob + p] = c;
      if (v1) {  // folded pair: {a1, a2} interleaved
        tv2[2 * static_cast<long long>(ob + p)] = a;
        tv2[2 * static_cast<long long>(ob + p) + 1] = b;
      } else {   // one system
        tv2[ob + p] = a;
      }
    }
  }
}

// tiles per vector (tile = 4*VS padded entries) -> counts for the first-tile scan
__global__ void tile_counts_kernel(const int* __restrict__ tptr, long long n, int tile,
                                   int* __restrict__ cnt) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i <= n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    cnt[i] = i < n ? (tptr[i + 1] - tptr[i] + tile - 1) / tile : 0;
  }
}

// 16-bit tiled stream (see seg_dot2c): same permutation as tile_stream_kernel;
// per tile base = its smallest index (the tile's first entry in sorted order),
// per entry offset = index - base; padding repeats the base. Any offset that
// does not fit 16 bits raises *overflow (the plan then keeps int32 indices).
template <class T, class S>
__global__ void tile_stream16_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                                     const S* __restrict__ v0, const S* __restrict__ v1,
                                     long long nvec, const int* __restrict__ tptr,
                                     const int* __restrict__ tfirst, unsigned short* __restrict__ tofs,
                                     int* __restrict__ tbase, T* __restrict__ tv2, int tile,
                                     int* __restrict__ overflow) {
  const int lane = threadIdx.x & 31;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long s = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
       s < nvec; s += nw) {
    const int beg = ptr[s], len = ptr[s + 1] - beg;
    const int ob = tptr[s], lp = tptr[s + 1] - ob;
    const int tf = tfirst[s];
    for (int t = lane; t * tile < lp; t += 32) tbase[tf + t] = idx[beg + t * tile];
    bool bad = false;
    for (int p = lane; p < lp; p += 32) {
      const int t0 = (p / tile) * tile;
      const int r = min(tile, lp - t0) >> 2;
      const int w = p - t0;
      const int o = t0 + (w & 3) * r + (w >> 2);
      const int base = idx[beg + t0];
      int c = base;
      T a = T(0), b = T(0);
      if (o < len) {
        c = idx[beg + o];
        a = static_cast<T>(v0[beg + o]);
        if (v1) b = static_cast<T>(v1[beg + o]);
      }
      const unsigned d = static_cast<unsigned>(c - base);
      bad |= d > 0xffffu;
      tofs[ob + p] = static_cast<unsigned short>(d);
      if (v1) {
        tv2[2 * static_cast<long long>(ob + p)] = a;
        tv2[2 * static_cast<long long>(ob + p) + 1] = b;
      } else {
        tv2[ob + p] = a;
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(overflow, 1);
  }
}

// Does any tile of 4*VS entries span >= 65536 indices? (tiles cover stored
// entries [t0, t0 + tile) of a vector in sorted order; the 16-bit streams
// then cannot be built for this direction)
__global__ void tile_overflow_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                                     long long nvec, int tile, int* __restrict__ overflow) {
  for (long long s = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; s < nvec;
       s += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int beg = ptr[s], len = ptr[s + 1] - beg;
    bool bad = false;
    for (int t0 = 0; t0 < len && !bad; t0 += tile) {
      const int last = min(t0 + tile, len) - 1;
      bad = static_cast<unsigned>(idx[beg + last] - idx[beg + t0]) > 0xffffu;
    }
    if (bad) atomicOr(overflow, 1);
  }
}

// Bucket class of the mirror-coded stream in the plan type:
// 0 a1 == a2, 1 a1 == -a2 (both exact), 2 exception.
template <class T>
__device__ __forceinline__ int mirror_class(double a1, double a2) {
  const T a = static_cast<T>(a1), b = static_cast<T>(a2);
  if (a == b) return 0;
  if (a == -b) return 1;
  return 2;
}

// Mirror-coded 16-bit tiled stream (see seg_dot2m): the permutation and
// offsets of tile_stream16_kernel, one value (a2) per entry, and the tile's
// sign bits (bit w of the tile = padded position w) in its header words
// 1..; word 0 is the base. thdr must be zeroed (partial tiles, padding).
template <class T>
__global__ void tile_mirror_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                                   const double* __restrict__ v0, const double* __restrict__ v1,
                                   long long nvec, const int* __restrict__ tptr,
                                   const int* __restrict__ tfirst, unsigned short* __restrict__ tofs,
                                   int* __restrict__ tidx,
                                   unsigned* __restrict__ thdr, int hs, T* __restrict__ tv,
                                   int tile, int* __restrict__ overflow) {
  const int lane = threadIdx.x & 31;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long s = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
       s < nvec; s += nw) {
    const int beg = ptr[s], len = ptr[s + 1] - beg;
    const int ob = tptr[s], lp = tptr[s + 1] - ob;
    const int tf = tfirst[s];
    for (int t = lane; t * tile < lp; t += 32) {
      thdr[static_cast<long long>(tf + t) * hs] = static_cast<unsigned>(idx[beg + t * tile]);
    }
    bool bad = false;
    for (int p0 = 0; p0 < lp; p0 += 32) {
      const int p = p0 + lane;
      bool neg = false;
      if (p < lp) {
        const int t0 = (p / tile) * tile;
        const int r = min(tile, lp - t0) >> 2;
        const int w = p - t0;
        const int o = t0 + (w & 3) * r + (w >> 2);
        const int base = idx[beg + t0];
        int c = base;
        T v = T(0);
        if (o < len) {
          c = idx[beg + o];
          const int cls = mirror_class<T>(v0[beg + o], v1[beg + o]);
          if (cls < 2) {
            v = static_cast<T>(v1[beg + o]);
            neg = cls == 1;
          }
        }
        const unsigned d = static_cast<unsigned>(c - base);
        bad |= d > 0xffffu;
        if (tofs) tofs[ob + p] = static_cast<unsigned short>(d);
        else tidx[ob + p] = c;  // int32 indices (tiles too wide for 16 bits)
        tv[ob + p] = v;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, neg);
      if (lane == 0) {
        if (tile >= 32) {
          thdr[static_cast<long long>(tf + p0 / tile) * hs + 1 + (p0 % tile) / 32] = bal;
        } else {  // 16-entry tiles: two per ballot
          for (int h = 0; h < 2; ++h) {
            const int pp = p0 + 16 * h;
            if (pp < lp) thdr[static_cast<long long>(tf + pp / 16) * hs + 1] = (bal >> (16 * h)) & 0xffffu;
          }
        }
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(overflow, 1);
  }
}

// exception buckets per vector (counts for the pointer scan; cnt[n] stays 0)
template <class T>
__global__ void mirror_exc_count_kernel(const int* __restrict__ ptr, const double* __restrict__ v0,
                                        const double* __restrict__ v1, long long nvec,
                                        int* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long s = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
       s < nvec; s += nw) {
    int n = 0;
    for (int q = ptr[s] + lane; q < ptr[s + 1]; q += 32) n += mirror_class<T>(v0[q], v1[q]) == 2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if (lane == 0) cnt[s] = n;
  }
}

// exception lists in stored (sorted) order: index and {a1, a2} in the plan type
template <class T>
__global__ void mirror_exc_fill_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                                       const double* __restrict__ v0, const double* __restrict__ v1,
                                       long long nvec, const int* __restrict__ eptr,
                                       int* __restrict__ eidx, T* __restrict__ ev2) {
  const int lane = threadIdx.x & 31;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long s = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
       s < nvec; s += nw) {
    int at = eptr[s];
    if (at == eptr[s + 1]) continue;
    for (int q0 = ptr[s]; q0 < ptr[s + 1]; q0 += 32) {
      const int q = q0 + lane;
      const bool ex = q < ptr[s + 1] && mirror_class<T>(v0[q], v1[q]) == 2;
      const unsigned bal = __ballot_sync(0xffffffffu, ex);
      if (ex) {
        const int e = at + __popc(bal & ((1u << lane) - 1u));
        eidx[e] = idx[q];
        ev2[2 * static_cast<long long>(e)] = static_cast<T>(v0[q]);
        ev2[2 * static_cast<long long>(e) + 1] = static_cast<T>(v1[q]);
      }
      at += __popc(bal);
    }
  }
}

// padded vector lengths (multiple of 4) -> counts for the pointer scan
__global__ void pad4_counts_kernel(const int* __restrict__ ptr, long long n, int* __restrict__ cnt) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i <= n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    cnt[i] = i < n ? ((ptr[i + 1] - ptr[i] + 3) & ~3) : 0;
  }
}

// ------------------------------------------------------------ multi-RHS kernels
// Slices share A; X/W/P are [n][S] so a warp reads the S slices of one
// gathered row contiguously while the matrix entry is loaded once per warp and
// broadcast: matrix bytes amortise over S. Lane l owns the V consecutive slices
// q*32V + l*V .. +V-1 (q < Q) and moves them with one vector load, so a warp
// covers 32*V slices per gather instruction.
// The warp loads 32 (index, value) pairs coalesced, then broadcasts them 8 at
// a time so 8 independent slice-row gathers are in flight per lane. Entries
// past `end` carry value 0 and index 0 (a harmless gather).
template <class T, int V>
__device__ __forceinline__ void loadv(const T* __restrict__ p, T (&o)[V]) {
  if constexpr (V == 1) {
    o[0] = __ldg(p);
  } else if constexpr (V == 2 && sizeof(T) == 4) {
    const float2 t = __ldg(reinterpret_cast<const float2*>(p));
    o[0] = t.x; o[1] = t.y;
  } else if constexpr (V == 4 && sizeof(T) == 4) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
  } else {
#pragma unroll
    for (int h = 0; h < V; h += 2) {
      const double2 t = __ldg(reinterpret_cast<const double2*>(p) + h / 2);
      o[h] = t.x; o[h + 1] = t.y;
    }
  }
}

template <class T, int V, int Q>
__device__ __forceinline__ void multi_row_dot(const int* __restrict__ idx, const T* __restrict__ val,
                                              const T* __restrict__ X, int beg, int end,
                                              int lane, int S, T (&acc)[Q][V]) {
  for (int base = beg; base < end; base += 32) {
    const int kk = base + lane;
    const int c = kk < end ? __ldg(idx + kk) : 0;
    const T v = kk < end ? __ldg(val + kk) : T(0);
    const int cnt = min(32, end - base);
    for (int e0 = 0; e0 < cnt; e0 += 8) {
      int ce[8];
      T ve[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        ce[u] = __shfl_sync(0xffffffffu, c, (e0 + u) & 31);
        ve[u] = __shfl_sync(0xffffffffu, v, (e0 + u) & 31);
        if (e0 + u >= cnt) {
          ce[u] = 0;
          ve[u] = T(0);
        }
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int sl = (q * 32 + lane) * V;
        if (sl < S) {
          T g[8][V];
#pragma unroll
          for (int u = 0; u < 8; ++u) loadv<T, V>(X + static_cast<long long>(ce[u]) * S + sl, g[u]);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int t = 0; t < V; ++t) acc[q][t] += ve[u] * g[u][t];
          }
        }
      }
    }
  }
}

template <class T, int V, int Q>
__global__ void __launch_bounds__(kThreads) sart_fwd_multi_kernel(SartK<T> k, int it, int band) {
  // band: 0 = the whole row in one pass; with column bands 1 = first pass
  // (w <- partial), 2 = middle (w += partial), 3 = last (r from w + partial)
  it = pass_index(k, it, true);
  if (loop_over(k, true)) return;
  extern __shared__ double mred[];  // [kWarps][nsys*S]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int S = k.nrhs;
  const long long gw = (blockIdx.x * (long long)kThreads + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kThreads) >> 5;
  double r2a[Q][V], r2b[Q][V];
  bool ona[Q][V], onb[Q][V];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
#pragma unroll
    for (int t = 0; t < V; ++t) {
      const int sl = (q * 32 + lane) * V + t;
      r2a[q][t] = r2b[q][t] = 0.0;
      ona[q][t] = sl < S && sys_on(k.state, sl);
      onb[q][t] = sl < S && k.nsys > 1 && sys_on(k.state, S + sl);
    }
  }
  for (long long g = gw; g < k.rows_total; g += nw) {
    const int s = g >= k.rows0 ? 1 : 0;
    const SysK<T>& Sy = k.s[s];
    const int i = static_cast<int>(g - (s ? k.rows0 : 0));
    T acc[Q][V];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
#pragma unroll
      for (int t = 0; t < V; ++t) acc[q][t] = T(0);
    }
    const int beg = Sy.bb ? Sy.bb[i] : Sy.rp[i], end = Sy.be ? Sy.be[i] : Sy.rp[i + 1];
    multi_row_dot<T, V, Q>(Sy.ci, Sy.rv, Sy.x, beg, end, lane, S, acc);
    if (band == 1 || band == 2) {  // partial dot products of this column band
#pragma unroll
      for (int q = 0; q < Q; ++q) {
#pragma unroll
        for (int t = 0; t < V; ++t) {
          const int sl = (q * 32 + lane) * V + t;
          if (s ? onb[q][t] : ona[q][t]) {
            const long long o = static_cast<long long>(i) * S + sl;
            Sy.w[o] = band == 1 ? acc[q][t] : Sy.w[o] + acc[q][t];
          }
        }
      }
      continue;
    }
    if (band == 3) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
#pragma unroll
        for (int t = 0; t < V; ++t) {
          const int sl = (q * 32 + lane) * V + t;
          if (sl < S) acc[q][t] = Sy.w[static_cast<long long>(i) * S + sl] + acc[q][t];
        }
      }
    }
    const T ri = Sy.rinv[i];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
#pragma unroll
      for (int t = 0; t < V; ++t) {
        const int sl = (q * 32 + lane) * V + t;
        if (s ? onb[q][t] : ona[q][t]) {
          const long long o = static_cast<long long>(i) * S + sl;
          const T r = Sy.p[o] - acc[q][t];
          Sy.w[o] = ri * r;
          const double r2 = static_cast<double>(r) * static_cast<double>(r);
          if (s) r2b[q][t] += r2; else r2a[q][t] += r2;
        }
      }
    }
  }
  if (band == 1 || band == 2) return;
  const int nsr = k.nsys * S;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
#pragma unroll
    for (int t = 0; t < V; ++t) {
      const int sl = (q * 32 + lane) * V + t;
      if (sl < S) {
        mred[warp * nsr + sl] = r2a[q][t];
        if (k.nsys > 1) mred[warp * nsr + S + sl] = r2b[q][t];
      }
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
    loop_next(k, it);
    if (threadIdx.x == 0) *k.ticket = 0;
  }
}

// one slice pass (Q = 1): 4 CTAs per SM (63 registers, no spills), K2 0.68 ->
// 0.63 ms on config 4; Q = 2 and the forward kernel spill under that cap
template <class T, int V, int Q>
__global__ void __launch_bounds__(kThreads, Q == 1 ? 4 : 1) sart_back_multi_kernel(SartK<T> k, int it) {
  it = pass_index(k, it, false);
  if (loop_over(k, false)) return;
  const int lane = threadIdx.x & 31;
  const int S = k.nrhs;
  const long long gw = (blockIdx.x * (long long)kThreads + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kThreads) >> 5;
  bool ona[Q][V], onb[Q][V];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
#pragma unroll
    for (int t = 0; t < V; ++t) {
      const int sl = (q * 32 + lane) * V + t;
      ona[q][t] = sl < S && sys_on(k.state, sl);
      onb[q][t] = sl < S && k.nsys > 1 && sys_on(k.state, S + sl);
    }
  }
  for (long long g = gw; g < k.cols_total; g += nw) {
    const int s = g >= k.cols0 ? 1 : 0;
    const SysK<T>& Sy = k.s[s];
    const int j = static_cast<int>(g - (s ? k.cols0 : 0));
    T acc[Q][V];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
#pragma unroll
      for (int t = 0; t < V; ++t) acc[q][t] = T(0);
    }
    const int beg = Sy.cp[j], end = Sy.cp[j + 1];
    multi_row_dot<T, V, Q>(Sy.ri, Sy.cv, Sy.w, beg, end, lane, S, acc);
    const T ci = Sy.cinv[j];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
#pragma unroll
      for (int t = 0; t < V; ++t) {
        const int sl = (q * 32 + lane) * V + t;
        if (s ? onb[q][t] : ona[q][t]) {
          const long long o = static_cast<long long>(j) * S + sl;
          const T xn = upd(Sy.x[o], k.relax, acc[q][t], ci);
          Sy.x[o] = xn;
          if (!isfinite(static_cast<double>(xn))) {
            atomicCAS(&k.state[4 * (s * S + sl) + 2], 0, it + 1);
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------ block-merged multi-RHS
// Adjacent rays (rows) share most of their voxels, and adjacent voxels most of
// their rays: a block of R consecutive vectors touches ~2.2x fewer distinct
// indices than its R vectors together (config 4: 1,161 columns for 4 rows of
// 624). The plan merges each block's R vectors of BOTH folded systems into one
// sorted union list: per union index its 2R values (zero where a vector has no
// entry). A warp owns one block: it stages 32 union entries at a time in
// shared memory (read back as broadcasts), gathers each S-wide record of the
// dense operand once and applies it to all R vectors of both systems, whose
// accumulators stay in registers ([R][2][V] per lane, V slices per lane). The
// X (K1) / W (K2) record of an index is thus read once per block instead of
// once per vector and system. Summation order per vector: union order (=
// ascending index, as the vector's own CSR/CSC order), one product at a time.
template <class T>
struct BlockK {
  const int* ptr;  // [nblk + 1] union range of block b
  const int* idx;  // [nu] union indices
  const T* val;    // [nu][2][R] values: system s, vector r of the block
  long long nblk;
};

template <class T, int V>
__device__ __forceinline__ void ldv(const T* __restrict__ p, T (&o)[V], bool nc) {
  if (nc) {
    loadv<T, V>(p, o);
  } else {
#pragma unroll
    for (int t = 0; t < V; ++t) o[t] = p[t];
  }
}

constexpr int kBlockR = 4;     // vectors per block
constexpr int kBlockStage = 32;  // union entries staged per warp at a time

// acc[r][s][t] += sum over the block's union of val[s][r] * D_s[idx][slice t]
template <class T, int V, int E>
__device__ __forceinline__ void block_dot(const BlockK<T>& b, const T* __restrict__ d0,
                                          const T* __restrict__ d1, int u0, int u1, int lane,
                                          int S, int sl, int* sidx, T* sval,
                                          T (&acc)[kBlockR][2][V]) {
  constexpr int R = kBlockR;
  for (int ub = u0; ub < u1; ub += kBlockStage) {
    const int cnt = min(kBlockStage, u1 - ub);
    // stage: lane t copies entry ub + t (index + 2R values); zeros past the end
    {
      const int u = ub + lane;
      const bool on = lane < cnt;
      sidx[lane] = on ? __ldg(b.idx + u) : 0;
#pragma unroll
      for (int q = 0; q < 2 * R; ++q) {
        sval[lane * (2 * R) + q] = on ? __ldg(b.val + static_cast<long long>(u) * 2 * R + q) : T(0);
      }
    }
    __syncwarp();
    const bool act = sl < S;
    for (int t = 0; t < cnt; t += E) {  // E union entries' gathers in flight
      T g[E][2][V];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const long long o = static_cast<long long>(sidx[t + e]) * S + sl;
        if (act) {
          loadv<T, V>(d0 + o, g[e][0]);
          loadv<T, V>(d1 + o, g[e][1]);
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) g[e][0][v] = g[e][1][v] = T(0);
        }
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const T* vv = sval + (t + e) * (2 * R);
#pragma unroll
        for (int sy = 0; sy < 2; ++sy) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const T a = vv[sy * R + r];
#pragma unroll
            for (int v = 0; v < V; ++v) acc[r][sy][v] += a * g[e][sy][v];
          }
        }
      }
    }
    __syncwarp();
  }
}

template <class T, int V, int E>
__global__ void __launch_bounds__(kThreads, E <= 2 ? 3 : 1) sart_fwd_block_kernel(SartK<T> k, BlockK<T> b, int it) {
  constexpr int R = kBlockR;
  it = pass_index(k, it, true);
  if (loop_over(k, true)) return;
  extern __shared__ double mred[];  // [kWarps][2*S] then the staging buffers
  __shared__ int sidx_all[kWarps][kBlockStage];
  __shared__ T sval_all[kWarps][kBlockStage * 2 * R];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int S = k.nrhs;
  const int Q = (S + 32 * V - 1) / (32 * V);
  const long long gw = (blockIdx.x * (long long)kThreads + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kThreads) >> 5;
  const int nsr = 2 * S;
  for (int t = threadIdx.x; t < kWarps * nsr; t += kThreads) mred[t] = 0.0;
  __syncthreads();
  const long long rows = k.rows0;
  for (int q = 0; q < Q; ++q) {
    const int sl = (q * 32 + lane) * V;
    bool on[2][V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      on[0][v] = sl + v < S && sys_on(k.state, sl + v);
      on[1][v] = sl + v < S && sys_on(k.state, S + sl + v);
    }
    double r2[2][V];
#pragma unroll
    for (int v = 0; v < V; ++v) r2[0][v] = r2[1][v] = 0.0;
    for (long long blk = gw; blk < b.nblk; blk += nw) {
      T acc[R][2][V];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int sy = 0; sy < 2; ++sy)
#pragma unroll
          for (int v = 0; v < V; ++v) acc[r][sy][v] = T(0);
      block_dot<T, V, E>(b, k.s[0].x, k.s[1].x, __ldg(b.ptr + blk), __ldg(b.ptr + blk + 1), lane, S,
                      sl, sidx_all[warp], sval_all[warp], acc);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long i = blk * R + r;
        if (i >= rows) break;
#pragma unroll
        for (int sy = 0; sy < 2; ++sy) {
          const SysK<T>& Sy = k.s[sy];
          const T ri = Sy.rinv[i];
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if (!on[sy][v]) continue;
            const long long o = i * S + sl + v;
            const T rr = Sy.p[o] - acc[r][sy][v];
            Sy.w[o] = ri * rr;
            r2[sy][v] += static_cast<double>(rr) * static_cast<double>(rr);
          }
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (sl + v < S) {
        mred[warp * nsr + sl + v] = r2[0][v];
        mred[warp * nsr + S + sl + v] = r2[1][v];
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nsr; t += kThreads) {
    double a = 0.0;
    for (int q = 0; q < kWarps; ++q) a += mred[q * nsr + t];
    k.partial[static_cast<long long>(t) * gridDim.x + blockIdx.x] = a;
  }
  if (last_block(k.ticket)) {
    finish_norms(k.partial, gridDim.x, nsr, k.pnorm, k.tol, k.history, k.hstride, k.state, it);
    loop_next(k, it);
    if (threadIdx.x == 0) *k.ticket = 0;
  }
}

// ------------------------------------------------------------ X-staged multi-RHS K1
// Multi-RHS K1 with the gathered operand staged in shared memory by the bulk-
// copy (TMA) engine. A CTA owns blocks of kStageR consecutive rows (rays of one
// source, neighbouring detector bins) of one system. The rows of a block touch
// a sorted union U of columns (config 4: 3,303 for 16 rows of ~624 entries,
// reuse 3.0x), cut into chunks of kStageC union positions. The plan stores
// each block's entries chunk-major: per chunk a header of kStageR + 1 entry
// offsets (one run per pair of neighbouring rows) and the pair's merged
// entries {value of row a, value of row b (0 where absent), position in the
// chunk}: one X record read serves both rays (config 4: 803 merged positions
// per pair instead of 2 x 624 row entries).
// A producer warp fills a kStageNS-deep shared-memory ring: per chunk one bulk
// copy of its entry record and one bulk copy per run of consecutive union
// columns (contiguous X records [c][0..S) of the [n][S] layout; config 4
// unions run ~23 columns), completing on the slot's mbarrier (bytes counted);
// it runs ahead across block boundaries. Eight consumer warps (two rows each)
// apply a chunk with one broadcast shared-memory read per merged entry and one
// conflict-free read of its S-wide X record (V slices per lane) for two rows. X records
// thus move L2 -> shared memory once per block instead of once per row and
// never through L1; each row and slice is summed in CSR order, one product at
// a time, the padding adding exact zeros (bitwise equal to the per-row multi
// kernel).
constexpr int kStageR = 16;     // rows per block (2 per consumer warp)
constexpr int kStageC = 64;     // union positions per chunk
constexpr int kStageNS = 3;     // ring depth
constexpr int kStageThreads = kThreads + 32;  // 8 consumer warps + 1 producer warp
constexpr int kStageHdr = 32;   // (kStageR / 2 + 1) uint16 run offsets (row pairs), padded

template <class T>
struct StageK {
  const int* bptr;   // [nsys*nblk + 1] union range of each block (system-major)
  const int* buni;   // union columns
  const int* bch;    // [nsys*nblk] global index of each block's first chunk
  const long long* cofs;  // [nchunks + 1] byte offset of each chunk's entry record
  const char* ent;   // chunk records: header, then entries {T value, int position}
  long long nblk;    // blocks per system
  int slot_bytes;    // ring slot: kStageC X records + the largest entry record
};

// one union position of a row pair: both rows' values (0 where a row has no
// entry) and the position within the chunk
template <class T>
struct alignas(16) StageEnt {
  T va, vb;
  int u;
};

__device__ __forceinline__ void mbar_arrive(unsigned mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mb) : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes,
                                         unsigned mb) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(mb) : "memory");
}

template <class T, int V>
__device__ __forceinline__ void lds_v(const T* p, T (&o)[V]) {
  if constexpr (sizeof(T) * V == 16) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    const T* q = reinterpret_cast<const T*>(&t);
#pragma unroll
    for (int v = 0; v < V; ++v) o[v] = q[v];
  } else if constexpr (sizeof(T) * V == 32) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *(reinterpret_cast<const float4*>(p) + 1);
    const T* qa = reinterpret_cast<const T*>(&a);
    const T* qb = reinterpret_cast<const T*>(&b);
#pragma unroll
    for (int v = 0; v < V / 2; ++v) {
      o[v] = qa[v];
      o[V / 2 + v] = qb[v];
    }
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) o[v] = p[v];
  }
}

template <class T, int V, bool FWD>
__global__ void __launch_bounds__(kStageThreads, sizeof(T) == 4 ? 2 : 1)
    sart_stage_kernel(SartK<T> k, StageK<T> sk, int it) {
  it = pass_index(k, it, FWD);
  if (loop_over(k, FWD)) return;
  constexpr int RPW = kStageR / kWarps;  // rows per consumer warp
  static_assert(RPW == 2, "two rows per consumer warp");
  constexpr int S = 32 * V;               // slices (k.nrhs)
  constexpr int REC = S * static_cast<int>(sizeof(T));
  extern __shared__ __align__(128) char st_smem[];  // the ring; reused for the reductions
  __shared__ __align__(8) unsigned long long full[kStageNS], empty[kStageNS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int q = 0; q < kStageNS; ++q) {
      mbar_init(smem_u32(&full[q]), 1);
      mbar_init(smem_u32(&empty[q]), kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long nb_total = sk.nblk * k.nsys;
  const int sl = lane * V;
  double r2a[V], r2b[V];  // per-slice ||r||^2 of system 0 / 1
#pragma unroll
  for (int v = 0; v < V; ++v) r2a[v] = r2b[v] = 0.0;
  if (warp == kWarps) {
    // ---- producer: every chunk of every block of this CTA, NS slots ahead;
    // the next chunk's descriptors load while this one waits for its slot
    const unsigned ring_s = smem_u32(st_smem);
    struct Desc {
      long long e0, e1;
      int cu, nc, col0, col1;
      const T* X;
    };
    long long blk = blockIdx.x;
    int c = 0, nch = 0, u0 = 0, u1 = 0;
    long long gc = 0;
    const auto enter = [&]() {  // the block at blk (if any): its union and first chunk
      if (blk >= nb_total) return;
      u0 = __ldg(sk.bptr + blk);
      u1 = __ldg(sk.bptr + blk + 1);
      nch = (u1 - u0 + kStageC - 1) / kStageC;
      gc = __ldg(sk.bch + blk);
      c = 0;
    };
    const auto load = [&](Desc& d) {
      d.cu = u0 + c * kStageC;
      d.nc = min(kStageC, u1 - d.cu);
      d.e0 = __ldg(sk.cofs + gc);
      d.e1 = __ldg(sk.cofs + gc + 1);
      d.col0 = lane < d.nc ? __ldg(sk.buni + d.cu + lane) : 0;
      d.col1 = 32 + lane < d.nc ? __ldg(sk.buni + d.cu + 32 + lane) : 0;
      d.X = FWD ? k.s[blk >= sk.nblk ? 1 : 0].x : k.s[blk >= sk.nblk ? 1 : 0].w;
    };
    const auto advance = [&]() {  // to the next chunk of this CTA
      ++c;
      ++gc;
      while (blk < nb_total && c >= nch) {
        blk += gridDim.x;
        enter();
      }
    };
    enter();
    while (blk < nb_total && nch == 0) {
      blk += gridDim.x;
      enter();
    }
    Desc cur{};
    if (blk < nb_total) load(cur);
    for (unsigned q = 0; blk < nb_total; ++q) {
      advance();
      Desc nxt{};
      const bool more = blk < nb_total;
      if (more) load(nxt);
      const unsigned slot = q % kStageNS, use = q / kStageNS;
      const unsigned fb = smem_u32(&full[slot]);
      const unsigned base = ring_s + slot * sk.slot_bytes;
      if (use > 0) mbar_wait(smem_u32(&empty[slot]), (use - 1) & 1u);
      if (lane == 0) {
        mbar_expect(fb, static_cast<unsigned>(cur.nc * REC + (cur.e1 - cur.e0)));
        bulk_g2s(base + kStageC * REC, sk.ent + cur.e0, static_cast<unsigned>(cur.e1 - cur.e0),
                 fb);
      }
      // consecutive union columns are contiguous X records: one copy per run
#pragma unroll
      for (int h = 0; h < kStageC; h += 32) {
        const int m = min(32, cur.nc - h);
        const int col = h ? cur.col1 : cur.col0;
        const int prev = __shfl_up_sync(0xffffffffu, col, 1);
        const bool head = lane < m && (lane == 0 || col != prev + 1);
        const unsigned heads = __ballot_sync(0xffffffffu, head);
        if (head) {
          const unsigned later = heads & ~((2u << lane) - 1u);  // heads above this lane
          const int len = (later ? __ffs(later) - 1 : m) - lane;
          bulk_g2s(base + (h + lane) * REC, cur.X + static_cast<long long>(col) * S,
                   static_cast<unsigned>(len * REC), fb);
        }
      }
      if (!more) break;
      cur = nxt;
    }
  } else {
    // ---- consumers: warp w owns the neighbouring rows 2w and 2w + 1 of each block
    bool on0[V], on1[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      on0[v] = sys_on(k.state, sl + v);
      on1[v] = k.nsys > 1 && sys_on(k.state, S + sl + v);
    }
    unsigned q = 0;
    for (long long blk = blockIdx.x; blk < nb_total; blk += gridDim.x) {
      const int sy = blk >= sk.nblk ? 1 : 0;
      const SysK<T>& Sy = k.s[sy];
      const int u0 = __ldg(sk.bptr + blk), u1 = __ldg(sk.bptr + blk + 1);
      const int nch = (u1 - u0 + kStageC - 1) / kStageC;
      const int r0 = static_cast<int>((blk - sy * sk.nblk) * kStageR);
      const int nr = min(kStageR, static_cast<int>(FWD ? k.rows0 : k.cols0) - r0);
      T acc[RPW][V];
#pragma unroll
      for (int j = 0; j < RPW; ++j)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[j][v] = T(0);
      for (int c = 0; c < nch; ++c, ++q) {
        const unsigned slot = q % kStageNS, use = q / kStageNS;
        mbar_wait(smem_u32(&full[slot]), use & 1u);
        const char* sb = st_smem + slot * sk.slot_bytes;
        const T* xs = reinterpret_cast<const T*>(sb) + lane * V;
        const unsigned short* hdr = reinterpret_cast<const unsigned short*>(sb + kStageC * REC);
        const StageEnt<T>* ent = reinterpret_cast<const StageEnt<T>*>(sb + kStageC * REC + kStageHdr);
        const int eb = hdr[warp], ee = hdr[warp + 1];
        for (int e = eb; e < ee; e += 4) {
          StageEnt<T> en[4];
          T g[4][V];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (e + j < ee) {
              en[j] = ent[e + j];  // broadcast
              lds_v<T, V>(xs + en[j].u * S, g[j]);
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (e + j < ee) {
#pragma unroll
              for (int v = 0; v < V; ++v) {
                acc[0][v] += en[j].va * g[j][v];
                acc[1][v] += en[j].vb * g[j][v];
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&empty[slot]));
      }
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const int rl = 2 * warp + r;
        if (rl >= nr) continue;
        const long long i = r0 + rl;
        if constexpr (FWD) {  // r = p - A x, w = rinv r, per-slice ||r||^2
          const T ri = Sy.rinv[i];
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if (!(sy ? on1[v] : on0[v])) continue;
            const long long o = i * S + sl + v;
            const T rr = Sy.p[o] - acc[r][v];
            Sy.w[o] = ri * rr;
            const double d = static_cast<double>(rr) * static_cast<double>(rr);
            if (sy) r2b[v] += d;
            else r2a[v] += d;
          }
        } else {  // x += lambda * (u * cinv) (skipped for stopped slices)
          const T ci = Sy.cinv[i];
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if (!(sy ? on1[v] : on0[v])) continue;
            const long long o = i * S + sl + v;
            const T xn = upd(Sy.x[o], k.relax, acc[r][v], ci);
            Sy.x[o] = xn;
            if (!isfinite(static_cast<double>(xn))) {
              atomicCAS(&k.state[4 * (sy * S + sl + v) + 2], 0, it + 1);
            }
          }
        }
      }
    }
  }
  if constexpr (!FWD) return;
  __syncthreads();  // every chunk consumed: the ring is free
  double* mred = reinterpret_cast<double*>(st_smem);  // [kWarps][nsys*S]
  const int nsr = k.nsys * S;
  if (warp < kWarps) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      mred[warp * nsr + sl + v] = r2a[v];
      if (k.nsys > 1) mred[warp * nsr + S + sl + v] = r2b[v];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nsr; t += blockDim.x) {
    double a = 0.0;
    for (int w = 0; w < kWarps; ++w) a += mred[w * nsr + t];
    k.partial[static_cast<long long>(t) * gridDim.x + blockIdx.x] = a;
  }
  if (last_block(k.ticket)) {
    finish_norms(k.partial, gridDim.x, nsr, k.pnorm, k.tol, k.history, k.hstride, k.state, it);
    loop_next(k, it);
    if (threadIdx.x == 0) *k.ticket = 0;
  }
}

template <class T, int V, int E>
__global__ void __launch_bounds__(kThreads, E <= 2 ? 3 : 1) sart_back_block_kernel(SartK<T> k, BlockK<T> b, int it) {
  constexpr int R = kBlockR;
  it = pass_index(k, it, false);
  if (loop_over(k, false)) return;
  __shared__ int sidx_all[kWarps][kBlockStage];
  __shared__ T sval_all[kWarps][kBlockStage * 2 * R];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int S = k.nrhs;
  const int Q = (S + 32 * V - 1) / (32 * V);
  const long long gw = (blockIdx.x * (long long)kThreads + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * kThreads) >> 5;
  const long long cols = k.cols0;
  for (int q = 0; q < Q; ++q) {
    const int sl = (q * 32 + lane) * V;
    bool on[2][V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      on[0][v] = sl + v < S && sys_on(k.state, sl + v);
      on[1][v] = sl + v < S && sys_on(k.state, S + sl + v);
    }
    for (long long blk = gw; blk < b.nblk; blk += nw) {
      T acc[R][2][V];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int sy = 0; sy < 2; ++sy)
#pragma unroll
          for (int v = 0; v < V; ++v) acc[r][sy][v] = T(0);
      block_dot<T, V, E>(b, k.s[0].w, k.s[1].w, __ldg(b.ptr + blk), __ldg(b.ptr + blk + 1), lane, S,
                      sl, sidx_all[warp], sval_all[warp], acc);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const long long j = blk * R + r;
        if (j >= cols) break;
#pragma unroll
        for (int sy = 0; sy < 2; ++sy) {
          const SysK<T>& Sy = k.s[sy];
          const T ci = Sy.cinv[j];
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if (!on[sy][v]) continue;
            const long long o = j * S + sl + v;
            const T xn = upd(Sy.x[o], k.relax, acc[r][sy][v], ci);
            Sy.x[o] = xn;
            if (!isfinite(static_cast<double>(xn))) {
              atomicCAS(&k.state[4 * (sy * S + sl + v) + 2], 0, it + 1);
            }
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------ sharded update
// After the all-reduce of [A_g^T w_g | ||r_g||^2] every rank applies the same
// update (SURVEY §8e level 3) with the reference's check-before-update order.
template <class T>
__global__ void sart_sharded_update_kernel(T* x, const T* bp, const double* r2, const T* cinv,
                                           long long cols, const double* pnorm, double tol,
                                           double relax, double* history, int* state, int it) {
  if (!sys_on(state, 0)) return;
  const double res = sqrt(*r2);
  if (blockIdx.x == 0 && threadIdx.x == 0) history[it] = res;
  if (res <= tol * pnorm[0]) return;  // break before the update
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < cols;
       j += (long long)gridDim.x * blockDim.x) {
    const T xn = upd(x[j], relax, bp[j], cinv[j]);
    x[j] = xn;
    if (!isfinite(static_cast<double>(xn))) atomicCAS(&state[2], 0, it + 1);
  }
}

__global__ void sharded_stop_kernel(const double* r2, const double* pnorm, double tol, int* state,
                                    int it) {
  if (state[0] == 0 && state[2] == 0 && sqrt(*r2) <= tol * pnorm[0]) {
    state[0] = 1;
    state[1] = it;
  }
}

// Fixed-order sum of the forward kernel's per-block ||r_g||^2 partials into
// the fp64 all-reduce slot behind the back-projection (fp64 in every plan
// dtype, like the unsharded plans' residual).
__global__ void sharded_r2_kernel(const double* partial, int nblk, double* slot) {
  __shared__ double sh[kThreads];
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += partial[b];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *slot = sh[0];
}

// byte offset of the fp64 ||r_g||^2 slot behind the [cols] back-projection
inline std::size_t sharded_r2_offset(long long cols, std::size_t tsize) {
  return (static_cast<std::size_t>(cols) * tsize + 15) & ~static_cast<std::size_t>(15);
}
inline double* sharded_r2_slot(Plan& P) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(P.bp.get()) +
                                   sharded_r2_offset(P.cols[0], P.tsize()));
}

// ------------------------------------------------------------ peer exchange
// Row-sharded SART with the all-reduce replaced by peer-memory traffic
// (SURVEY §8e level 3; region layout in plan.hpp PeerExchange). Rank h owns
// the contiguous column range [h*own, (h+1)*own). Per iteration on rank me:
//   K1x  announces that this rank's previous reduce finished (one atomic per
//        rank into `xready`), waits until all G owners have pushed the
//        previous iteration's x range into this rank's replica, settles that
//        iteration's ||r|| (history, stop test) from the ranks' ||r_g||^2,
//        then runs the usual K1 over the local rows; its last block stores
//        ||r_me||^2 into every rank's slot.
//   K2x  the usual K2 over the local row block's CSC, except that each
//        column's partial (A_me^T w_me)_j goes straight into row `me` of the
//        owner's receive buffer — NVLink stores issued from the SpMV as the
//        columns complete, so the reduce-scatter's transfer overlaps the math.
//   Rx   (owner side) announces that this rank's K2x finished (`done`), waits
//        for all G ranks' K2x, sums the G partials of its columns in rank
//        order (the same bits on every run, independent of timing), applies
//        the update unless the iteration stopped and stores the new x range
//        into every replica.
// Every signal is issued by the kernel *after* the one whose stores it
// announces: stream order has completed those stores (kernel boundary), so no
// system-scope fence is needed on the data path (measured: fences at the end
// of every K2x / reduce CTA cost 13-16 us per iteration). Counters are
// monotone over solves (epoch base in `local`); no kernel resets a peer's
// state, and every wait is bounded (timeout flag, reported by Plan::finish) so
// a lost rank fails the solve instead of hanging the GPU.
template <class T>
struct XK {
  char* const* peers;
  int G, me;
  long long cols, own;  // columns, columns owned per rank
  int rgrid;            // CTAs of the reduce kernel
  unsigned long long off_recv, off_x, off_r2, off_done, off_xready, off_dflag;
  long long* local;     // {epoch base, iterations proceeded, timeout, reduces announced}
  int inline_signal;    // 1: kernels announce; 0 (emulated group): announce kernels do
};

template <class T>
__device__ __forceinline__ char* xbase(const XK<T>& x, int r) {
  return reinterpret_cast<char*>(
      __ldg(reinterpret_cast<const unsigned long long*>(x.peers) + r));
}
template <class T>
__device__ __forceinline__ T* xrecv(const XK<T>& x, int r) {
  return reinterpret_cast<T*>(xbase(x, r) + x.off_recv);
}
template <class T>
__device__ __forceinline__ T* xrep(const XK<T>& x, int r) {
  return reinterpret_cast<T*>(xbase(x, r) + x.off_x);
}
template <class T>
__device__ __forceinline__ double* xr2(const XK<T>& x, int r) {
  return reinterpret_cast<double*>(xbase(x, r) + x.off_r2);
}
template <class T>
__device__ __forceinline__ unsigned long long* xdone(const XK<T>& x, int r) {
  return reinterpret_cast<unsigned long long*>(xbase(x, r) + x.off_done);
}
template <class T>
__device__ __forceinline__ unsigned long long* xready(const XK<T>& x, int r) {
  return reinterpret_cast<unsigned long long*>(xbase(x, r) + x.off_xready);
}
template <class T>
__device__ __forceinline__ int* xdflag(const XK<T>& x, int r) {
  return reinterpret_cast<int*>(xbase(x, r) + x.off_dflag);
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float ld_sys(const float* p) {
  float v;
  asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_sys(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_sys(const int* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// one count into counter `off` of every rank. The stores being announced
// belong to an earlier, completed kernel of this stream (or to this thread);
// one system-scope fence in the announcing thread makes them cumulatively
// visible before any count lands, so a consumer's ld.acquire.sys of the
// counter pairs with it (PTX memory model) -- no per-CTA fences on the data
// path, one fence per rank per announcement.
template <class T>
__device__ void signal_all(const XK<T>& x, unsigned long long off) {
  __threadfence_system();
  for (int r = 0; r < x.G; ++r) {
    atomicAdd_system(reinterpret_cast<unsigned long long*>(xbase(x, r) + off), 1ull);
  }
}

// ~4 s at 1.9 GHz: far beyond any healthy exchange wait (microseconds)
constexpr long long kSpinCycles = 8000000000LL;

__device__ bool wait_geq(const unsigned long long* p, unsigned long long target,
                         long long* timeout) {
  if (ld_acquire_sys(p) >= target) return true;
  const long long t0 = clock64();
  while (ld_acquire_sys(p) < target) {
    if (*reinterpret_cast<volatile long long*>(timeout) != 0) return false;
    if (clock64() - t0 > kSpinCycles) {
      if (atomicExch(reinterpret_cast<unsigned long long*>(timeout), 1ull) == 0ull) {
        printf("symsplit_b200: exchange wait timed out (counter %llu, want %llu, block %d, "
               "grid %d)\n", ld_acquire_sys(p), target, static_cast<int>(blockIdx.x),
               static_cast<int>(gridDim.x));
      }
      return false;
    }
    __nanosleep(100);
  }
  return true;
}

// ||r||^2 of absolute iteration e: the ranks' contributions in rank order
template <class T>
__device__ double xr2_sum(const XK<T>& x, long long e) {
  const double* s = xr2(x, x.me) + (e & 1) * x.G;
  double t = 0.0;
  for (int g = 0; g < x.G; ++g) t += ld_sys(s + g);
  return t;
}

template <class T>
__device__ __forceinline__ unsigned long long xready_target(const XK<T>& x, long long epochs) {
  return static_cast<unsigned long long>(x.G) * epochs;
}

// K1x prologue (thread 0 of every block; every block decides alike): wait for
// the previous iteration's x, settle its residual / stop / divergence.
template <class T>
__device__ int xchg_enter(const SartK<T>& k, const XK<T>& x, int it) {
  volatile int* st = k.state;
  // reduce it-1 ran iff K1x(it-1) proceeded; announce its x pushes (block 0)
  if (x.inline_signal && blockIdx.x == 0 && it > 0 && x.local[1] == it) {
    signal_all(x, x.off_xready);
    x.local[3] = it;
  }
  if (st[0] != 0 || st[2] != 0) return 0;
  const long long base = x.local[0];
  if (!wait_geq(xready(x, x.me), xready_target(x, base + it), x.local + 2)) return 0;
  if (it > 0) {
    const int d = ld_sys(xdflag(x, x.me));
    if (d != 0) {
      if (blockIdx.x == 0) st[2] = d;
      return 0;
    }
    const double res = sqrt(xr2_sum(x, base + it - 1));
    if (blockIdx.x == 0) k.history[it - 1] = res;
    if (res <= k.tol * k.pnorm[0]) {
      if (blockIdx.x == 0) {
        st[0] = 1;
        st[1] = it - 1;
      }
      return 0;
    }
  }
  if (blockIdx.x == 0) x.local[1] = it + 1;
  return 1;
}

template <class T, int VS, int UF, bool U16>
__global__ void __launch_bounds__(kThreads, kDirectMinBlocks)
    sart_fwd_xchg_kernel(SartK<T> k, XK<T> x, int it) {
  cudaGridDependencySynchronize();
  __shared__ double red[kWarps];
  __shared__ int go;
  if (threadIdx.x == 0) go = xchg_enter(k, x, it);
  __syncthreads();
  if (!go) return;
  const SysK<T>& S = k.s[0];
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const int n = static_cast<int>(k.rows0);
  const int gstep = static_cast<int>((long long)gridDim.x * kThreads / VS);
  int g = static_cast<int>((blockIdx.x * (long long)kThreads + threadIdx.x) / VS);
  double r2 = 0.0;
  int beg = 0, end = 0, tf = 0;
  if (g < n) {
    beg = __ldg(k.tpf + g);
    end = __ldg(k.tpf + g + 1);
    if (U16) tf = __ldg(k.tff + g);
  }
  for (; g < n; g += gstep) {
    const int gn = g + gstep;
    int nbeg = 0, nend = 0, ntf = 0;
    if (gn < n) {
      nbeg = __ldg(k.tpf + gn);
      nend = __ldg(k.tpf + gn + 1);
      if (U16) ntf = __ldg(k.tff + gn);
    }
    T pv = T(0), ri = T(0);
    if (lane == 0) {
      pv = S.p[g];
      ri = S.rinv[g];
    }
    const T dot = seg_dot1<T, VS, UF, U16>(k.tif, k.tof, k.tbf, tf, k.rv2, S.x, beg, end, lane,
                                           mask);
    if (lane == 0) {
      const T r = pv - dot;
      S.w[g] = ri * r;
      r2 += static_cast<double>(r) * static_cast<double>(r);
    }
    beg = nbeg;
    end = nend;
    tf = ntf;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < kWarps; ++q) t += red[q];
    k.partial[blockIdx.x] = t;
  }
  if (last_block(k.ticket)) {
    // fixed-order ||r_me||^2, stored into slot [parity][me] of every rank
    __shared__ double sh[kThreads];
    double s = 0.0;
    for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += kThreads) s += k.partial[b];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = kThreads / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
      __syncthreads();
    }
    const long long e = x.local[0] + it;
    if (threadIdx.x < x.G) xr2(x, threadIdx.x)[(e & 1) * x.G + x.me] = sh[0];
    if (threadIdx.x == 0) *k.ticket = 0;
  }
}

template <class T, int VS, int UF, bool U16>
__global__ void __launch_bounds__(kThreads, kDirectMinBlocks)
    sart_back_xchg_kernel(SartK<T> k, XK<T> x, int it) {
  cudaGridDependencySynchronize();
  if (!sys_on_cg(k.state, 0)) return;
  const SysK<T>& S = k.s[0];
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const int n = static_cast<int>(k.cols0);
  const int gstep = static_cast<int>((long long)gridDim.x * kThreads / VS);
  int g = static_cast<int>((blockIdx.x * (long long)kThreads + threadIdx.x) / VS);
  const long long row = static_cast<long long>(x.me) * x.cols;
  int beg = 0, end = 0, tf = 0;
  if (g < n) {
    beg = __ldg(k.tpb + g);
    end = __ldg(k.tpb + g + 1);
    if (U16) tf = __ldg(k.tfb + g);
  }
  for (; g < n; g += gstep) {
    const int gn = g + gstep;
    int nbeg = 0, nend = 0, ntf = 0;
    if (gn < n) {
      nbeg = __ldg(k.tpb + gn);
      nend = __ldg(k.tpb + gn + 1);
      if (U16) ntf = __ldg(k.tfb + gn);
    }
    const T u = seg_dot1<T, VS, UF, U16>(k.tib, k.tob, k.tbb, tf, k.cv2, S.w, beg, end, lane,
                                         mask);
    if (lane == 0) {  // NVLink store into the owner's receive row
      xrecv(x, static_cast<int>(static_cast<unsigned>(g) / static_cast<unsigned>(x.own)))[row + g] = u;
    }
    beg = nbeg;
    end = nend;
    tf = ntf;
  }
}

// Owner side: rank-order sum of the G partials of this rank's columns,
// update (unless the iteration stopped), push the new range to every replica.
template <class T>
__global__ void __launch_bounds__(kThreads) xchg_reduce_kernel(SartK<T> k, XK<T> x, int it) {
  cudaGridDependencySynchronize();  // K2x of this rank has completed
  if (!sys_on(k.state, 0)) return;
  __shared__ int go;
  const long long e = x.local[0] + it;
  if (threadIdx.x == 0) {
    if (x.inline_signal && blockIdx.x == 0) signal_all(x, x.off_done);
    go = wait_geq(xdone(x, x.me), static_cast<unsigned long long>(x.G) * (e + 1), x.local + 2);
  }
  __syncthreads();
  if (!go) return;
  const bool stop = sqrt(xr2_sum(x, e)) <= k.tol * k.pnorm[0];
  if (!stop) {
    const long long j0 = x.me * x.own, j1 = min(j0 + x.own, x.cols);
    const T* src = xrecv(x, x.me);
    const T* xl = xrep(x, x.me);
    const T* ci = k.s[0].cinv;
    bool bad = false;
    for (long long j = j0 + blockIdx.x * (long long)kThreads + threadIdx.x; j < j1;
         j += (long long)gridDim.x * kThreads) {
      T s = ld_sys(src + j);
      for (int g = 1; g < x.G; ++g) s += ld_sys(src + g * x.cols + j);
      const T xn = upd(ld_sys(xl + j), k.relax, s, ci[j]);
      for (int r = 0; r < x.G; ++r) xrep(x, r)[j] = xn;  // local + NVLink stores
      bad |= !isfinite(static_cast<double>(xn));
    }
    if (bad) {
      for (int r = 0; r < x.G; ++r) atomicCAS_system(xdflag(x, r), 0, it + 1);
    }
  }
}

// Emulated group: the announcements the kernels make inline on real ranks,
// as separate launches issued for every rank before any rank's next waiting
// kernel (kind 0: before K1x, 1: before the reduce, 2: before the final kernel).
template <class T>
__global__ void xchg_announce_kernel(SartK<T> k, XK<T> x, int it, int kind) {
  if (threadIdx.x != 0) return;
  if (kind == 0 && it > 0 && x.local[1] == it) {
    signal_all(x, x.off_xready);
    x.local[3] = it;
  }
  if (kind == 1 && sys_on(k.state, 0)) signal_all(x, x.off_done);
  if (kind == 2 && x.local[3] < x.local[1]) signal_all(x, x.off_xready);
}

// After the last pass: wait for the final iteration's x, settle its residual /
// stop state, advance the epoch base by the iterations run.
template <class T>
__global__ void xchg_final_kernel(SartK<T> k, XK<T> x) {
  if (threadIdx.x != 0) return;
  volatile int* st = k.state;
  const long long base = x.local[0], L = x.local[1];
  // the last reduce is announced here unless a K1x already did (a solve cut
  // short by the stop test, or a partial pass count as in Plan::profile)
  if (x.inline_signal && x.local[3] < L) signal_all(x, x.off_xready);
  if (!wait_geq(xready(x, x.me), xready_target(x, base + L), x.local + 2)) return;
  if (L > 0 && st[0] == 0 && st[2] == 0) {
    const int d = ld_sys(xdflag(x, x.me));
    if (d != 0) {
      st[2] = d;
    } else {
      const double res = sqrt(xr2_sum(x, base + L - 1));
      k.history[L - 1] = res;
      if (res <= k.tol * k.pnorm[0]) {
        st[0] = 1;
        st[1] = static_cast<int>(L - 1);
      }
    }
  }
  x.local[0] = base + L;
  x.local[1] = 0;
  x.local[3] = 0;
}

// ---------------------------------------------------------- paired peer exchange
// The folded pair row-sharded over all G ranks (not one system per GPU half):
// rank `me` keeps rows [rb, re) of A1 and A2 on the paired mirror-coded
// streams, so every rank streams 1/G of the bytes of the single-GPU paired
// plan. Same protocol as the single-system exchange above, with both systems
// in every message: receive rows hold {u1, u2} pairs ([G][cols][2]), the x
// replica is the interleaved iterate ([cols][2]), the ||r_g||^2 slots are
// [2 parity][G][2 systems], the divergence flags one per system. Each system
// keeps its own stop / divergence state (the two branches of solve_split stay
// independent solves, solvers.cpp:212-233); a pass runs while either is on.

// K1x-pair prologue (thread 0 of every block; every block decides alike):
// settle the previous iteration of each system, return the systems to run
// (bit 0: system 1, bit 1: system 2; 0 = nothing this pass)
template <class T>
__device__ int xchg_enter_pair(const SartK<T>& k, const XK<T>& x, int it) {
  volatile int* st = k.state;
  if (x.inline_signal && blockIdx.x == 0 && it > 0 && x.local[1] == it) {
    signal_all(x, x.off_xready);
    x.local[3] = it;
  }
  bool on[2] = {st[0] == 0 && st[2] == 0, st[4] == 0 && st[6] == 0};
  if (!on[0] && !on[1]) return 0;
  const long long base = x.local[0];
  if (!wait_geq(xready(x, x.me), xready_target(x, base + it), x.local + 2)) return 0;
  if (it > 0) {
    const double* r2 = xr2(x, x.me) + ((base + it - 1) & 1) * 2 * x.G;
    for (int q = 0; q < 2; ++q) {
      if (!on[q]) continue;
      const int d = ld_sys(xdflag(x, x.me) + q);
      if (d != 0) {
        if (blockIdx.x == 0) st[4 * q + 2] = d;
        on[q] = false;
        continue;
      }
      double t = 0.0;
      for (int g = 0; g < x.G; ++g) t += ld_sys(r2 + 2 * g + q);
      const double res = sqrt(t);
      if (blockIdx.x == 0) k.history[q * k.hstride + it - 1] = res;
      if (res <= k.tol * k.pnorm[q]) {
        if (blockIdx.x == 0) {
          st[4 * q + 0] = 1;
          st[4 * q + 1] = it - 1;
        }
        on[q] = false;
      }
    }
  }
  if (!on[0] && !on[1]) return 0;
  if (blockIdx.x == 0) x.local[1] = it + 1;
  return (on[0] ? 1 : 0) | (on[1] ? 2 : 0);
}

template <class T, int VS, int UF, int TL>
__global__ void __launch_bounds__(kThreads, kDirectMinBlocks)
    sart_fwd_xchg_pair_kernel(SartK<T> k, XK<T> x, int it) {
  using T2 = typename Vec2<T>::type;
  cudaGridDependencySynchronize();
  __shared__ double red[2][kWarps];
  __shared__ int go;
  if (threadIdx.x == 0) go = xchg_enter_pair(k, x, it);
  __syncthreads();
  if (!go) return;
  const bool on0 = (go & 1) != 0, on1 = (go & 2) != 0;
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const int n = static_cast<int>(k.rows0);
  const int gstep = static_cast<int>((long long)gridDim.x * kThreads / VS);
  double r2a = 0.0, r2b = 0.0;
  for (int g = static_cast<int>((blockIdx.x * (long long)kThreads + threadIdx.x) / VS); g < n;
       g += gstep) {
    const int beg = __ldg(k.tpf + g), end = __ldg(k.tpf + g + 1), tf = __ldg(k.tff + g);
    int eb = 0, ee = 0;
    if (k.epf) {
      eb = __ldg(k.epf + g);
      ee = __ldg(k.epf + g + 1);
    }
    T e[4] = {T(0), T(0), T(0), T(0)};
    if (lane == 0) load4(k.pe + 4 * static_cast<long long>(g), e);
    T da, db;
    seg_dot2m<T, VS, UF, TL == 5, TL != 6>(k.tof, k.tif, k.thf, tf, k.rv2,
                                            reinterpret_cast<const T2*>(k.xx), beg, end, eb, ee,
                                            k.eif, k.evf, lane, mask, da, db);
    if (lane == 0) {
      const T ra = e[0] - da, rb = e[1] - db;
      T2 wo;
      wo.x = on0 ? e[2] * ra : T(0);
      wo.y = on1 ? e[3] * rb : T(0);
      reinterpret_cast<T2*>(k.ww)[g] = wo;
      if (on0) r2a += static_cast<double>(ra) * static_cast<double>(ra);
      if (on1) r2b += static_cast<double>(rb) * static_cast<double>(rb);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r2a += __shfl_xor_sync(0xffffffffu, r2a, o);
    r2b += __shfl_xor_sync(0xffffffffu, r2b, o);
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][warp] = r2a;
    red[1][warp] = r2b;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double t = 0.0;
    for (int q = 0; q < kWarps; ++q) t += red[threadIdx.x][q];
    k.partial[threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
  if (last_block(k.ticket)) {
    // fixed-order ||r_me||^2 of both systems into slot [parity][me][q] of every rank
    __shared__ double sh[kThreads];
    __shared__ double tot[2];
    for (int q = 0; q < 2; ++q) {
      double s = 0.0;
      for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += kThreads)
        s += k.partial[q * gridDim.x + b];
      sh[threadIdx.x] = s;
      __syncthreads();
      for (int o = kThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
      }
      if (threadIdx.x == 0) tot[q] = sh[0];
      __syncthreads();
    }
    const long long e = x.local[0] + it;
    if (threadIdx.x < x.G) {
      double* slot = xr2(x, threadIdx.x) + (e & 1) * 2 * x.G + 2 * x.me;
      slot[0] = tot[0];
      slot[1] = tot[1];
    }
    if (threadIdx.x == 0) *k.ticket = 0;
  }
}

template <class T, int VS, int UF, int TL>
__global__ void __launch_bounds__(kThreads, kDirectMinBlocks)
    sart_back_xchg_pair_kernel(SartK<T> k, XK<T> x, int it) {
  using T2 = typename Vec2<T>::type;
  cudaGridDependencySynchronize();
  const bool on0 = sys_on_cg(k.state, 0), on1 = sys_on_cg(k.state, 1);
  if (!on0 && !on1) return;
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const int n = static_cast<int>(k.cols0);
  const int gstep = static_cast<int>((long long)gridDim.x * kThreads / VS);
  const long long row = static_cast<long long>(x.me) * x.cols;
  for (int g = static_cast<int>((blockIdx.x * (long long)kThreads + threadIdx.x) / VS); g < n;
       g += gstep) {
    const int beg = __ldg(k.tpb + g), end = __ldg(k.tpb + g + 1), tf = __ldg(k.tfb + g);
    int eb = 0, ee = 0;
    if (k.epb) {
      eb = __ldg(k.epb + g);
      ee = __ldg(k.epb + g + 1);
    }
    T ua, ub;
    seg_dot2m<T, VS, UF, TL == 5, TL != 6>(k.tob, k.tib, k.thb, tf, k.cv2,
                                            reinterpret_cast<const T2*>(k.ww), beg, end, eb, ee,
                                            k.eib, k.evb, lane, mask, ua, ub);
    if (lane == 0) {  // {u1, u2} into the owner's receive row (NVLink store)
      T2 u;
      u.x = ua;
      u.y = ub;
      T2* recv = reinterpret_cast<T2*>(
          xrecv(x, static_cast<int>(static_cast<unsigned>(g) / static_cast<unsigned>(x.own))));
      recv[row + g] = u;
    }
  }
}

// Owner side, both systems: rank-order sums of the G partial pairs of this
// rank's columns, per-system update (unless that system stopped this pass),
// the new {x1, x2} range pushed into every replica.
template <class T>
__global__ void __launch_bounds__(kThreads) xchg_reduce_pair_kernel(SartK<T> k, XK<T> x, int it) {
  using T2 = typename Vec2<T>::type;
  cudaGridDependencySynchronize();
  const bool on0 = sys_on_cg(k.state, 0), on1 = sys_on_cg(k.state, 1);
  if (!on0 && !on1) return;
  __shared__ int go;
  const long long e = x.local[0] + it;
  if (threadIdx.x == 0) {
    if (x.inline_signal && blockIdx.x == 0) signal_all(x, x.off_done);
    go = wait_geq(xdone(x, x.me), static_cast<unsigned long long>(x.G) * (e + 1), x.local + 2);
  }
  __syncthreads();
  if (!go) return;
  bool up[2] = {on0, on1};
  const double* r2 = xr2(x, x.me) + (e & 1) * 2 * x.G;
  for (int q = 0; q < 2; ++q) {
    if (!up[q]) continue;
    double t = 0.0;
    for (int g = 0; g < x.G; ++g) t += ld_sys(r2 + 2 * g + q);
    if (sqrt(t) <= k.tol * k.pnorm[q]) up[q] = false;  // check before update
  }
  if (!up[0] && !up[1]) return;
  const long long j0 = x.me * x.own, j1 = min(j0 + x.own, x.cols);
  const T* src = xrecv(x, x.me);
  const T* xl = xrep(x, x.me);
  const T2* ci = reinterpret_cast<const T2*>(k.cc);
  bool bad[2] = {false, false};
  for (long long j = j0 + blockIdx.x * (long long)kThreads + threadIdx.x; j < j1;
       j += (long long)gridDim.x * kThreads) {
    T sa = ld_sys(src + 2 * j), sb = ld_sys(src + 2 * j + 1);
    for (int g = 1; g < x.G; ++g) {
      sa += ld_sys(src + 2 * (g * x.cols + j));
      sb += ld_sys(src + 2 * (g * x.cols + j) + 1);
    }
    T2 xo;
    xo.x = ld_sys(xl + 2 * j);
    xo.y = ld_sys(xl + 2 * j + 1);
    const T2 c = __ldg(ci + j);
    if (up[0]) xo.x = upd(xo.x, k.relax, sa, c.x);
    if (up[1]) xo.y = upd(xo.y, k.relax, sb, c.y);
    for (int r = 0; r < x.G; ++r) reinterpret_cast<T2*>(xrep(x, r))[j] = xo;  // local + NVLink
    bad[0] |= up[0] && !isfinite(static_cast<double>(xo.x));
    bad[1] |= up[1] && !isfinite(static_cast<double>(xo.y));
  }
  for (int q = 0; q < 2; ++q) {
    if (bad[q]) {
      for (int r = 0; r < x.G; ++r) atomicCAS_system(xdflag(x, r) + q, 0, it + 1);
    }
  }
}

// Emulated group, pairs: the announcements the kernels make inline on real ranks.
template <class T>
__global__ void xchg_announce_pair_kernel(SartK<T> k, XK<T> x, int it, int kind) {
  if (threadIdx.x != 0) return;
  if (kind == 0 && it > 0 && x.local[1] == it) {
    signal_all(x, x.off_xready);
    x.local[3] = it;
  }
  if (kind == 1 && (sys_on(k.state, 0) || sys_on(k.state, 1))) signal_all(x, x.off_done);
  if (kind == 2 && x.local[3] < x.local[1]) signal_all(x, x.off_xready);
}

// After the last pass, pairs: wait for the final x, settle each system's last
// residual / stop / divergence, advance the epoch base.
template <class T>
__global__ void xchg_final_pair_kernel(SartK<T> k, XK<T> x) {
  if (threadIdx.x != 0) return;
  volatile int* st = k.state;
  const long long base = x.local[0], L = x.local[1];
  if (x.inline_signal && x.local[3] < L) signal_all(x, x.off_xready);
  if (!wait_geq(xready(x, x.me), xready_target(x, base + L), x.local + 2)) return;
  if (L > 0) {
    const double* r2 = xr2(x, x.me) + ((base + L - 1) & 1) * 2 * x.G;
    for (int q = 0; q < 2; ++q) {
      if (st[4 * q] != 0 || st[4 * q + 2] != 0) continue;
      const int d = ld_sys(xdflag(x, x.me) + q);
      if (d != 0) {
        st[4 * q + 2] = d;
        continue;
      }
      double t = 0.0;
      for (int g = 0; g < x.G; ++g) t += ld_sys(r2 + 2 * g + q);
      const double res = sqrt(t);
      k.history[q * k.hstride + L - 1] = res;
      if (res <= k.tol * k.pnorm[q]) {
        st[4 * q] = 1;
        st[4 * q + 1] = static_cast<int>(L - 1);
      }
    }
  }
  x.local[0] = base + L;
  x.local[1] = 0;
  x.local[3] = 0;
}

// Column-band boundaries inside every CSR row (columns ascending): out[b][i] =
// first position of row i whose column is >= b*cols/nband (b = nband: row end).
__global__ void band_ptr_kernel(const int* __restrict__ rp, const int* __restrict__ ci,
                                long long rows, long long cols, int nband, int* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows;
       i += (long long)gridDim.x * blockDim.x) {
    const int beg = rp[i], end = rp[i + 1];
    out[i] = beg;
    out[static_cast<long long>(nband) * rows + i] = end;
    for (int b = 1; b < nband; ++b) {
      const long long c0 = cols * b / nband;
      int lo = beg, hi = end;  // first position with ci >= c0
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ci[mid] < c0) lo = mid + 1;
        else hi = mid;
      }
      out[static_cast<long long>(b) * rows + i] = lo;
    }
  }
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

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

bool pdl_enabled() {
  static const bool on = env_int("SSB_PDL", 1) != 0;
  return on;
}

// Lanes per compressed vector. Several vectors per warp keep independent
// dependency chains in flight; adjacent rows (rays) share x lines in L1.
int pick_vs(double avg) {
  if (avg >= 384) return 16;
  if (avg >= 160) return 8;
  return 4;
}

int pick_vs_mirror(double avg) {
  if (avg >= 1024) return 16;
  if (avg >= 96) return 8;
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
  k.sys_blocks[0] = P.sys_blocks_f;
  k.sys_blocks[1] = P.sys_blocks_b;
  k.xx = reinterpret_cast<T*>(P.xx.get());
  k.ww = reinterpret_cast<T*>(P.ww.get());
  k.rv2 = reinterpret_cast<const T*>(P.rv2.get());
  k.cv2 = reinterpret_cast<const T*>(P.cv2.get());
  k.pe = reinterpret_cast<const T*>(P.pe.get());
  k.cc = reinterpret_cast<const T*>(P.cc.get());
  k.tpf = P.tptr_f.get();
  k.tif = P.tidx_f.get();
  k.tpb = P.tptr_b.get();
  k.tib = P.tidx_b.get();
  k.tof = P.tofs_f.get();
  k.tbf = P.tbase_f.get();
  k.tff = P.tfirst_f.get();
  k.tob = P.tofs_b.get();
  k.tbb = P.tbase_b.get();
  k.tfb = P.tfirst_b.get();
  k.thf = P.thdr_f.get();
  k.thb = P.thdr_b.get();
  k.epf = P.eptr_f.get();
  k.eif = P.eidx_f.get();
  k.evf = reinterpret_cast<const T*>(P.ev2_f.get());
  k.epb = P.eptr_b.get();
  k.eib = P.eidx_b.get();
  k.evb = reinterpret_cast<const T*>(P.ev2_b.get());
  if (P.sharded && !P.px) {
    k.bp_out = reinterpret_cast<T*>(P.bp.get());
  }
  if (P.px && !P.paired) {
    k.s[0].x = reinterpret_cast<T*>(static_cast<char*>(P.px->region) + P.px->off_x);
  }
  if (P.px && P.paired) {  // the interleaved iterate is this rank's replica
    k.xx = reinterpret_cast<T*>(static_cast<char*>(P.px->region) + P.px->off_x);
  }
  if (P.while_capture) {
    k.iter = P.iter_dev.get();
    k.cond = P.cond;
  }
  k.max_iters = P.opts.max_iters;
  return k;
}

template <class T, int VS>
void launch_fwd1(Plan& P, const SartK<T>& k, int it) {
  auto* fn = P.uf_fwd >= 4 ? sart_fwd_kernel<T, VS, 4> : sart_fwd_kernel<T, VS, 2>;
  fn<<<P.fwd_blocks, kThreads, 0, P.ctx->stream>>>(k, it);
}
template <class T, int VS>
void launch_back1(Plan& P, const SartK<T>& k, int it) {
  auto* fn = P.uf_back >= 4 ? sart_back_kernel<T, VS, 4> : sart_back_kernel<T, VS, 2>;
  fn<<<P.back_blocks, kThreads, 0, P.ctx->stream>>>(k, it);
}

template <class T>
using PairFn = void (*)(SartK<T>, int);

// the paired kernel a plan launches (layout x VS x UF) and its
// dynamic shared memory
template <class T>
PairFn<T> pair_kernel(const Plan& P, bool fwd, int* smem) {
  const int vs = fwd ? P.vs_fwd : P.vs_back;
  const int uf = fwd ? P.uf_fwd : P.uf_back;
  *smem = 0;
#define SSB_PAIR(V, U)                                                                        \
  if (vs == V && uf == U) {                                                                   \
    if (!P.tiled) return fwd ? sart_fwd_pair_kernel<T, V, U, 0> : sart_back_pair_kernel<T, V, U, 0>; \
    if ((fwd ? P.mir_f : P.mir_b) && !(fwd ? P.c16f : P.c16b))                                \
      return fwd ? sart_fwd_pair_kernel<T, V, U, 6> : sart_back_pair_kernel<T, V, U, 6>;      \
    if ((fwd ? P.mir_f : P.mir_b) && P.stream_cs)                                            \
      return fwd ? sart_fwd_pair_kernel<T, V, U, 5> : sart_back_pair_kernel<T, V, U, 5>;      \
    if (fwd ? P.mir_f : P.mir_b)                                                              \
      return fwd ? sart_fwd_pair_kernel<T, V, U, 4> : sart_back_pair_kernel<T, V, U, 4>;      \
    if ((fwd ? P.c16f : P.c16b) && P.stream_cs)                                              \
      return fwd ? sart_fwd_pair_kernel<T, V, U, 3> : sart_back_pair_kernel<T, V, U, 3>;      \
    if (fwd ? P.c16f : P.c16b)                                                                \
      return fwd ? sart_fwd_pair_kernel<T, V, U, 2> : sart_back_pair_kernel<T, V, U, 2>;      \
    return fwd ? sart_fwd_pair_kernel<T, V, U, 1> : sart_back_pair_kernel<T, V, U, 1>;        \
  }
  SSB_PAIR(4, 1) SSB_PAIR(8, 1) SSB_PAIR(16, 1) SSB_PAIR(32, 1)
  SSB_PAIR(4, 2) SSB_PAIR(8, 2) SSB_PAIR(16, 2) SSB_PAIR(32, 2)
  SSB_PAIR(4, 4) SSB_PAIR(8, 4) SSB_PAIR(16, 4) SSB_PAIR(32, 4)
#undef SSB_PAIR
  fail("plan: unsupported paired kernel shape");
  return nullptr;
}

// single-system tiled kernel of a plan
template <class T>
PairFn<T> single_kernel(const Plan& P, bool fwd) {
  const int vs = fwd ? P.vs_fwd : P.vs_back;
  const int uf = fwd ? P.uf_fwd : P.uf_back;
  const bool u16 = fwd ? P.c16f : P.c16b;
#define SSB_ONE(V, U)                                                                          \
  if (vs == V && uf == U) {                                                                    \
    if (u16) return fwd ? sart_fwd_tiled_kernel<T, V, U, true> : sart_back_tiled_kernel<T, V, U, true>; \
    return fwd ? sart_fwd_tiled_kernel<T, V, U, false> : sart_back_tiled_kernel<T, V, U, false>; \
  }
  SSB_ONE(4, 2) SSB_ONE(8, 2) SSB_ONE(16, 2) SSB_ONE(32, 2)
  SSB_ONE(4, 4) SSB_ONE(8, 4) SSB_ONE(16, 4) SSB_ONE(32, 4)
#undef SSB_ONE
  fail("plan: unsupported single-system kernel shape");
  return nullptr;
}

bool single_tiled(const Plan& P) { return !P.paired && P.tiled && P.nrhs == 1 && P.nsys == 1; }

// Launch with programmatic dependent launch: the kernel's CTAs are scheduled
// while the previous pass's tail drains and wait in cudaGridDependencySynchronize
// (the first statement of every kernel launched this way) for its results.
template <class T>
void launch_pdl(PairFn<T> fn, int grid, int block, std::size_t smem, cudaStream_t st,
                const SartK<T>& k, int it, const void* hot = nullptr, std::size_t hot_bytes = 0) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (hot && hot_bytes) {  // keep the gathered vector L2-resident (persisting window)
    attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[na].val.accessPolicyWindow.base_ptr = const_cast<void*>(hot);
    attr[na].val.accessPolicyWindow.num_bytes = hot_bytes;
    attr[na].val.accessPolicyWindow.hitRatio = 1.0f;
    attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  SSB_CUDA(cudaLaunchKernelEx(&cfg, fn, k, it));
}

template <class T>
void launch_pair(Plan& P, const SartK<T>& k, int it, bool fwd) {
  int smem = 0;
  const PairFn<T> fn = pair_kernel<T>(P, fwd, &smem);
  const void* hot = nullptr;
  std::size_t hb = 0;
  if (P.l2_window) {
    hot = fwd ? P.xx.get() : P.ww.get();
    hb = 2 * (fwd ? P.cols[0] : P.rows[0]) * sizeof(T);
  }
  launch_pdl<T>(fn, fwd ? P.fwd_blocks : P.back_blocks, kThreads, smem, P.ctx->stream, k, it,
                hot, hb);
}

// multi-RHS kernel: V consecutive slices per lane (vector loads; S % V == 0),
// Q passes of 32*V slices
template <class T>
using MultiFwdFn = void (*)(SartK<T>, int, int);

template <class T>
PairFn<T> multi_back_kernel(const Plan& P) {
  const int S = P.nrhs;
  const int v = S % 4 == 0 && S >= 128 ? 4 : (S % 2 == 0 && S >= 64 ? 2 : 1);
  const int q = (S + 32 * v - 1) / (32 * v);
#define SSB_MULTI(V, Q) \
  if (v == V && q <= Q) return sart_back_multi_kernel<T, V, Q>;
  SSB_MULTI(1, 1) SSB_MULTI(1, 2) SSB_MULTI(2, 1) SSB_MULTI(2, 2) SSB_MULTI(4, 1) SSB_MULTI(4, 2)
#undef SSB_MULTI
  fail("plan: unsupported multi-RHS shape");
  return nullptr;
}

template <class T>
MultiFwdFn<T> multi_fwd_kernel(const Plan& P) {
  const int S = P.nrhs;
  const int v = S % 4 == 0 && S >= 128 ? 4 : (S % 2 == 0 && S >= 64 ? 2 : 1);
  const int q = (S + 32 * v - 1) / (32 * v);
#define SSB_MULTI(V, Q) \
  if (v == V && q <= Q) return sart_fwd_multi_kernel<T, V, Q>;
  SSB_MULTI(1, 1) SSB_MULTI(1, 2) SSB_MULTI(2, 1) SSB_MULTI(2, 2) SSB_MULTI(4, 1) SSB_MULTI(4, 2)
#undef SSB_MULTI
  fail("plan: unsupported multi-RHS shape");
  return nullptr;
}

// Multi-RHS K1 over column bands (X of all slices larger than a share of L2):
// one pass per band so each pass's gathered X records stay L2-resident; the
// partial dot products accumulate in w (band 1 stores, 2 adds, the last pass
// adds and forms r). Rows' band boundaries are positions inside the CSR rows
// (columns ascending), so the matrix is still streamed once per iteration.
template <class T>
void launch_multi_fwd(Plan& P, const SartK<T>& k, int it) {
  const std::size_t sh = sizeof(double) * kWarps * P.nsys * P.nrhs;
  const MultiFwdFn<T> fn = multi_fwd_kernel<T>(P);
  if (P.nband <= 1) {
    fn<<<P.fwd_blocks, kThreads, sh, P.ctx->stream>>>(k, it, 0);
    return;
  }
  for (int b = 0; b < P.nband; ++b) {
    SartK<T> kb = k;
    for (int s = 0; s < P.nsys; ++s) {
      const int* bp = P.band_ptr[s].get();  // [nband + 1][rows]
      kb.s[s].bb = bp + static_cast<std::size_t>(b) * P.rows[s];
      kb.s[s].be = bp + static_cast<std::size_t>(b + 1) * P.rows[s];
    }
    if (P.nsys == 1) kb.s[1] = kb.s[0];
    const int band = b == 0 ? 1 : (b == P.nband - 1 ? 3 : 2);
    fn<<<P.fwd_blocks, kThreads, sh, P.ctx->stream>>>(kb, it, band);
    if (b + 1 < P.nband) P.ctx->check_launch("sart_fwd_multi_kernel(band)");
  }
}

template <class T>
BlockK<T> block_args(const Plan& P, bool fwd) {
  BlockK<T> b{};
  b.ptr = fwd ? P.bptr_f.get() : P.bptr_b.get();
  b.idx = fwd ? P.bidx_f.get() : P.bidx_b.get();
  b.val = reinterpret_cast<const T*>(fwd ? P.bval_f.get() : P.bval_b.get());
  b.nblk = fwd ? P.nblk_f : P.nblk_b;
  return b;
}

template <class T>
using BlockFn = void (*)(SartK<T>, BlockK<T>, int);

template <class T>
BlockFn<T> block_kernel(const Plan& P, bool fwd) {
  const int S = P.nrhs;
  const int v = S % 4 == 0 && S >= 128 ? 4 : (S % 2 == 0 && S >= 64 ? 2 : 1);
  const int e = fwd ? P.block_e_f : P.block_e_b;
#define SSB_BLK(V, E) \
  if (v == V && e == E) return fwd ? sart_fwd_block_kernel<T, V, E> : sart_back_block_kernel<T, V, E>;
  SSB_BLK(4, 2) SSB_BLK(4, 4) SSB_BLK(2, 2) SSB_BLK(2, 4) SSB_BLK(1, 2) SSB_BLK(1, 4)
#undef SSB_BLK
  fail("plan: unsupported block-merged kernel shape");
  return nullptr;
}

template <class T>
void launch_block(Plan& P, const SartK<T>& k, int it, bool fwd) {
  const std::size_t sh = fwd ? sizeof(double) * kWarps * 2 * P.nrhs : 0;
  block_kernel<T>(P, fwd)<<<fwd ? P.fwd_blocks : P.back_blocks, kThreads, sh, P.ctx->stream>>>(
      k, block_args<T>(P, fwd), it);
}

template <class T>
StageK<T> stage_args(const Plan& P, bool fwd) {
  const Plan::StageBufs& b = P.stg[fwd ? 0 : 1];
  StageK<T> sk{};
  sk.bptr = b.bptr.get();
  sk.buni = b.buni.get();
  sk.bch = b.bch.get();
  sk.cofs = b.cofs.get();
  sk.ent = b.ent.get();
  sk.nblk = b.nblk;
  sk.slot_bytes = b.slot;
  return sk;
}

template <class T>
using StageFn = void (*)(SartK<T>, StageK<T>, int);

template <class T>
StageFn<T> stage_kernel(int nrhs, bool fwd) {
  switch (nrhs) {
    case 32: return fwd ? sart_stage_kernel<T, 1, true> : sart_stage_kernel<T, 1, false>;
    case 64: return fwd ? sart_stage_kernel<T, 2, true> : sart_stage_kernel<T, 2, false>;
    case 128: return fwd ? sart_stage_kernel<T, 4, true> : sart_stage_kernel<T, 4, false>;
    default: return nullptr;
  }
}

template <class T>
void launch_stage(Plan& P, const SartK<T>& k, int it, bool fwd) {
  const Plan::StageBufs& b = P.stg[fwd ? 0 : 1];
  stage_kernel<T>(P.nrhs, fwd)<<<b.blocks, kStageThreads, b.smem, P.ctx->stream>>>(
      k, stage_args<T>(P, fwd), it);
}

template <class T>
void launch_fwd(Plan& P, const SartK<T>& k, int it) {
  if (P.stg[0].on) {
    launch_stage<T>(P, k, it, true);
    return;
  }
  if (P.blocked_f) {
    launch_block<T>(P, k, it, true);
    return;
  }
  if (P.paired) {
    launch_pair<T>(P, k, it, true);
    return;
  }
  if (single_tiled(P)) {
    launch_pdl<T>(single_kernel<T>(P, true), P.fwd_blocks, kThreads, 0, P.ctx->stream, k, it);
    return;
  }
  if (P.nrhs > 1) {
    launch_multi_fwd<T>(P, k, it);
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
  if (P.stg[1].on) {
    launch_stage<T>(P, k, it, false);
    return;
  }
  if (P.blocked_b) {
    launch_block<T>(P, k, it, false);
    return;
  }
  if (P.paired) {
    launch_pair<T>(P, k, it, false);
    return;
  }
  if (single_tiled(P)) {
    launch_pdl<T>(single_kernel<T>(P, false), P.back_blocks, kThreads, 0, P.ctx->stream, k, it);
    return;
  }
  if (P.nrhs > 1) {
    multi_back_kernel<T>(P)<<<P.back_blocks, kThreads, 0, P.ctx->stream>>>(k, it);
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
    e = fwd ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, multi_fwd_kernel<T>(P),
                                                            kThreads, sh)
            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, multi_back_kernel<T>(P),
                                                            kThreads, sh);
  } else {
    e = fwd ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sart_fwd_kernel<T, 32, 4>,
                                                            kThreads, 0)
            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sart_back_kernel<T, 8, 4>,
                                                            kThreads, 0);
  }
  SSB_CUDA(e);
  return std::max(1, per_sm) * P.ctx->sm_count;
}

template <class T>
int occupancy_pair_t(Plan& P, bool fwd) {
  int smem = 0, per_sm = 0;
  const PairFn<T> fn = pair_kernel<T>(P, fwd, &smem);
  if (smem > 0) {  // static + dynamic may pass 48 KB
    SSB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem));
  return std::max(1, per_sm) * P.ctx->sm_count;
}

// resident-CTA grids of a single-system tiled plan (never more blocks than groups)
template <class T>
void size_single_grid_t(Plan& P) {
  for (int f = 0; f < 2; ++f) {
    const bool fwd = f == 0;
    int per_sm = 0;
    SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, single_kernel<T>(P, fwd),
                                                           kThreads, 0));
    const long long groups = static_cast<long long>(fwd ? P.rows[0] : P.cols[0]) *
                             (fwd ? P.vs_fwd : P.vs_back);
    const int b = static_cast<int>(std::max<long long>(1, std::min<long long>(
        std::max(1, per_sm) * static_cast<long long>(P.ctx->sm_count),
        (groups + kThreads - 1) / kThreads)));
    (fwd ? P.fwd_blocks : P.back_blocks) = b;
  }
}

void size_single_grid(Plan& P) {
  if (P.dtype == SS_F32) size_single_grid_t<float>(P);
  else size_single_grid_t<double>(P);
  if (static_cast<std::size_t>(P.fwd_blocks) * P.nsys * P.nrhs > P.partial.size()) {
    P.partial.alloc(static_cast<std::size_t>(P.fwd_blocks) * P.nsys * P.nrhs);
  }
}

int occupancy_pair_blocks(Plan& P, bool fwd) {
  return P.dtype == SS_F32 ? occupancy_pair_t<float>(P, fwd) : occupancy_pair_t<double>(P, fwd);
}

template <class T>
XK<T> make_xargs(const Plan& P) {
  const PeerExchange& X = *P.px;
  XK<T> x{};
  x.peers = X.peers.get();
  x.G = X.G;
  x.me = X.me;
  x.cols = X.cols;
  x.own = X.own;
  x.rgrid = X.rgrid;
  x.off_recv = X.off_recv;
  x.off_x = X.off_x;
  x.off_r2 = X.off_r2;
  x.off_done = X.off_done;
  x.off_xready = X.off_xready;
  x.off_dflag = X.off_dflag;
  x.local = X.local.get();
  x.inline_signal = X.emulated ? 0 : 1;
  return x;
}

template <class T>
using XchgFn = void (*)(SartK<T>, XK<T>, int);

template <class T>
XchgFn<T> xchg_kernel(const Plan& P, bool fwd) {
  const int vs = fwd ? P.vs_fwd : P.vs_back;
  const int uf = fwd ? P.uf_fwd : P.uf_back;
  const bool u16 = fwd ? P.c16f : P.c16b;
#define SSB_X(V, U)                                                                           \
  if (vs == V && uf == U) {                                                                   \
    if (u16) return fwd ? sart_fwd_xchg_kernel<T, V, U, true> : sart_back_xchg_kernel<T, V, U, true>; \
    return fwd ? sart_fwd_xchg_kernel<T, V, U, false> : sart_back_xchg_kernel<T, V, U, false>; \
  }
  SSB_X(4, 2) SSB_X(8, 2) SSB_X(16, 2) SSB_X(32, 2)
  SSB_X(4, 4) SSB_X(8, 4) SSB_X(16, 4) SSB_X(32, 4)
#undef SSB_X
  fail("plan: unsupported peer-exchange kernel shape");
  return nullptr;
}

// phase: K1x (fwd), else K2x then (with_reduce) the owner-side reduce; an
// emulated group issues every rank's K2x before any rank's reduce
template <class T>
void launch_xchg(Plan& P, const SartK<T>& k, int it, bool fwd, bool with_reduce = true,
                 bool with_back = true) {
  const XK<T> x = make_xargs<T>(P);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(fwd ? P.fwd_blocks : P.back_blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = P.ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  if (!with_back) {
    cfg.gridDim = dim3(P.px->rgrid);
    SSB_CUDA(cudaLaunchKernelEx(&cfg, xchg_reduce_kernel<T>, k, x, it));
    P.ctx->check_launch("xchg_reduce_kernel");
    return;
  }
  SSB_CUDA(cudaLaunchKernelEx(&cfg, xchg_kernel<T>(P, fwd), k, x, it));
  P.ctx->check_launch(fwd ? "sart_fwd_xchg_kernel" : "sart_back_xchg_kernel");
  if (fwd || !with_reduce) return;
  cfg.gridDim = dim3(P.px->rgrid);  // owner-side reduce + push of x
  SSB_CUDA(cudaLaunchKernelEx(&cfg, xchg_reduce_kernel<T>, k, x, it));
  P.ctx->check_launch("xchg_reduce_kernel");
}

template <class T>
XchgFn<T> xchg_pair_kernel(const Plan& P, bool fwd) {
  const int vs = fwd ? P.vs_fwd : P.vs_back;
  const int uf = fwd ? P.uf_fwd : P.uf_back;
  const int tl = P.layout_mode(fwd);
#define SSB_XP(V, U)                                                                          \
  if (vs == V && uf == U) {                                                                   \
    if (tl == 4) return fwd ? sart_fwd_xchg_pair_kernel<T, V, U, 4> : sart_back_xchg_pair_kernel<T, V, U, 4>; \
    if (tl == 5) return fwd ? sart_fwd_xchg_pair_kernel<T, V, U, 5> : sart_back_xchg_pair_kernel<T, V, U, 5>; \
    if (tl == 6) return fwd ? sart_fwd_xchg_pair_kernel<T, V, U, 6> : sart_back_xchg_pair_kernel<T, V, U, 6>; \
  }
  SSB_XP(4, 2) SSB_XP(8, 2) SSB_XP(16, 2) SSB_XP(32, 2)
  SSB_XP(4, 4) SSB_XP(8, 4) SSB_XP(16, 4) SSB_XP(32, 4)
#undef SSB_XP
  fail("plan: unsupported paired peer-exchange kernel shape");
  return nullptr;
}

// paired variant of launch_xchg (same phases)
template <class T>
void launch_xchg_pair(Plan& P, const SartK<T>& k, int it, bool fwd, bool with_reduce = true,
                      bool with_back = true) {
  const XK<T> x = make_xargs<T>(P);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(fwd ? P.fwd_blocks : P.back_blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = P.ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  if (!with_back) {
    cfg.gridDim = dim3(P.px->rgrid);
    SSB_CUDA(cudaLaunchKernelEx(&cfg, xchg_reduce_pair_kernel<T>, k, x, it));
    P.ctx->check_launch("xchg_reduce_pair_kernel");
    return;
  }
  SSB_CUDA(cudaLaunchKernelEx(&cfg, xchg_pair_kernel<T>(P, fwd), k, x, it));
  P.ctx->check_launch(fwd ? "sart_fwd_xchg_pair_kernel" : "sart_back_xchg_pair_kernel");
  if (fwd || !with_reduce) return;
  cfg.gridDim = dim3(P.px->rgrid);
  SSB_CUDA(cudaLaunchKernelEx(&cfg, xchg_reduce_pair_kernel<T>, k, x, it));
  P.ctx->check_launch("xchg_reduce_pair_kernel");
}

template <class T>
void launch_announce(Plan& P, int it, int kind) {
  if (P.paired) {
    xchg_announce_pair_kernel<T><<<1, 32, 0, P.ctx->stream>>>(make_args<T>(P), make_xargs<T>(P),
                                                              it, kind);
    P.ctx->check_launch("xchg_announce_pair_kernel");
    return;
  }
  xchg_announce_kernel<T><<<1, 32, 0, P.ctx->stream>>>(make_args<T>(P), make_xargs<T>(P), it,
                                                       kind);
  P.ctx->check_launch("xchg_announce_kernel");
}

template <class T>
void launch_xchg_final(Plan& P) {
  const SartK<T> k = make_args<T>(P);
  if (P.paired) {
    xchg_final_pair_kernel<T><<<1, 32, 0, P.ctx->stream>>>(k, make_xargs<T>(P));
    P.ctx->check_launch("xchg_final_pair_kernel");
    return;
  }
  xchg_final_kernel<T><<<1, 32, 0, P.ctx->stream>>>(k, make_xargs<T>(P));
  P.ctx->check_launch("xchg_final_kernel");
}

template <class T>
using PersistFn = void (*)(SartK<T>, int, int, unsigned*);

// the persistent kernel of a paired plan's shape, or nullptr (not instantiated)
template <class T>
PersistFn<T> persistent_kernel(const Plan& P) {
  const bool u16 = P.c16f && P.c16b;
  if (!(P.mir_f && P.mir_b) || !u16 || P.c16f != P.c16b || P.stream_cs) return nullptr;
#define SSB_PERSIST(F, B) \
  if (P.vs_fwd == F && P.vs_back == B) return sart_persistent_pair_kernel<T, F, B, 2, 4>;
  SSB_PERSIST(8, 4) SSB_PERSIST(8, 8) SSB_PERSIST(8, 16)
  SSB_PERSIST(16, 4) SSB_PERSIST(16, 8) SSB_PERSIST(16, 16)
  SSB_PERSIST(32, 4) SSB_PERSIST(32, 8) SSB_PERSIST(32, 16)
#undef SSB_PERSIST
  return nullptr;
}

template <class T>
using ClusterFn = void (*)(SartK<T>, int, int);

// the cluster-persistent kernel of a paired plan's shape, or nullptr
template <class T>
ClusterFn<T> cluster_kernel(int vsf, int vsb) {
#define SSB_CLUSTER(F, B) \
  if (vsf == F && vsb == B) return sart_cluster_pair_kernel<T, F, B, 2>;
  SSB_CLUSTER(8, 4) SSB_CLUSTER(8, 8) SSB_CLUSTER(8, 16)
  SSB_CLUSTER(16, 4) SSB_CLUSTER(16, 8) SSB_CLUSTER(16, 16)
  SSB_CLUSTER(32, 4) SSB_CLUSTER(32, 8) SSB_CLUSTER(32, 16)
#undef SSB_CLUSTER
  return nullptr;
}

// largest cluster (16, else 8) of 1024-thread CTAs with `smem` bytes of
// dynamic shared memory this device can co-schedule (0: none)
template <class T>
int cluster_size_for(ClusterFn<T> fn, int smem) {
  if (!fn) return 0;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  for (int c = kMaxCluster; c >= 8; c /= 2) {
    if (c > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                     cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) == cudaSuccess && n >= 1) return c;
    cudaGetLastError();
  }
  return 0;
}

template <class T>
void launch_cluster(Plan& P, const SartK<T>& k, int first, int count) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.ccluster);
  cfg.blockDim = dim3(kClusterThreads);
  cfg.dynamicSmemBytes = P.csmem;
  cfg.stream = P.ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P.ccluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SSB_CUDA(cudaLaunchKernelEx(&cfg, cluster_kernel<T>(P.vs_fwd, P.vs_back), k, first, count));
  P.ctx->check_launch("sart_cluster_pair_kernel");
}

// Cluster-persistent loop of a small paired plan (see sart_cluster_pair_kernel):
// every CTA's staged share must fit kClusterSmemMax and one pass of the
// cluster must cover every row and column; otherwise the plan keeps ccluster 0.
template <class T>
void setup_cluster(Plan& P) {
  const int c0 = P.ccluster;
  P.ccluster = 0;
  ClusterFn<T> fn = cluster_kernel<T>(P.vs_fwd, P.vs_back);
  if (!fn || c0 <= 0 || !P.mir_f || !P.mir_b || !P.c16f || !P.c16b || P.stream_cs) return;
  const int nr = static_cast<int>(P.rows[0]), nc = static_cast<int>(P.cols[0]);
  std::vector<int> tpf(nr + 1), tff(nr + 1), epf(nr + 1, 0), tpb(nc + 1), tfb(nc + 1),
      epb(nc + 1, 0);
  P.ctx->copy(tpf.data(), P.tptr_f.get(), (nr + 1) * sizeof(int));
  P.ctx->copy(tff.data(), P.tfirst_f.get(), (nr + 1) * sizeof(int));
  P.ctx->copy(tpb.data(), P.tptr_b.get(), (nc + 1) * sizeof(int));
  P.ctx->copy(tfb.data(), P.tfirst_b.get(), (nc + 1) * sizeof(int));
  if (P.eptr_f.get()) P.ctx->copy(epf.data(), P.eptr_f.get(), (nr + 1) * sizeof(int));
  if (P.eptr_b.get()) P.ctx->copy(epb.data(), P.eptr_b.get(), (nc + 1) * sizeof(int));
  const auto blk = [](const std::vector<int>& tp, const std::vector<int>& tf,
                      const std::vector<int>& ep, int n, int per, int b) {
    CBlock c;
    c.v0 = std::min(b * per, n);
    c.v1 = std::min(c.v0 + per, n);
    c.e0 = tp[c.v0];
    c.e1 = tp[c.v1];
    c.t0 = tf[c.v0];
    c.t1 = tf[c.v1];
    c.x0 = ep[c.v0];
    c.x1 = ep[c.v1];
    return c;
  };
  for (int c = c0; c >= 8; c /= 2) {
    const int pf = (nr + c - 1) / c, pb = (nc + c - 1) / c;  // the kernel's blocks
    if (pf > kClusterThreads / P.vs_fwd || pb > kClusterThreads / P.vs_back) break;
    long long need = 0;
    for (int b = 0; b < c; ++b) {
      need = std::max(need, cstage_bytes<T>(blk(tpf, tff, epf, nr, pf, b), P.hs_f, 4) +
                                cstage_bytes<T>(blk(tpb, tfb, epb, nc, pb, b), P.hs_b, 2));
    }
    need += (2ll * sizeof(T) * (nr + nc) + 15) & ~15ll;  // x / w replicas
    if (need > kClusterSmemMax) break;
    const int smem = static_cast<int>(need);
    if (cluster_size_for<T>(fn, smem) >= c) {
      P.ccluster = c;
      P.csmem = smem;
      if (static_cast<std::size_t>(c) * 2 > P.partial.size()) P.partial.alloc(2 * c);
      return;
    }
  }
}

// the stream-resident kernel of a paired plan's shape, or nullptr
template <class T>
PersistFn<T> resident_kernel(int vsf, int vsb, bool sb) {
#define SSB_RESIDENT(F, B)                                                    \
  if (vsf == F && vsb == B) {                                                 \
    return sb ? sart_resident_pair_kernel<T, F, B, 2, true>                   \
              : sart_resident_pair_kernel<T, F, B, 2, false>;                 \
  }
  SSB_RESIDENT(8, 4) SSB_RESIDENT(8, 8) SSB_RESIDENT(8, 16)
  SSB_RESIDENT(16, 4) SSB_RESIDENT(16, 8) SSB_RESIDENT(16, 16)
  SSB_RESIDENT(32, 4) SSB_RESIDENT(32, 8) SSB_RESIDENT(32, 16)
#undef SSB_RESIDENT
  return nullptr;
}

// Stream-resident persistent loop of a paired plan (see
// sart_resident_pair_kernel): one CTA per SM, every CTA's share of both
// streams must fit kResSmemMax and the grid must be co-resident; otherwise the
// plan keeps resident = false.
template <class T>
void setup_resident(Plan& P) {
  P.resident = false;
  if (!resident_kernel<T>(P.vs_fwd, P.vs_back, true) || !P.mir_f || !P.mir_b || !P.c16f ||
      !P.c16b || P.stream_cs) {
    return;
  }
  const int nr = static_cast<int>(P.rows[0]), nc = static_cast<int>(P.cols[0]);
  std::vector<int> tpf(nr + 1), tff(nr + 1), epf(nr + 1, 0), tpb(nc + 1), tfb(nc + 1),
      epb(nc + 1, 0);
  P.ctx->copy(tpf.data(), P.tptr_f.get(), (nr + 1) * sizeof(int));
  P.ctx->copy(tff.data(), P.tfirst_f.get(), (nr + 1) * sizeof(int));
  P.ctx->copy(tpb.data(), P.tptr_b.get(), (nc + 1) * sizeof(int));
  P.ctx->copy(tfb.data(), P.tfirst_b.get(), (nc + 1) * sizeof(int));
  if (P.eptr_f.get()) P.ctx->copy(epf.data(), P.eptr_f.get(), (nr + 1) * sizeof(int));
  if (P.eptr_b.get()) P.ctx->copy(epb.data(), P.eptr_b.get(), (nc + 1) * sizeof(int));
  const auto blk = [](const std::vector<int>& tp, const std::vector<int>& tf,
                      const std::vector<int>& ep, int n, int per, int b) {
    CBlock c;
    c.v0 = std::min(b * per, n);
    c.v1 = std::min(c.v0 + per, n);
    c.e0 = tp[c.v0];
    c.e1 = tp[c.v1];
    c.t0 = tf[c.v0];
    c.t1 = tf[c.v1];
    c.x0 = ep[c.v0];
    c.x1 = ep[c.v1];
    return c;
  };
  const int g = P.ctx->sm_count;
  const int pf = (nr + g - 1) / g, pb = (nc + g - 1) / g;
  long long need = 0, need_f = 0;
  for (int b = 0; b < g; ++b) {
    const long long f = cstage_bytes<T>(blk(tpf, tff, epf, nr, pf, b), P.hs_f, 4);
    need_f = std::max(need_f, f);
    need = std::max(need, f + cstage_bytes<T>(blk(tpb, tfb, epb, nc, pb, b), P.hs_b, 2));
  }
  // both streams resident, else K1's only (config 2 fp64: K2 streams from L2)
  P.res_back = need <= kResSmemMax;
  if (!P.res_back) need = need_f;
  if (need > kResSmemMax) return;
  PersistFn<T> fn = resident_kernel<T>(P.vs_fwd, P.vs_back, P.res_back);
  const int smem = static_cast<int>(need);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
      cudaSuccess) {
    cudaGetLastError();
    return;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kResThreads, smem) !=
          cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return;
  }
  P.pgrid = g;
  P.csmem = smem;
  P.gbar.alloc(2);
  SSB_CUDA(cudaMemsetAsync(P.gbar.get(), 0, 2 * sizeof(unsigned), P.ctx->stream));
  if (static_cast<std::size_t>(g) * 2 > P.partial.size()) P.partial.alloc(2 * g);
  P.ctx->sync();
  P.resident = P.persistent = true;
}

template <class T>
void launch_resident(Plan& P, const SartK<T>& k, int first, int count) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.pgrid);
  cfg.blockDim = dim3(kResThreads);
  cfg.dynamicSmemBytes = P.csmem;
  cfg.stream = P.ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SSB_CUDA(cudaLaunchKernelEx(&cfg, resident_kernel<T>(P.vs_fwd, P.vs_back, P.res_back), k, first,
                              count, P.gbar.get()));
  P.ctx->check_launch("sart_resident_pair_kernel");
#ifdef SSB_RES_TIMING
  {
    cudaStreamCaptureStatus cs;
    cudaStreamIsCapturing(P.ctx->stream, &cs);
    if (cs == cudaStreamCaptureStatusNone) {
      unsigned long long h[8];
      cudaStreamSynchronize(P.ctx->stream);
      cudaMemcpyFromSymbol(h, res_ticks, sizeof h);
      std::fprintf(stderr, "[res ticks] head %llu K1 %llu sync1 %llu norm %llu K2 %llu sync2 %llu (count %d)\n",
                   h[0], h[1], h[2], h[3], h[4], h[5], count);
      unsigned long long z[8] = {};
      cudaMemcpyToSymbol(res_ticks, z, sizeof z);
    }
  }
#endif
}

// one cooperative launch runs passes [first, first + count) (all CTAs resident)
template <class T>
void launch_persistent(Plan& P, const SartK<T>& k, int first, int count) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.pgrid);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = P.ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SSB_CUDA(cudaLaunchKernelEx(&cfg, persistent_kernel<T>(P), k, first, count, P.gbar.get()));
  P.ctx->check_launch("sart_persistent_pair_kernel");
}

template <class T>
void do_iterations(Plan& P, int first, int count) {
  const SartK<T> k = make_args<T>(P);
  if (P.cluster) {
    launch_cluster<T>(P, k, first, count);
    return;
  }
  if (P.resident) {
    launch_resident<T>(P, k, first, count);
    return;
  }
  if (P.persistent) {
    launch_persistent<T>(P, k, first, count);
    return;
  }
  for (int it = first; it < first + count; ++it) {
    if (P.px && P.paired) {  // the row-sharded pair: K1x, K2x + reduce, both systems
      launch_xchg_pair<T>(P, k, it, true);
      launch_xchg_pair<T>(P, k, it, false);
      continue;
    }
    if (P.px) {  // K1x over local rows, K2x with the fused peer exchange
      launch_xchg<T>(P, k, it, true);
      launch_xchg<T>(P, k, it, false);
      continue;
    }
    if (P.sharded) {
      // K1 over local rows, fixed-order ||r_g||^2, K2 partial back-projection,
      // all-reduce [bp | r2], identical update on every rank.
      T* bp = reinterpret_cast<T*>(P.bp.get());
      const long long cols = P.cols[0];
      double* r2 = sharded_r2_slot(P);
      launch_fwd<T>(P, k, it);
      P.ctx->check_launch("sart_fwd(sharded)");
      sharded_r2_kernel<<<1, kThreads, 0, P.ctx->stream>>>(P.partial.get(), P.fwd_blocks, r2);
      P.ctx->check_launch("sharded_r2_kernel");
      launch_back<T>(P, k, it);
      P.ctx->check_launch("sart_back(sharded)");
      // [bp] in the plan dtype and ||r_g||^2 in fp64, fused into one NCCL launch
      nccl_check(nccl().GroupStart(), "ncclGroupStart");
      nccl_check(nccl().AllReduce(bp, bp, static_cast<std::size_t>(cols),
                                  sizeof(T) == 4 ? ncclFloat32 : ncclFloat64, ncclSum,
                                  static_cast<ncclComm_t>(P.ctx->comm), P.ctx->stream),
                 "ncclAllReduce");
      nccl_check(nccl().AllReduce(r2, r2, 1, ncclFloat64, ncclSum,
                                  static_cast<ncclComm_t>(P.ctx->comm), P.ctx->stream),
                 "ncclAllReduce(r2)");
      nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
      sart_sharded_update_kernel<T><<<P.back_blocks, kThreads, 0, P.ctx->stream>>>(
          reinterpret_cast<T*>(P.x[0].get()), bp, r2,
          reinterpret_cast<const T*>(P.cinv[0].get()), cols, P.pnorm.get(), P.opts.tol,
          P.opts.relaxation, P.history.get(), P.state.get(), it);
      P.ctx->check_launch("sart_sharded_update_kernel");
      sharded_stop_kernel<<<1, 1, 0, P.ctx->stream>>>(r2, P.pnorm.get(), P.opts.tol,
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
  delete px;
  delete own;
  delete own2;
  delete pair_own[0];
  delete pair_own[1];
}

void Plan::enqueue_reset() {
  for (int s = 0; s < nsys; ++s) {
    SSB_CUDA(cudaMemsetAsync(x[s].get(), 0, cols[s] * nrhs * tsize(), ctx->stream));
  }
  if (paired) SSB_CUDA(cudaMemsetAsync(xx.get(), 0, 2 * cols[0] * tsize(), ctx->stream));
  if (px) {  // own replica and divergence flag only: peers never touch them
    // before this rank's first arrival of the solve (see sart.cu peer exchange)
    char* r = static_cast<char*>(px->region);
    const std::size_t ns = paired ? 2 : 1;
    SSB_CUDA(cudaMemsetAsync(r + px->off_x, 0, cols[0] * tsize() * ns, ctx->stream));
    SSB_CUDA(cudaMemsetAsync(r + px->off_dflag, 0, ns * sizeof(int), ctx->stream));
    SSB_CUDA(cudaMemsetAsync(px->local.get() + 1, 0, sizeof(long long), ctx->stream));
    SSB_CUDA(cudaMemsetAsync(px->local.get() + 3, 0, sizeof(long long), ctx->stream));
  }
  SSB_CUDA(cudaMemsetAsync(state.get(), 0, state.size() * sizeof(int), ctx->stream));
  SSB_CUDA(cudaMemsetAsync(ticket.get(), 0, 2 * sizeof(unsigned), ctx->stream));
}

void Plan::enqueue_iterations(int first, int count) {
  if (dtype == SS_F32) do_iterations<float>(*this, first, count);
  else do_iterations<double>(*this, first, count);
}

void Plan::enqueue_epilogue() {
  if (px) {  // settle the last iteration, then the replica is the solution
    if (dtype == SS_F32) launch_xchg_final<float>(*this);
    else launch_xchg_final<double>(*this);
    if (paired) {  // interleaved replica -> xx -> x1, x2 (below)
      SSB_CUDA(cudaMemcpyAsync(xx.get(), static_cast<char*>(px->region) + px->off_x,
                               2 * cols[0] * tsize(), cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
      SSB_CUDA(cudaMemcpyAsync(x[0].get(), static_cast<char*>(px->region) + px->off_x,
                               cols[0] * tsize(), cudaMemcpyDeviceToDevice, ctx->stream));
      return;
    }
  }
  if (!paired) return;
  const int g = grid1(ctx, cols[0]);
  if (dtype == SS_F32) {
    deinterleave_kernel<float><<<g, 256, 0, ctx->stream>>>(
        reinterpret_cast<const float*>(xx.get()), reinterpret_cast<float*>(x[0].get()),
        reinterpret_cast<float*>(x[1].get()), cols[0]);
  } else {
    deinterleave_kernel<double><<<g, 256, 0, ctx->stream>>>(
        reinterpret_cast<const double*>(xx.get()), reinterpret_cast<double*>(x[0].get()),
        reinterpret_cast<double*>(x[1].get()), cols[0]);
  }
  ctx->check_launch("deinterleave_kernel");
}

// passes unrolled per WHILE-body execution (amortises the per-body scheduling)
constexpr int kPassesPerBody = 8;

void Plan::build_graph() {
  // NCCL calls stay out of the captured graph; a peer-exchange plan is captured
  // when the pass count is fixed (an emulated group launches rank by rank)
  if (graph || (sharded && !(px && !px->emulated && !(opts.tol > 0.0)))) return;
  if (!(opts.tol > 0.0) || persistent) {
    // fixed iteration count (tol = 0 can never stop early): every pass
    // unrolled into the graph, the cheapest replay (a WHILE node's per-pass
    // scheduling costs ~5% on config 3)
    cudaGraph_t g = nullptr;
    SSB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    const std::int64_t before = ctx->launches;
    try {
      enqueue_reset();
      enqueue_iterations(0, opts.max_iters);
      enqueue_epilogue();
    } catch (...) {
      cudaStreamEndCapture(ctx->stream, &g);
      if (g) cudaGraphDestroy(g);
      ctx->launches = before;
      throw;
    }
    ctx->launches = before;  // captured, not launched
    SSB_CUDA(cudaStreamEndCapture(ctx->stream, &g));
    SSB_CUDA(cudaGraphInstantiate(&graph, g, 0));
    cudaGraphDestroy(g);
    return;
  }
  // tol > 0: reset nodes, then a WHILE node whose body is one pass (K1 + K2) and whose
  // condition K1's last block sets, then the epilogue: the loop stops on the
  // device at the reference's stop test (tol > 0) or after max_iters passes
  cudaGraph_t g = nullptr;
  SSB_CUDA(cudaGraphCreate(&g, 0));
  const std::int64_t before = ctx->launches;
  cudaStreamCaptureStatus cs;
  try {
    SSB_CUDA(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault));
    SSB_CUDA(cudaStreamBeginCaptureToGraph(ctx->stream, g, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    enqueue_reset();
    SSB_CUDA(cudaMemsetAsync(iter_dev.get(), 0, 2 * sizeof(int), ctx->stream));
    const cudaGraphNode_t* deps = nullptr;
    std::size_t nd = 0;
    SSB_CUDA(cudaStreamGetCaptureInfo(ctx->stream, &cs, nullptr, nullptr, &deps, &nd));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    SSB_CUDA(cudaGraphAddNode(&cnode, g, deps, nd, &cp));
    SSB_CUDA(cudaStreamUpdateCaptureDependencies(ctx->stream, &cnode, 1,
                                                 cudaStreamSetCaptureDependencies));
    enqueue_epilogue();
    SSB_CUDA(cudaStreamEndCapture(ctx->stream, &g));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    SSB_CUDA(cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    while_capture = true;
    enqueue_iterations(0, std::min(opts.max_iters, kPassesPerBody));
    while_capture = false;
    SSB_CUDA(cudaStreamEndCapture(ctx->stream, &body));
    SSB_CUDA(cudaGraphInstantiate(&graph, g, 0));
  } catch (...) {
    while_capture = false;
    if (cudaStreamIsCapturing(ctx->stream, &cs) == cudaSuccess &&
        cs != cudaStreamCaptureStatusNone) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(ctx->stream, &junk);
      if (junk && junk != g) cudaGraphDestroy(junk);
    }
    cudaGraphDestroy(g);
    ctx->launches = before;
    throw;
  }
  ctx->launches = before;  // captured, not launched
  cudaGraphDestroy(g);
}

void Plan::launch() {
  if (px && px->emulated) fail("plan: an emulated exchange rank runs through ss_plan_group_run");
  group_ms = -1.0f;
  SSB_CUDA(cudaEventRecord(ev0, ctx->stream));
  if (graph) {
    SSB_CUDA(cudaGraphLaunch(graph, ctx->stream));
    ctx->launches += persistent ? 2
                                : static_cast<std::int64_t>(px ? 3 : 1 + nband) * opts.max_iters +
                                      (paired || px ? 1 : 0);
  } else {
    enqueue_reset();
    enqueue_iterations(0, opts.max_iters);
    enqueue_epilogue();
  }
  SSB_CUDA(cudaEventRecord(ev1, ctx->stream));
  launched = true;
}

void Plan::finish(ss_solve_report* rep) {
  if (!launched) fail("plan: finish without launch");
  SSB_CUDA(cudaEventSynchronize(ev1));
  SSB_CUDA(cudaEventElapsedTime(&last_ms, ev0, ev1));
  if (group_ms >= 0.0f) last_ms = group_ms;  // emulated group: one clock for all ranks
  std::vector<int> st(state.size());
  ctx->copy(st.data(), state.get(), st.size() * sizeof(int));
  if (px) {
    long long loc[3];
    ctx->copy(loc, px->local.get(), sizeof loc);
    if (loc[2] != 0) {
      fail("sart_solve: peer exchange timed out (a rank of the sharded system stopped "
           "responding)", SS_ERR_CUDA);
    }
  }
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
  if (paired) {  // p of this system into slot `which` of the {p1, p2, rinv1, rinv2} records
    const int g = grid1(ctx, rows[which]);
    if (dtype == SS_F32) {
      interleave_kernel<float, float><<<g, 256, 0, ctx->stream>>>(
          reinterpret_cast<const float*>(p[which].get()), reinterpret_cast<float*>(pe.get()),
          rows[which], 4, which);
    } else {
      interleave_kernel<double, double><<<g, 256, 0, ctx->stream>>>(
          reinterpret_cast<const double*>(p[which].get()), reinterpret_cast<double*>(pe.get()),
          rows[which], 4, which);
    }
    ctx->check_launch("interleave_kernel<p>");
  }
  if (dtype == SS_F32) {
    pnorm_kernel<float><<<nrhs, kThreads, 0, ctx->stream>>>(
        reinterpret_cast<const float*>(p[which].get()), rows[which], nrhs, pn);
  } else {
    pnorm_kernel<double><<<nrhs, kThreads, 0, ctx->stream>>>(
        reinterpret_cast<const double*>(p[which].get()), rows[which], nrhs, pn);
  }
  ctx->check_launch("pnorm_kernel");
  if (sharded && px && px->emulated) {
    // emulated ranks: run_group combines the ranks' local ||p_g||
    ctx->copy(&pn_local[which], pn, sizeof(double));
  } else if (sharded) {
    // ||p||^2 = sum over ranks of the local ||p_g||^2
    square_kernel<<<1, 32, 0, ctx->stream>>>(pn, nrhs);
    ctx->check_launch("square_kernel");
    nccl_check(nccl().AllReduce(pn, pn, nrhs, ncclFloat64, ncclSum,
                                static_cast<ncclComm_t>(ctx->comm), ctx->stream),
               "ncclAllReduce");
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
  ctx->copy(st, state.get() + 4 * which * nrhs, sizeof st);
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
  ctx->copy(st, state.get() + 4 * q, sizeof st);
  const int n = st[0] ? st[1] + 1 : opts.max_iters;
  if (h) {
    ctx->copy(h, history.get() + static_cast<std::int64_t>(q) * (opts.max_iters + 1),
                        n * sizeof(double));
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
  if (px && px->emulated) fail("plan: an emulated exchange rank runs through ss_plan_group_run");
  cudaEvent_t e[3];
  for (auto& q : e) SSB_CUDA(cudaEventCreate(&q));
  float tf = 0.f, tb = 0.f;
  enqueue_reset();
  for (int it = 0; it < iters; ++it) {
    const int i = it % std::max(1, opts.max_iters);
    if (px && i == 0 && it > 0) {  // exchange epochs: whole solves only
      enqueue_epilogue();
      enqueue_reset();
    }
    SSB_CUDA(cudaEventRecord(e[0], ctx->stream));
    if (px) {  // K1x | K2x + reduce (the exchange's share lands in "back")
      if (dtype == SS_F32) {
        const SartK<float> k = make_args<float>(*this);
        launch_xchg<float>(*this, k, i, true);
        SSB_CUDA(cudaEventRecord(e[1], ctx->stream));
        launch_xchg<float>(*this, k, i, false);
      } else {
        const SartK<double> k = make_args<double>(*this);
        launch_xchg<double>(*this, k, i, true);
        SSB_CUDA(cudaEventRecord(e[1], ctx->stream));
        launch_xchg<double>(*this, k, i, false);
      }
      --ctx->launches;  // launch_xchg counted its own; check_launch below adds one
    } else if (dtype == SS_F32) {
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
  if (px) {
    enqueue_epilogue();
    ctx->sync();
  }
  for (auto& q : e) cudaEventDestroy(q);
  *fwd_ms = tf;
  *back_ms = tb;
}

// One SART kernel launched `reps` times back to back on the plan stream (the
// same launch configuration and programmatic dependent launch as inside the
// loop), CUDA events around the batch: the kernel's in-loop time per launch
// without per-launch events between launches. The iterate changes (K2) but
// the work per launch does not; the plan is reset afterwards.
void Plan::time_kernel(bool fwd, int reps, float* ms) {
  if (px) fail("plan: time_kernel is not available for peer-exchange plans");
  if (reps < 1) fail("plan: reps must be >= 1");
  enqueue_reset();
  SSB_CUDA(cudaEventRecord(ev0, ctx->stream));
  for (int r = 0; r < reps; ++r) {
    if (dtype == SS_F32) {
      const SartK<float> k = make_args<float>(*this);
      if (fwd) launch_fwd<float>(*this, k, 0);
      else launch_back<float>(*this, k, 0);
    } else {
      const SartK<double> k = make_args<double>(*this);
      if (fwd) launch_fwd<double>(*this, k, 0);
      else launch_back<double>(*this, k, 0);
    }
    ctx->check_launch(fwd ? "sart_fwd_kernel" : "sart_back_kernel");
  }
  SSB_CUDA(cudaEventRecord(ev1, ctx->stream));
  SSB_CUDA(cudaEventSynchronize(ev1));
  float t = 0.f;
  SSB_CUDA(cudaEventElapsedTime(&t, ev0, ev1));
  *ms = t / reps;
  enqueue_reset();
  ctx->sync();
  launched = false;
}

void Plan::kernel_bytes(std::int64_t* fwd, std::int64_t* back) const {
  // bytes of matrix data each kernel must stream per launch, in this plan's format
  const std::int64_t b = static_cast<std::int64_t>(tsize());
  std::int64_t f = 0, k = 0;
  if (paired) {
    const std::int64_t nf = tiled ? tnnz_f : a[0]->nnz, nb = tiled ? tnnz_b : a[0]->nnz;
    // uint16 offsets + int32 tile bases + padded and first-tile pointers, or int32 indices
    f = c16f ? nf * (2 + 2 * b) + 4 * ntile_f + 8 * (rows[0] + 1)
             : nf * (4 + 2 * b) + 4 * (rows[0] + 1);
    k = c16b ? nb * (2 + 2 * b) + 4 * ntile_b + 8 * (cols[0] + 1)
             : nb * (4 + 2 * b) + 4 * (cols[0] + 1);
    // mirror-coded: offsets + one value per entry + tile headers + exceptions
    if (mir_f) {
      f = nf * ((c16f ? 2 : 4) + b) + 4 * hs_f * ntile_f + 8 * (rows[0] + 1) +
          (nexc_f ? nexc_f * (4 + 2 * b) + 4 * (rows[0] + 1) : 0);
    }
    if (mir_b) {
      k = nb * ((c16b ? 2 : 4) + b) + 4 * hs_b * ntile_b + 8 * (cols[0] + 1) +
          (nexc_b ? nexc_b * (4 + 2 * b) + 4 * (cols[0] + 1) : 0);
    }
  } else if (blocked_f || blocked_b || stg[0].on || stg[1].on) {  // union indices + 2R values per entry + pointers
    for (int s2 = 0; s2 < nsys; ++s2) {
      f += a[s2]->nnz * (4 + b) + 4 * (rows[s2] + 1);
      k += a[s2]->nnz * (4 + b) + 4 * (cols[s2] + 1);
    }
    if (blocked_f) f = nu_f * (4 + 2 * kBlockR * b) + 4 * (nblk_f + 1);
    if (blocked_b) k = nu_b * (4 + 2 * kBlockR * b) + 4 * (nblk_b + 1);
    // staged: chunk records + unions (+ pointers); the operand moves via L2
    if (stg[0].on) f = stg[0].entb + 4 * stg[0].nu + 4 * (stg[0].nblk * nsys + 1);
    if (stg[1].on) k = stg[1].entb + 4 * stg[1].nu + 4 * (stg[1].nblk * nsys + 1);
  } else if (tiled && nsys == 1 && nrhs == 1) {
    f = c16f ? tnnz_f * (2 + b) + 4 * ntile_f + 8 * (rows[0] + 1)
             : tnnz_f * (4 + b) + 4 * (rows[0] + 1);
    k = c16b ? tnnz_b * (2 + b) + 4 * ntile_b + 8 * (cols[0] + 1)
             : tnnz_b * (4 + b) + 4 * (cols[0] + 1);
  } else {
    for (int s = 0; s < nsys; ++s) {
      f += a[s]->nnz * (4 + b) + 4 * (rows[s] + 1);
      k += a[s]->nnz * (4 + b) + 4 * (cols[s] + 1);
    }
  }
  if (fwd) *fwd = f;
  if (back) *back = k;
}

std::string Plan::describe() const {
  const char* t = dtype == SS_F32 ? "float" : "double";
  std::string fk, bk;
  if (!paired && tiled && nrhs == 1 && nsys == 1) {
    fk = "sart_fwd_tiled_kernel<" + std::string(t) + ", " + std::to_string(vs_fwd) + ", " +
         std::to_string(uf_fwd) + ", " + (c16f ? "true" : "false") + ">";
    bk = "sart_back_tiled_kernel<" + std::string(t) + ", " + std::to_string(vs_back) + ", " +
         std::to_string(uf_back) + ", " + (c16b ? "true" : "false") + ">";
  } else if (sharded || nrhs > 1 || !paired) {
    fk = stg[0].on ? "sart_stage_kernel<fwd>"
                   : (blocked_f ? "sart_fwd_block_kernel"
                                : (nrhs > 1 ? "sart_fwd_multi_kernel" : "sart_fwd_kernel"));
    bk = stg[1].on ? "sart_stage_kernel<back>"
                   : (blocked_b ? "sart_back_block_kernel"
                                : (nrhs > 1 ? "sart_back_multi_kernel" : "sart_back_kernel"));
  } else {
    fk = "sart_fwd_pair_kernel<" + std::string(t) + ", " + std::to_string(vs_fwd) + ", " +
         std::to_string(uf_fwd) + ", " + std::to_string(layout_mode(true)) + ">";
    bk = "sart_back_pair_kernel<" + std::string(t) + ", " + std::to_string(vs_back) + ", " +
         std::to_string(uf_back) + ", " + std::to_string(layout_mode(false)) + ">";
  }
  std::string pk = cluster ? "sart_cluster_pair_kernel<" + std::string(t) + ", " +
                                 std::to_string(vs_fwd) + ", " + std::to_string(vs_back) +
                                 ", 2>"
                   : resident ? "sart_resident_pair_kernel<" + std::string(t) + ", " +
                                    std::to_string(vs_fwd) + ", " + std::to_string(vs_back) +
                                    (res_back ? ", 2, true>" : ", 2, false>")
                   : persistent ? "sart_persistent_pair_kernel<" + std::string(t) + ", " +
                                      std::to_string(vs_fwd) + ", " + std::to_string(vs_back) +
                                      ", 2, 4>"
                                : "";
  std::int64_t f = 0, b = 0;
  kernel_bytes(&f, &b);
  char buf[2048];
  std::snprintf(buf, sizeof buf,
                "{\"layout\": \"%s\", \"dtype\": \"%s\", \"nsys\": %d, \"nrhs\": %d, "
                "\"vs_fwd\": %d, \"uf_fwd\": %d, \"vs_back\": %d, \"uf_back\": %d, "
                "\"fwd_blocks\": %d, \"back_blocks\": %d, \"threads\": %d, "
                "\"fwd_kernel\": \"%s\", \"back_kernel\": \"%s\", \"fwd_bytes\": %lld, "
                "\"back_bytes\": %lld, \"exceptions\": [%lld, %lld], \"graph\": %s, "
                "\"persistent_kernel\": \"%s\", \"persistent_grid\": %d, "
                "\"staged_union\": [%lld, %lld]}",
                sharded ? (tiled ? "row-sharded-tiled" : "row-sharded")
                        : (paired ? (tiled ? (mir_f || mir_b ? "paired-tiled-u16-mirror"
                                                                    : (c16f || c16b ? "paired-tiled-u16" : "paired-tiled"))
                                         : "paired")
                                  : (tiled ? "single-tiled" : "separate")),
                t, nsys, nrhs, vs_fwd, uf_fwd, vs_back, uf_back, fwd_blocks, back_blocks, kThreads,
                fk.c_str(), bk.c_str(), static_cast<long long>(f), static_cast<long long>(b),
                static_cast<long long>(nexc_f), static_cast<long long>(nexc_b),
                graph ? "true" : "false", pk.c_str(), cluster ? ccluster : (persistent ? pgrid : 0),
                static_cast<long long>(stg[0].on ? stg[0].nu : 0),
                static_cast<long long>(stg[1].on ? stg[1].nu : 0));
  return buf;
}

void Plan::stats(std::int64_t* mbytes, std::int64_t* vbytes, int* kernels) const {
  std::int64_t f = 0, k = 0, vb = 0;
  kernel_bytes(&f, &k);
  const std::int64_t b = static_cast<std::int64_t>(tsize());
  for (int s = 0; s < nsys; ++s) vb += (3 * rows[s] + 4 * cols[s]) * b * nrhs;
  if (mbytes) *mbytes = f + k;
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
  if (P.paired) {
    P.xx.alloc(2 * P.cols[0] * tb);
    P.ww.alloc(2 * P.rows[0] * tb);
    SSB_CUDA(cudaMemsetAsync(P.xx.get(), 0, 2 * P.cols[0] * tb, P.ctx->stream));
    SSB_CUDA(cudaMemsetAsync(P.ww.get(), 0, 2 * P.rows[0] * tb, P.ctx->stream));
  }
  const int nsr = P.nsys * P.nrhs;
  P.partial.alloc(static_cast<std::size_t>(nsr) * P.fwd_blocks);
  P.pnorm.alloc(nsr);
  SSB_CUDA(cudaMemsetAsync(P.pnorm.get(), 0, nsr * sizeof(double), P.ctx->stream));
  P.history.alloc(static_cast<std::size_t>(nsr) * (P.opts.max_iters + 1));
  P.state.alloc(4 * nsr);
  P.ticket.alloc(2);  // K1 last block, K2x last block
  P.iter_dev.alloc(2);  // WHILE loop: pass counter, loop-over flag
  SSB_CUDA(cudaMemsetAsync(P.state.get(), 0, 4 * nsr * sizeof(int), P.ctx->stream));
  SSB_CUDA(cudaMemsetAsync(P.ticket.get(), 0, 2 * sizeof(unsigned), P.ctx->stream));
  SSB_CUDA(cudaEventCreate(&P.ev0));
  SSB_CUDA(cudaEventCreate(&P.ev1));
}

// Normalisers (solvers.cpp:156-168): absolute row/column sums in fp64 in
// the reference order, inverses with the zero guard, cast to the plan type.
void normalisers(Plan& P, int s, double* max_row_sum) {
  Matrix* a = P.a[s];
  DBuf<double> rs(P.rows[s]), cs(P.cols[s]);
  if (a->ctx != P.ctx) P.ctx->sync();  // matrix on another context's stream
  abs_sums(*a, rs.get(), cs.get());
  if (a->ctx != P.ctx) a->ctx->sync();
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


namespace {
// padded pointer of one compressed direction; returns the padded entry count
std::int64_t tiled_ptr(Plan& P, const int* ptr, long long n, DBuf<int>& tptr) {
  DBuf<int> cnt(n + 1);
  tptr.alloc(n + 1);
  pad4_counts_kernel<<<grid1(P.ctx, n + 1), 256, 0, P.ctx->stream>>>(ptr, n, cnt.get());
  P.ctx->check_launch("pad4_counts_kernel");
  scan_counts(P.ctx, cnt.get(), tptr.get(), n);
  int total = 0;
  P.ctx->copy(&total, tptr.get() + n, sizeof(int));
  return total;
}

// Tiled streams (see seg_dot2t / seg_dot1) of a[0]'s pattern in both
// directions, with the values of w systems (2 = the folded pair interleaved):
// padded pointers, then per direction 16-bit offsets + tile bases when every
// tile spans < 65536 indices, else int32 indices. Returns false if the padded
// offsets would overflow int32 (the plan then keeps the plain layout).
// Exception buckets (a1 != +-a2 in the plan type) of one direction, per vector.
template <class T>
void build_exceptions(Plan& P, bool fwd, const int* ptr, const int* idx, const double* v0,
                      const double* v1, long long n, int gw) {
  DBuf<int>& eptr = fwd ? P.eptr_f : P.eptr_b;
  std::int64_t& nexc = fwd ? P.nexc_f : P.nexc_b;
  DBuf<int> cnt(n + 1);
  SSB_CUDA(cudaMemsetAsync(cnt.get(), 0, (n + 1) * sizeof(int), P.ctx->stream));
  mirror_exc_count_kernel<T><<<gw, 256, 0, P.ctx->stream>>>(ptr, v0, v1, n, cnt.get());
  P.ctx->check_launch("mirror_exc_count_kernel");
  eptr.alloc(n + 1);
  scan_counts(P.ctx, cnt.get(), eptr.get(), n);
  int ne = 0;
  P.ctx->copy(&ne, eptr.get() + n, sizeof(int));
  nexc = ne;
  if (ne == 0) {
    eptr.release();
    return;
  }
  DBuf<int>& eidx = fwd ? P.eidx_f : P.eidx_b;
  DBuf<char>& ev2 = fwd ? P.ev2_f : P.ev2_b;
  eidx.alloc(ne);
  ev2.alloc(2 * static_cast<std::size_t>(ne) * sizeof(T));
  mirror_exc_fill_kernel<T><<<gw, 256, 0, P.ctx->stream>>>(ptr, idx, v0, v1, n, eptr.get(),
                                                           eidx.get(), reinterpret_cast<T*>(ev2.get()));
  P.ctx->check_launch("mirror_exc_fill_kernel");
}

template <class T>
bool build_tiled_streams(Plan& P, int w) {
  const long long nnz = P.a[0]->nnz, rows = P.rows[0], cols = P.cols[0];
  if (nnz + 3 * std::max(rows, cols) >= (1LL << 31)) return false;
  P.tnnz_f = tiled_ptr(P, P.a[0]->rowptr.get(), rows, P.tptr_f);
  P.tnnz_b = tiled_ptr(P, P.a[0]->colptr.get(), cols, P.tptr_b);
  const std::size_t tb = sizeof(T);
  // straight from the fp64 CSR/CSC values (no fp32 matrix copies)
  const auto vals = [&](int s, bool csr) -> const double* {
    if (s >= w) return nullptr;
    return csr ? P.a[s]->val.get() : P.a[s]->cval.get();
  };
  const int gw = std::max(1, static_cast<int>(std::min<long long>(
                                 P.ctx->sm_count * 16LL, (std::max(rows, cols) + 7) / 8)));
  const auto build_dir = [&](bool fwd) {
    const Matrix& m = *P.a[0];
    const int* ptr = fwd ? m.rowptr.get() : m.colptr.get();
    const int* idx = fwd ? m.colidx.get() : m.rowidx.get();
    const long long n = fwd ? rows : cols;
    const DBuf<int>& tptr = fwd ? P.tptr_f : P.tptr_b;
    const std::int64_t tn = fwd ? P.tnnz_f : P.tnnz_b;
    DBuf<char>& vbuf = fwd ? P.rv2 : P.cv2;
    DBuf<int>& tidx = fwd ? P.tidx_f : P.tidx_b;
    bool& u16 = fwd ? P.c16f : P.c16b;
    bool& mir = fwd ? P.mir_f : P.mir_b;
    mir = mir && w == 2;
    int tile = 4 * (fwd ? P.vs_fwd : P.vs_back);
    if (u16) {  // 16 bits fit every tile? (decided before any stream buffer exists)
      // a paired plan first narrows its lane groups (smaller tiles span fewer
      // indices): config 5's K2 fits at 4 lanes, 0.83 -> 0.71 ms vs int32 at 8
      const bool narrow = w == 2 && std::getenv(fwd ? "SSB_VS_FWD" : "SSB_VS_BACK") == nullptr;
      const int vs0 = fwd ? P.vs_fwd : P.vs_back;
      for (;;) {
        DBuf<int> of(1);
        SSB_CUDA(cudaMemsetAsync(of.get(), 0, sizeof(int), P.ctx->stream));
        tile_overflow_kernel<<<grid1(P.ctx, n), 256, 0, P.ctx->stream>>>(ptr, idx, n, tile,
                                                                          of.get());
        P.ctx->check_launch("tile_overflow_kernel");
        int bad = 0;
        P.ctx->copy(&bad, of.get(), sizeof(int));
        if (!bad) break;
        int& vs = fwd ? P.vs_fwd : P.vs_back;
        if (!narrow || vs <= 4) {  // no width fits: int32 indices at the picked width
          u16 = false;
          vs = vs0;
          tile = 4 * vs;
          break;
        }
        vs /= 2;
        tile = 4 * vs;
      }
    }
    if (u16 || mir) {  // per-tile data: first tile of every vector
      DBuf<int>& tfirst = fwd ? P.tfirst_f : P.tfirst_b;
      std::int64_t& ntile = fwd ? P.ntile_f : P.ntile_b;
      DBuf<int> cnt(n + 1), overflow(1);
      tfirst.alloc(n + 1);
      tile_counts_kernel<<<grid1(P.ctx, n + 1), 256, 0, P.ctx->stream>>>(tptr.get(), n, tile,
                                                                        cnt.get());
      P.ctx->check_launch("tile_counts_kernel");
      scan_counts(P.ctx, cnt.get(), tfirst.get(), n);
      int total = 0;
      P.ctx->copy(&total, tfirst.get() + n, sizeof(int));
      ntile = total;
      SSB_CUDA(cudaMemsetAsync(overflow.get(), 0, sizeof(int), P.ctx->stream));
      DBuf<unsigned short>& tofs = fwd ? P.tofs_f : P.tofs_b;
      if (mir) {  // one value + sign bits; 16-bit offsets or int32 indices
        DBuf<unsigned>& thdr = fwd ? P.thdr_f : P.thdr_b;
        int& hs = fwd ? P.hs_f : P.hs_b;
        hs = tile <= 32 ? 2 : (tile == 64 ? 4 : 8);
        thdr.alloc(static_cast<std::size_t>(ntile) * hs);
        SSB_CUDA(cudaMemsetAsync(thdr.get(), 0, static_cast<std::size_t>(ntile) * hs * 4,
                                 P.ctx->stream));
        vbuf.alloc(tn * tb);
        if (u16) tofs.alloc(tn);
        else tidx.alloc(tn);
        tile_mirror_kernel<T><<<gw, 256, 0, P.ctx->stream>>>(
            ptr, idx, vals(0, fwd), vals(1, fwd), n, tptr.get(), tfirst.get(),
            u16 ? tofs.get() : nullptr, u16 ? nullptr : tidx.get(), thdr.get(), hs,
            reinterpret_cast<T*>(vbuf.get()), tile, overflow.get());
        P.ctx->check_launch("tile_mirror_kernel");
        build_exceptions<T>(P, fwd, ptr, idx, vals(0, fwd), vals(1, fwd), n, gw);
        return;
      }
      DBuf<int>& tbase = fwd ? P.tbase_f : P.tbase_b;  // interleaved values, 16-bit offsets
      tofs.alloc(tn);
      tbase.alloc(ntile);
      vbuf.alloc(w * tn * tb);
      tile_stream16_kernel<T, double><<<gw, 256, 0, P.ctx->stream>>>(
          ptr, idx, vals(0, fwd), vals(1, fwd), n, tptr.get(), tfirst.get(), tofs.get(),
          tbase.get(), reinterpret_cast<T*>(vbuf.get()), tile, overflow.get());
      P.ctx->check_launch("tile_stream16_kernel");
      return;
    }
    tidx.alloc(tn);
    vbuf.alloc(w * tn * tb);
    tile_stream_kernel<T, double><<<gw, 256, 0, P.ctx->stream>>>(
        ptr, idx, vals(0, fwd), vals(1, fwd), n, tptr.get(), tidx.get(),
        reinterpret_cast<T*>(vbuf.get()), tile);
    P.ctx->check_launch("tile_stream_kernel");
  };
  build_dir(true);
  build_dir(false);
  P.ctx->sync();
  return true;
}

template <class T>
void build_paired_t(Plan& P) {
  const long long nnz = P.a[0]->nnz, rows = P.rows[0], cols = P.cols[0];
  const std::size_t tb = sizeof(T);
  if (P.tiled && !build_tiled_streams<T>(P, 2)) P.tiled = false;
  if (!P.tiled) {
    P.c16f = P.c16b = false;
    P.rv2.alloc(2 * nnz * tb);
    P.cv2.alloc(2 * nnz * tb);
  }
  P.pe.alloc(4 * rows * tb);
  P.cc.alloc(2 * cols * tb);
  SSB_CUDA(cudaMemsetAsync(P.pe.get(), 0, 4 * rows * tb, P.ctx->stream));
  T* rv2 = reinterpret_cast<T*>(P.rv2.get());
  T* cv2 = reinterpret_cast<T*>(P.cv2.get());
  const int gn = grid1(P.ctx, nnz), gr = grid1(P.ctx, rows), gc = grid1(P.ctx, cols);
  for (int s = 0; s < 2; ++s) {
    if (!P.tiled) {
      const T* rv = nullptr;
      const T* cv = nullptr;
      if constexpr (sizeof(T) == 4) {
        P.a[s]->ensure_f32();
        rv = P.a[s]->val32.get();
        cv = P.a[s]->cval32.get();
      } else {
        rv = P.a[s]->val.get();
        cv = P.a[s]->cval.get();
      }
      interleave_kernel<T, T><<<gn, 256, 0, P.ctx->stream>>>(rv, rv2, nnz, 2, s);
      interleave_kernel<T, T><<<gn, 256, 0, P.ctx->stream>>>(cv, cv2, nnz, 2, s);
    }
    interleave_kernel<T, T><<<gr, 256, 0, P.ctx->stream>>>(
        reinterpret_cast<const T*>(P.rinv[s].get()), reinterpret_cast<T*>(P.pe.get()), rows, 4,
        2 + s);
    interleave_kernel<T, T><<<gc, 256, 0, P.ctx->stream>>>(
        reinterpret_cast<const T*>(P.cinv[s].get()), reinterpret_cast<T*>(P.cc.get()), cols, 2,
        s);
    P.ctx->check_launch("interleave_kernel");
  }
  P.ctx->sync();
}

// single-system plans: tiled streams when enabled (else the plain CSR/CSC kernels)
void build_single(Plan& P) {
  if (!P.tiled) return;
  const bool ok = P.dtype == SS_F32 ? build_tiled_streams<float>(P, 1)
                                    : build_tiled_streams<double>(P, 1);
  if (!ok) P.tiled = false;
  if (!P.tiled) P.c16f = P.c16b = false;
}
}  // namespace

// Block-merged multi-RHS streams of one direction (see sart_fwd_block_kernel):
// vectors of both folded systems in blocks of kBlockR, each block's sorted
// union of indices with its 2*kBlockR values per index (zero where absent).
template <class T>
void build_blocks_dir(Plan& P, bool fwd) {
  constexpr int R = kBlockR;
  const std::int64_t n = fwd ? P.rows[0] : P.cols[0];
  std::vector<int> ptr[2], idx[2];
  std::vector<double> val[2];
  for (int s = 0; s < 2; ++s) {
    Matrix* a = P.a[s];
    a->ensure_csc();
    const std::int64_t nnz = a->nnz;
    ptr[s].resize(n + 1);
    idx[s].resize(nnz);
    val[s].resize(nnz);
    P.ctx->copy(ptr[s].data(), fwd ? a->rowptr.get() : a->colptr.get(), (n + 1) * sizeof(int));
    P.ctx->copy(idx[s].data(), fwd ? a->colidx.get() : a->rowidx.get(), nnz * sizeof(int));
    P.ctx->copy(val[s].data(), fwd ? a->val.get() : a->cval.get(), nnz * sizeof(double));
  }
  const std::int64_t nblk = (n + R - 1) / R;
  std::vector<int> bptr(nblk + 1, 0), bidx;
  std::vector<T> bval;
  std::vector<int> uni;
  for (std::int64_t b = 0; b < nblk; ++b) {
    uni.clear();
    for (int s = 0; s < 2; ++s) {
      for (int r = 0; r < R && b * R + r < n; ++r) {
        const std::int64_t v = b * R + r;
        uni.insert(uni.end(), idx[s].begin() + ptr[s][v], idx[s].begin() + ptr[s][v + 1]);
      }
    }
    std::sort(uni.begin(), uni.end());
    uni.erase(std::unique(uni.begin(), uni.end()), uni.end());
    const std::size_t base = bidx.size();
    bidx.insert(bidx.end(), uni.begin(), uni.end());
    bval.resize(bidx.size() * 2 * R, T(0));
    for (int s = 0; s < 2; ++s) {
      for (int r = 0; r < R && b * R + r < n; ++r) {
        const std::int64_t v = b * R + r;
        std::size_t u = 0;  // both lists ascending: one merge walk
        for (int q = ptr[s][v]; q < ptr[s][v + 1]; ++q) {
          while (uni[u] != idx[s][q]) ++u;
          bval[(base + u) * 2 * R + s * R + r] = static_cast<T>(val[s][q]);
        }
      }
    }
    if (bidx.size() >= (std::size_t{1} << 31)) fail("plan: block-merged stream exceeds int32");
    bptr[b + 1] = static_cast<int>(bidx.size());
  }
  DBuf<int>& dp = fwd ? P.bptr_f : P.bptr_b;
  DBuf<int>& di = fwd ? P.bidx_f : P.bidx_b;
  DBuf<char>& dv = fwd ? P.bval_f : P.bval_b;
  dp.alloc(nblk + 1);
  di.alloc(bidx.size());
  dv.alloc(bval.size() * sizeof(T));
  SSB_CUDA(cudaMemcpyAsync(dp.get(), bptr.data(), bptr.size() * sizeof(int),
                           cudaMemcpyHostToDevice, P.ctx->stream));
  SSB_CUDA(cudaMemcpyAsync(di.get(), bidx.data(), bidx.size() * sizeof(int),
                           cudaMemcpyHostToDevice, P.ctx->stream));
  SSB_CUDA(cudaMemcpyAsync(dv.get(), bval.data(), bval.size() * sizeof(T),
                           cudaMemcpyHostToDevice, P.ctx->stream));
  P.ctx->sync();
  (fwd ? P.nblk_f : P.nblk_b) = nblk;
  (fwd ? P.nu_f : P.nu_b) = static_cast<std::int64_t>(bidx.size());
}

// multi-RHS plans over the folded pair use the block-merged kernels
// (SSB_BLOCKED=0: the per-vector multi kernels)
template <class T>
void build_blocks(Plan& P) {
  if (P.nrhs < 2 || P.nsys != 2 || P.nband > 1) return;
  // measured on config 4 (profiles/r02_notes.md): the merged blocks win for
  // K2 (0.61 -> 0.43 ms), the per-vector kernel stays faster for K1
  const int all = env_int("SSB_BLOCKED", -1);
  P.blocked_f = all >= 0 ? all != 0 : env_int("SSB_BLOCKED_FWD", 0) != 0;
  P.blocked_b = all >= 0 ? all != 0 : env_int("SSB_BLOCKED_BACK", 1) != 0;
  P.block_e_f = env_int("SSB_BLOCK_E_FWD", 4) <= 2 ? 2 : 4;
  P.block_e_b = env_int("SSB_BLOCK_E_BACK", 2) <= 2 ? 2 : 4;
  for (int f = 0; f < 2; ++f) {
    const bool fwd = f == 0;
    if (!(fwd ? P.blocked_f : P.blocked_b)) continue;
    build_blocks_dir<T>(P, fwd);
    int per_sm = 0;
    const std::size_t sh = fwd ? sizeof(double) * kWarps * 2 * P.nrhs : 0;
    SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, block_kernel<T>(P, fwd),
                                                           kThreads, sh));
    const long long warps = fwd ? P.nblk_f : P.nblk_b;
    (fwd ? P.fwd_blocks : P.back_blocks) = static_cast<int>(std::max<long long>(
        1, std::min<long long>(static_cast<long long>(std::max(1, per_sm)) * P.ctx->sm_count,
                               (warps + kWarps - 1) / kWarps)));
  }
  const std::size_t need = static_cast<std::size_t>(P.fwd_blocks) * 2 * P.nrhs;
  if (need > P.partial.size()) P.partial.alloc(need);
}

// Staged multi-RHS streams of one direction (see sart_stage_kernel): blocks of
// kStageR rows (K1) / columns (K2) per system, each block's sorted index union
// and its entries chunk-major, neighbouring vector pairs merged.
template <class T>
void build_stage_dir(Plan& P, bool fwd) {
  Plan::StageBufs& B = P.stg[fwd ? 0 : 1];
  B.on = false;
  constexpr int R = kStageR, C = kStageC;
  const std::int64_t n = fwd ? P.rows[0] : P.cols[0];
  for (int s = 1; s < P.nsys; ++s) {
    if ((fwd ? P.rows[s] : P.cols[s]) != n) return;
  }
  const std::int64_t nblk = (n + R - 1) / R;
  std::vector<int> bptr(1, 0), buni, bch;
  std::vector<long long> cofs(1, 0);
  std::vector<char> ent;
  std::vector<int> uni, pos;
  long long maxrec = 0;
  const auto put = [&](const void* p, std::size_t nb) {
    const char* c = static_cast<const char*>(p);
    ent.insert(ent.end(), c, c + nb);
  };
  for (int s = 0; s < P.nsys; ++s) {
    Matrix* a = P.a[s];
    if (!fwd) a->ensure_csc();
    std::vector<int> rp(n + 1), ci(a->nnz);
    std::vector<double> va(a->nnz);
    P.ctx->copy(rp.data(), fwd ? a->rowptr.get() : a->colptr.get(), (n + 1) * sizeof(int));
    P.ctx->copy(ci.data(), fwd ? a->colidx.get() : a->rowidx.get(), a->nnz * sizeof(int));
    P.ctx->copy(va.data(), fwd ? a->val.get() : a->cval.get(), a->nnz * sizeof(double));
    pos.resize(a->nnz);
    for (std::int64_t b = 0; b < nblk; ++b) {
      const std::int64_t r0 = b * R, r1 = std::min<std::int64_t>(r0 + R, n);
      uni.assign(ci.begin() + rp[r0], ci.begin() + rp[r1]);
      std::sort(uni.begin(), uni.end());
      uni.erase(std::unique(uni.begin(), uni.end()), uni.end());
      for (std::int64_t i = r0; i < r1; ++i) {
        std::size_t u = 0;  // both ascending: one merge walk
        for (int e = rp[i]; e < rp[i + 1]; ++e) {
          while (uni[u] != ci[e]) ++u;
          pos[e] = static_cast<int>(u);
        }
      }
      const int nch = (static_cast<int>(uni.size()) + C - 1) / C;
      bch.push_back(static_cast<int>(cofs.size() - 1));
      std::vector<int> cur(R, 0);  // next entry of each row
      for (int rl = 0; rl < R; ++rl) cur[rl] = r0 + rl < r1 ? rp[r0 + rl] : 0;
      for (int c = 0; c < nch; ++c) {
        // header: kStageR / 2 + 1 run offsets (row pairs), then per pair the
        // merged positions {value a, value b, position - c*C}
        const std::size_t h0 = ent.size();
        ent.resize(h0 + kStageHdr, 0);
        unsigned short off = 0;
        for (int pr = 0; pr < R / 2; ++pr) {
          std::memcpy(&ent[h0 + 2 * pr], &off, 2);
          const int ra = 2 * pr, rb = ra + 1;
          const int ea = r0 + ra < r1 ? rp[r0 + ra + 1] : 0;
          const int ebd = r0 + rb < r1 ? rp[r0 + rb + 1] : 0;
          int& ia = cur[ra];
          int& ib = cur[rb];
          while (true) {
            const int pa = ia < ea && pos[ia] < (c + 1) * C ? pos[ia] : INT32_MAX;
            const int pb = ib < ebd && pos[ib] < (c + 1) * C ? pos[ib] : INT32_MAX;
            const int pm = std::min(pa, pb);
            if (pm == INT32_MAX) break;
            StageEnt<T> se;
            std::memset(&se, 0, sizeof se);
            se.u = pm - c * C;
            if (pa == pm) se.va = static_cast<T>(va[ia++]);
            if (pb == pm) se.vb = static_cast<T>(va[ib++]);
            put(&se, sizeof se);
            ++off;
          }
        }
        std::memcpy(&ent[h0 + 2 * (R / 2)], &off, 2);
        ent.resize((ent.size() + 15) & ~std::size_t{15}, 0);
        maxrec = std::max<long long>(maxrec, static_cast<long long>(ent.size() - h0));
        cofs.push_back(static_cast<long long>(ent.size()));
      }
      buni.insert(buni.end(), uni.begin(), uni.end());
      if (buni.size() >= (std::size_t{1} << 31)) return;
      bptr.push_back(static_cast<int>(buni.size()));
    }
  }
  const auto up = [&](auto& dbuf, const auto& v) {
    dbuf.alloc(std::max<std::size_t>(v.size(), 1));
    SSB_CUDA(cudaMemcpyAsync(dbuf.get(), v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice,
                             P.ctx->stream));
  };
  up(B.bptr, bptr);
  up(B.buni, buni);
  up(B.bch, bch);
  up(B.cofs, cofs);
  up(B.ent, ent);
  P.ctx->sync();
  B.nblk = nblk;
  B.nu = static_cast<std::int64_t>(buni.size());
  B.entb = static_cast<std::int64_t>(ent.size());
  // ring slots: kStageC X records + the largest chunk record; the ring is
  // reused for the per-slice reductions at the end
  const long long rec = static_cast<long long>(P.nrhs) * sizeof(T);
  B.slot = static_cast<int>((C * rec + maxrec + 127) & ~127ll);
  B.smem = static_cast<int>(std::max<long long>(static_cast<long long>(kStageNS) * B.slot,
                                                8ll * kWarps * P.nsys * P.nrhs));
  StageFn<T> fn = stage_kernel<T>(P.nrhs, fwd);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, B.smem) !=
      cudaSuccess) {
    cudaGetLastError();
    return;
  }
  int per_sm = 0;
  SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kStageThreads, B.smem));
  if (per_sm < 1) return;
  B.blocks = static_cast<int>(std::max<long long>(
      1, std::min<long long>(static_cast<long long>(per_sm) * P.ctx->sm_count, nblk * P.nsys)));
  if (fwd) {
    P.fwd_blocks = B.blocks;
    const std::size_t need = static_cast<std::size_t>(B.blocks) * P.nsys * P.nrhs;
    if (need > P.partial.size()) P.partial.alloc(need);
    P.blocked_f = false;
  } else {
    P.back_blocks = B.blocks;
    P.blocked_b = false;
  }
  B.on = true;
}

// multi-RHS plans of 32 / 64 / 128 slices without column bands stage the
// gathered operand (SSB_STAGED=0: neither direction; SSB_STAGED_FWD /
// SSB_STAGED_BACK per direction)
template <class T>
void build_stage(Plan& P) {
  if (P.nrhs < 2 || P.nband > 1 || !stage_kernel<T>(P.nrhs, true)) return;
  const int all = env_int("SSB_STAGED", -1);
  if (all == 0) return;
  if (all == 1 || env_int("SSB_STAGED_FWD", 1) != 0) build_stage_dir<T>(P, true);
  if (all == 1 || env_int("SSB_STAGED_BACK", 1) != 0) build_stage_dir<T>(P, false);
}

// Persistent loop of a paired plan (see sart_persistent_pair_kernel): the
// grid is every co-resident CTA the work can use; the barrier words are
// zeroed once (the barrier leaves its count at 0).
template <class T>
void setup_persistent(Plan& P) {
  PersistFn<T> fn = persistent_kernel<T>(P);
  if (!fn) return;
  int per_sm = 0;
  SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0));
  if (per_sm < 1) return;
  const long long need = std::max<long long>(static_cast<long long>(P.rows[0]) * P.vs_fwd,
                                             static_cast<long long>(P.cols[0]) * P.vs_back);
  P.pgrid = static_cast<int>(std::max<long long>(1, std::min<long long>(
      static_cast<long long>(per_sm) * P.ctx->sm_count, (need + kThreads - 1) / kThreads)));
  P.gbar.alloc(2);
  SSB_CUDA(cudaMemsetAsync(P.gbar.get(), 0, 2 * sizeof(unsigned), P.ctx->stream));
  if (static_cast<std::size_t>(P.pgrid) * 2 > P.partial.size()) P.partial.alloc(2 * P.pgrid);
  P.ctx->sync();
  P.persistent = true;
}

Plan* make_plan(Context* ctx, Matrix* a1, Matrix* a2, const ss_solve_options& o, int nrhs,
                bool reusable) {
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
  PhaseTrace tr(ctx);
  if (a2 && nrhs == 1 && env_int("SSB_PAIRED", 1) != 0) {
    // one shared index stream for the folded pair (identical patterns unless
    // the fold pruned cancellations; then the union with explicit zeros)
    if (!same_pattern(*a1, *a2)) {
      union_pattern(*a1, *a2, P->pair_own[0], P->pair_own[1]);
      P->a[0] = P->pair_own[0];
      P->a[1] = P->pair_own[1];
    }
    P->paired = true;
    P->tiled = env_int("SSB_TILED", 1) != 0;
    P->c16f = P->c16b = env_int("SSB_U16", 1) != 0;
    P->mir_f = P->mir_b = env_int("SSB_MIRROR", 1) != 0;
    tr.mark("pair pattern");
  }
  for (int s = 0; s < P->nsys; ++s) {
    Matrix* a = P->a[s];
    if (P->paired && s == 1) {
      a->csc_like(*P->a[0]);  // same CSR pattern: a[0]'s column ordering, own values
      P->a[0]->csc_perm.release();
    } else {
      a->ensure_csc(P->paired && !P->a[1]->has_csc);
    }
    tr.mark("csc");
    if (o.dtype == SS_F32 && !P->paired) a->ensure_f32();  // paired streams convert on build
    tr.mark("f32 copies");
    P->rows[s] = a->rows;
    P->cols[s] = a->cols;
    nnz_total += a->nnz;
    rows_total += a->rows;
    cols_total += a->cols;
  }
  P->vs_fwd = env_int("SSB_VS_FWD", pick_vs(rows_total > 0 ? nnz_total / rows_total : 0));
  P->vs_back = env_int("SSB_VS_BACK", pick_vs(cols_total > 0 ? nnz_total / cols_total : 0));
  if (P->paired) {
    // measured best for the paired streams (config 3 sweeps, profiles/r01_notes.md):
    // fp32 mirror-coded streams carry 6 bytes per entry and prefer 8-lane groups
    // down to ~100 entries per vector; fp64 mirror-coded K1 spills at UF = 4
    const bool mir32 = P->mir_f && o.dtype == SS_F32;
    const auto vs_of = [&](double avg) { return mir32 ? pick_vs_mirror(avg) : pick_vs(avg); };
    P->vs_fwd = env_int("SSB_VS_FWD", vs_of(nnz_total / std::max(rows_total, 1.0)));
    P->vs_back = env_int("SSB_VS_BACK", vs_of(nnz_total / std::max(cols_total, 1.0)));
    // too few vectors to give every SM one CTA: wider lane groups (config 1,
    // 640 x 2048 per system: 75.7K -> 86.6K it/s at 32 / 16 lanes; config 2's
    // 6,144 rows already fill the SMs and measure slower when widened)
    const double fill = static_cast<double>(ctx->sm_count) * kThreads;
    while (!std::getenv("SSB_VS_FWD") && P->vs_fwd < 32 && P->rows[0] * P->vs_fwd < fill) {
      P->vs_fwd *= 2;
    }
    while (!std::getenv("SSB_VS_BACK") && P->vs_back < 16 && P->cols[0] * P->vs_back < fill) {
      P->vs_back *= 2;
    }
    P->uf_fwd = env_int("SSB_UF_FWD", P->mir_f && o.dtype == SS_F64 ? 2 : 4);
    P->uf_back = env_int("SSB_UF_BACK", 2);
    // the smallest pairs (one pass of 8-lane rows / 4-lane columns fits one
    // 16-CTA cluster: config 1) run the whole loop in one cluster-persistent
    // kernel; its lane groups are widened to cover every vector in one pass
    // (SSB_PERSIST: -1 auto, 0 two launches per pass, 1 grid-persistent
    // kernel, 2 cluster kernel whenever the shape allows)
    const int want = env_int("SSB_PERSIST", -1);
    if (P->mir_f && P->c16f && (want == 2 || want == -1)) {
      const int c = o.dtype == SS_F32
                        ? cluster_size_for<float>(cluster_kernel<float>(16, 8), kClusterSmemMax)
                        : cluster_size_for<double>(cluster_kernel<double>(16, 8), kClusterSmemMax);
      const long long cap = static_cast<long long>(c) * kClusterThreads;
      if (c > 0 && (want == 2 || (P->rows[0] * 8 <= cap && P->cols[0] * 4 <= cap))) {
        P->ccluster = c;
        if (!std::getenv("SSB_VS_FWD")) {
          P->vs_fwd = 8;
          while (P->vs_fwd < 32 && P->rows[0] * P->vs_fwd * 2 <= cap) P->vs_fwd *= 2;
        }
        if (!std::getenv("SSB_VS_BACK")) {
          P->vs_back = 4;
          while (P->vs_back < 16 && P->cols[0] * P->vs_back * 2 <= cap) P->vs_back *= 2;
        }
        P->uf_fwd = P->uf_back = 2;
      }
    }
  }
  if (!P->paired) {
    P->uf_fwd = env_int("SSB_UF_FWD", 4);
    P->uf_back = env_int("SSB_UF_BACK", 4);
  }
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
  if (nrhs > 1) {
    // K1 over column bands (SSB_BANDS > 1) keeps each pass's X records
    // L2-resident; measured slower on config 4 at every band count (2: -3%,
    // 3: -7%, 4: -12%; profiles/r01_notes.md), so one pass is the default
    const int nb = std::min(8, std::max(1, env_int("SSB_BANDS", 1)));
    P->nband = nb;
    if (nb > 1) {
      for (int s = 0; s < P->nsys; ++s) {
        P->band_ptr[s].alloc(static_cast<std::size_t>(nb + 1) * P->rows[s]);
        band_ptr_kernel<<<grid1(ctx, P->rows[s]), 256, 0, ctx->stream>>>(
            P->a[s]->rowptr.get(), P->a[s]->colidx.get(), P->rows[s], P->cols[s], nb,
            P->band_ptr[s].get());
        ctx->check_launch("band_ptr_kernel");
      }
    }
  }
  if (P->paired) {
    const long long fg = static_cast<long long>(P->rows[0]) * P->vs_fwd;
    const long long bg = static_cast<long long>(P->cols[0]) * P->vs_back;
    P->fwd_blocks = static_cast<int>(std::max<long long>(1, std::min<long long>(
        occupancy_pair_blocks(*P, true), (fg + kThreads - 1) / kThreads)));
    P->back_blocks = static_cast<int>(std::max<long long>(1, std::min<long long>(
        occupancy_pair_blocks(*P, false), (bg + kThreads - 1) / kThreads)));
  } else if (nrhs == 1 && P->nsys == 2) {
    // CTA-uniform systems: split the grid in proportion to each system's work
    const auto split = [&](int& blocks, double w0, double w1) {
      blocks = std::max(blocks, 2);
      const int b0 = static_cast<int>(std::llround(blocks * w0 / std::max(w0 + w1, 1.0)));
      return std::max(1, std::min(blocks - 1, b0));
    };
    const double n0 = static_cast<double>(a1->nnz), n1 = static_cast<double>(a2->nnz);
    P->sys_blocks_f = split(P->fwd_blocks, n0 + 16.0 * a1->rows, n1 + 16.0 * a2->rows);
    P->sys_blocks_b = split(P->back_blocks, n0 + 16.0 * a1->cols, n1 + 16.0 * a2->cols);
  }
  alloc_common(*P);
  tr.mark("occupancy + alloc");
  for (int s = 0; s < P->nsys; ++s) {
    double mx = 0;
    normalisers(*P, s, &mx);
    P->empty_rows[s] = !(mx > 0.0);
  }
  tr.mark("normalisers");
  if (o.dtype == SS_F32) build_blocks<float>(*P);
  else build_blocks<double>(*P);
  if (o.dtype == SS_F32) build_stage<float>(*P);
  else build_stage<double>(*P);
  if (P->paired) {
    if (o.dtype == SS_F32) build_paired_t<float>(*P);
    else build_paired_t<double>(*P);
    // the final layout (16-bit fit, lane groups) picks the kernels: size their grids
    P->fwd_blocks = static_cast<int>(std::max<long long>(1, std::min<long long>(
        occupancy_pair_blocks(*P, true),
        (static_cast<long long>(P->rows[0]) * P->vs_fwd + kThreads - 1) / kThreads)));
    P->back_blocks = static_cast<int>(std::max<long long>(1, std::min<long long>(
        occupancy_pair_blocks(*P, false),
        (static_cast<long long>(P->cols[0]) * P->vs_back + kThreads - 1) / kThreads)));
    if (static_cast<std::size_t>(P->fwd_blocks) * P->nsys * P->nrhs > P->partial.size()) {
      P->partial.alloc(static_cast<std::size_t>(P->fwd_blocks) * P->nsys * P->nrhs);
    }
    // fp32 streams of 1-16x the L2 carry the evict-first hint (see lds):
    // measured +2.5% at 5.3x (config 3), -2.6% at 92x (config 5)
    std::int64_t fb = 0, bb = 0;
    P->kernel_bytes(&fb, &bb);
    const std::size_t sb = static_cast<std::size_t>(fb + bb);
    P->stream_cs = o.dtype == SS_F32 && env_int("SSB_STREAM_CS", 1) != 0 &&
                   sb > ctx->l2_bytes && sb <= 16 * ctx->l2_bytes;
    P->l2_window = env_int("SSB_L2WIN", 0) != 0;
    if (P->l2_window) {
      SSB_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize,
                                  static_cast<std::size_t>(env_int("SSB_L2WIN_MB", 16)) << 20));
    }
    // L2-resident pairs (configs 1-2) run the loop as one persistent kernel
    // (SSB_PERSIST=0: the two launches per pass; 1: whenever the shape allows)
    if (P->ccluster > 0) {
      if (o.dtype == SS_F32) setup_cluster<float>(*P);
      else setup_cluster<double>(*P);
      P->cluster = P->persistent = P->ccluster > 0;
    }
    if (!P->cluster) {
      const int want = env_int("SSB_PERSIST", -1);
      const bool small = static_cast<std::size_t>(fb + bb) * 2 <= ctx->l2_bytes;
      // streams that fit the shared memory of the whole GPU stay resident
      // there (3: whenever the shape allows; 1: the L2-streamed grid kernel)
      if (want == 3 || (want == -1 && small)) {
        if (o.dtype == SS_F32) setup_resident<float>(*P);
        else setup_resident<double>(*P);
      }
      if (!P->resident && want != 0 && want != 2 && (want == 1 || want == 3 || small)) {
        if (o.dtype == SS_F32) setup_persistent<float>(*P);
        else setup_persistent<double>(*P);
      }
    }
    tr.mark("paired streams");
  } else if (P->nsys == 1 && nrhs == 1) {
    P->tiled = env_int("SSB_TILED", 1) != 0;
    P->c16f = P->c16b = env_int("SSB_U16", 1) != 0;
    build_single(*P);
    if (P->tiled) size_single_grid(*P);
    tr.mark("tiled streams");
  }
  if (P->nsys == 1 && P->empty_rows[0]) fail("sart_solve: matrix has no nonzero rows");
  // a reusable plan replays one captured graph; a one-shot solve enqueues its
  // launches directly (the host stays ahead of the 2*max_iters kernels)
  // SSB_GRAPH=0: direct launches (ncu lists graph-replayed K1 nodes of this
  // loop incompletely, so launch lists are taken with it)
  if (reusable && env_int("SSB_GRAPH", 1) != 0) P->build_graph();
  tr.mark("graph capture");
  return P.release();
}

void exchange_owned_columns(std::int64_t cols, int parts, int rank, std::int64_t* begin,
                            std::int64_t* end) {
  if (parts < 1 || rank < 0 || rank >= parts || cols < 0) fail("exchange: bad rank / parts");
  const std::int64_t own = (cols + parts - 1) / parts;  // as setup_exchange
  *begin = std::min(cols, rank * own);
  *end = std::min(cols, *begin + own);
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
namespace {

std::size_t align256(std::size_t v) { return (v + 255) & ~static_cast<std::size_t>(255); }

// All-gather of the ranks' IPC handles plus one status byte each: every rank
// fills its slot of a zeroed table (handle, status 1) -- or only zeros when its
// local setup failed -- and one byte-wise sum over the communicator combines
// them. Every rank of a peer-exchange plan calls this exactly once, whether or
// not its own setup succeeded, so no rank can block the others.
std::vector<unsigned char> exchange_table(Context* ctx, int G, int me,
                                          const cudaIpcMemHandle_t* h) {
  const std::size_t hs = sizeof(cudaIpcMemHandle_t);
  std::vector<unsigned char> tab(static_cast<std::size_t>(G) * (hs + 1), 0);
  if (h) {
    std::memcpy(tab.data() + me * hs, h, hs);
    tab[static_cast<std::size_t>(G) * hs + me] = 1;
  }
  DBuf<unsigned char> dt(tab.size());
  SSB_CUDA(cudaMemcpyAsync(dt.get(), tab.data(), tab.size(), cudaMemcpyHostToDevice,
                           ctx->stream));
  nccl_check(nccl().AllReduce(dt.get(), dt.get(), tab.size(), ncclUint8, ncclSum,
                              static_cast<ncclComm_t>(ctx->comm), ctx->stream),
             "ncclAllReduce(ipc handles)");
  ctx->copy(tab.data(), dt.get(), tab.size());
  return tab;
}

// Exchange region of a peer-exchange rank (layout in plan.hpp). Ownership and
// the reduce grid depend only on the column count, G and the SM count, so
// every rank derives the same ones.
void setup_exchange(Plan& P, int G, int me, bool emulated, bool* joined) {
  Context* ctx = P.ctx;
  const std::size_t ns = P.paired ? 2 : 1;  // systems per message (paired: {s1, s2} pairs)
  auto X = std::make_unique<PeerExchange>();
  X->G = G;
  X->me = me;
  X->emulated = emulated;
  X->cols = P.cols[0];
  X->own = (X->cols + G - 1) / G;  // owner of column j: j / own (exchange_owned_columns)
  // about one owned column per reduce thread (latency-bound gathers of G rows)
  X->rgrid = static_cast<int>(std::min<std::int64_t>(
      8LL * ctx->sm_count, std::max<std::int64_t>(ctx->sm_count, (X->own + 255) / 256)));
  const std::size_t tb = P.tsize();
  X->off_recv = 0;
  X->off_x = align256(static_cast<std::size_t>(G) * X->cols * tb * ns + kSlackBytes);
  X->off_r2 = align256(X->off_x + X->cols * tb * ns + kSlackBytes);
  X->off_done = align256(X->off_r2 + 2 * G * ns * sizeof(double));
  X->off_xready = X->off_done + 64;
  X->off_dflag = X->off_xready + 64;
  X->bytes = align256(X->off_dflag + 64);
  // Local setup first (allocation, IPC export). A failure here must not
  // leave the other ranks blocked in the handle exchange below: it is
  // reported through the exchange's status bytes and every rank fails alike.
  std::vector<char*> bases(G, nullptr);
  cudaIpcMemHandle_t h{};
  std::string local_err;
  try {
    // plain cudaMalloc: pool (cudaMallocAsync) memory cannot be exported over IPC
    SSB_CUDA(cudaMalloc(&X->region, X->bytes));
    SSB_CUDA(cudaMemsetAsync(X->region, 0, X->bytes, ctx->stream));
    X->local.alloc(4);
    SSB_CUDA(cudaMemsetAsync(X->local.get(), 0, 4 * sizeof(long long), ctx->stream));
    X->peers.alloc(G);
    bases[me] = static_cast<char*>(X->region);
    if (!emulated && G > 1) SSB_CUDA(cudaIpcGetMemHandle(&h, X->region));
  } catch (const std::exception& e) {
    local_err = e.what();
  }
  if (emulated || G == 1) {
    if (!local_err.empty()) fail("peer exchange setup: " + local_err);
  } else {
    *joined = true;
    std::vector<unsigned char> tab = exchange_table(ctx, G, me, local_err.empty() ? &h : nullptr);
    const unsigned char* status = tab.data() + static_cast<std::size_t>(G) * sizeof h;
    if (!local_err.empty()) fail("peer exchange setup: " + local_err);
    for (int r = 0; r < G; ++r) {
      if (status[r] != 1) fail("peer exchange setup failed on rank " + std::to_string(r));
    }
    for (int r = 0; r < G; ++r) {
      if (r == me) continue;
      cudaIpcMemHandle_t hr;
      std::memcpy(&hr, tab.data() + r * sizeof hr, sizeof hr);
      void* q = nullptr;
      SSB_CUDA(cudaIpcOpenMemHandle(&q, hr, cudaIpcMemLazyEnablePeerAccess));
      X->opened.push_back(q);
      bases[r] = static_cast<char*>(q);
    }
  }
  if (!emulated) {
    SSB_CUDA(cudaMemcpyAsync(X->peers.get(), bases.data(), G * sizeof(char*),
                             cudaMemcpyHostToDevice, ctx->stream));
  }
  ctx->sync();
  P.px = X.release();
}

}  // namespace

PeerExchange::~PeerExchange() {
  for (void* q : opened) cudaIpcCloseMemHandle(q);
  if (region) cudaFree(region);
}

void link_group(Plan* const* plans, int parts) {
  std::vector<char*> bases(parts);
  for (int g = 0; g < parts; ++g) {
    if (!plans[g]->px || !plans[g]->px->emulated || plans[g]->px->G != parts ||
        plans[g]->px->me != g) {
      fail("plan: not rank " + std::to_string(g) + " of an emulated group of " +
           std::to_string(parts));
    }
    bases[g] = static_cast<char*>(plans[g]->px->region);
  }
  for (int g = 0; g < parts; ++g) {
    Context* ctx = plans[g]->ctx;
    SSB_CUDA(cudaMemcpyAsync(plans[g]->px->peers.get(), bases.data(), parts * sizeof(char*),
                             cudaMemcpyHostToDevice, ctx->stream));
    ctx->sync();
  }
}

void run_group(Plan* const* plans, int parts) {
  if (parts < 1) fail("plan: empty group");
  Plan& P0 = *plans[0];
  for (int g = 0; g < parts; ++g) {
    Plan& P = *plans[g];
    if (!P.px || !P.px->emulated || P.ctx != P0.ctx || P.opts.max_iters != P0.opts.max_iters) {
      fail("plan: group plans must be one emulated exchange on one context");
    }
  }
  Context* ctx = P0.ctx;
  // ||p||^2 = sum of the ranks' local ||p_g||^2, in rank order (per system)
  const int ns = P0.paired ? 2 : 1;
  double pn[2] = {0.0, 0.0};
  for (int q = 0; q < ns; ++q) {
    double sq = 0.0;
    for (int g = 0; g < parts; ++g) {
      const double v = plans[g]->pn_local[q];
      if (v < 0.0) fail("plan: group rank " + std::to_string(g) + " has no rhs");
      sq += v * v;
    }
    pn[q] = std::sqrt(sq);
  }
  for (int g = 0; g < parts; ++g) {
    SSB_CUDA(cudaMemcpyAsync(plans[g]->pnorm.get(), pn, ns * sizeof(double),
                             cudaMemcpyHostToDevice, ctx->stream));
  }
  ctx->sync();
  for (int g = 0; g < parts; ++g) plans[g]->enqueue_reset();
  SSB_CUDA(cudaEventRecord(P0.ev0, ctx->stream));
  // rank order inside each phase (K1x, K2x, reduce): every wait a kernel
  // performs is on launches issued, and completed, before it
  auto announce = [&](int it, int kind) {
    for (int g = 0; g < parts; ++g) {
      if (plans[g]->dtype == SS_F32) launch_announce<float>(*plans[g], it, kind);
      else launch_announce<double>(*plans[g], it, kind);
    }
  };
  for (int it = 0; it < P0.opts.max_iters; ++it) {
    announce(it, 0);
    // phase: 0 K1x, 1 K2x, 2 reduce
    const auto phase = [&](Plan& P, int ph) {
      const bool fwd = ph == 0, red = ph == 2;
      if (P.dtype == SS_F32) {
        const SartK<float> k = make_args<float>(P);
        if (P.paired) launch_xchg_pair<float>(P, k, it, fwd, false, !red);
        else launch_xchg<float>(P, k, it, fwd, false, !red);
      } else {
        const SartK<double> k = make_args<double>(P);
        if (P.paired) launch_xchg_pair<double>(P, k, it, fwd, false, !red);
        else launch_xchg<double>(P, k, it, fwd, false, !red);
      }
    };
    for (int g = 0; g < parts; ++g) phase(*plans[g], 0);
    for (int g = 0; g < parts; ++g) phase(*plans[g], 1);
    announce(it, 1);
    for (int g = 0; g < parts; ++g) phase(*plans[g], 2);
  }
  announce(P0.opts.max_iters, 2);
  for (int g = 0; g < parts; ++g) plans[g]->enqueue_epilogue();
  SSB_CUDA(cudaEventRecord(P0.ev1, ctx->stream));
  SSB_CUDA(cudaEventSynchronize(P0.ev1));
  float ms = 0.0f;
  SSB_CUDA(cudaEventElapsedTime(&ms, P0.ev0, P0.ev1));
  for (int g = 0; g < parts; ++g) {
    Plan& P = *plans[g];
    SSB_CUDA(cudaEventRecord(P.ev0, ctx->stream));  // finish() re-reads the pair
    SSB_CUDA(cudaEventRecord(P.ev1, ctx->stream));
    P.launched = true;
  }
  ctx->sync();
  for (int g = 0; g < parts; ++g) plans[g]->group_ms = ms;

}

Plan* make_sharded_plan_local(Context* ctx, Matrix* a, std::int64_t rb, std::int64_t re,
                              const ss_solve_options& o, int exchange, int emul_parts,
                              int emul_rank, bool* joined);

Plan* make_sharded_plan(Context* ctx, Matrix* a, std::int64_t rb, std::int64_t re,
                        const ss_solve_options& o, int exchange, int emul_parts, int emul_rank) {
  if (exchange != SS_XCHG_NCCL && exchange != SS_XCHG_PEER) fail("plan: unknown exchange");
  if (emul_parts > 0) {
    if (exchange != SS_XCHG_PEER) fail("plan: only the peer exchange can be emulated");
    if (emul_rank < 0 || emul_rank >= emul_parts) fail("plan: emulated rank out of range");
  } else if (!ctx->comm) {
    fail("plan: context has no NCCL communicator");
  }
  // A real peer-exchange rank that fails before its handle exchange still
  // joins it (with status 0), so the other ranks fail too instead of blocking.
  const bool joins = exchange == SS_XCHG_PEER && emul_parts == 0 && ctx->nranks > 1;
  bool joined = false;  // set once this rank took part in the handle exchange
  try {
    return make_sharded_plan_local(ctx, a, rb, re, o, exchange, emul_parts, emul_rank, &joined);
  } catch (...) {
    if (joins && !joined) {
      try {
        exchange_table(ctx, ctx->nranks, ctx->rank, nullptr);
      } catch (...) {
      }
    }
    throw;
  }
}

Plan* make_sharded_plan_local(Context* ctx, Matrix* a, std::int64_t rb, std::int64_t re,
                              const ss_solve_options& o, int exchange, int emul_parts,
                              int emul_rank, bool* joined) {
  if (rb < 0 || re > a->rows || rb > re) fail("plan: row range out of bounds");
  if (o.relaxation <= 0 || o.relaxation > 2) fail("sart_solve: relaxation must be in (0, 2]");
  if (o.max_iters < 1) fail("sart_solve: max_iters must be >= 1");
  a->ensure_csc();
  // host-side slice of the CSR row block, then a local matrix on device
  std::vector<int> ptr(a->rows + 1);
  ctx->copy(ptr.data(), a->rowptr.get(), ptr.size() * sizeof(int));
  const std::int64_t k0 = ptr[rb], k1 = ptr[re], nloc = k1 - k0, rloc = re - rb;
  std::vector<int> lptr(rloc + 1), lcol(nloc), lrow(nloc);
  std::vector<double> lval(nloc);
  for (std::int64_t r = 0; r <= rloc; ++r) lptr[r] = static_cast<int>(ptr[rb + r] - k0);
  ctx->copy(lcol.data(), a->colidx.get() + k0, nloc * sizeof(int));
  ctx->copy(lval.data(), a->val.get() + k0, nloc * sizeof(double));
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
  P->vs_fwd = env_int("SSB_VS_FWD", pick_vs(rloc > 0 ? double(nloc) / rloc : 0));
  P->vs_back = env_int("SSB_VS_BACK", pick_vs(a->cols > 0 ? double(nloc) / a->cols : 0));
  // the single-system tiled kernels' measured best (as make_plan): UF 2 in K1
  // costs ~10 us per launch on a config-3 system (62 vs 52 us)
  P->uf_fwd = env_int("SSB_UF_FWD", 4);
  P->uf_back = env_int("SSB_UF_BACK", 4);
  if (o.dtype == SS_F32) {
    P->fwd_blocks = occupancy_blocks<float>(*P, true);
    P->back_blocks = occupancy_blocks<float>(*P, false);
  } else {
    P->fwd_blocks = occupancy_blocks<double>(*P, true);
    P->back_blocks = occupancy_blocks<double>(*P, false);
  }
  alloc_common(*P);
  if (exchange == SS_XCHG_NCCL) P->bp.alloc(sharded_r2_offset(a->cols, P->tsize()) + sizeof(double));
  // normalisers: rows from the local block, columns from the full matrix
  DBuf<double> rs_full(a->rows), cs_full(a->cols);
  // `a` may live on another context (stream): order the buffers' allocation
  // before, and the sums' completion after, the work on a->ctx's stream.
  ctx->sync();
  abs_sums(*a, rs_full.get(), cs_full.get());
  a->ctx->sync();
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
  P->tiled = env_int("SSB_TILED", 1) != 0;  // the row block on the tiled streams
  P->c16f = P->c16b = env_int("SSB_U16", 1) != 0;
  if (exchange == SS_XCHG_PEER) P->tiled = true;  // the exchange kernels are tiled-only
  build_single(*P);
  if (P->tiled) size_single_grid(*P);
  if (exchange == SS_XCHG_PEER) {
    if (emul_parts > 0) setup_exchange(*P, emul_parts, emul_rank, true, joined);
    else setup_exchange(*P, ctx->nranks, ctx->rank, false, joined);
  }
  ctx->sync();
  return P.release();
}

// Rows [rb, re) of matrix a as a local matrix on ctx (host-side CSR slice).
Matrix* row_block(Context* ctx, Matrix* a, std::int64_t rb, std::int64_t re) {
  std::vector<int> ptr(a->rows + 1);
  ctx->copy(ptr.data(), a->rowptr.get(), ptr.size() * sizeof(int));
  const std::int64_t k0 = ptr[rb], k1 = ptr[re], nloc = k1 - k0, rloc = re - rb;
  std::vector<int> lcol(nloc), lrow(nloc);
  std::vector<double> lval(nloc);
  ctx->copy(lcol.data(), a->colidx.get() + k0, nloc * sizeof(int));
  ctx->copy(lval.data(), a->val.get() + k0, nloc * sizeof(double));
  for (std::int64_t r = 0; r < rloc; ++r) {
    for (int k = ptr[rb + r]; k < ptr[rb + r + 1]; ++k) lrow[k - k0] = static_cast<int>(r);
  }
  return matrix_from_triplets_host(ctx, rloc, a->cols, nloc, lrow.data(), lcol.data(),
                                   lval.data());
}

// The folded pair row-sharded over all ranks of the exchange (see "paired
// peer exchange"): rows [rb, re) of A1 and A2 on the paired mirror-coded
// streams of an ordinary paired plan over the local row blocks; the column
// normalisers come from the full matrices (every rank holds the same ones).
Plan* make_sharded_pair_plan_local(Context* ctx, Matrix* a1, Matrix* a2, std::int64_t rb,
                                   std::int64_t re, const ss_solve_options& o, int emul_parts,
                                   int emul_rank, bool* joined) {
  if (!a2 || a1->rows != a2->rows || a1->cols != a2->cols) {
    fail("plan: folded systems must have equal shapes");
  }
  if (rb < 0 || re > a1->rows || rb > re) fail("plan: row range out of bounds");
  if (o.relaxation <= 0 || o.relaxation > 2) fail("sart_solve: relaxation must be in (0, 2]");
  if (o.max_iters < 1) fail("sart_solve: max_iters must be >= 1");
  std::unique_ptr<Matrix> l1(row_block(ctx, a1, rb, re)), l2(row_block(ctx, a2, rb, re));
  std::unique_ptr<Plan> P(make_plan(ctx, l1.get(), l2.get(), o, 1, false));
  if (!P->paired || !P->tiled || !P->mir_f || !P->mir_b) {
    fail("plan: the row-sharded pair needs the paired mirror-coded streams");
  }
  P->own = l1.release();
  P->own2 = l2.release();
  P->persistent = false;  // the exchange kernels run the loop
  P->resident = false;
  P->cluster = false;
  P->ccluster = 0;
  P->sharded = true;
  P->row_begin = rb;
  P->row_end = re;
  // column normalisers of the full matrices, then the interleaved {cinv1, cinv2}
  const std::int64_t cols = a1->cols;
  for (int s = 0; s < 2; ++s) {
    Matrix* a = s ? a2 : a1;
    DBuf<double> rs_full(a->rows), cs_full(cols);
    ctx->sync();
    abs_sums(*a, rs_full.get(), cs_full.get());
    a->ctx->sync();
    const int gc = grid1(ctx, cols);
    if (o.dtype == SS_F32) {
      inv_kernel<float><<<gc, 256, 0, ctx->stream>>>(
          cs_full.get(), reinterpret_cast<float*>(P->cinv[s].get()), cols);
      interleave_kernel<float, float><<<gc, 256, 0, ctx->stream>>>(
          reinterpret_cast<const float*>(P->cinv[s].get()), reinterpret_cast<float*>(P->cc.get()),
          cols, 2, s);
    } else {
      inv_kernel<double><<<gc, 256, 0, ctx->stream>>>(
          cs_full.get(), reinterpret_cast<double*>(P->cinv[s].get()), cols);
      interleave_kernel<double, double><<<gc, 256, 0, ctx->stream>>>(
          reinterpret_cast<const double*>(P->cinv[s].get()),
          reinterpret_cast<double*>(P->cc.get()), cols, 2, s);
    }
    ctx->check_launch("inv_kernel(full columns)");
    if (!(max_dev(ctx, rs_full.get(), a->rows) > 0.0)) P->empty_rows[s] = true;
    else P->empty_rows[s] = false;
  }
  ctx->sync();
  if (emul_parts > 0) setup_exchange(*P, emul_parts, emul_rank, true, joined);
  else setup_exchange(*P, ctx->nranks, ctx->rank, false, joined);
  ctx->sync();
  // real ranks, fixed pass count: the 3 launches per pass replay from one
  // captured graph (the host would otherwise pace a many-GPU loop)
  if (emul_parts == 0 && env_int("SSB_GRAPH", 1) != 0) P->build_graph();
  return P.release();
}

Plan* make_sharded_pair_plan(Context* ctx, Matrix* a1, Matrix* a2, std::int64_t rb,
                             std::int64_t re, const ss_solve_options& o, int emul_parts,
                             int emul_rank) {
  if (emul_parts > 0) {
    if (emul_rank < 0 || emul_rank >= emul_parts) fail("plan: emulated rank out of range");
  } else if (!ctx->comm) {
    fail("plan: context has no NCCL communicator");
  }
  const bool joins = emul_parts == 0 && ctx->nranks > 1;
  bool joined = false;
  try {
    return make_sharded_pair_plan_local(ctx, a1, a2, rb, re, o, emul_parts, emul_rank, &joined);
  } catch (...) {
    if (joins && !joined) {
      try {
        exchange_table(ctx, ctx->nranks, ctx->rank, nullptr);
      } catch (...) {
      }
    }
    throw;
  }
}

// ====================================================================== paired CGLS
// CGLS (reference cgls_solve, solvers.cpp:99-146) on both folded systems at
// once, over the SART plan's paired tiled streams: one index stream and
// interleaved {a1, a2} values, iterates interleaved {x1, x2}, each system with
// its own scalars and stop / break state (the two branches stay independent
// solves, as in the reference). The loop is a CUDA-graph WHILE node; the last
// block of the transposed product decides whether another pass runs.
namespace {

template <class T>
struct CgPairK {
  SartK<T> sk;     // stream layout (tiled pointers, indices / offsets, values)
  T *x, *r, *s, *d, *q;  // interleaved [n][2]
  long long rows, cols;
  double* part;    // [2][grid]
  double* sc;      // [2][5] gamma, alpha, beta, stop, rnorm2
  int* st;         // [2][5] done, iterations, err_step_at, err_res_at, -
  int* loop;       // pass counter, loop-over flag (the WHILE body unrolls passes)
  unsigned* ticket;
  double* hist;    // [2][hstride]
  int hstride;
  double tol;
  int max_iters;
  cudaGraphConditionalHandle cond;
};

__device__ __forceinline__ bool cg_on(const int* st, int s) {
  return *(volatile const int*)(st + 5 * s) == 0;
}

// fixed-order block sums of two values, then of the per-block partials by the
// last block (returns true there, with the totals)
__device__ __forceinline__ bool two_sums(double va, double vb, double* part, unsigned* ticket,
                                         double& ta, double& tb) {
  __shared__ double red[2][kWarps];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    va += __shfl_xor_sync(0xffffffffu, va, o);
    vb += __shfl_xor_sync(0xffffffffu, vb, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = va;
    red[1][threadIdx.x >> 5] = vb;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double t = 0.0;
    for (int w = 0; w < kWarps; ++w) t += red[threadIdx.x][w];
    part[threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
  if (!last_block(ticket)) return false;
  __shared__ double sh[2][kThreads];
  for (int q = 0; q < 2; ++q) {
    double t = 0.0;
    for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += blockDim.x) t += part[q * gridDim.x + b];
    sh[q][threadIdx.x] = t;
  }
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + o];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + o];
    }
    __syncthreads();
  }
  ta = sh[0][0];
  tb = sh[1][0];
  if (threadIdx.x == 0) *ticket = 0;
  return true;
}

// grid-stride sweep of the paired stream of one direction: (a, b) = dot
// products of vector g with the interleaved vector `vec`, handed to epi on lane 0
template <class T, int VS, int UF, int TL, bool FWD, class Epi>
__device__ __forceinline__ void pair_sweep(const SartK<T>& k, long long n,
                                           const typename Vec2<T>::type* __restrict__ vec,
                                           Epi&& epi) {
  const int lane = threadIdx.x & (VS - 1);
  const unsigned mask = group_mask<VS>();
  const int* __restrict__ ptr = FWD ? k.tpf : k.tpb;
  const int* __restrict__ tfp = FWD ? k.tff : k.tfb;
  const int gstep = static_cast<int>((long long)gridDim.x * kThreads / VS);
  int g = static_cast<int>((blockIdx.x * (long long)kThreads + threadIdx.x) / VS);
  const int* __restrict__ ep = FWD ? k.epf : k.epb;
  int beg = 0, end = 0, tf = 0, eb = 0, ee = 0;
  if (g < n) {
    beg = __ldg(ptr + g);
    end = __ldg(ptr + g + 1);
    if (TL >= 2) tf = __ldg(tfp + g);
    if ((TL == 4 || TL == 6) && ep) {
      eb = __ldg(ep + g);
      ee = __ldg(ep + g + 1);
    }
  }
  for (; g < n; g += gstep) {
    const int gn = g + gstep;
    int nbeg = 0, nend = 0, ntf = 0, neb = 0, nee = 0;
    if (gn < n) {
      nbeg = __ldg(ptr + gn);
      nend = __ldg(ptr + gn + 1);
      if (TL >= 2) ntf = __ldg(tfp + gn);
      if ((TL == 4 || TL == 6) && ep) {
        neb = __ldg(ep + gn);
        nee = __ldg(ep + gn + 1);
      }
    }
    T a, b;
    if (TL == 4 || TL == 6) {
      seg_dot2m<T, VS, UF, false, TL == 4>(FWD ? k.tof : k.tob, FWD ? k.tif : k.tib,
                                           FWD ? k.thf : k.thb, tf, FWD ? k.rv2 : k.cv2,
                           vec, beg, end, eb, ee, FWD ? k.eif : k.eib, FWD ? k.evf : k.evb, lane,
                           mask, a, b);
    } else if (TL == 2) {
      seg_dot2c<T, VS, UF>(FWD ? k.tof : k.tob, FWD ? k.tbf : k.tbb, tf, FWD ? k.rv2 : k.cv2,
                           vec, beg, end, lane, mask, a, b);
    } else {
      seg_dot2t<T, VS, UF>(FWD ? k.tif : k.tib, FWD ? k.rv2 : k.cv2, vec, beg, end, lane, mask,
                           a, b);
    }
    if (lane == 0) epi(g, a, b);
    beg = nbeg;
    end = nend;
    tf = ntf;
    eb = neb;
    ee = nee;
  }
}

// q = A d (both systems); alpha = gamma / ||q||^2, or break when ||q|| = 0
template <class T, int VS, int UF, int TL>
__global__ void __launch_bounds__(kThreads, kDirectMinBlocks) cgp_fwd_kernel(CgPairK<T> k) {
  using T2 = typename Vec2<T>::type;
  if (*(volatile const int*)(k.loop + 1)) return;
  const int it = *(volatile const int*)k.loop;
  const bool on0 = cg_on(k.st, 0), on1 = cg_on(k.st, 1);
  double qa = 0.0, qb = 0.0;
  if (on0 || on1) {
    pair_sweep<T, VS, UF, TL, true>(k.sk, k.rows, reinterpret_cast<const T2*>(k.d),
                                    [&](int g, T a, T b) {
      T2 o;
      o.x = a;
      o.y = b;
      reinterpret_cast<T2*>(k.q)[g] = o;
      qa += static_cast<double>(a) * static_cast<double>(a);
      qb += static_cast<double>(b) * static_cast<double>(b);
    });
  }
  double ta, tb;
  if (!two_sums(qa, qb, k.part, k.ticket, ta, tb) || threadIdx.x != 0) return;
  for (int s = 0; s < 2; ++s) {
    if (!cg_on(k.st, s)) continue;
    const double tot = s ? tb : ta;
    double* sc = k.sc + 5 * s;
    int* st = k.st + 5 * s;
    if (tot == 0.0) {
      st[0] = 1;  // d in the null space: break (solvers.cpp:124-126)
    } else {
      const double alpha = sc[0] / tot;
      sc[1] = alpha;
      if (!isfinite(alpha)) {
        st[2] = it + 1;
        st[0] = 1;
      }
    }
  }
}

// x += alpha d, r -= alpha q, ||r||^2 (solvers.cpp:130-131, :142)
template <class T>
__global__ void __launch_bounds__(kThreads) cgp_axpy_kernel(CgPairK<T> k) {
  if (*(volatile const int*)(k.loop + 1)) return;
  const bool on[2] = {cg_on(k.st, 0), cg_on(k.st, 1)};
  if (!on[0] && !on[1]) return;
  const T al[2] = {static_cast<T>(k.sc[1]), static_cast<T>(k.sc[5 + 1])};
  const long long tid = blockIdx.x * (long long)kThreads + threadIdx.x;
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long j = tid; j < 2 * k.cols; j += stride) {
    const int s = static_cast<int>(j & 1);
    if (on[s]) k.x[j] = k.x[j] + al[s] * k.d[j];
  }
  double ra = 0.0, rb = 0.0;
  for (long long i = tid; i < 2 * k.rows; i += stride) {
    const int s = static_cast<int>(i & 1);
    if (!on[s]) continue;
    const T ri = k.r[i] - al[s] * k.q[i];
    k.r[i] = ri;
    const double r2 = static_cast<double>(ri) * static_cast<double>(ri);
    if (s) rb += r2; else ra += r2;
  }
  double ta, tb;
  if (!two_sums(ra, rb, k.part, k.ticket, ta, tb) || threadIdx.x != 0) return;
  if (on[0]) k.sc[4] = ta;
  if (on[1]) k.sc[5 + 4] = tb;
}

// s = A^T r (both systems). init: gamma0 and the stop level (solvers.cpp:
// 115-120); else beta, gamma, history, stop test (:132-141) and the WHILE
// condition of the next pass
template <class T, int VS, int UF, int TL>
__global__ void __launch_bounds__(kThreads, kDirectMinBlocks) cgp_back_kernel(CgPairK<T> k, int init) {
  using T2 = typename Vec2<T>::type;
  if (!init && *(volatile const int*)(k.loop + 1)) return;
  const int it = *(volatile const int*)k.loop;
  const bool on0 = cg_on(k.st, 0), on1 = cg_on(k.st, 1);
  double sa = 0.0, sb = 0.0;
  if (init || on0 || on1) {
    pair_sweep<T, VS, UF, TL, false>(k.sk, k.cols, reinterpret_cast<const T2*>(k.r),
                                     [&](int g, T a, T b) {
      T2 o;
      o.x = a;
      o.y = b;
      reinterpret_cast<T2*>(k.s)[g] = o;
      sa += static_cast<double>(a) * static_cast<double>(a);
      sb += static_cast<double>(b) * static_cast<double>(b);
    });
  }
  double ta, tb;
  if (!two_sums(sa, sb, k.part, k.ticket, ta, tb) || threadIdx.x != 0) return;
  bool any = false;
  for (int s = 0; s < 2; ++s) {
    const double tot = s ? tb : ta;
    double* sc = k.sc + 5 * s;
    int* st = k.st + 5 * s;
    if (init) {
      sc[0] = tot;
      sc[3] = k.tol * sqrt(tot);
      st[1] = 0;
      if (!(sqrt(tot) > sc[3])) st[0] = 1;
    } else if (cg_on(k.st, s)) {
      if (!isfinite(tot)) {
        st[3] = it + 1;
        st[0] = 1;
      } else {
        sc[2] = tot / sc[0];
        sc[0] = tot;
        st[1] = it + 1;
        k.hist[s * k.hstride + it] = sqrt(sc[4]);
        if (!(sqrt(tot) > sc[3])) st[0] = 1;
      }
    }
    any = any || cg_on(k.st, s);
  }
  if (!init) {
    const int nit = it + 1;
    const bool more = any && nit < k.max_iters;
    k.loop[0] = nit;
    k.loop[1] = more ? 0 : 1;
    cudaGraphSetConditional(k.cond, more ? 1u : 0u);
  }
}

// d = s + beta d (d = s before the loop)
template <class T>
__global__ void cgp_dupdate_kernel(CgPairK<T> k, int init) {
  if (!init && *(volatile const int*)(k.loop + 1)) return;
  const bool on[2] = {init || cg_on(k.st, 0), init || cg_on(k.st, 1)};
  const T be[2] = {static_cast<T>(k.sc[2]), static_cast<T>(k.sc[5 + 2])};
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < 2 * k.cols;
       j += (long long)gridDim.x * blockDim.x) {
    const int s = static_cast<int>(j & 1);
    if (on[s]) k.d[j] = init ? k.s[j] : k.s[j] + be[s] * k.d[j];
  }
}

// rhs of system s into slot s of the interleaved r
__global__ void cgp_rhs_kernel(const double* p, long long n, int slot, float* r) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    r[2 * i + slot] = static_cast<float>(p[i]);
  }
}
__global__ void cgp_rhs_kernel(const double* p, long long n, int slot, double* r) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    r[2 * i + slot] = p[i];
  }
}

template <class T>
__global__ void cgp_out_kernel(const T* x, long long n, double* f0, double* f1) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    f0[j] = static_cast<double>(x[2 * j]);
    f1[j] = static_cast<double>(x[2 * j + 1]);
  }
}

constexpr int kCgPassesPerBody = 4;  // passes unrolled per WHILE-body execution

template <class T>
void run_cgls_pair(Plan& P, const double* p[2], const ss_solve_options& o, double* f[2],
                   ss_solve_report rep[2], std::string errs[2], int codes[2]) {
  Context* ctx = P.ctx;
  const long long rows = P.rows[0], cols = P.cols[0];
  DBuf<T> x(2 * cols), r(2 * rows), sv(2 * cols), d(2 * cols), q(2 * rows);
  const int gv = grid1(ctx, 2 * std::max(rows, cols));
  const int grid = std::max({P.fwd_blocks, P.back_blocks, gv});
  DBuf<double> part(2 * static_cast<std::size_t>(grid)), sc(10), hist(2 * (o.max_iters + 1));
  DBuf<int> st(10), loop(2);
  DBuf<unsigned> ticket(1);
  CgPairK<T> k{};
  k.sk = make_args<T>(P);
  k.x = x.get();
  k.r = r.get();
  k.s = sv.get();
  k.d = d.get();
  k.q = q.get();
  k.rows = rows;
  k.cols = cols;
  k.part = part.get();
  k.sc = sc.get();
  k.st = st.get();
  k.loop = loop.get();
  k.ticket = ticket.get();
  k.hist = hist.get();
  k.hstride = o.max_iters + 1;
  k.tol = o.tol;
  k.max_iters = o.max_iters;
  // kernels of this plan's layout
  void (*fwd)(CgPairK<T>) = nullptr;
  void (*back)(CgPairK<T>, int) = nullptr;
  const int vsf = P.vs_fwd, vsb = P.vs_back;
  const int mf = P.mir_f ? (P.c16f ? 4 : 6) : (P.c16f ? 2 : 1);
  const int mb = P.mir_b ? (P.c16b ? 4 : 6) : (P.c16b ? 2 : 1);
#define SSB_CGF(V, M) if (vsf == V && mf == M) fwd = cgp_fwd_kernel<T, V, 4, M>;
#define SSB_CGB(V, M) if (vsb == V && mb == M) back = cgp_back_kernel<T, V, 2, M>;
  SSB_CGF(4, 1) SSB_CGF(8, 1) SSB_CGF(16, 1) SSB_CGF(32, 1)
  SSB_CGF(4, 2) SSB_CGF(8, 2) SSB_CGF(16, 2) SSB_CGF(32, 2)
  SSB_CGF(4, 4) SSB_CGF(8, 4) SSB_CGF(16, 4) SSB_CGF(32, 4)
  SSB_CGF(4, 6) SSB_CGF(8, 6) SSB_CGF(16, 6) SSB_CGF(32, 6)
  SSB_CGB(4, 1) SSB_CGB(8, 1) SSB_CGB(16, 1) SSB_CGB(32, 1)
  SSB_CGB(4, 2) SSB_CGB(8, 2) SSB_CGB(16, 2) SSB_CGB(32, 2)
  SSB_CGB(4, 4) SSB_CGB(8, 4) SSB_CGB(16, 4) SSB_CGB(32, 4)
  SSB_CGB(4, 6) SSB_CGB(8, 6) SSB_CGB(16, 6) SSB_CGB(32, 6)
#undef SSB_CGF
#undef SSB_CGB
  if (!fwd || !back) fail("cgls: unsupported paired kernel shape");
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  SSB_CUDA(cudaGraphCreate(&g, 0));
  cudaStreamCaptureStatus cs;
  try {
    SSB_CUDA(cudaGraphConditionalHandleCreate(&k.cond, g, 1, cudaGraphCondAssignDefault));
    SSB_CUDA(cudaStreamBeginCaptureToGraph(ctx->stream, g, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    SSB_CUDA(cudaMemsetAsync(x.get(), 0, 2 * cols * sizeof(T), ctx->stream));
    SSB_CUDA(cudaMemsetAsync(st.get(), 0, 10 * sizeof(int), ctx->stream));
    SSB_CUDA(cudaMemsetAsync(loop.get(), 0, 2 * sizeof(int), ctx->stream));
    SSB_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned), ctx->stream));
    for (int s = 0; s < 2; ++s) {
      cgp_rhs_kernel<<<grid1(ctx, rows), 256, 0, ctx->stream>>>(p[s], rows, s, r.get());
    }
    back<<<P.back_blocks, kThreads, 0, ctx->stream>>>(k, 1);
    cgp_dupdate_kernel<T><<<gv, 256, 0, ctx->stream>>>(k, 1);
    const cudaGraphNode_t* deps = nullptr;
    std::size_t nd = 0;
    SSB_CUDA(cudaStreamGetCaptureInfo(ctx->stream, &cs, nullptr, nullptr, &deps, &nd));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = k.cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    SSB_CUDA(cudaGraphAddNode(&cnode, g, deps, nd, &cp));
    SSB_CUDA(cudaStreamUpdateCaptureDependencies(ctx->stream, &cnode, 1,
                                                 cudaStreamSetCaptureDependencies));
    SSB_CUDA(cudaStreamEndCapture(ctx->stream, &g));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    SSB_CUDA(cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    for (int pass = 0; pass < std::min(o.max_iters, kCgPassesPerBody); ++pass) {
      fwd<<<P.fwd_blocks, kThreads, 0, ctx->stream>>>(k);
      cgp_axpy_kernel<T><<<gv, kThreads, 0, ctx->stream>>>(k);
      back<<<P.back_blocks, kThreads, 0, ctx->stream>>>(k, 0);
      cgp_dupdate_kernel<T><<<gv, 256, 0, ctx->stream>>>(k, 0);
    }
    SSB_CUDA(cudaStreamEndCapture(ctx->stream, &body));
    SSB_CUDA(cudaGraphInstantiate(&ge, g, 0));
  } catch (...) {
    if (cudaStreamIsCapturing(ctx->stream, &cs) == cudaSuccess &&
        cs != cudaStreamCaptureStatusNone) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(ctx->stream, &junk);
      if (junk && junk != g) cudaGraphDestroy(junk);
    }
    cudaGraphDestroy(g);
    throw;
  }
  cudaGraphDestroy(g);
  cudaEvent_t e0, e1;
  SSB_CUDA(cudaEventCreate(&e0));
  SSB_CUDA(cudaEventCreate(&e1));
  SSB_CUDA(cudaEventRecord(e0, ctx->stream));
  SSB_CUDA(cudaGraphLaunch(ge, ctx->stream));
  SSB_CUDA(cudaEventRecord(e1, ctx->stream));
  SSB_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  SSB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaGraphExecDestroy(ge);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  int hs[10];
  int passes = 0;
  ctx->copy(hs, st.get(), sizeof hs);
  ctx->copy(&passes, loop.get(), sizeof(int));
  ctx->launches += 4 + 4LL * std::max(passes, 1);
  for (int s = 0; s < 2; ++s) {
    const int* h = hs + 5 * s;
    if (h[2]) {
      errs[s] = "cgls_solve: diverged (non-finite step at iteration " + std::to_string(h[2]) + ")";
      codes[s] = SS_ERR_DIVERGED;
    } else if (h[3]) {
      errs[s] = "cgls_solve: diverged (non-finite residual at iteration " + std::to_string(h[3]) + ")";
      codes[s] = SS_ERR_DIVERGED;
    }
    rep[s].iterations = h[1];
    rep[s].history_len = h[1];
    rep[s].wall_time_seconds = ms * 1e-3;
  }
  cgp_out_kernel<T><<<grid1(ctx, cols), 256, 0, ctx->stream>>>(x.get(), cols, f[0], f[1]);
  ctx->check_launch("cgp_out_kernel");
  ctx->sync();
}

}  // namespace

// both folded systems' CGLS in one loop over the paired streams
void cgls_device_paired(Matrix* a1, Matrix* a2, const double* p[2], const ss_solve_options& o,
                        double* f[2], ss_solve_report rep[2], std::string errs[2], int codes[2]) {
  if (o.tol <= 0) fail("cgls_solve: tol must be positive");
  if (o.max_iters < 1) fail("cgls_solve: max_iters must be >= 1");
  ss_solve_options so = o;
  so.relaxation = 1.0;  // unused by CGLS; the plan builder validates it
  so.method = SS_METHOD_SART;
  so.tol = 0.0;
  std::unique_ptr<Plan> P(make_plan(a1->ctx, a1, a2, so, 1, false));
  if (!P->paired || !P->tiled) fail("cgls: paired tiled streams unavailable");
  if (o.dtype == SS_F32) run_cgls_pair<float>(*P, p, o, f, rep, errs, codes);
  else run_cgls_pair<double>(*P, p, o, f, rep, errs, codes);
}

}  // namespace ssb
