// Device operations of the build side of the path: Siddon tracer, CSR/CSC
// construction, centrosymmetric fold, symmetry check, normalisers, phantom
// rasterisation and folded forward projection.
//
// Bit-exactness contract: every floating-point operation
// here reproduces the reference's scalar expression with round-to-nearest
// and no contraction. The file is compiled with -fmad=false and the
// arithmetic is spelled with __d*_rn intrinsics so that a flag change cannot
// silently introduce an FMA. Integer/index work is exact by construction.
#include <cub/cub.cuh>

#include <algorithm>
#include <limits>
#include <cmath>

#include "internal.hpp"

namespace ssb {

cudaStream_t& alloc_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}

namespace {

constexpr int kT = 256;

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

int grid_for(Context* ctx, std::int64_t n, int threads = kT) {
  const std::int64_t want = (n + threads - 1) / threads;
  const std::int64_t cap = static_cast<std::int64_t>(ctx->sm_count) * 16;
  return static_cast<int>(std::max<std::int64_t>(1, std::min(want, cap)));
}

int bits_for(std::int64_t v) {  // bits needed to represent values in [0, v)
  int b = 1;
  while ((std::int64_t{1} << b) < v) ++b;
  return b;
}

// ------------------------------------------------------------------ tracer
struct TraceArgs {
  const double *sx, *sy, *dx, *dy, *seg, *tin, *tout;
  const double *xb, *yb;  // boundary abscissae k = 0..n_x, ordinates k = 0..n_y
  int nx, ny;
  double vs, x_left, y_bottom;
  std::int64_t mh;
};

// Next parametric crossing of one axis strictly inside (t_in, t_out), or +inf.
// The boundary sequence is monotone in k and so is (b_k - p0)/d, hence the
// in-range candidates are one contiguous run that this cursor walks in
// increasing t (reference collects all k and std::sorts; equal values are
// bitwise identical so their relative order cannot matter).
struct AxisCursor {
  const double* b;
  double p0, d, tin, tout;
  int k, kend, step;
  __device__ double next() {
    while (k != kend) {
      const double t = dvd(sub(b[k], p0), d);
      k += step;
      if (t > tin) {
        if (t < tout) return t;
        k = kend;
        break;
      }
    }
    return __longlong_as_double(0x7ff0000000000000LL);
  }
};

// Walk of reference ray_weights (geometry.cpp:175-225) for traced ray i:
// sorted crossings -> per-segment midpoint cell -> snake column, lengths
// of consecutive equal cells merged with +=. emit(col0, len) per entry.
template <class Emit>
__device__ void walk_ray(const TraceArgs& a, std::int64_t i, Emit&& emit) {
  const double sx = a.sx[i], sy = a.sy[i], dx = a.dx[i], dy = a.dy[i];
  const double seg = a.seg[i], tin = a.tin[i], tout = a.tout[i];
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  AxisCursor cx{a.xb, sx, dx, tin, tout, 0, 0, 1};
  if (dx > 0.0) {
    cx.k = 0; cx.kend = a.nx + 1; cx.step = 1;
  } else if (dx < 0.0) {
    cx.k = a.nx; cx.kend = -1; cx.step = -1;
  }
  AxisCursor cy{a.yb, sy, dy, tin, tout, 0, 0, 1};
  if (dy > 0.0) {
    cy.k = 0; cy.kend = a.ny + 1; cy.step = 1;
  } else if (dy < 0.0) {
    cy.k = a.ny; cy.kend = -1; cy.step = -1;
  }
  double tx = cx.next(), ty = cy.next();
  double ta = tin;
  int pc = -1;
  double plen = 0.0;
  for (;;) {
    double tb;
    bool last = false;
    if (tx <= ty) {
      if (tx == INF) {
        tb = tout;
        last = true;
      } else {
        tb = tx;
        tx = cx.next();
      }
    } else {
      tb = ty;
      ty = cy.next();
    }
    if (tb > ta) {
      const double tm = mul(0.5, add(ta, tb));
      const double xm = add(sx, mul(tm, dx));
      const double ym = add(sy, mul(tm, dy));
      int c = static_cast<int>(floor(dvd(sub(xm, a.x_left), a.vs)));
      c = min(max(c, 0), a.nx - 1);
      int fb = static_cast<int>(floor(dvd(sub(ym, a.y_bottom), a.vs)));
      fb = min(max(fb, 0), a.ny - 1);
      // snake_index(c+1, n_y-fb) - 1: odd 1-based columns run top->bottom
      const int col = (c & 1) ? c * a.ny + fb : c * a.ny + (a.ny - 1 - fb);
      const double len = mul(sub(tb, ta), seg);
      if (col == pc) {
        plen = add(plen, len);
      } else {
        if (pc >= 0) emit(pc, plen);
        pc = col;
        plen = len;
      }
    }
    ta = tb;
    if (last) break;
  }
  if (pc >= 0) emit(pc, plen);
}

__global__ void trace_count_kernel(TraceArgs a, int* counts) {
  for (std::int64_t i = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; i < a.mh;
       i += (std::int64_t)gridDim.x * blockDim.x) {
    int n = 0;
    walk_ray(a, i, [&](int, double) { ++n; });
    counts[i] = n;
  }
}

__global__ void trace_fill_kernel(TraceArgs a, const std::int64_t* offsets,
                                  unsigned long long* keys, double* vals) {
  for (std::int64_t i = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; i < a.mh;
       i += (std::int64_t)gridDim.x * blockDim.x) {
    std::int64_t o = offsets[i];
    const unsigned long long rowkey = static_cast<unsigned long long>(i) << 32;
    walk_ray(a, i, [&](int col, double len) {
      keys[o] = rowkey | static_cast<unsigned int>(col);
      vals[o] = len;
      ++o;
    });
  }
}

// ------------------------------------------------------------------ sorted triplets -> CSR
__global__ void head_flags_kernel(const unsigned long long* keys, std::int64_t n, int* head) {
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    head[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1 : 0;
  }
}

// Repeated (row,col) runs are summed left to right in stable (insertion)
// order — Eigen collapseDuplicates: first slot kept, value = acc + next.
__global__ void collapse_kernel(const unsigned long long* keys, const double* vals,
                                const int* head, const std::int64_t* pos, std::int64_t n,
                                int* col_out, int* row_out, double* val_out) {
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    if (!head[k]) continue;
    double acc = vals[k];
    std::int64_t e = k + 1;
    while (e < n && keys[e] == keys[k]) {
      acc = add(acc, vals[e]);
      ++e;
    }
    const std::int64_t o = pos[k];
    col_out[o] = static_cast<int>(keys[k] & 0xffffffffull);
    row_out[o] = static_cast<int>(keys[k] >> 32);
    val_out[o] = acc;
  }
}

__global__ void split_keys_kernel(const unsigned long long* keys, std::int64_t n, int* col_out,
                                  int* row_out) {
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    col_out[k] = static_cast<int>(keys[k] & 0xffffffffull);
    row_out[k] = static_cast<int>(keys[k] >> 32);
  }
}

// ptr[r] = first position whose (sorted) outer index is >= r.
__global__ void ptr_from_sorted_kernel(const int* outer_of, std::int64_t n, std::int64_t outer,
                                       int* ptr) {
  for (std::int64_t u = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; u <= n;
       u += (std::int64_t)gridDim.x * blockDim.x) {
    const std::int64_t prev = (u == 0) ? -1 : outer_of[u - 1];
    const std::int64_t cur = (u == n) ? outer : outer_of[u];
    for (std::int64_t r = prev + 1; r <= cur; ++r) ptr[r] = static_cast<int>(u);
  }
}

__global__ void iota_kernel(int* v, std::int64_t n) {
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    v[k] = static_cast<int>(k);
  }
}

__global__ void expand_ptr_kernel(const int* ptr, std::int64_t outer, int* outer_of) {
  for (std::int64_t r = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; r < outer;
       r += (std::int64_t)gridDim.x * blockDim.x) {
    for (int k = ptr[r]; k < ptr[r + 1]; ++k) outer_of[k] = static_cast<int>(r);
  }
}

__global__ void gather_kernel(const int* perm, const int* src_idx, const double* src_val,
                              std::int64_t n, int* dst_idx, double* dst_val) {
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    const int s = perm[k];
    dst_idx[k] = src_idx[s];
    dst_val[k] = src_val[s];
  }
}

// Full A from the traced half by the mirror rule (geometry.cpp:257-269):
// row M-1-i holds (N-1-j, len) of row i, so the mirrored half of the CSR
// arrays is the traced half reversed with columns reflected.
__global__ void mirror_fill_kernel(int* col, double* val, std::int64_t half, std::int64_t n) {
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < half;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    const std::int64_t d = 2 * half - 1 - k;
    col[d] = static_cast<int>(n - 1 - col[k]);
    val[d] = val[k];
  }
}

__global__ void mirror_ptr_kernel(int* ptr, std::int64_t mh, std::int64_t half) {
  // ptr[mh + t] = 2H - ptr[mh - t] for t = 1..mh
  for (std::int64_t t = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x + 1; t <= mh;
       t += (std::int64_t)gridDim.x * blockDim.x) {
    ptr[mh + t] = static_cast<int>(2 * half - ptr[mh - t]);
  }
}

template <class T>
__global__ void cast_kernel(const double* s, T* d, std::int64_t n) {
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    d[k] = static_cast<T>(s[k]);
  }
}

__global__ void finite_kernel(const double* v, std::int64_t n, int* bad) {
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    if (!isfinite(v[k])) atomicOr(bad, 1);
  }
}

__global__ void count_nonzero_kernel(const double* v, std::int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    c += v[k] != 0.0 ? 1ull : 0ull;
  }
  using BR = cub::BlockReduce<unsigned long long, kT>;
  __shared__ typename BR::TempStorage tmp;
  c = BR(tmp).Sum(c);
  if (threadIdx.x == 0 && c) atomicAdd(out, c);
}

// ------------------------------------------------------------------ symmetry
// Row i against the reflected row M-1-i (centro.cpp:46-66): for every stored
// (i,j,v), d = |v - a(M-1-i, N-1-j)| (0 if absent; the mirror coefficient is
// found by binary search in the mirror row, like SparseMatrix::coeff). Keeps
// the row maximum and the smallest column reaching it — the first entry in
// column-major order with strict '>'. One warp per row.
constexpr int kSymCap = 1536;  // mirror-row columns staged per warp (6 KB)

__global__ void symmetry_rows_kernel(const int* ptr, const int* col, const double* val,
                                     std::int64_t m, std::int64_t n, double* rmax, int* rarg) {
  extern __shared__ int sym_sm[];
  int* wsm = sym_sm + (threadIdx.x >> 5) * kSymCap;
  const int lane = threadIdx.x & 31;
  const std::int64_t w0 = (blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x) >> 5;
  const std::int64_t nw = ((std::int64_t)gridDim.x * blockDim.x) >> 5;
  for (std::int64_t i = w0; i < m; i += nw) {
    const std::int64_t mi = m - 1 - i;
    const int mb = ptr[mi], me = ptr[mi + 1];
    // the mirror row's columns in shared memory when they fit: the per-entry
    // binary searches then run at shared-memory latency
    const int* mc = col;
    __syncwarp();
    if (me - mb <= kSymCap) {
      for (int q = lane; q < me - mb; q += 32) wsm[q] = col[mb + q];
      __syncwarp();
      mc = wsm - mb;
    }
    double best = 0.0;
    int arg = 0x7fffffff;
    for (int k = ptr[i] + lane; k < ptr[i + 1]; k += 32) {
      const int j = col[k];
      const std::int64_t target = n - 1 - j;
      int lo = mb, hi = me;
      while (lo < hi) {
        const int mid = lo + ((hi - lo) >> 1);
        if (mc[mid] < target) lo = mid + 1; else hi = mid;
      }
      const double mv = (lo < me && mc[lo] == target) ? val[lo] : 0.0;
      const double d = fabs(sub(val[k], mv));
      if (d > best) {  // entries of a lane ascend in j: first maximum kept
        best = d;
        arg = j;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, off);
      if (ob > best || (ob == best && oa < arg)) {
        best = ob;
        arg = oa;
      }
    }
    if (lane == 0) {
      rmax[i] = best;
      rarg[i] = best > 0.0 ? arg : -1;
    }
  }
}

struct Worst {
  double d;
  int j;
  long long i;
};

__device__ __forceinline__ bool better(const Worst& a, const Worst& b) {
  if (a.d != b.d) return a.d > b.d;
  if (a.j != b.j) return a.j < b.j;
  return a.i < b.i;
}

__global__ void symmetry_reduce_kernel(const double* rmax, const int* rarg, std::int64_t m,
                                       Worst* out) {
  __shared__ Worst sh[1024];
  Worst w{0.0, 0x7fffffff, 0x7fffffffffffffffLL};
  for (std::int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    if (rarg[i] >= 0) {
      Worst c{rmax[i], rarg[i], i};
      if (better(c, w)) w = c;
    }
  }
  sh[threadIdx.x] = w;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s && better(sh[threadIdx.x + s], sh[threadIdx.x])) {
      sh[threadIdx.x] = sh[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// worst (value, column, row) over the fold's per-output-row candidates
__global__ void symmetry_reduce3_kernel(const double* d, const int* j, const int* i,
                                        std::int64_t n, Worst* out) {
  __shared__ Worst sh[1024];
  Worst w{0.0, 0x7fffffff, 0x7fffffffffffffffLL};
  for (std::int64_t t = threadIdx.x; t < n; t += blockDim.x) {
    if (j[t] >= 0) {
      Worst c{d[t], j[t], i[t]};
      if (better(c, w)) w = c;
    }
  }
  sh[threadIdx.x] = w;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s && better(sh[threadIdx.x + s], sh[threadIdx.x])) {
      sh[threadIdx.x] = sh[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// ------------------------------------------------------------------ fold
struct FoldArgs {
  const int* ptr;
  const int* col;
  const double* val;
  std::int64_t m, n, mh, nh;
  const int* ptr1;  // fill pass: output row pointers
  const int* ptr2;
  int* cnt1;        // per-lane bucket counts [mh][32] (count pass out, fill pass in)
  int* cnt2;
  int* rcnt1;       // per-row counts (count pass)
  int* rcnt2;
  int* col1;
  double* val1;
  int* col2;
  double* val2;
  // count pass, optional: the symmetry check fused into the merge (per output
  // row bi the worst violation of rows bi and M-1-bi: value, column, row)
  double* sym_d;
  int* sym_j;
  int* sym_i;
};

__device__ __forceinline__ int first_at_least(const int* col, int b, int e, std::int64_t v) {
  while (b < e) {
    const int mid = b + ((e - b) >> 1);
    if (col[mid] < v) b = mid + 1; else e = mid;
  }
  return b;
}

// Output row bi merges the four quadrant streams of buckets (bi, bj):
// TL = a(bi,bj), BL = a(M-1-bi,bj), TR = a(bi,N-1-bj), BR = a(M-1-bi,N-1-bj)
// (centro.cpp:109-128 visits them in this column-major triplet order). Each
// term enters as h = 0.5*v (A1 signs +,-,-,+; A2 all +), summed left to right
// from the first present term, then exact zeros (either sign) are pruned.
// One warp per output row: the row's bucket range is cut into 32 equal bj
// segments, lane q merges segment q (cursors placed by binary search). The
// count pass records per-lane counts; the fill pass writes each lane's
// buckets at the row offset plus the exclusive prefix of the lanes before it,
// so the output is sorted by bj exactly as a sequential merge would be.
// Column indices of the two source rows are staged in shared memory (when
// they fit) so the 32 per-lane merges chase indices at shared-memory latency.
constexpr int kFoldCap = 1536;  // staged columns per warp (6 KB; 48 KB per 256-thread block)

template <bool FILL>
__global__ void fold_kernel(FoldArgs a) {
  extern __shared__ int fold_sm[];
  int* wsm = fold_sm + (threadIdx.x >> 5) * kFoldCap;
  const int lane = threadIdx.x & 31;
  const std::int64_t w0 = (blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x) >> 5;
  const std::int64_t nw = ((std::int64_t)gridDim.x * blockDim.x) >> 5;
  const std::int64_t nm1 = a.n - 1;
  for (std::int64_t bi = w0; bi < a.mh; bi += nw) {
    const std::int64_t top = bi, bot = a.m - 1 - bi;
    const int tb = a.ptr[top], te = a.ptr[top + 1];
    const int bb = a.ptr[bot], be = a.ptr[bot + 1];
    const int* ct = a.col;  // column lists of the top / bottom row
    const int* cb = a.col;
    const int lt = te - tb, lb = be - bb;
    __syncwarp();  // previous row's reads of the staging area are done
    if (lt + lb <= kFoldCap) {
      for (int q = lane; q < lt; q += 32) wsm[q] = a.col[tb + q];
      for (int q = lane; q < lb; q += 32) wsm[lt + q] = a.col[bb + q];
      __syncwarp();
      ct = wsm - tb;
      cb = wsm + lt - bb;
    }
    const int tmid = first_at_least(ct, tb, te, a.nh);  // first TR entry of top
    const int bmid = first_at_least(cb, bb, be, a.nh);
    // bucket span of the row (all four lists)
    std::int64_t lo = a.nh, hi = -1;
    if (tmid > tb) { lo = min(lo, (std::int64_t)ct[tb]); hi = max(hi, (std::int64_t)ct[tmid - 1]); }
    if (bmid > bb) { lo = min(lo, (std::int64_t)cb[bb]); hi = max(hi, (std::int64_t)cb[bmid - 1]); }
    if (te > tmid) { lo = min(lo, nm1 - ct[te - 1]); hi = max(hi, nm1 - ct[tmid]); }
    if (be > bmid) { lo = min(lo, nm1 - cb[be - 1]); hi = max(hi, nm1 - cb[bmid]); }
    int n1 = 0, n2 = 0;
    double wd = 0.0;  // fused symmetry check: worst (value, column, row) of this lane
    std::int64_t wj = 0x7fffffff, wi = 0x7fffffffffffffffLL;
    if (hi >= lo) {
      const std::int64_t span = hi - lo + 1;
      const std::int64_t s_lo = lo + span * lane / 32, s_hi = lo + span * (lane + 1) / 32;
      // TL/BL: columns in [s_lo, s_hi); TR/BR: columns in [n-s_hi, n-1-s_lo], walked down
      int tl = first_at_least(ct, tb, tmid, s_lo);
      const int tl_end = first_at_least(ct, tl, tmid, s_hi);
      int bl = first_at_least(cb, bb, bmid, s_lo);
      const int bl_end = first_at_least(cb, bl, bmid, s_hi);
      const int tr_stop = first_at_least(ct, tmid, te, a.n - s_hi);
      int tr = first_at_least(ct, tr_stop, te, a.n - s_lo) - 1;
      const int br_stop = first_at_least(cb, bmid, be, a.n - s_hi);
      int br = first_at_least(cb, br_stop, be, a.n - s_lo) - 1;
      int o1 = 0, o2 = 0;
      if (FILL) {
        const int c1 = a.cnt1[bi * 32 + lane], c2 = a.cnt2[bi * 32 + lane];
        int x1 = c1, x2 = c2;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int y1 = __shfl_up_sync(0xffffffffu, x1, off);
          const int y2 = __shfl_up_sync(0xffffffffu, x2, off);
          if (lane >= off) {
            x1 += y1;
            x2 += y2;
          }
        }
        o1 = a.ptr1[bi] + x1 - c1;
        o2 = a.ptr2[bi] + x2 - c2;
      }
      for (;;) {
        std::int64_t bj = s_hi;
        if (tl < tl_end) bj = min(bj, (std::int64_t)ct[tl]);
        if (bl < bl_end) bj = min(bj, (std::int64_t)cb[bl]);
        if (tr >= tr_stop) bj = min(bj, nm1 - ct[tr]);
        if (br >= br_stop) bj = min(bj, nm1 - cb[br]);
        if (bj == s_hi) break;
        bool have = false;
        double s1 = 0.0, s2 = 0.0;
        auto term = [&](double v, bool neg) {
          const double h = mul(0.5, v);
          const double t1 = neg ? -h : h;
          if (!have) {
            s1 = t1;
            s2 = h;
            have = true;
          } else {
            s1 = add(s1, t1);
            s2 = add(s2, h);
          }
        };
        const bool hTL = tl < tl_end && ct[tl] == bj;
        const bool hBL = bl < bl_end && cb[bl] == bj;
        const bool hTR = tr >= tr_stop && nm1 - ct[tr] == bj;
        const bool hBR = br >= br_stop && nm1 - cb[br] == bj;
        const double vTL = hTL ? a.val[tl++] : 0.0, vBL = hBL ? a.val[bl++] : 0.0;
        const double vTR = hTR ? a.val[tr--] : 0.0, vBR = hBR ? a.val[br--] : 0.0;
        if (hTL) term(vTL, false);
        if (hBL) term(vBL, true);
        if (hTR) term(vTR, true);
        if (hBR) term(vBR, false);
        if (!FILL && a.sym_d) {
          // verify_symmetry's per-entry test (centro.cpp:27-42): every stored
          // entry against its mirror (absent = 0); TL<->BR and BL<->TR pair up
          const auto cand = [&](bool h, double v, double mv, std::int64_t j, std::int64_t i) {
            if (!h) return;
            const double d = fabs(sub(v, mv));
            if (d > 0.0 && (d > wd || (d == wd && (j < wj || (j == wj && i < wi))))) {
              wd = d;
              wj = j;
              wi = i;
            }
          };
          cand(hTL, vTL, vBR, bj, top);
          cand(hBR, vBR, vTL, nm1 - bj, bot);
          cand(hBL, vBL, vTR, bj, bot);
          cand(hTR, vTR, vBL, nm1 - bj, top);
        }
        if (s1 != 0.0) {
          if (FILL) {
            a.col1[o1] = static_cast<int>(bj);
            a.val1[o1] = s1;
            ++o1;
          }
          ++n1;
        }
        if (s2 != 0.0) {
          if (FILL) {
            a.col2[o2] = static_cast<int>(bj);
            a.val2[o2] = s2;
            ++o2;
          }
          ++n2;
        }
      }
    }
    if (!FILL && a.sym_d) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, wd, off);
        const long long oj = __shfl_xor_sync(0xffffffffu, static_cast<long long>(wj), off);
        const long long oi = __shfl_xor_sync(0xffffffffu, static_cast<long long>(wi), off);
        if (od > wd || (od == wd && (oj < wj || (oj == wj && oi < wi)))) {
          wd = od;
          wj = oj;
          wi = oi;
        }
      }
      if (lane == 0) {
        a.sym_d[bi] = wd;
        a.sym_j[bi] = wd > 0.0 ? static_cast<int>(wj) : -1;
        a.sym_i[bi] = static_cast<int>(wi);
      }
    }
    if (!FILL) {
      a.cnt1[bi * 32 + lane] = n1;
      a.cnt2[bi * 32 + lane] = n2;
      int t1 = n1, t2 = n2;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        t1 += __shfl_xor_sync(0xffffffffu, t1, off);
        t2 += __shfl_xor_sync(0xffffffffu, t2, off);
      }
      if (lane == 0) {
        a.rcnt1[bi] = t1;
        a.rcnt2[bi] = t2;
      }
    }
  }
}

// ------------------------------------------------------------------ small vectors
__global__ void split_rhs_kernel(const double* p, double* p1, double* p2, std::int64_t mh) {
  for (std::int64_t i = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; i < mh;
       i += (std::int64_t)gridDim.x * blockDim.x) {
    const double a = p[i], b = p[2 * mh - 1 - i];
    p1[i] = sub(a, b);
    p2[i] = add(a, b);
  }
}

// f[s*N + j] = (f2+f1)/2, f[s*N + N-1-j] = (f2-f1)/2 with f1/f2 laid out
// [nh][nrhs] (centro.cpp:170-185).
__global__ void recombine_kernel(const double* f1, const double* f2, double* f, std::int64_t nh,
                                 std::int64_t nrhs) {
  const std::int64_t total = nh * nrhs;
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < total;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    const std::int64_t j = k / nrhs, s = k % nrhs;
    const double a = f1[k], b = f2[k];
    f[s * 2 * nh + j] = mul(0.5, add(b, a));
    f[s * 2 * nh + 2 * nh - 1 - j] = mul(0.5, sub(b, a));
  }
}

__global__ void decompose_kernel(const double* f, double* f1, double* f2, std::int64_t nh) {
  for (std::int64_t j = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; j < nh;
       j += (std::int64_t)gridDim.x * blockDim.x) {
    const double a = f[j], b = f[2 * nh - 1 - j];
    f1[j] = sub(a, b);
    f2[j] = add(a, b);
  }
}

// Sum of |v| over a compressed outer vector in stored (ascending) order —
// the reference accumulates row_sums[i] and col_sums[j] in column-major
// for_each order (solvers.cpp:156-160), i.e. ascending j per row and
// ascending i per column, starting from 0.0.
__global__ void abs_sum_kernel(const int* ptr, const double* val, std::int64_t outer, double* out) {
  for (std::int64_t r = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; r < outer;
       r += (std::int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = ptr[r]; k < ptr[r + 1]; ++k) s = add(s, fabs(val[k]));
    out[r] = s;
  }
}

// y[i] (-= p[i]) = sum_k val*x over row i, warp per row (residual / apply).
__global__ void csr_apply_kernel(const int* ptr, const int* col, const double* val,
                                 const double* x, const double* p, std::int64_t m, double* y) {
  const int lane = threadIdx.x & 31;
  const std::int64_t warp = (blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x) >> 5;
  const std::int64_t nw = ((std::int64_t)gridDim.x * blockDim.x) >> 5;
  for (std::int64_t i = warp; i < m; i += nw) {
    double s = 0.0;
    for (int k = ptr[i] + lane; k < ptr[i + 1]; k += 32) s = add(s, mul(val[k], x[col[k]]));
    for (int o = 16; o > 0; o >>= 1) s = add(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (lane == 0) y[i] = p ? sub(s, p[i]) : s;
  }
}

__global__ void sq_partial_kernel(const double* v, std::int64_t n, double* part) {
  double s = 0.0;
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    s = add(s, mul(v[k], v[k]));
  }
  using BR = cub::BlockReduce<double, kT, cub::BLOCK_REDUCE_RAKING_COMMUTATIVE_ONLY>;
  __shared__ typename BR::TempStorage tmp;
  s = BR(tmp).Sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_partial_kernel(const double* v, std::int64_t n, double* part) {
  double s = 0.0;
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    s = add(s, v[k]);
  }
  using BR = cub::BlockReduce<double, kT, cub::BLOCK_REDUCE_RAKING_COMMUTATIVE_ONLY>;
  __shared__ typename BR::TempStorage tmp;
  s = BR(tmp).Sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void max_partial_kernel(const double* v, std::int64_t n, double* part) {
  double s = -__longlong_as_double(0x7ff0000000000000LL);
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    s = fmax(s, v[k]);
  }
  using BR = cub::BlockReduce<double, kT>;
  __shared__ typename BR::TempStorage tmp;
  s = BR(tmp).Reduce(s, cub::Max());
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// ------------------------------------------------------------------ phantom
struct EllipseDev {
  double x0, y0, a, b, ca, sa, density;
};

struct RasterArgs {
  const EllipseDev* e;
  int count, nx, ny;
  double vs, center_x, y_bottom, half_w, half_h, y_mid;
  double* out;
};

// reference phantom.cpp:34-58 with Ellipse::contains (:8-16); cos/sin of the
// ellipse angle come from the host libm.
__global__ void rasterize_kernel(RasterArgs a) {
  const std::int64_t total = static_cast<std::int64_t>(a.nx) * a.ny;
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < total;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(k / a.ny) + 1;  // 1-based column
    const int r = static_cast<int>(k % a.ny) + 1;  // 1-based row
    const double x = add(a.center_x, mul(sub(static_cast<double>(c) - 0.5, 0.5 * a.nx), a.vs));
    const double y = add(a.y_bottom, mul(static_cast<double>(a.ny - r) + 0.5, a.vs));
    const double u = dvd(sub(x, a.center_x), a.half_w);
    const double v = dvd(sub(y, a.y_mid), a.half_h);
    double value = 0.0;
    for (int q = 0; q < a.count; ++q) {
      const EllipseDev& e = a.e[q];
      const double dx = sub(u, e.x0), dy = sub(v, e.y0);
      const double uu = dvd(add(mul(dx, e.ca), mul(dy, e.sa)), e.a);
      const double vv = dvd(add(mul(-dx, e.sa), mul(dy, e.ca)), e.b);
      if (add(mul(uu, uu), mul(vv, vv)) <= 1.0) value = add(value, e.density);
    }
    const int base = (c - 1) * a.ny;
    const int j = (c & 1) ? base + r : base + (a.ny - r + 1);
    a.out[j - 1] = value;
  }
}

// reference phantom.cpp:75-104: two-pointer walk pairing column j with its
// mirror N-1-j so a centrosymmetric A maps mirror images to mirror data.
__global__ void forward_project_kernel(const int* ptr, const int* col, const double* val,
                                       const double* f, std::int64_t m, std::int64_t n,
                                       double* p) {
  for (std::int64_t i = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; i < m;
       i += (std::int64_t)gridDim.x * blockDim.x) {
    const std::int64_t begin = ptr[i], end = ptr[i + 1];
    double acc = 0.0;
    std::int64_t l = begin, r = end - 1;
    while (l <= r && l < end) {
      const std::int64_t cl = col[l];
      const std::int64_t crm = n - 1 - col[r];
      if (l == r) {
        acc = add(acc, mul(val[l], f[cl]));
        break;
      }
      if (cl < crm) {
        acc = add(acc, mul(val[l], f[cl]));
        ++l;
      } else if (cl > crm) {
        acc = add(acc, mul(val[r], f[col[r]]));
        --r;
      } else {
        acc = add(acc, add(mul(val[l], f[cl]), mul(val[r], f[col[r]])));
        ++l;
        --r;
      }
    }
    p[i] = acc;
  }
}


// ------------------------------------------------------------------ paired pattern
__global__ void diff_kernel(const int* a, const int* b, std::int64_t n, int* flag) {
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    if (a[k] != b[k]) {
      atomicOr(flag, 1);
      return;
    }
  }
}

// Union of the row patterns of two CSR matrices of equal shape; the value of
// an entry missing from one of them is 0.0 (exactly what the fold pruned).
template <bool FILL>
__global__ void union_rows_kernel(const int* pa, const int* ca, const double* va, const int* pb,
                                  const int* cb, const double* vb, std::int64_t rows, int* cnt,
                                  const int* up, int* uc, double* ua, double* ub) {
  for (std::int64_t i = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (std::int64_t)gridDim.x * blockDim.x) {
    int x = pa[i], xe = pa[i + 1], y = pb[i], ye = pb[i + 1];
    int o = FILL ? up[i] : 0, n = 0;
    while (x < xe || y < ye) {
      const int cx = x < xe ? ca[x] : 0x7fffffff, cy = y < ye ? cb[y] : 0x7fffffff;
      const int c = min(cx, cy);
      if (FILL) {
        uc[o] = c;
        ua[o] = cx == c ? va[x] : 0.0;
        ub[o] = cy == c ? vb[y] : 0.0;
        ++o;
      }
      if (cx == c) ++x;
      if (cy == c) ++y;
      ++n;
    }
    if (!FILL) cnt[i] = n;
  }
}

// ------------------------------------------------------------------ host helpers
template <class T>
void upload(Context* ctx, T* dst, const T* src, std::size_t n) {
  if (n) SSB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
}

void exclusive_scan_int_to_i64(Context* ctx, const int* in, std::int64_t* out, std::int64_t n) {
  std::size_t bytes = 0;
  SSB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, static_cast<int>(n + 1),
                                         ctx->stream));
  void* t = ctx->temp(bytes);
  SSB_CUDA(cub::DeviceScan::ExclusiveSum(t, bytes, in, out, static_cast<int>(n + 1), ctx->stream));
  ctx->launched(1);
}

// counts[0..n) -> ptr[0..n] (int, exclusive scan incl. the total)
void counts_to_ptr(Context* ctx, const int* counts_np1, int* ptr, std::int64_t n) {
  std::size_t bytes = 0;
  SSB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, counts_np1, ptr, static_cast<int>(n + 1),
                                         ctx->stream));
  void* t = ctx->temp(bytes);
  SSB_CUDA(cub::DeviceScan::ExclusiveSum(t, bytes, counts_np1, ptr, static_cast<int>(n + 1),
                                         ctx->stream));
  ctx->launched(1);
}

template <class T>
T read_scalar(Context* ctx, const T* dev) {
  T h{};
  SSB_CUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  return h;
}

}  // namespace

// counts[0..n] -> exclusive-scan pointer (shared with the plan builder)
void scan_counts(Context* ctx, const int* counts_np1, int* ptr, std::int64_t n) {
  counts_to_ptr(ctx, counts_np1, ptr, n);
}

// ====================================================================== API
template <class T>
void cast_dev(Context* ctx, const double* src, T* dst, std::int64_t n) {
  if (n <= 0) return;
  cast_kernel<T><<<grid_for(ctx, n), kT, 0, ctx->stream>>>(src, dst, n);
  ctx->check_launch("cast_kernel");
}
template void cast_dev<float>(Context*, const double*, float*, std::int64_t);
template void cast_dev<double>(Context*, const double*, double*, std::int64_t);

Matrix* matrix_from_csr_device(Context* ctx, std::int64_t rows, std::int64_t cols,
                               std::int64_t nnz, DBuf<int>&& rowptr, DBuf<int>&& colidx,
                               DBuf<double>&& val) {
  auto* a = new Matrix();
  a->ctx = ctx;
  a->rows = rows;
  a->cols = cols;
  a->nnz = nnz;
  a->rowptr = std::move(rowptr);
  a->colidx = std::move(colidx);
  a->val = std::move(val);
  return a;
}

// Stable-sorted (row<<32|col) keys with values -> CSR; repeats collapse in
// insertion order. keys/vals are consumed (device, `count` entries).
Matrix* matrix_from_sorted_triplets(Context* ctx, std::int64_t rows, std::int64_t cols,
                                    std::int64_t count, unsigned long long* keys, double* vals) {
  DBuf<int> rowptr(rows + 1);
  if (count == 0) {
    SSB_CUDA(cudaMemsetAsync(rowptr.get(), 0, (rows + 1) * sizeof(int), ctx->stream));
    return matrix_from_csr_device(ctx, rows, cols, 0, std::move(rowptr), DBuf<int>(1),
                                  DBuf<double>(1));
  }
  DBuf<int> head(count + 1);
  head_flags_kernel<<<grid_for(ctx, count), kT, 0, ctx->stream>>>(keys, count, head.get());
  ctx->check_launch("head_flags_kernel");
  SSB_CUDA(cudaMemsetAsync(head.get() + count, 0, sizeof(int), ctx->stream));
  DBuf<std::int64_t> pos(count + 1);
  exclusive_scan_int_to_i64(ctx, head.get(), pos.get(), count);
  const std::int64_t uniq = read_scalar(ctx, pos.get() + count);
  DBuf<int> col(uniq), row(uniq);
  DBuf<double> val(uniq);
  if (uniq == count) {
    split_keys_kernel<<<grid_for(ctx, count), kT, 0, ctx->stream>>>(keys, count, col.get(),
                                                                   row.get());
    ctx->check_launch("split_keys_kernel");
    SSB_CUDA(cudaMemcpyAsync(val.get(), vals, count * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
  } else {
    collapse_kernel<<<grid_for(ctx, count), kT, 0, ctx->stream>>>(
        keys, vals, head.get(), pos.get(), count, col.get(), row.get(), val.get());
    ctx->check_launch("collapse_kernel");
  }
  ptr_from_sorted_kernel<<<grid_for(ctx, uniq + 1), kT, 0, ctx->stream>>>(row.get(), uniq, rows,
                                                                          rowptr.get());
  ctx->check_launch("ptr_from_sorted_kernel");
  return matrix_from_csr_device(ctx, rows, cols, uniq, std::move(rowptr), std::move(col),
                                std::move(val));
}

namespace {
void sort_pairs_u64(Context* ctx, unsigned long long* kin, unsigned long long* kout,
                    double* vin, double* vout, std::int64_t n, int end_bit) {
  std::size_t bytes = 0;
  SSB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout,
                                           static_cast<int>(n), 0, end_bit, ctx->stream));
  void* t = ctx->temp(bytes);
  SSB_CUDA(cub::DeviceRadixSort::SortPairs(t, bytes, kin, kout, vin, vout, static_cast<int>(n), 0,
                                           end_bit, ctx->stream));
  ctx->launched(1);
}

__global__ void make_keys_kernel(const int* r, const int* c, std::int64_t n,
                                 unsigned long long* keys) {
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    keys[k] = (static_cast<unsigned long long>(r[k]) << 32) | static_cast<unsigned int>(c[k]);
  }
}
}  // namespace

Matrix* matrix_from_triplets_host(Context* ctx, std::int64_t rows, std::int64_t cols,
                                  std::int64_t count, const int* r, const int* c,
                                  const double* v) {
  if (rows < 0 || cols < 0) fail("matrix shape must be non-negative");
  for (std::int64_t k = 0; k < count; ++k) {
    if (r[k] < 0 || r[k] >= rows || c[k] < 0 || c[k] >= cols) fail("triplet index out of range");
  }
  DBuf<int> dr(count), dc(count);
  DBuf<double> dv(count), dv2(count);
  DBuf<unsigned long long> k1(count), k2(count);
  upload(ctx, dr.get(), r, count);
  upload(ctx, dc.get(), c, count);
  upload(ctx, dv.get(), v, count);
  Matrix* a = nullptr;
  if (count > 0) {
    make_keys_kernel<<<grid_for(ctx, count), kT, 0, ctx->stream>>>(dr.get(), dc.get(), count,
                                                                  k1.get());
    ctx->check_launch("make_keys_kernel");
    sort_pairs_u64(ctx, k1.get(), k2.get(), dv.get(), dv2.get(), count, 32 + bits_for(rows));
    a = matrix_from_sorted_triplets(ctx, rows, cols, count, k2.get(), dv2.get());
  } else {
    a = matrix_from_sorted_triplets(ctx, rows, cols, 0, nullptr, nullptr);
  }
  ctx->sync();
  check_finite(*a);
  return a;
}

Matrix* matrix_from_csc_host(Context* ctx, std::int64_t rows, std::int64_t cols,
                             std::int64_t nnz, const int* outer, const int* inner,
                             const double* v) {
  if (rows < 0 || cols < 0 || nnz < 0) fail("matrix shape must be non-negative");
  if (outer[0] != 0 || outer[cols] != nnz) fail("invalid compressed column pointers");
  for (std::int64_t j = 0; j < cols; ++j) {
    if (outer[j + 1] < outer[j]) fail("invalid compressed column pointers");
    for (int k = outer[j]; k < outer[j + 1]; ++k) {
      if (inner[k] < 0 || inner[k] >= rows) fail("row index out of range");
      if (k > outer[j] && inner[k] <= inner[k - 1]) fail("row indices must ascend within a column");
    }
  }
  // Column-major triplets are already in (col,row) order; a stable sort by
  // row gives the CSR with columns ascending.
  std::vector<int> r(inner, inner + nnz), c(static_cast<std::size_t>(nnz));
  for (std::int64_t j = 0; j < cols; ++j) {
    for (int k = outer[j]; k < outer[j + 1]; ++k) c[k] = static_cast<int>(j);
  }
  Matrix* a = matrix_from_triplets_host(ctx, rows, cols, nnz, r.data(), c.data(), v);
  a->colptr.alloc(cols + 1);
  a->rowidx.alloc(nnz);
  a->cval.alloc(nnz);
  upload(ctx, a->colptr.get(), outer, cols + 1);
  upload(ctx, a->rowidx.get(), inner, nnz);
  upload(ctx, a->cval.get(), v, nnz);
  a->has_csc = true;
  ctx->sync();
  return a;
}

void Matrix::ensure_csc(bool keep_perm) {
  if (has_csc) return;
  Context* c = ctx;
  colptr.alloc(cols + 1);
  rowidx.alloc(nnz);
  cval.alloc(nnz);
  if (nnz == 0) {
    SSB_CUDA(cudaMemsetAsync(colptr.get(), 0, (cols + 1) * sizeof(int), c->stream));
    has_csc = true;
    return;
  }
  DBuf<int> rowof(nnz), keys_in(nnz), keys_out(nnz), perm_in(nnz), perm_out(nnz);
  expand_ptr_kernel<<<grid_for(c, rows), kT, 0, c->stream>>>(rowptr.get(), rows, rowof.get());
  c->check_launch("expand_ptr_kernel");
  SSB_CUDA(cudaMemcpyAsync(keys_in.get(), colidx.get(), nnz * sizeof(int),
                           cudaMemcpyDeviceToDevice, c->stream));
  iota_kernel<<<grid_for(c, nnz), kT, 0, c->stream>>>(perm_in.get(), nnz);
  c->check_launch("iota_kernel");
  // Stable radix sort by column: CSR order has rows ascending, so rows stay
  // ascending inside every column (Eigen's compressed CSC invariant).
  std::size_t bytes = 0;
  const int eb = bits_for(std::max<std::int64_t>(cols, 2));
  SSB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys_in.get(), keys_out.get(),
                                           perm_in.get(), perm_out.get(), static_cast<int>(nnz), 0,
                                           eb, c->stream));
  void* t = c->temp(bytes);
  SSB_CUDA(cub::DeviceRadixSort::SortPairs(t, bytes, keys_in.get(), keys_out.get(), perm_in.get(),
                                           perm_out.get(), static_cast<int>(nnz), 0, eb,
                                           c->stream));
  c->launched(1);
  gather_kernel<<<grid_for(c, nnz), kT, 0, c->stream>>>(perm_out.get(), rowof.get(), val.get(),
                                                        nnz, rowidx.get(), cval.get());
  c->check_launch("gather_kernel");
  ptr_from_sorted_kernel<<<grid_for(c, nnz + 1), kT, 0, c->stream>>>(keys_out.get(), nnz, cols,
                                                                    colptr.get());
  c->check_launch("ptr_from_sorted_kernel");
  if (keep_perm) csc_perm = std::move(perm_out);
  c->sync();
  has_csc = true;
}

__global__ void permute_values_kernel(const int* __restrict__ perm, const double* __restrict__ src,
                                      std::int64_t n, double* __restrict__ dst) {
  for (std::int64_t k = blockIdx.x * (std::int64_t)blockDim.x + threadIdx.x; k < n;
       k += (std::int64_t)gridDim.x * blockDim.x) {
    dst[k] = src[perm[k]];
  }
}

void Matrix::csc_like(const Matrix& ref) {
  if (has_csc) return;
  if (ref.ctx != ctx || !ref.has_csc || ref.nnz != nnz || ref.rows != rows || ref.cols != cols ||
      ref.csc_perm.size() != static_cast<std::size_t>(std::max<std::int64_t>(nnz, 1)) ||
      nnz == 0) {
    ensure_csc();
    return;
  }
  Context* c = ctx;
  colptr.alloc(cols + 1);
  rowidx.alloc(nnz);
  cval.alloc(nnz);
  SSB_CUDA(cudaMemcpyAsync(colptr.get(), ref.colptr.get(), (cols + 1) * sizeof(int),
                           cudaMemcpyDeviceToDevice, c->stream));
  SSB_CUDA(cudaMemcpyAsync(rowidx.get(), ref.rowidx.get(), nnz * sizeof(int),
                           cudaMemcpyDeviceToDevice, c->stream));
  permute_values_kernel<<<grid_for(c, nnz), kT, 0, c->stream>>>(ref.csc_perm.get(), val.get(),
                                                               nnz, cval.get());
  c->check_launch("permute_values_kernel");
  has_csc = true;
}

void Matrix::ensure_f32() {
  if (has_f32) return;
  ensure_csc();
  val32.alloc(nnz);
  cval32.alloc(nnz);
  cast_dev<float>(ctx, val.get(), val32.get(), nnz);
  cast_dev<float>(ctx, cval.get(), cval32.get(), nnz);
  ctx->sync();
  has_f32 = true;
}

void check_finite(Matrix& a) {
  Context* ctx = a.ctx;
  if (a.nnz == 0) return;
  DBuf<int> bad(1);
  SSB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), ctx->stream));
  finite_kernel<<<grid_for(ctx, a.nnz), kT, 0, ctx->stream>>>(a.val.get(), a.nnz, bad.get());
  ctx->check_launch("finite_kernel");
  if (read_scalar(ctx, bad.get())) fail("matrix contains non-finite values");
}

std::int64_t nonzeros(Matrix& a) {
  Context* ctx = a.ctx;
  if (a.nnz == 0) return 0;
  DBuf<unsigned long long> out(1);
  SSB_CUDA(cudaMemsetAsync(out.get(), 0, sizeof(unsigned long long), ctx->stream));
  count_nonzero_kernel<<<grid_for(ctx, a.nnz), kT, 0, ctx->stream>>>(a.val.get(), a.nnz,
                                                                    out.get());
  ctx->check_launch("count_nonzero_kernel");
  return static_cast<std::int64_t>(read_scalar(ctx, out.get()));
}

// GPU build_system (geometry.cpp:227-275): count -> scan -> fill of the
// traced half, stable (row,col) radix sort (repeats collapse in traversal
// order, as setFromTriplets would sum them), then the mirror half.
void ray_weights_dev(Context* ctx, double sx, double sy, double ex, double ey, const Grid& g,
                     std::vector<int>& cols, std::vector<double>& lens) {
  g.validate();
  cols.clear();
  lens.clear();
  const double dx = ex - sx, dy = ey - sy;
  const double seg = std::hypot(dx, dy);
  if (seg == 0.0) fail("ray_weights: degenerate ray");
  double tin = 0.0, tout = 0.0;
  if (!clip_ray(sx, sy, ex, ey, g, tin, tout)) return;
  std::vector<double> xb(g.n_x + 1), yb(g.n_y + 1);
  for (int k = 0; k <= g.n_x; ++k) xb[k] = g.center_x + (k - g.n_x / 2) * g.voxel_size;
  for (int k = 0; k <= g.n_y; ++k) yb[k] = g.y_bottom + k * g.voxel_size;
  const double ray7[7] = {sx, sy, dx, dy, seg, tin, tout};
  DBuf<double> d_ray(7), d_xb(xb.size()), d_yb(yb.size());
  upload(ctx, d_ray.get(), ray7, 7);
  upload(ctx, d_xb.get(), xb.data(), xb.size());
  upload(ctx, d_yb.get(), yb.data(), yb.size());
  TraceArgs ta{d_ray.get(),     d_ray.get() + 1, d_ray.get() + 2, d_ray.get() + 3,
               d_ray.get() + 4, d_ray.get() + 5, d_ray.get() + 6, d_xb.get(),
               d_yb.get(),      g.n_x,           g.n_y,           g.voxel_size,
               g.x_left(),      g.y_bottom,      1};
  DBuf<int> count(1);
  trace_count_kernel<<<1, 32, 0, ctx->stream>>>(ta, count.get());
  ctx->check_launch("trace_count_kernel");
  const int n = read_scalar(ctx, count.get());
  DBuf<std::int64_t> off(1);
  SSB_CUDA(cudaMemsetAsync(off.get(), 0, sizeof(std::int64_t), ctx->stream));
  DBuf<unsigned long long> keys(std::max(n, 1));
  DBuf<double> vals(std::max(n, 1));
  trace_fill_kernel<<<1, 32, 0, ctx->stream>>>(ta, off.get(), keys.get(), vals.get());
  ctx->check_launch("trace_fill_kernel");
  std::vector<unsigned long long> hk(n);
  lens.resize(n);
  if (n) {
    SSB_CUDA(cudaMemcpyAsync(hk.data(), keys.get(), n * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, ctx->stream));
    SSB_CUDA(cudaMemcpyAsync(lens.data(), vals.get(), n * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
  }
  ctx->sync();
  cols.resize(n);
  for (int q = 0; q < n; ++q) cols[q] = static_cast<int>(hk[q] & 0xffffffffull) + 1;
}

Matrix* build_system(Context* ctx, const ss_scan_config& cfg) {
  return build_system(ctx, cfg, make_grid(cfg));
}

// reference build_system(const ScanGeometry&, const GridSpec&, int)
// (geometry.cpp:227-275): the grid is the caller's (cfg.grid_nx / grid_ny unused)
Matrix* build_system(Context* ctx, const ss_scan_config& cfg, const Grid& g) {
  const RayTable rt = enumerate_rays(cfg, g, false);
  const std::int64_t mh = rt.m / 2, m = rt.m, n = g.cell_count();
  std::vector<double> xb(g.n_x + 1), yb(g.n_y + 1);
  for (int k = 0; k <= g.n_x; ++k) xb[k] = g.center_x + (k - g.n_x / 2) * g.voxel_size;
  for (int k = 0; k <= g.n_y; ++k) yb[k] = g.y_bottom + k * g.voxel_size;

  DBuf<double> d_rays(7 * mh), d_xb(xb.size()), d_yb(yb.size());
  const std::vector<double>* cols7[7] = {&rt.sx, &rt.sy, &rt.dx, &rt.dy,
                                         &rt.seg_len, &rt.t_in, &rt.t_out};
  for (int q = 0; q < 7; ++q) upload(ctx, d_rays.get() + q * mh, cols7[q]->data(), mh);
  upload(ctx, d_xb.get(), xb.data(), xb.size());
  upload(ctx, d_yb.get(), yb.data(), yb.size());
  TraceArgs ta{d_rays.get(),          d_rays.get() + mh,     d_rays.get() + 2 * mh,
               d_rays.get() + 3 * mh, d_rays.get() + 4 * mh, d_rays.get() + 5 * mh,
               d_rays.get() + 6 * mh, d_xb.get(),            d_yb.get(),
               g.n_x,                 g.n_y,                 g.voxel_size,
               g.x_left(),            g.y_bottom,            mh};
  DBuf<int> counts(mh + 1);
  SSB_CUDA(cudaMemsetAsync(counts.get() + mh, 0, sizeof(int), ctx->stream));
  trace_count_kernel<<<grid_for(ctx, mh, 128), 128, 0, ctx->stream>>>(ta, counts.get());
  ctx->check_launch("trace_count_kernel");
  DBuf<std::int64_t> offs(mh + 1);
  exclusive_scan_int_to_i64(ctx, counts.get(), offs.get(), mh);
  const std::int64_t half = read_scalar(ctx, offs.get() + mh);
  if (2 * half >= (std::int64_t{1} << 31)) fail("build_system: nnz exceeds int32 storage");
  Matrix* a = nullptr;
  {
    DBuf<unsigned long long> k1(half), k2(half);
    DBuf<double> v1(half), v2(half);
    trace_fill_kernel<<<grid_for(ctx, mh, 128), 128, 0, ctx->stream>>>(ta, offs.get(), k1.get(),
                                                                      v1.get());
    ctx->check_launch("trace_fill_kernel");
    sort_pairs_u64(ctx, k1.get(), k2.get(), v1.get(), v2.get(), half, 32 + bits_for(mh));
    a = matrix_from_sorted_triplets(ctx, mh, n, half, k2.get(), v2.get());
  }
  // Grow the traced-half CSR into the full M x N matrix.
  const std::int64_t h = a->nnz;
  DBuf<int> ptr(m + 1), col(2 * h);
  DBuf<double> val(2 * h);
  SSB_CUDA(cudaMemcpyAsync(ptr.get(), a->rowptr.get(), (mh + 1) * sizeof(int),
                           cudaMemcpyDeviceToDevice, ctx->stream));
  SSB_CUDA(cudaMemcpyAsync(col.get(), a->colidx.get(), h * sizeof(int), cudaMemcpyDeviceToDevice,
                           ctx->stream));
  SSB_CUDA(cudaMemcpyAsync(val.get(), a->val.get(), h * sizeof(double), cudaMemcpyDeviceToDevice,
                           ctx->stream));
  mirror_ptr_kernel<<<grid_for(ctx, mh), kT, 0, ctx->stream>>>(ptr.get(), mh, h);
  ctx->check_launch("mirror_ptr_kernel");
  mirror_fill_kernel<<<grid_for(ctx, h), kT, 0, ctx->stream>>>(col.get(), val.get(), h, n);
  ctx->check_launch("mirror_fill_kernel");
  ctx->sync();
  delete a;
  return matrix_from_csr_device(ctx, m, n, 2 * h, std::move(ptr), std::move(col), std::move(val));
}

ss_symmetry_report verify_symmetry(Matrix& a, double tol) {
  if (tol < 0) fail("verify_symmetry: tol must be non-negative");
  Context* ctx = a.ctx;
  ss_symmetry_report rep{};
  rep.status = a.rows % 2 != 0 ? 1 : (a.cols % 2 != 0 ? 2 : 0);
  rep.max_violation = 0.0;
  rep.worst_row = 1;
  rep.worst_col = 1;
  if (a.rows > 0 && a.nnz > 0) {
    DBuf<double> rmax(a.rows);
    DBuf<int> rarg(a.rows);
    DBuf<Worst> w(1);
    symmetry_rows_kernel<<<grid_for(ctx, a.rows * 32), kT,
                           (kT / 32) * kSymCap * static_cast<int>(sizeof(int)), ctx->stream>>>(
        a.rowptr.get(), a.colidx.get(), a.val.get(), a.rows, a.cols, rmax.get(), rarg.get());
    ctx->check_launch("symmetry_rows_kernel");
    symmetry_reduce_kernel<<<1, 1024, 0, ctx->stream>>>(rmax.get(), rarg.get(), a.rows, w.get());
    ctx->check_launch("symmetry_reduce_kernel");
    const Worst hw = read_scalar(ctx, w.get());
    if (hw.j != 0x7fffffff && hw.d > 0.0) {
      rep.max_violation = hw.d;
      rep.worst_row = hw.i + 1;
      rep.worst_col = hw.j + 1;
    }
  }
  rep.holds = (rep.status == 0 && rep.max_violation <= tol) ? 1 : 0;
  return rep;
}

constexpr int kFoldSmem = (kT / 32) * kFoldCap * static_cast<int>(sizeof(int));
static_assert(kFoldSmem <= 48 * 1024, "fold staging must fit the default shared memory");

// The fold with verify_symmetry fused into its count pass (one read of A
// instead of two): the count pass also reports, per output row, the worst
// mirror violation of the two source rows; if the reduced maximum exceeds tol
// the report is returned before the fill pass (a1 = a2 = nullptr), with the
// same value and first column-major arg-max verify_symmetry gives.
ss_symmetry_report fold_checked(Matrix& a, double tol, Matrix*& a1, Matrix*& a2) {
  if (tol < 0) fail("verify_symmetry: tol must be non-negative");
  ss_symmetry_report rep{};
  rep.status = a.rows % 2 != 0 ? 1 : (a.cols % 2 != 0 ? 2 : 0);
  rep.max_violation = 0.0;
  rep.worst_row = 1;
  rep.worst_col = 1;
  a1 = a2 = nullptr;
  if (rep.status != 0) {
    rep.holds = 0;
    return rep;
  }
  Context* ctx = a.ctx;
  const std::int64_t mh = a.rows / 2, nh = a.cols / 2;
  DBuf<int> lane1(mh * 32), lane2(mh * 32), c1(mh + 1), c2(mh + 1);
  DBuf<double> sd(std::max<std::int64_t>(mh, 1));
  DBuf<int> sj(std::max<std::int64_t>(mh, 1)), si(std::max<std::int64_t>(mh, 1));
  SSB_CUDA(cudaMemsetAsync(c1.get() + mh, 0, sizeof(int), ctx->stream));
  SSB_CUDA(cudaMemsetAsync(c2.get() + mh, 0, sizeof(int), ctx->stream));
  FoldArgs fa{a.rowptr.get(), a.colidx.get(), a.val.get(), a.rows, a.cols, mh, nh,
              nullptr, nullptr, lane1.get(), lane2.get(), c1.get(), c2.get(),
              nullptr, nullptr, nullptr, nullptr, sd.get(), sj.get(), si.get()};
  if (mh > 0) {
    fold_kernel<false><<<grid_for(ctx, mh * 32), kT, kFoldSmem, ctx->stream>>>(fa);
    ctx->check_launch("fold_kernel<count>");
    DBuf<Worst> w(1);
    symmetry_reduce3_kernel<<<1, 1024, 0, ctx->stream>>>(sd.get(), sj.get(), si.get(), mh,
                                                         w.get());
    ctx->check_launch("symmetry_reduce3_kernel");
    const Worst hw = read_scalar(ctx, w.get());
    if (hw.j != 0x7fffffff && hw.d > 0.0) {
      rep.max_violation = hw.d;
      rep.worst_row = hw.i + 1;
      rep.worst_col = hw.j + 1;
    }
  }
  rep.holds = rep.max_violation <= tol ? 1 : 0;
  if (!rep.holds) return rep;
  DBuf<int> p1(mh + 1), p2(mh + 1);
  counts_to_ptr(ctx, c1.get(), p1.get(), mh);
  counts_to_ptr(ctx, c2.get(), p2.get(), mh);
  const int n1 = read_scalar(ctx, p1.get() + mh);
  const int n2 = read_scalar(ctx, p2.get() + mh);
  DBuf<int> col1(n1), col2(n2);
  DBuf<double> val1(n1), val2(n2);
  fa.ptr1 = p1.get();
  fa.ptr2 = p2.get();
  fa.col1 = col1.get();
  fa.val1 = val1.get();
  fa.col2 = col2.get();
  fa.val2 = val2.get();
  fa.sym_d = nullptr;
  if (mh > 0) {
    fold_kernel<true><<<grid_for(ctx, mh * 32), kT, kFoldSmem, ctx->stream>>>(fa);
    ctx->check_launch("fold_kernel<fill>");
  }
  ctx->sync();
  a1 = matrix_from_csr_device(ctx, mh, nh, n1, std::move(p1), std::move(col1), std::move(val1));
  a2 = matrix_from_csr_device(ctx, mh, nh, n2, std::move(p2), std::move(col2), std::move(val2));
  return rep;
}

void fold(Matrix& a, Matrix*& a1, Matrix*& a2) {
  if (a.rows % 2 != 0 || a.cols % 2 != 0) fail("split_matrix: dimensions must be even");
  // no tolerance: the fold of any even-sized matrix (split_matrix semantics)
  const ss_symmetry_report r = fold_checked(a, std::numeric_limits<double>::infinity(), a1, a2);
  (void)r;
}

void split_rhs_dev(Context* ctx, const double* p, double* p1, double* p2, std::int64_t mh) {
  if (mh <= 0) return;
  split_rhs_kernel<<<grid_for(ctx, mh), kT, 0, ctx->stream>>>(p, p1, p2, mh);
  ctx->check_launch("split_rhs_kernel");
}

void recombine_dev(Context* ctx, const double* f1, const double* f2, double* f, std::int64_t nh,
                   std::int64_t nrhs) {
  if (nh * nrhs <= 0) return;
  recombine_kernel<<<grid_for(ctx, nh * nrhs), kT, 0, ctx->stream>>>(f1, f2, f, nh, nrhs);
  ctx->check_launch("recombine_kernel");
}

void decompose_dev(Context* ctx, const double* f, double* f1, double* f2, std::int64_t nh) {
  if (nh <= 0) return;
  decompose_kernel<<<grid_for(ctx, nh), kT, 0, ctx->stream>>>(f, f1, f2, nh);
  ctx->check_launch("decompose_kernel");
}

void abs_sums(Matrix& a, double* row_sums, double* col_sums) {
  Context* ctx = a.ctx;
  a.ensure_csc();
  if (a.rows > 0) {
    abs_sum_kernel<<<grid_for(ctx, a.rows), kT, 0, ctx->stream>>>(a.rowptr.get(), a.val.get(),
                                                                 a.rows, row_sums);
    ctx->check_launch("abs_sum_kernel<rows>");
  }
  if (a.cols > 0) {
    abs_sum_kernel<<<grid_for(ctx, a.cols), kT, 0, ctx->stream>>>(a.colptr.get(), a.cval.get(),
                                                                 a.cols, col_sums);
    ctx->check_launch("abs_sum_kernel<cols>");
  }
}

void apply_dev(Matrix& a, const double* x, double* y) {
  if (a.rows <= 0) return;
  csr_apply_kernel<<<grid_for(a.ctx, a.rows * 32), kT, 0, a.ctx->stream>>>(
      a.rowptr.get(), a.colidx.get(), a.val.get(), x, nullptr, a.rows, y);
  a.ctx->check_launch("csr_apply_kernel");
}

void apply_transpose_dev(Matrix& a, const double* y, double* x) {
  a.ensure_csc();
  if (a.cols <= 0) return;
  csr_apply_kernel<<<grid_for(a.ctx, a.cols * 32), kT, 0, a.ctx->stream>>>(
      a.colptr.get(), a.rowidx.get(), a.cval.get(), y, nullptr, a.cols, x);
  a.ctx->check_launch("csr_apply_kernel<T>");
}

void residual_dev(Matrix& a, const double* x, const double* p, double* r) {
  if (a.rows <= 0) return;
  csr_apply_kernel<<<grid_for(a.ctx, a.rows * 32), kT, 0, a.ctx->stream>>>(
      a.rowptr.get(), a.colidx.get(), a.val.get(), x, p, a.rows, r);
  a.ctx->check_launch("csr_apply_kernel<res>");
}

double norm2_dev(Context* ctx, const double* v, std::int64_t n) {
  if (n <= 0) return 0.0;
  const int blocks = 256;
  DBuf<double> part(blocks), out(1);
  sq_partial_kernel<<<blocks, kT, 0, ctx->stream>>>(v, n, part.get());
  ctx->check_launch("sq_partial_kernel");
  sum_partial_kernel<<<1, kT, 0, ctx->stream>>>(part.get(), blocks, out.get());
  ctx->check_launch("sum_partial_kernel");
  return read_scalar(ctx, out.get());
}

double max_dev(Context* ctx, const double* v, std::int64_t n) {
  if (n <= 0) return 0.0;
  const int blocks = 256;
  DBuf<double> part(blocks), out(1);
  max_partial_kernel<<<blocks, kT, 0, ctx->stream>>>(v, n, part.get());
  ctx->check_launch("max_partial_kernel");
  max_partial_kernel<<<1, kT, 0, ctx->stream>>>(part.get(), blocks, out.get());
  ctx->check_launch("max_partial_kernel<final>");
  return read_scalar(ctx, out.get());
}

bool all_finite_dev(Context* ctx, const double* v, std::int64_t n) {
  if (n <= 0) return true;
  DBuf<int> bad(1);
  SSB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), ctx->stream));
  finite_kernel<<<grid_for(ctx, n), kT, 0, ctx->stream>>>(v, n, bad.get());
  ctx->check_launch("finite_kernel");
  return read_scalar(ctx, bad.get()) == 0;
}

void rasterize_dev(Context* ctx, const double* ell6, int count, const Grid& g, double* out) {
  g.validate();
  std::vector<EllipseDev> es(static_cast<std::size_t>(count));
  for (int q = 0; q < count; ++q) {
    const double* e = ell6 + 6 * q;
    es[q] = EllipseDev{e[0], e[1], e[2], e[3], std::cos(e[4]), std::sin(e[4]), e[5]};
  }
  DBuf<EllipseDev> d(es.size());
  upload(ctx, d.get(), es.data(), es.size());
  const double half_w = 0.5 * g.width(), half_h = 0.5 * g.height();
  RasterArgs ra{d.get(), count, g.n_x, g.n_y, g.voxel_size, g.center_x, g.y_bottom,
                half_w, half_h, g.y_bottom + half_h, out};
  const std::int64_t total = static_cast<std::int64_t>(g.n_x) * g.n_y;
  rasterize_kernel<<<grid_for(ctx, total), kT, 0, ctx->stream>>>(ra);
  ctx->check_launch("rasterize_kernel");
  ctx->sync();
}

void forward_project_dev(Matrix& a, const double* f, double* p) {
  if (a.rows <= 0) return;
  forward_project_kernel<<<grid_for(a.ctx, a.rows), kT, 0, a.ctx->stream>>>(
      a.rowptr.get(), a.colidx.get(), a.val.get(), f, a.rows, a.cols, p);
  a.ctx->check_launch("forward_project_kernel");
}


bool same_pattern(Matrix& a, Matrix& b) {
  if (a.rows != b.rows || a.cols != b.cols || a.nnz != b.nnz) return false;
  Context* ctx = a.ctx;
  DBuf<int> flag(1);
  SSB_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), ctx->stream));
  diff_kernel<<<grid_for(ctx, a.rows + 1), kT, 0, ctx->stream>>>(a.rowptr.get(), b.rowptr.get(),
                                                               a.rows + 1, flag.get());
  ctx->check_launch("diff_kernel<ptr>");
  if (a.nnz > 0) {
    diff_kernel<<<grid_for(ctx, a.nnz), kT, 0, ctx->stream>>>(a.colidx.get(), b.colidx.get(),
                                                             a.nnz, flag.get());
    ctx->check_launch("diff_kernel<idx>");
  }
  return read_scalar(ctx, flag.get()) == 0;
}

void union_pattern(Matrix& a, Matrix& b, Matrix*& ua, Matrix*& ub) {
  if (a.rows != b.rows || a.cols != b.cols) fail("union_pattern: shapes differ");
  Context* ctx = a.ctx;
  const std::int64_t rows = a.rows;
  DBuf<int> cnt(rows + 1), ptr(rows + 1), ptr2(rows + 1);
  SSB_CUDA(cudaMemsetAsync(cnt.get() + rows, 0, sizeof(int), ctx->stream));
  union_rows_kernel<false><<<grid_for(ctx, rows), kT, 0, ctx->stream>>>(
      a.rowptr.get(), a.colidx.get(), a.val.get(), b.rowptr.get(), b.colidx.get(), b.val.get(),
      rows, cnt.get(), nullptr, nullptr, nullptr, nullptr);
  ctx->check_launch("union_rows_kernel<count>");
  counts_to_ptr(ctx, cnt.get(), ptr.get(), rows);
  const int n = read_scalar(ctx, ptr.get() + rows);
  DBuf<int> col(n), col2(n);
  DBuf<double> va(n), vb(n);
  union_rows_kernel<true><<<grid_for(ctx, rows), kT, 0, ctx->stream>>>(
      a.rowptr.get(), a.colidx.get(), a.val.get(), b.rowptr.get(), b.colidx.get(), b.val.get(),
      rows, nullptr, ptr.get(), col.get(), va.get(), vb.get());
  ctx->check_launch("union_rows_kernel<fill>");
  SSB_CUDA(cudaMemcpyAsync(ptr2.get(), ptr.get(), (rows + 1) * sizeof(int),
                           cudaMemcpyDeviceToDevice, ctx->stream));
  SSB_CUDA(cudaMemcpyAsync(col2.get(), col.get(), n * sizeof(int), cudaMemcpyDeviceToDevice,
                           ctx->stream));
  ctx->sync();
  ua = matrix_from_csr_device(ctx, rows, a.cols, n, std::move(ptr), std::move(col), std::move(va));
  ub = matrix_from_csr_device(ctx, rows, a.cols, n, std::move(ptr2), std::move(col2),
                              std::move(vb));
}

}  // namespace ssb
