// TMA-fed SART kernels over the paired mirror-coded streams (included by
// sart.cu inside its anonymous namespace; uses its helpers and SartK).
//
// K1 (rows, FWD) and K2 (columns, !FWD) of reference sart_solve
// (proj/src/solvers.cpp:178-191) for both folded systems per launch, with the
// matrix stream moved by the copy engine instead of by the threads that use it:
//
//   * the plan cuts each direction's stream into chunks of whole vectors
//     (<= cap entries and tiles) and gives every CTA (one per SM) a contiguous,
//     byte-balanced run of chunks;
//   * one producer thread streams the CTA's chunks into a ring of `stages`
//     shared-memory slots with 1-D bulk copies (cp.async.bulk, completion
//     counted in bytes on a per-slot mbarrier): index offsets, values and tile
//     headers of a chunk are three copies. The first `stages` chunks are issued
//     before the grid-dependency wait (the matrix does not depend on the
//     previous pass), so they land while the previous kernel drains;
//   * consumer lane groups (VS lanes, the tiled layout of seg_dot2m) take the
//     CTA's vectors in order from a shared counter (dynamic balance inside the
//     CTA), wait for their chunk's slot, read offsets / values / sign bits from
//     shared memory and only gather x (K1) or w (K2) through L1/L2. The last
//     group to finish a chunk releases its slot to the producer.
//
// Consumers therefore never wait on DRAM latency for the stream: the bytes in
// flight per SM are the ring's, not the registers'. Each vector is reduced by
// one group in a fixed order (the same tile order and butterfly as seg_dot2m),
// so results are bitwise reproducible run to run and independent of which
// group took which vector.

// CTA size NT: 512 (15 consumer warps + 1 producer warp, up to 128 registers)
// or 1024 (31 consumer warps at 64 registers)
constexpr int kRingMaxStages = 8;

// One chunk of a direction's stream, precomputed by the plan: the vector
// range and, per array, the 16-byte-aligned global byte range the producer
// copies (aligned down / up; the slack stays inside the allocations' padding).
struct RingDesc {
  long long i0, v0, h0, e0;   // aligned byte starts: indices, values, headers, epilogue operands
  unsigned ib, vb, hb, eb;    // aligned byte counts
  int vbeg, vend;             // vectors [vbeg, vend)
  int pad[2];
};
static_assert(sizeof(RingDesc) == 64, "RingDesc layout");

struct RingArgs {
  const RingDesc* desc;   // [nchunk]
  const int* cta_chunk;   // [grid + 1] first chunk of every CTA
  const int4* vmeta;      // [n + 1] per vector {stream begin, first tile, first exception, 0}
  const unsigned char* epi;  // constant per-vector epilogue operands (K1: {p1,p2,rinv1,rinv2})
  int stages;
  unsigned off_v, off_h, off_m, off_e, stage_bytes;  // regions inside a slot
  int evict_first;        // L2 evict-first policy on the bulk copies
  int prefetch;           // L1 prefetch of the next round's gather lines
  int nchunk;             // chunks of the direction
  int interleave;         // CTA b takes chunks b, b+G, ... (else its contiguous run)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// ~2 s at 1.9 GHz: far beyond any healthy wait; a broken ring protocol traps
// (a launch failure the host reports) instead of hanging the GPU
constexpr long long kRingSpinCycles = 4000000000LL;

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(bar, parity)) {
    if (clock64() - t0 > kRingSpinCycles) __trap();
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, bool evict_first, uint64_t pol) {
  if (evict_first) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
  }
}

// header words per tile of a VS-lane layout (load_hdr)
template <int VS>
constexpr int ring_hs() {
  return VS <= 8 ? 2 : (VS == 16 ? 4 : 8);
}

// Dot products of one vector against the interleaved iterate, stream from the
// slot (same tile order, sign coding and exception handling as seg_dot2m).
template <class T, int VS, int UF, bool U16>
__device__ __forceinline__ void ring_dot(const unsigned char* __restrict__ si,
                                         const unsigned char* __restrict__ sv,
                                         const unsigned char* __restrict__ sh, int tf,
                                         const typename Vec2<T>::type* __restrict__ xv, int beg,
                                         int end, int eb, int ee, const int* __restrict__ eidx,
                                         const T* __restrict__ ev2, int lane, unsigned mask,
                                         bool pf, T& acc_a, T& acc_b) {
  using T2 = typename Vec2<T>::type;
  constexpr int isz = U16 ? 2 : 4;
  constexpr int hsz = 4 * ring_hs<VS>();
  T sa = T(0), sb = T(0);
  const int nvec = (end - beg) >> 2;
  const auto hdr = [&](int t, int& base, unsigned& nib) {
    const unsigned char* h = sh + static_cast<long long>(t) * hsz;
    if constexpr (VS <= 8) {
      const uint2 w = *reinterpret_cast<const uint2*>(h);
      base = static_cast<int>(w.x);
      nib = w.y >> (4 * lane);
    } else if constexpr (VS == 16) {
      const uint4 w = *reinterpret_cast<const uint4*>(h);
      base = static_cast<int>(w.x);
      nib = (lane < 8 ? w.y : w.z) >> (4 * (lane & 7));
    } else {
      const unsigned* hw = reinterpret_cast<const unsigned*>(h);
      base = static_cast<int>(hw[0]);
      nib = hw[1 + (lane >> 3)] >> (4 * (lane & 7));
    }
  };
  const auto quad = [&](int k0, int base, int4& c, T (&v)[4]) {
    if constexpr (U16) {
      c = decode16(*reinterpret_cast<const uint2*>(si + static_cast<long long>(k0) * isz), base);
    } else {
      c = *reinterpret_cast<const int4*>(si + static_cast<long long>(k0) * isz);
    }
    if constexpr (sizeof(T) == 4) {
      const float4 t = *reinterpret_cast<const float4*>(sv + static_cast<long long>(k0) * 4);
      v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else {
      const double2 a = *reinterpret_cast<const double2*>(sv + static_cast<long long>(k0) * 8);
      const double2 b = *reinterpret_cast<const double2*>(sv + static_cast<long long>(k0) * 8 + 16);
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
      int b;
      hdr(t0 + u, b, s[u]);
      quad(beg + ((q + u * VS) << 2), b, c[u], v[u]);
    }
    if (pf && q + (2 * UF - 1) * VS < nvec) {
      // the next round's gather lines into L1 while this round's are in flight
#pragma unroll
      for (int u = 0; u < UF; ++u) {
        int b;
        unsigned sn;
        hdr(t0 + UF + u, b, sn);
        int4 cn;
        T vn[4];
        quad(beg + ((q + (UF + u) * VS) << 2), b, cn, vn);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(xv + cn.x));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(xv + cn.y));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(xv + cn.z));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(xv + cn.w));
      }
    }
    T2 g[UF][4];
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      g[u][0] = __ldg(xv + c[u].x);
      g[u][1] = __ldg(xv + c[u].y);
      g[u][2] = __ldg(xv + c[u].z);
      g[u][3] = __ldg(xv + c[u].w);
    }
#pragma unroll
    for (int u = 0; u < UF; ++u) {
      sa += flip(v[u][0], s[u], 0) * g[u][0].x + flip(v[u][1], s[u], 1) * g[u][1].x +
            flip(v[u][2], s[u], 2) * g[u][2].x + flip(v[u][3], s[u], 3) * g[u][3].x;
      sb += v[u][0] * g[u][0].y + v[u][1] * g[u][1].y + v[u][2] * g[u][2].y +
            v[u][3] * g[u][3].y;
    }
  }
  for (; q < nvec; q += VS) {
    int b;
    unsigned s;
    hdr(tf + (q - lane) / VS, b, s);
    int4 c;
    T v[4];
    quad(beg + (q << 2), b, c, v);
    const T2 g0 = __ldg(xv + c.x), g1 = __ldg(xv + c.y), g2 = __ldg(xv + c.z),
             g3 = __ldg(xv + c.w);
    sa += flip(v[0], s, 0) * g0.x + flip(v[1], s, 1) * g1.x + flip(v[2], s, 2) * g2.x +
          flip(v[3], s, 3) * g3.x;
    sb += v[0] * g0.y + v[1] * g1.y + v[2] * g2.y + v[3] * g3.y;
  }
  for (int e = eb + lane; e < ee; e += VS) {  // exception buckets (rare), from global
    const int c = __ldg(eidx + e);
    const T2 a = __ldg(reinterpret_cast<const T2*>(ev2) + e);
    const T2 gg = __ldg(xv + c);
    sa += a.x * gg.x;
    sb += a.y * gg.y;
  }
#pragma unroll
  for (int off2 = VS / 2; off2 > 0; off2 >>= 1) {
    sa += __shfl_xor_sync(mask, sa, off2, VS);
    sb += __shfl_xor_sync(mask, sb, off2, VS);
  }
  acc_a = sa;
  acc_b = sb;
}

template <class T, int VS, int UF, bool U16, bool FWD, int NT>
__global__ void __launch_bounds__(NT, 1) sart_ring_kernel(SartK<T> k, int it, RingArgs R) {
  constexpr int kRingThreads = NT;
  constexpr int kRingWarps = NT / 32;
  using T2 = typename Vec2<T>::type;
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ uint64_t full[kRingMaxStages], empty[kRingMaxStages];
  __shared__ int done[kRingMaxStages];
  // slot bookkeeping written by the producer before `loaded` (fenced)
  __shared__ volatile int loaded[kRingMaxStages];
  __shared__ volatile int slot_v0[kRingMaxStages], slot_v1[kRingMaxStages];
  __shared__ volatile long long slot_i0[kRingMaxStages], slot_v0b[kRingMaxStages],
      slot_h0[kRingMaxStages], slot_e0[kRingMaxStages];
  __shared__ int next_v, vend_cta, go, pass;
  __shared__ double red[2][kRingWarps];

  const unsigned char* gidx = reinterpret_cast<const unsigned char*>(
      U16 ? static_cast<const void*>(FWD ? k.tof : k.tob)
          : static_cast<const void*>(FWD ? k.tif : k.tib));
  const unsigned char* gval = reinterpret_cast<const unsigned char*>(FWD ? k.rv2 : k.cv2);
  const unsigned char* ghdr = reinterpret_cast<const unsigned char*>(FWD ? k.thf : k.thb);
  const unsigned char* gmeta = reinterpret_cast<const unsigned char*>(R.vmeta);
  const int* __restrict__ eidx = FWD ? k.eif : k.eib;
  const T* __restrict__ ev2 = FWD ? k.evf : k.evb;
  const int S = R.stages;
  // the CTA's chunks: a contiguous run [cb, cb + nloc), or (interleave) the
  // sweep b, b + G, b + 2G, ... so that all SMs stream neighbouring bytes
  const int G = gridDim.x, b = blockIdx.x;
  const int cb = R.interleave ? b : __ldg(R.cta_chunk + b);
  const int nloc = R.interleave ? (R.nchunk > b ? (R.nchunk - b + G - 1) / G : 0)
                                : __ldg(R.cta_chunk + b + 1) - cb;
  const int cstep = R.interleave ? G : 1;
  const int warp = threadIdx.x >> 5, wl = threadIdx.x & 31;
  const bool producer = warp == kRingWarps - 1;

  // behind the slots: per local chunk j its first vector gv[j] and the
  // prefix lp[j] of the CTA's vector counts (local vector l of chunk j is
  // global vector gv[j] + l - lp[j]); groups take local vectors in order
  int* lp = reinterpret_cast<int*>(ring + static_cast<size_t>(S) * R.stage_bytes);
  int* gv = lp + nloc + 1;
  if (warp == 0) {
    int carry = 0;
    for (int base = 0; base < nloc; base += 32) {
      const int j = base + wl;
      int cnt = 0;
      if (j < nloc) {
        const RingDesc& d = R.desc[cb + j * cstep];
        gv[j] = d.vbeg;
        cnt = d.vend - d.vbeg;
      }
      int inc = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (wl >= o) inc += t;
      }
      if (j < nloc) lp[j + 1] = carry + inc;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (wl == 0) {
      lp[0] = 0;
      vend_cta = carry;
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      done[s] = 0;
      loaded[s] = -1;
    }
    next_v = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  uint64_t pol = 0;
  if (R.evict_first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  // producer lane 0: chunk descriptor d into slot i % S (five bulk copies:
  // indices, values, tile headers, vector metadata, epilogue operands)
  const auto issue = [&](int i, const RingDesc& d) {
    const int s = i % S;
    unsigned char* slot = ring + static_cast<size_t>(s) * R.stage_bytes;
    const long long m0 = static_cast<long long>(d.vbeg) * 16;
    const unsigned mb = static_cast<unsigned>(d.vend + 1 - d.vbeg) * 16u;
    slot_v0[s] = d.vbeg;
    slot_v1[s] = d.vend;
    slot_i0[s] = d.i0;
    slot_v0b[s] = d.v0;
    slot_h0[s] = d.h0;
    slot_e0[s] = d.e0;
    __threadfence_block();
    loaded[s] = i;
    mbar_expect_tx(&full[s], d.ib + d.vb + d.hb + mb + d.eb);
    if (d.ib) bulk_g2s(slot, gidx + d.i0, d.ib, &full[s], R.evict_first, pol);
    if (d.vb) bulk_g2s(slot + R.off_v, gval + d.v0, d.vb, &full[s], R.evict_first, pol);
    if (d.hb) bulk_g2s(slot + R.off_h, ghdr + d.h0, d.hb, &full[s], R.evict_first, pol);
    bulk_g2s(slot + R.off_m, gmeta + m0, mb, &full[s], false, pol);
    if (d.eb) bulk_g2s(slot + R.off_e, R.epi + d.e0, d.eb, &full[s], false, pol);
  };
  // descriptors are read 32 at a time by the producer warp (one per lane) so
  // issuing a chunk never waits on a global load
  RingDesc dl{};
  const int pre = min(S, nloc);
  if (producer) {
    if (wl < nloc) dl = R.desc[cb + wl * cstep];
    for (int i = 0; i < pre; ++i) {  // the matrix is constant: before the dependency wait
      RingDesc d;
      const long long* src = reinterpret_cast<const long long*>(&dl);
      long long* dst = reinterpret_cast<long long*>(&d);
#pragma unroll
      for (int q = 0; q < 8; ++q) dst[q] = __shfl_sync(0xffffffffu, src[q], i & 31);
      if (wl == 0) issue(i, d);
    }
  }

  cudaGridDependencySynchronize();
  if (threadIdx.x == 0) {
    pass = pass_index(k, it, FWD);
    go = loop_over(k) ? 0 : ((sys_on(k.state, 0) || sys_on(k.state, 1)) ? 2 : 1);
  }
  __syncthreads();
  it = pass;
  if (go < 2) {
    // no work this pass: let the prefetched copies land before the CTA exits
    if (producer && wl == 0) {
      for (int i = 0; i < pre; ++i) mbar_wait(&full[i % S], 0);
    }
    if (go == 0 || !FWD) return;
  }

  double r2a = 0.0, r2b = 0.0;
  if (go == 2) {
    if (producer) {
      for (int i = pre; i < nloc; ++i) {
        if ((i & 31) == 0) dl = i + wl < nloc ? R.desc[cb + (i + wl) * cstep] : RingDesc{};
        RingDesc d;
        const long long* src = reinterpret_cast<const long long*>(&dl);
        long long* dst = reinterpret_cast<long long*>(&d);
#pragma unroll
        for (int q = 0; q < 8; ++q) dst[q] = __shfl_sync(0xffffffffu, src[q], i & 31);
        if (wl == 0) {
          mbar_wait(&empty[i % S], ((i / S) - 1) & 1);
          issue(i, d);
        }
        __syncwarp();
      }
    } else {
      const bool on0 = sys_on(k.state, 0), on1 = sys_on(k.state, 1);
      const int lane = threadIdx.x & (VS - 1);
      const unsigned mask = group_mask<VS>();
      const T2* __restrict__ xv = reinterpret_cast<const T2*>(FWD ? k.xx : k.ww);
      const int vend = vend_cta;
      int ci = 0, s = 0;
      for (;;) {
        int l = 0;
        if (lane == 0) l = atomicAdd(&next_v, 1);
        l = __shfl_sync(mask, l, 0, VS);
        if (l >= vend) break;
        // v's chunk (vectors are taken in order, so ci only moves forward),
        // then its slot once the producer has started that chunk in it (a
        // group may run up to S chunks ahead of the slowest one)
        while (lp[ci + 1] <= l) ++ci;
        const int v = gv[ci] + l - lp[ci];
        s = ci % S;
        if (loaded[s] != ci) {
          const long long t0 = clock64();
          while (loaded[s] != ci) {
            __nanosleep(32);
            if (clock64() - t0 > kRingSpinCycles) __trap();
          }
        }
        T e[4] = {T(0), T(0), T(0), T(0)};
        if (!FWD && lane == 0) {  // the iterate changes every pass: from global
          const T2 xo = reinterpret_cast<const T2*>(k.xx)[v];
          e[0] = xo.x;
          e[1] = xo.y;
        }
        mbar_wait(&full[s], (ci / S) & 1);
        const unsigned char* slot = ring + static_cast<size_t>(s) * R.stage_bytes;
        const int vl = v - slot_v0[s];
        const int4 m0 = *reinterpret_cast<const int4*>(slot + R.off_m + 16 * vl);
        const int4 m1 = *reinterpret_cast<const int4*>(slot + R.off_m + 16 * vl + 16);
        if (lane == 0) {
          const unsigned char* ep = slot + R.off_e;
          if (FWD) {  // {p1, p2, rinv1, rinv2}
            const T* pe = reinterpret_cast<const T*>(ep) + 4 * vl;
            e[0] = pe[0];
            e[1] = pe[1];
            e[2] = pe[2];
            e[3] = pe[3];
          } else {
            const long long off = static_cast<long long>(v) * 2 * sizeof(T) - slot_e0[s];
            const T2 cc = *reinterpret_cast<const T2*>(ep + off);
            e[2] = cc.x;
            e[3] = cc.y;
          }
        }
        T da, db;
        ring_dot<T, VS, UF, U16>(slot - slot_i0[s], slot + R.off_v - slot_v0b[s],
                                 slot + R.off_h - slot_h0[s], m0.y, xv, m0.x, m1.x, m0.z, m1.z,
                                 eidx, ev2, lane, mask, R.prefetch != 0, da, db);
        __syncwarp(mask);
        if (lane == 0) {
          if (FWD) {
            const T ra = e[0] - da, rb = e[1] - db;
            T2 wo;
            wo.x = on0 ? e[2] * ra : T(0);
            wo.y = on1 ? e[3] * rb : T(0);
            reinterpret_cast<T2*>(k.ww)[v] = wo;
            if (on0) r2a += static_cast<double>(ra) * static_cast<double>(ra);
            if (on1) r2b += static_cast<double>(rb) * static_cast<double>(rb);
          } else {
            T2 xo;
            xo.x = on0 ? upd(e[0], k.relax, da, e[2]) : e[0];
            xo.y = on1 ? upd(e[1], k.relax, db, e[3]) : e[1];
            reinterpret_cast<T2*>(k.xx)[v] = xo;
            if (on0 && !isfinite(static_cast<double>(xo.x))) atomicCAS(&k.state[2], 0, it + 1);
            if (on1 && !isfinite(static_cast<double>(xo.y))) atomicCAS(&k.state[4 + 2], 0, it + 1);
          }
          if (atomicAdd(&done[s], 1) + 1 == slot_v1[s] - slot_v0[s]) {
            done[s] = 0;
            mbar_arrive(&empty[s]);
          }
        }
      }
    }
  }
  if constexpr (FWD) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      r2a += __shfl_xor_sync(0xffffffffu, r2a, o);
      r2b += __shfl_xor_sync(0xffffffffu, r2b, o);
    }
    if (wl == 0) {
      red[0][warp] = r2a;
      red[1][warp] = r2b;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
      double t = 0.0;
      for (int q = 0; q < kRingWarps; ++q) t += red[threadIdx.x][q];
      k.partial[threadIdx.x * gridDim.x + blockIdx.x] = t;
    }
    if (last_block(k.ticket)) {
      finish_norms<kRingThreads>(k.partial, gridDim.x, 2, k.pnorm, k.tol, k.history, k.hstride,
                                 k.state, it);
      loop_next(k, it);
      if (threadIdx.x == 0) *k.ticket = 0;
    }
  }
}
