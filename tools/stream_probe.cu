// Microbenchmark (not product code): how fast can a B200 stream two large
// arrays (index int32 + value fp32, like a CSR matrix) under different
// work-partition patterns, with and without dependent gathers?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

// A: grid-stride, each warp instruction reads 32 consecutive elements (lane-strided)
template <bool GATHER>
__global__ void grid_stride(const int* __restrict__ idx, const float* __restrict__ val,
                            const float* __restrict__ x, long long n, float* out) {
  float acc = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    int c0 = __ldg(idx + i), c1 = __ldg(idx + i + stride), c2 = __ldg(idx + i + 2 * stride), c3 = __ldg(idx + i + 3 * stride);
    float v0 = __ldg(val + i), v1 = __ldg(val + i + stride), v2 = __ldg(val + i + 2 * stride), v3 = __ldg(val + i + 3 * stride);
    if (GATHER) acc += v0 * __ldg(x + c0) + v1 * __ldg(x + c1) + v2 * __ldg(x + c2) + v3 * __ldg(x + c3);
    else acc += v0 * c0 + v1 * c1 + v2 * c2 + v3 * c3;
  }
  for (; i < n; i += stride) acc += __ldg(val + i) * (GATHER ? __ldg(x + __ldg(idx + i)) : (float)__ldg(idx + i));
  if (acc == 12345.f) *out = acc;
}

// B: each warp owns a contiguous range [w*L, (w+1)*L) and walks it in 32*Q batches
template <bool GATHER, int Q>
__global__ void warp_ranges(const int* __restrict__ idx, const float* __restrict__ val,
                            const float* __restrict__ x, long long n, long long L, float* out) {
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  long long b = w * L, e = b + L < n ? b + L : n;
  float acc = 0.f;
  for (long long B = b; B < e; B += 32 * Q) {
    int c[Q]; float v[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      long long k = B + lane + 32 * q;
      c[q] = k < e ? __ldg(idx + k) : 0;
      v[q] = k < e ? __ldg(val + k) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) acc += v[q] * (GATHER ? __ldg(x + c[q]) : (float)c[q]);
  }
  if (acc == 12345.f) *out = acc;
}

// C: like B but ranges interleaved at 4 KB granularity across warps (neighbouring
// warps read neighbouring pages at the same time)
template <bool GATHER, int Q>
__global__ void warp_interleaved(const int* __restrict__ idx, const float* __restrict__ val,
                                 const float* __restrict__ x, long long n, float* out) {
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (long long B = w * 32 * Q; B < n; B += W * 32 * Q) {
    int c[Q]; float v[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      long long k = B + lane + 32 * q;
      c[q] = k < n ? __ldg(idx + k) : 0;
      v[q] = k < n ? __ldg(val + k) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) acc += v[q] * (GATHER ? __ldg(x + c[q]) : (float)c[q]);
  }
  if (acc == 12345.f) *out = acc;
}

int main(int argc, char** argv) {
  const long long n = 130LL * 1000 * 1000;  // ~1 GB for idx+val (config-3 scale per kernel is 0.5 GB)
  const int nx = 262144;
  int* idx; float* val; float* x; float* out;
  CK(cudaMalloc(&idx, n * 4)); CK(cudaMalloc(&val, n * 4)); CK(cudaMalloc(&x, nx * 4)); CK(cudaMalloc(&out, 4));
  // snake-like index pattern: runs of 8 consecutive columns then a jump of 512
  std::vector<int> h(n < 1 << 24 ? n : 1 << 24);
  for (size_t k = 0; k < h.size(); ++k) h[k] = (int)(((k / 8) * 512 + (k % 8)) % nx);
  for (long long o = 0; o < n; o += h.size()) CK(cudaMemcpy(idx + o, h.data(), 4 * std::min<long long>(h.size(), n - o), cudaMemcpyHostToDevice));
  CK(cudaMemset(val, 0, n * 4)); CK(cudaMemset(x, 0, nx * 4));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    const int reps = 20;
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-48s %8.1f GB/s  (%.1f us)\n", name, 8.0 * n * reps / (ms * 1e-3) / 1e9, ms * 1e3 / reps);
  };
  for (int bps : {4, 8}) {
    const int blocks = sms * bps, threads = 256;
    const long long W = (long long)blocks * threads / 32;
    const long long L = (n + W - 1) / W;
    char nm[128];
    snprintf(nm, 128, "grid_stride nogather bps=%d", bps);
    run(nm, [&] { grid_stride<false><<<blocks, threads>>>(idx, val, x, n, out); });
    snprintf(nm, 128, "grid_stride gather bps=%d", bps);
    run(nm, [&] { grid_stride<true><<<blocks, threads>>>(idx, val, x, n, out); });
    snprintf(nm, 128, "warp_ranges Q4 nogather bps=%d", bps);
    run(nm, [&] { warp_ranges<false, 4><<<blocks, threads>>>(idx, val, x, n, L, out); });
    snprintf(nm, 128, "warp_ranges Q4 gather bps=%d", bps);
    run(nm, [&] { warp_ranges<true, 4><<<blocks, threads>>>(idx, val, x, n, L, out); });
    snprintf(nm, 128, "warp_ranges Q8 gather bps=%d", bps);
    run(nm, [&] { warp_ranges<true, 8><<<blocks, threads>>>(idx, val, x, n, L, out); });
    snprintf(nm, 128, "warp_interleaved Q4 nogather bps=%d", bps);
    run(nm, [&] { warp_interleaved<false, 4><<<blocks, threads>>>(idx, val, x, n, out); });
    snprintf(nm, 128, "warp_interleaved Q4 gather bps=%d", bps);
    run(nm, [&] { warp_interleaved<true, 4><<<blocks, threads>>>(idx, val, x, n, out); });
    snprintf(nm, 128, "warp_interleaved Q8 gather bps=%d", bps);
    run(nm, [&] { warp_interleaved<true, 8><<<blocks, threads>>>(idx, val, x, n, out); });
  }
  return 0;
}
