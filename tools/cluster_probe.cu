// Microbenchmark (not product code): cost of a cluster barrier and of the
// first shared-memory / global access after it, 16 CTAs x 512 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_probe cluster_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(long long* out, double* g, int iters) {
  __shared__ double red[32];
  __shared__ double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += 512) buf[i] = i;
  if (threadIdx.x < 32) red[threadIdx.x] = threadIdx.x;
  __syncthreads();
  long long t_bar = 0, t_after = 0;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    // some global traffic before the barrier, like the SART phases
    if (MODE & 1) {
      for (int i = threadIdx.x; i < 2048; i += 512) acc += __ldg(g + blockIdx.x * 2048 + i);
      g[blockIdx.x * 2048 + threadIdx.x] = acc;
    }
    long long t0 = clock64();
    if (MODE & 2) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    } else {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    long long t1 = clock64();
    double v = red[threadIdx.x & 31];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    acc += v;
    long long t2 = clock64();
    t_bar += t1 - t0;
    t_after += t2 - t1;
  }
  if (threadIdx.x == 0) {
    out[3 * blockIdx.x] = t_bar / iters;
    out[3 * blockIdx.x + 1] = t_after / iters;
    out[3 * blockIdx.x + 2] = (long long)acc;
  }
}

template <int MODE>
void run(long long* d, double* g) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16);
  cfg.blockDim = dim3(512);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 16;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, probe<MODE>, d, g, 1000);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[48];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("mode %d (%s%s): %.2f us/iter  barrier %lld cyc  LDS+shfl after %lld cyc  err=%s\n", MODE,
           MODE & 2 ? "relaxed arrive" : "release/acquire", MODE & 1 ? ", global traffic" : "",
           ms * 1000 / 1000, h[0], h[1], cudaGetErrorString(err));
  }
}

int main() {
  long long* d;
  double* g;
  cudaMalloc(&d, 48 * 8);
  cudaMalloc(&g, 16 * 2048 * 8 * 2);
  cudaMemset(g, 0, 16 * 2048 * 8 * 2);
  run<0>(d, g);
  run<1>(d, g);
  run<2>(d, g);
  run<3>(d, g);
  return 0;
}
