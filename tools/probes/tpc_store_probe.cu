// tpc_store_probe.cu -- dev microbenchmark: is HBM write bandwidth of the radio output pattern
// (128-byte line stores from registers, one beam row per warp store, [2B][M][N] fp32) limited per
// SM, per TPC (SM pair), or by lock-stepped CTA pairs?  Same bytes in every mode:
//   0  148 CTAs, no cluster, all store (free-running, like the single-CTA sample-major kernel)
//   1  148 CTAs in clusters of 2, only rank 0 stores (one storing SM per cluster)
//   2  148 CTAs in clusters of 2, both store, cluster barrier after every 128x128 tile (lock-step,
//      like the cta_group::2 kernel's shared TMEM buffers)
//   3  74 CTAs, no cluster, all store
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tpc_store_probe.cu -o /tmp/tpc_probe
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// tile = 128 samples x 128 beams x 2 planes; 8 warps: warp w -> lane quadrant q = w & 3 (samples),
// half = w >> 2 (plane); each thread stores 4 chunks x 32 rows
template <int MODE>
__global__ void __launch_bounds__(256, 1) store_kernel(float* out, int B, int M, int N, int storers,
                                                       unsigned* sm_of) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, half = warp >> 2;
  const int tiles_m = M / 128, tiles_n = N / 128;
  const long long num_tiles = (long long)B * tiles_m * tiles_n;
  int worker, nworkers;
  bool active = true;
  if (MODE == 1) {
    worker = blockIdx.x >> 1;
    nworkers = gridDim.x >> 1;
    active = cluster_rank() == 0;
  } else {
    worker = blockIdx.x;
    nworkers = gridDim.x;
  }
  if (threadIdx.x == 0) sm_of[blockIdx.x] = smid();
  const float v = 1.0f + lane;
  const long long my_tiles = (num_tiles - worker + nworkers - 1) / nworkers;
  for (long long i = 0; i < my_tiles; ++i) {
    const long long t = worker + i * nworkers;
    if (active) {
      const int b = (int)(t / (tiles_m * tiles_n));
      const int r = (int)(t % (tiles_m * tiles_n));
      const int nt = r / tiles_m, mt = r % tiles_m;
      const int n = nt * 128 + q * 32 + lane;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float* dst = out + ((size_t)(2 * b + half) * M + mt * 128 + c * 32) * N + n;
#pragma unroll
        for (int j = 0; j < 32; ++j) dst[(size_t)j * N] = v;
      }
    }
    if (MODE == 2) cluster_barrier();
  }
}

template <int MODE>
float run(float* out, int B, int M, int N, int grid, int cluster, unsigned* sm_of) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) cudaLaunchKernelEx(&cfg, store_kernel<MODE>, out, B, M, N, 0, sm_of);
  cudaEventRecord(e0);
  const int it = 20;
  for (int w = 0; w < it; ++w) cudaLaunchKernelEx(&cfg, store_kernel<MODE>, out, B, M, N, 0, sm_of);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms / it;
}

int main() {
  const int B = 256, M = 1024, N = 1024;
  const size_t bytes = (size_t)2 * B * M * N * 4;
  float* out;
  unsigned* sm_of;
  cudaMalloc(&out, bytes);
  cudaMalloc(&sm_of, 1024 * 4);
  const char* names[4] = {"148 CTAs free-running", "74 clusters of 2, rank 0 stores", "74 clusters of 2, lock-step",
                          "74 CTAs free-running"};
  for (int rep = 0; rep < 2; ++rep) {
    float t[4];
    t[0] = run<0>(out, B, M, N, 148, 1, sm_of);
    t[1] = run<1>(out, B, M, N, 148, 2, sm_of);
    if (rep == 0) {
      unsigned h[148];
      cudaMemcpy(h, sm_of, sizeof(h), cudaMemcpyDeviceToHost);
      int same_tpc = 0;
      for (int c = 0; c < 74; ++c) same_tpc += (h[2 * c] >> 1) == (h[2 * c + 1] >> 1);
      printf("clusters of 2 whose CTAs share smid>>1: %d / 74 (e.g. %u,%u %u,%u)\n", same_tpc, h[0], h[1], h[2], h[3]);
    }
    t[2] = run<2>(out, B, M, N, 148, 2, sm_of);
    t[3] = run<0>(out, B, M, N, 74, 1, sm_of);
    for (int m = 0; m < 4; ++m)
      printf("%-36s %8.1f us  %6.2f TB/s\n", names[m], t[m] * 1e3, bytes / (t[m] * 1e-3) / 1e12);
  }
  return 0;
}
