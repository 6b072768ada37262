// store_probe.cu -- dev microbenchmark: HBM write bandwidth of TMA bulk-tensor stores in the
// radio fp16 output pattern ([2B][M][N] fp32, 128 x 128 tiles, 32-column x 128-row boxes,
// 128-byte swizzle), no loads and no MMAs, against plain vector stores of the same bytes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2505_03269_b200/csrc
//        store_probe.cu -o /tmp/store_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"

using namespace tcbf;

template <int ROWS, int COLS>
__global__ void __launch_bounds__(128, 1) tma_store_kernel(const __grid_constant__ CUtensorMap tmC, int B, int M, int N,
                                                           int inflight) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tiles_m = M / 128, tiles_n = N / 128;
  const int num_tiles = B * tiles_m * tiles_n;
  constexpr int BOX = ROWS * COLS * 4;
  constexpr int PER_TILE = (128 / ROWS) * (128 / COLS) * 2;
  int buf = 0;
  if (threadIdx.x == 0) {
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int b = t / (tiles_m * tiles_n), r = t % (tiles_m * tiles_n);
      const int mt = r % tiles_m, nt = r / tiles_m;
      for (int c = 0; c < PER_TILE; ++c) {
        const int part = c / (PER_TILE / 2), cc = c % (PER_TILE / 2);
        const int rb = cc / (128 / COLS), cb = cc % (128 / COLS);
        if (inflight == 1) bulk_wait_group_read<0>(); else bulk_wait_group_read<3>();
        tma_store_3d(&tmC, smem + buf * BOX, nt * 128 + cb * COLS, mt * 128 + rb * ROWS, 2 * b + part);
        bulk_commit_group();
        buf = (buf + 1) & 3;
      }
    }
    bulk_wait_group<0>();
  }
}

// per-warp issue (as the 1-bit / fp16 epilogues): each of W warps stores 32-row x 32-column boxes of
// its own 32-row quarter, with up to INFL boxes in flight per warp
template <int W, int INFL>
__global__ void __launch_bounds__(W * 32, 1) tma_store_warps_kernel(const __grid_constant__ CUtensorMap tmC, int B,
                                                                   int M, int N) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = M / 128, tiles_n = N / 128;
  const int num_tiles = B * tiles_m * tiles_n;
  uint8_t* bufs = smem + warp * INFL * 4096;
  int buf = 0;
  if (lane == 0) {
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int b = t / (tiles_m * tiles_n), r = t % (tiles_m * tiles_n);
      const int mt = r % tiles_m, nt = r / tiles_m;
      // this warp's share of the tile's 2 planes x 4 row quarters x 4 column chunks of 32
      for (int i = warp; i < 32; i += W) {
        const int part = i >> 4, q = (i >> 2) & 3, c = i & 3;
        bulk_wait_group_read<INFL - 1>();
        tma_store_3d(&tmC, bufs + buf * 4096, nt * 128 + c * 32, mt * 128 + q * 32, 2 * b + part);
        bulk_commit_group();
        buf = (buf + 1) % INFL;
      }
    }
    bulk_wait_group<0>();
  }
}
// sample-major epilogue pattern (gemm_f16_smaj.cu): unit = (b, 128 samples); per 128-beam tile
// every thread owns one sample and writes 32 beams per chunk with row stride N: one 128-byte line
// per warp instruction.  W warps: 4 (one per 32-sample quadrant) or 8 (quadrant x Re/Im half).
template <int W, int CS>
__global__ void __launch_bounds__(W * 32, 1) smaj_store_kernel(float* out, int B, int M, int N) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, half = warp >> 2;
  const int tiles_n = N / 128, tiles_m = M / 128;
  const int units = B * tiles_n;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int b = u / tiles_n, n = (u % tiles_n) * 128 + q * 32 + lane;
    for (int mt = 0; mt < tiles_m; ++mt) {
#pragma unroll 1
      for (int ch = half * (8 / (W / 4)); ch < (half + 1) * (8 / (W / 4)); ++ch) {
        const int part = ch >> 2, m0 = mt * 128 + (ch & 3) * 32;
        float* dst = out + ((size_t)(2 * b + part) * M + m0) * N + n;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (CS) __stcs(dst + (size_t)j * N, (float)j);
          else dst[(size_t)j * N] = (float)j;
        }
      }
    }
  }
}
// same tiles, but each warp writes whole 512-byte tile rows with 16-byte stores (what a staged,
// transposed epilogue would issue): warp w of W handles rows w, w+W, ... of the 256 tile rows
template <int W>
__global__ void __launch_bounds__(W * 32, 1) rows_store_kernel(float* out, int B, int M, int N) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = N / 128, tiles_m = M / 128;
  const int units = B * tiles_n;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int b = u / tiles_n, n0 = (u % tiles_n) * 128;
    for (int mt = 0; mt < tiles_m; ++mt) {
      for (int r = warp; r < 256; r += W) {
        const int part = r >> 7, m = mt * 128 + (r & 127);
        float4* dst = reinterpret_cast<float4*>(out + ((size_t)(2 * b + part) * M + m) * N + n0) + lane;
        *dst = make_float4(1.f, 2.f, 3.f, (float)r);
      }
    }
  }
}
__global__ void vec_store_kernel(float4* out, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    out[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int B = 256, M = 1024, N = 1024;
  const size_t bytes = (size_t)2 * B * M * N * 4;
  float* out;
  cudaMalloc(&out, bytes);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    const int it = 10;
    for (int i = 0; i < it; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-48s %8.1f us  %7.0f GB/s  (%s)\n", name, ms * 1e3 / it, bytes / (ms / it * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  auto make_map = [&](uint32_t bc, uint32_t br, CUtensorMapSwizzle sw) {
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)2 * B};
    cuuint64_t strides[2] = {(cuuint64_t)N * 4, (cuuint64_t)N * M * 4};
    cuuint32_t box[3] = {bc, br, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     sw, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return m;
  };
  run("vector float4 stores (grid-stride)", [&] { vec_store_kernel<<<sms * 8, 512>>>((float4*)out, bytes / 16); });
  run("smaj st.global.f32 lines, 4 warps", [&] { smaj_store_kernel<4, 0><<<sms, 128>>>(out, B, M, N); });
  run("smaj st.global.f32 lines, 8 warps", [&] { smaj_store_kernel<8, 0><<<sms, 256>>>(out, B, M, N); });
  run("smaj st.global.cs.f32 lines, 8 warps", [&] { smaj_store_kernel<8, 1><<<sms, 256>>>(out, B, M, N); });
  run("smaj st.global.f32 lines, 16 warps", [&] { smaj_store_kernel<16, 0><<<sms, 512>>>(out, B, M, N); });
  run("smaj st.global.f32 lines, 8 warps x 2 CTA/SM", [&] { smaj_store_kernel<8, 0><<<2 * sms, 256>>>(out, B, M, N); });
  run("tile rows st.global.v4 (512 B), 8 warps", [&] { rows_store_kernel<8><<<sms, 256>>>(out, B, M, N); });
  run("tile rows st.global.v4 (512 B), 16 warps", [&] { rows_store_kernel<16><<<sms, 512>>>(out, B, M, N); });
  {
    CUtensorMap m = make_map(32, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    auto k = tma_store_kernel<128, 32>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384 + 1024);
    run("TMA box 32c x 128r swz128 (kernel pattern), 2 inflight", [&] { k<<<sms, 128, 4 * 16384 + 1024>>>(m, B, M, N, 0); });
    run("TMA box 32c x 128r swz128, 1 inflight", [&] { k<<<sms, 128, 4 * 16384 + 1024>>>(m, B, M, N, 1); });
  }
  {
    CUtensorMap m = make_map(128, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    auto k = tma_store_kernel<32, 128>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384 + 1024);
    run("TMA box 128c x 32r no swizzle (512 B rows)", [&] { k<<<sms, 128, 4 * 16384 + 1024>>>(m, B, M, N, 0); });
  }
  {
    CUtensorMap m = make_map(32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    auto k = tma_store_kernel<32, 32>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 4096 + 1024);
    run("TMA box 32c x 32r swz128", [&] { k<<<sms, 128, 4 * 4096 + 1024>>>(m, B, M, N, 0); });
  }
  {
    CUtensorMap m = make_map(32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    auto k1 = tma_store_warps_kernel<8, 2>;
    auto k2 = tma_store_warps_kernel<8, 4>;
    auto k3 = tma_store_warps_kernel<8, 6>;
    auto k4 = tma_store_warps_kernel<16, 4>;
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 2 * 4096 + 1024);
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * 4096 + 1024);
    cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 6 * 4096 + 1024);
    cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4 * 4096 + 1024);
    run("TMA 32x32 boxes, 8 warps x 2 in flight", [&] { k1<<<sms, 256, 8 * 2 * 4096 + 1024>>>(m, B, M, N); });
    run("TMA 32x32 boxes, 8 warps x 4 in flight", [&] { k2<<<sms, 256, 8 * 4 * 4096 + 1024>>>(m, B, M, N); });
    run("TMA 32x32 boxes, 8 warps x 6 in flight", [&] { k3<<<sms, 256, 8 * 6 * 4096 + 1024>>>(m, B, M, N); });
    run("TMA 32x32 boxes, 16 warps x 4 in flight", [&] { k4<<<sms, 512, 16 * 4 * 4096 + 1024>>>(m, B, M, N); });
  }
  return 0;
}
