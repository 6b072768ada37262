// tma_read_probe.cu -- dev probe: HBM read bandwidth of the swapped 1-bit kernel's packed-word
// stream alone (TMA boxes into a shared-memory ring, no consumers), for box shapes / ring depths.
// Tensor: uint32 [2 planes][N rows][Kw words] (K-contiguous rows, the packed data layout).
// Each CTA streams one 128-row tile over all of K; box = {bw words, br rows} per plane.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2505_03269_b200/csrc
//        tools/probes/tma_read_probe.cu -o tools/probes/tma_read_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace tcbf;

__global__ void __launch_bounds__(32, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, int kw, int bw, int br,
                                                       int stages, int stage_bytes, int rows_per_cta) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
  fence_barrier_init();
  const int row0 = blockIdx.x * rows_per_cta;
  // work items: (row block, K chunk) in K-inner order
  const int kchunks = kw / bw, rblocks = rows_per_cta / br;
  const int items = kchunks * rblocks;
  int issued = 0, done = 0;
  uint32_t phase_bits = 0;
  while (done < items) {
    while (issued < items && issued - done < stages) {
      const int s = issued % stages;
      const int rb = issued / kchunks, kc = issued % kchunks;
      uint8_t* dst = smem + s * stage_bytes;
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      tma_load_3d(dst, &tm, &full[s], kc * bw, row0 + rb * br, 0);
      tma_load_3d(dst + stage_bytes / 2, &tm, &full[s], kc * bw, row0 + rb * br, 1);
      ++issued;
    }
    const int s = done % stages;
    mbar_wait(&full[s], (phase_bits >> s) & 1);
    phase_bits ^= 1u << s;
    ++done;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q);
  if (!encode) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  const int N = 16384, KW = 512;  // K = 16384 bits per row and plane
  constexpr int COPIES = 4;  // rotate over 256 MB so the stream comes from HBM, not the 126 MB L2
  uint32_t* bufs[COPIES];
  const size_t bytes = 2ull * N * KW * 4;
  for (int i = 0; i < COPIES; ++i) {
    cudaMalloc(&bufs[i], bytes);
    cudaMemset(bufs[i], 0x5A, bytes);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct Case { int bw, br, stages, ctas; CUtensorMapSwizzle sw; CUtensorMapL2promotion pr; const char* name; bool blocked = false; };
  const Case cases[] = {
      {32, 128, 3, 128, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "kernel today: 128 B x 128 rows, 3 deep"},
      {32, 128, 4, 128, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "128 B x 128 rows, 4 deep"},
      {32, 128, 5, 128, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "128 B x 128 rows, 5 deep"},
      {32, 128, 4, 128, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, "128 B x 128 rows, 4 deep, no promotion"},
      {32, 128, 4, 128, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, "128 B x 128 rows, 4 deep, 128B promotion"},
      {64, 64, 4, 128, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "256 B x 64 rows, 4 deep"},
      {128, 32, 4, 128, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "512 B x 32 rows, 4 deep"},
      {256, 16, 4, 128, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "1 KB x 16 rows, 4 deep"},
      {256, 16, 4, 128, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "tile-blocked layout: contiguous 16 KB boxes, 4 deep", true},
      {256, 16, 6, 128, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "tile-blocked layout: contiguous 16 KB boxes, 6 deep", true},
  };
  for (const Case& c : cases) {
    CUtensorMap tms[COPIES];
    // blocked: each plane as [N * KW / 256][256] words, i.e. 1 KB rows; CTA c owns the contiguous
    // rows of its tile (128 samples x KW words = 256 KB per plane) and reads them 16 rows at a time
    const cuuint64_t dims[3] = {(cuuint64_t)(c.blocked ? 256 : KW), (cuuint64_t)(c.blocked ? (size_t)N * KW / 256 : N), 2};
    const cuuint64_t strides[2] = {(cuuint64_t)(c.blocked ? 1024 : KW * 4), (cuuint64_t)N * KW * 4};
    const cuuint32_t box[3] = {(cuuint32_t)c.bw, (cuuint32_t)c.br, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = CUDA_SUCCESS;
    for (int i = 0; i < COPIES && r == CUDA_SUCCESS; ++i)
      r = encode(&tms[i], CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, bufs[i], dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw, c.pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", c.name, (int)r); continue; }
    const int stage_bytes = 2 * c.bw * c.br * 4;
    const int smem = 1024 + c.stages * stage_bytes + 256;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int rows_per_cta = c.blocked ? 128 * KW / 256 : 128;
    int rot = 0;
    auto run = [&]() {
      stream_kernel<<<c.ctas, 32, smem>>>(tms[rot++ % COPIES], c.blocked ? 256 : KW, c.bw, c.br, c.stages, stage_bytes,
                                          rows_per_cta);
    };
    run();
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", c.name, cudaGetErrorString(e)); return 1; }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 50; ++i) run();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / 50;
    printf("%-52s %7.2f us  %7.1f GB/s  (%d KB per stage, %d in flight per SM)\n", c.name, us, bytes / us / 1e3,
           stage_bytes / 1024, c.stages * stage_bytes / 1024);
  }
  (void)sms;
  return 0;
}
