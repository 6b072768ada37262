// gemm_f16_ileave.cu -- 16-bit-mode beamformer GEMM on INTERLEAVED fp16 data, no data pack
// (the paper's future work "a matrix-matrix multiplication kernel that does not
// require this transpose", for producers that emit fp16 directly).
//
// The interleaved data X[b][k][n] = (x_r, x_i) is read as a REAL matrix Xr[b][k][2n + c]
// (K x 2N, row-contiguous) and fed to the tensor cores MN-major exactly as stored.  Two real
// GEMMs per K step against the same data tile,
//     D1 = A_r Xr ,  D2 = A_i Xr        (A_r, A_i: packed weight planes, K-major)
// give, column pair (2n, 2n+1) = (x_r, x_i) of sample n,
//     D1[2n] = sum A_r x_r, D1[2n+1] = sum A_r x_i, D2[2n] = sum A_i x_r, D2[2n+1] = sum A_i x_i,
// and the epilogue forms the complex result (Eq. 3):
//     Re = D1[2n] - D2[2n+1],   Im = D1[2n+1] + D2[2n].
// Same products as the planar kernel (exact fp16 x fp16, fp32 accumulation); the final
// subtraction / addition of two fp32 accumulators is the only change of rounding order.
//
// Tile = 128 beams x 64 samples (128 real data columns): D1 and D2 take 128 TMEM columns each,
// so two accumulator sets fit (epilogue of tile i overlaps the MMAs of tile i+1).
//   warp 0      TMA producer (A_r, A_i K-major boxes; the data tile as two 64-column MN-major boxes)
//   warp 1      MMA issuer: 2 x tcgen05.mma (M=128, N=128, K=16) per K step
//   warps 2-5   epilogue: tcgen05.ld D1 / D2 -> recombination -> 32 x 32 TMA store boxes of the
//               planar fp32 output (Re plane and Im plane)
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BM = 128;
constexpr int BNC = 64;        // complex samples per tile
constexpr int BNR = 2 * BNC;   // real data columns per tile (MMA N)
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int EPI_WARPS = 4;
constexpr int NUM_THREADS = (2 + EPI_WARPS) * 32;
constexpr int A_BYTES = BM * BK * 2;   // one weight plane
constexpr int B_BYTES = BNR * BK * 2;  // the interleaved data tile (2 blocks of 64 real columns)
constexpr int STAGE_BYTES = 2 * A_BYTES + B_BYTES;
constexpr int EPI_BYTES = EPI_WARPS * 2 * 4096;  // per warp: Re box + Im box (32 x 32 fp32)
constexpr int BAR_OFFSET = STAGES * STAGE_BYTES + EPI_BYTES;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
static_assert(SMEM_BYTES <= 232448, "smem budget");

__device__ __forceinline__ uint64_t desc_a128(const void* tile, uint32_t k_byte_off) {
  uint32_t addr = smem_u32(tile) + k_byte_off;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__device__ __forceinline__ uint64_t desc_b_mn(const void* tile, uint32_t k_row) {
  uint32_t addr = smem_u32(tile) + k_row * 128u;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((BK * 128u) >> 4) << 16;  // LBO: next 64-column block
  d |= (uint64_t)(1024u >> 4) << 32;        // SBO: next 8 k-rows
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_ileave_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
                            const __grid_constant__ CUtensorMap tmC, GemmF16Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_base = smem + STAGES * STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull = empty_bar + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmC);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x) {
        int b, mt, nt;
        tile_coords(t, args.tiles_m, args.tiles_n, args.group_m, b, mt, nt);
        for (int kb = 0; kb < args.num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
          tma_load_3d(st, &tmA, &full_bar[stage], kb * BK, mt * BM, 2 * b);
          tma_load_3d(st + A_BYTES, &tmA, &full_bar[stage], kb * BK, mt * BM, 2 * b + 1);
          uint8_t* sb = st + 2 * A_BYTES;
          tma_load_3d(sb, &tmX, &full_bar[stage], nt * BNR, kb * BK, b);
          tma_load_3d(sb + BK * 128, &tmX, &full_bar[stage], nt * BNR + 64, kb * BK, b);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // f16 A (K-major) and B (MN-major, bit 16), f32 D, M = 128, N = 128 real columns
      constexpr uint32_t IDESC = (1u << 4) | (1u << 16) | ((uint32_t)(BNR >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x, ++it) {
        const int abuf = it & 1;
        mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d1 = tmem_base + abuf * 2 * BNR;
        const uint32_t d2 = d1 + BNR;
        for (int kb = 0; kb < args.num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          uint8_t* st = smem + stage * STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ar = desc_a128(st, kk * 32), ai = desc_a128(st + A_BYTES, kk * 32);
            const uint64_t bx = desc_b_mn(st + 2 * A_BYTES, kk * 16);
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            mma_f16_ss(d1, ar, bx, IDESC, acc);  // A_r [x_r x_i ...]
            mma_f16_ss(d2, ai, bx, IDESC, acc);  // A_i [x_r x_i ...]
          }
          mma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[abuf]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    uint8_t* bufs = epi_base + (warp - 2) * 2 * 4096;  // [Re box][Im box], 32 rows x 128 B
    int it = 0;
    for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x, ++it) {
      int b, mt, nt;
      tile_coords(t, args.tiles_m, args.tiles_n, args.group_m, b, mt, nt);
      const int m0 = mt * BM + q * 32;
      const int abuf = it & 1;
      mbar_wait(&tfull[abuf], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 2 * BNR;
#pragma unroll 1
      for (int box = 0; box < BNC / 32; ++box) {  // 32 complex samples per output box
        if (lane == 0) bulk_wait_group_read<0>();  // both boxes of the previous round read
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // 16 complex samples = 32 real columns of D1 and D2
          uint32_t v1[32], v2[32];
          const uint32_t col = (uint32_t)(box * 64 + h * 32);
          tmem_ld_32x32b_x32(tb + col, v1);
          tmem_ld_32x32b_x32(tb + BNR + col, v2);
          tmem_wait_ld();
          if (box == BNC / 32 - 1 && h == 1) {  // last TMEM read of this tile
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[abuf]);
          }
          uint32_t re[16], im[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            re[j] = __float_as_uint(__uint_as_float(v1[2 * j]) - __uint_as_float(v2[2 * j + 1]));
            im[j] = __float_as_uint(__uint_as_float(v1[2 * j + 1]) + __uint_as_float(v2[2 * j]));
          }
          // columns h*16 .. h*16+15 of the 32-column boxes: 16-byte chunks 4h .. 4h+3, 128-B swizzle
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int pos = (4 * h + j) ^ (lane & 7);
            *reinterpret_cast<uint4*>(bufs + lane * 128 + pos * 16) =
                make_uint4(re[4 * j], re[4 * j + 1], re[4 * j + 2], re[4 * j + 3]);
            *reinterpret_cast<uint4*>(bufs + 4096 + lane * 128 + pos * 16) =
                make_uint4(im[4 * j], im[4 * j + 1], im[4 * j + 2], im[4 * j + 3]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const int n0 = nt * BNC + box * 32;
          tma_store_3d(&tmC, bufs, n0, m0, 2 * b);
          tma_store_3d(&tmC, bufs + 4096, n0, m0, 2 * b + 1);
          bulk_commit_group();
        }
      }
    }
    if (lane == 0) bulk_wait_group<0>();
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace

int gemm_f16_ileave_block_k() { return BK; }
int gemm_f16_ileave_block_n() { return BNC; }

cudaError_t launch_gemm_f16_ileave(const CUtensorMap& tmA, const CUtensorMap& tmX, const CUtensorMap& tmC,
                                   const GemmF16Args& args, int num_sms, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(cgemm_f16_ileave_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int grid = args.num_tiles < num_sms ? args.num_tiles : num_sms;
  cgemm_f16_ileave_kernel<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(tmA, tmX, tmC, args);
  return cudaGetLastError();
}

}  // namespace tcbf
