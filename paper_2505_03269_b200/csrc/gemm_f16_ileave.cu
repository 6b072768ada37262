// gemm_f16_ileave.cu -- 16-bit-mode beamformer on INTERLEAVED fp16 data, no data pack
// (the paper's future work "a matrix-matrix multiplication kernel that does not
// require this transpose", for producers that emit fp16 directly).
//
// Sample-major: the interleaved data X[b][k][n] = (x_r, x_i) is read as the REAL matrix
// Xr[b][k][2n + p] (K x 2N, row-contiguous) and used AS STORED as the MN-major A operand -- its
// 128 rows are 64 complex samples, real and imaginary part on adjacent TMEM lanes -- against the
// stacked weights [W_r ; W_i] (K-major B operand, N = 256).  ONE MMA per K=16 step,
//     D[2n + p][m]       = sum_k x_p[k][n] W_r[m][k]        (columns 0..127)
//     D[2n + p][128 + m] = sum_k x_p[k][n] W_i[m][k]        (columns 128..255)
// and the complex result (Eq. 3) pairs adjacent lanes:
//     Re[m][n] = D[2n][m] - D[2n+1][128+m],      Im[m][n] = D[2n][128+m] + D[2n+1][m].
// Each lane swaps its W_i-column value with its partner lane (one shfl.xor 1) and forms its part
// with one fused multiply-add by +-1 (exact: the sum / difference of two fp32 accumulators, the
// only rounding-order change against the planar kernels).  Even lanes then hold Re, odd lanes Im of
// the same sample, so a warp store writes two 64-byte runs (Re row, Im row) straight from registers.
//
// Per K step and 64 x 128 complex tile: one M=128 N=256 MMA reading 12 KB (24 KB per 128 x 128
// complex, against 28 KB for the fp32-data sample-major kernel and 32 KB for four N=128 MMAs), no
// data conversion, no smem staging of the output.  Any K (data and weights both stream through a
// 4-stage TMA ring); two 256-column TMEM accumulators.
//
//   warp 0      TMA producer: W_r, W_i boxes {64 K, 128 beams} + the data tile as two {64, 64 K}
//               MN-major boxes (128-byte swizzle; zero fill beyond K / 2N / M)
//   warp 1      MMA issuer: tcgen05.mma.kind::f16, A MN-major, M = 128, N = 256
//   warps 2-9   epilogue: 2 warps per TMEM lane quadrant (16 samples), 64 beams each
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BB = 128;        // beams per tile (stacked N = 256)
constexpr int BSR = 128;       // real data rows per tile (MMA M) = 64 complex samples
constexpr int BSC = BSR / 2;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int EPI_WARPS = 8;
constexpr int NUM_THREADS = (2 + EPI_WARPS) * 32;
constexpr int W_TILE = BB * BK * 2;     // one weight plane (16 KB)
constexpr int X_TILE = BSR * BK * 2;    // the interleaved data tile (16 KB)
constexpr int STAGE_BYTES = 2 * W_TILE + X_TILE;
constexpr int BAR_OFFSET = STAGES * STAGE_BYTES;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
static_assert(SMEM_BYTES <= 232448, "smem budget");

// K-major stacked weights: 8-row groups 1024 B apart, W_i directly after W_r (N = 256)
__device__ __forceinline__ uint64_t desc_w(const void* tile, uint32_t k_byte_off) {
  uint32_t addr = smem_u32(tile) + k_byte_off;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// MN-major data: 64-row (128 B) blocks BK k-rows deep (LBO = BK * 128 B), 8 k-rows per 1024 B
__device__ __forceinline__ uint64_t desc_x(const void* tile, uint32_t k_row) {
  uint32_t addr = smem_u32(tile) + k_row * 128u;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((BK * 128u) >> 4) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}


// tile t of this CTA: MC pairs walk pair tiles (b, mt, nt pair) and take sample tile 2 * pair + rank
__device__ __forceinline__ void my_tile(int t, const GemmF16Args& a, bool mc, int rank, int& b, int& mt, int& nt) {
  if (mc) {
    tile_coords(t, a.tiles_m, a.tiles_n >> 1, a.group_m, b, mt, nt);
    nt = 2 * nt + rank;
  } else {
    tile_coords(t, a.tiles_m, a.tiles_n, a.group_m, b, mt, nt);
  }
}

// MC: CTA pairs (clusters of 2) take the two sample tiles of a (batch, beam tile, sample-tile pair)
// and stream identical weight stages: each CTA TMA-loads one weight plane and multicasts it into both
// (half the L2 -> SM weight traffic, which bounds the loads of 64-sample tiles); a stage is refilled
// only when the MMAs of both CTAs have retired.
template <bool MC>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_ileave_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                            GemmF16Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull = empty_bar + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rank = MC ? (int)cluster_ctarank() : 0;
  const int t_first = MC ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int t_step = MC ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int n_tiles = MC ? args.num_tiles >> 1 : args.num_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], MC ? 2 : 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  if (MC) cluster_sync(); else __syncthreads();  // peers signal this CTA's barriers
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = t_first; t < n_tiles; t += t_step) {
        int b, mt, nt;
        my_tile(t, args, MC, rank, b, mt, nt);
        for (int kb = 0; kb < args.num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
          if (MC) {
            tma_load_3d_mc(st + rank * W_TILE, &tmW, &full_bar[stage], kb * BK, mt * BB, 2 * b + rank);
          } else {
            tma_load_3d(st, &tmW, &full_bar[stage], kb * BK, mt * BB, 2 * b);
            tma_load_3d(st + W_TILE, &tmW, &full_bar[stage], kb * BK, mt * BB, 2 * b + 1);
          }
          uint8_t* sx = st + 2 * W_TILE;
          tma_load_3d(sx, &tmX, &full_bar[stage], nt * BSR, kb * BK, b);
          tma_load_3d(sx + BK * 128, &tmX, &full_bar[stage], nt * BSR + 64, kb * BK, b);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (converged warp, one
    // elected lane issues: descriptors stay in uniform registers)
    {
      // kind::f16: fp16 A (MN-major, bit 15) and B (K-major), fp32 D, M = 128, N = 256
      constexpr uint32_t IDESC = (1u << 4) | (1u << 15) | ((uint32_t)((2 * BB) >> 3) << 17) |
                                 ((uint32_t)(BSR >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = t_first; t < n_tiles; t += t_step, ++it) {
        const int abuf = it & 1;
        mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + abuf * 2 * BB;
        for (int kb = 0; kb < args.num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint8_t* st = smem + stage * STAGE_BYTES;
          // K advance per MMA: 16 k-rows of the MN-major data (+128), 32 bytes of the weights (+2)
          const uint64_t x0 = desc_x(st + 2 * W_TILE, 0), w0 = desc_w(st, 0);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              if (TCBF_ABLATE(args, 2)) continue;
              mma_f16_ss(d, x0 + (uint64_t)(128 * kk), w0 + (uint64_t)(2 * kk), IDESC, (kb | kk) ? 1u : 0u);
            }
            if (MC) mma_commit_mc(&empty_bar[stage]);  // the stage is free in both CTAs
            else mma_commit(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit(&tfull[abuf]);
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;                 // TMEM lane quadrant: real rows 32q..32q+31
    const int half = (warp - 2) >> 2;       // beams 64*half .. 64*half+63 of the tile
    const int p = lane & 1;                 // 0: real row (even lane), 1: imaginary row (odd lane)
    const float sgn = p ? 1.0f : -1.0f;     // Re = D_r[2n] - D_i[2n+1], Im = D_r[2n+1] + D_i[2n]
    const size_t N = (size_t)args.N;
    const int M = args.M;
    int it = 0;
    for (int t = t_first; t < n_tiles; t += t_step, ++it) {
      int b, mt, nt;
      my_tile(t, args, MC, rank, b, mt, nt);
      const int n = nt * BSC + q * 16 + (lane >> 1);  // this lane's sample
      const bool n_ok = n < args.N;
      const int abuf = it & 1;
      mbar_wait(&tfull[abuf], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 2 * BB + half * 64;
#pragma unroll
      for (int c = 0; c < 2; ++c) {          // 2 chunks of 32 beams
        uint32_t vr[32], vi[32];
        tmem_ld_32x32b_x32(tbase + c * 32, vr);        // D[row][m]        (W_r columns)
        tmem_ld_32x32b_x32(tbase + BB + c * 32, vi);   // D[row][128 + m]  (W_i columns)
        tmem_wait_ld();
        if (c == 1) {  // all TMEM reads of this tile done: release the accumulator buffer
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[abuf]);
        }
        const int m0 = mt * BB + half * 64 + c * 32;
        float* dst = args.out + ((size_t)(2 * b + p) * M + m0) * N + n;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float other = __shfl_xor_sync(0xffffffffu, __uint_as_float(vi[j]), 1);
          vr[j] = __float_as_uint(fmaf(sgn, other, __uint_as_float(vr[j])));
        }
        if (TCBF_ABLATE(args, 1)) continue;
        if (n_ok) {
          if (m0 + 32 <= M) {
#pragma unroll
            for (int j = 0; j < 32; ++j) dst[(size_t)j * N] = __uint_as_float(vr[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (m0 + j < M) dst[(size_t)j * N] = __uint_as_float(vr[j]);
          }
        }
      }
    }
  }

  tc_fence_before();
  if (MC) cluster_sync(); else __syncthreads();  // no CTA exits while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace

int gemm_f16_ileave_block_k() { return BK; }
int gemm_f16_ileave_block_n() { return BSC; }

// args: tiles_m = 128-beam tiles, tiles_n = 64-sample tiles, num_kb = ceil(K / 64)
cudaError_t launch_gemm_f16_ileave(const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmC,
                                   const GemmF16Args& args, int num_sms, cudaStream_t stream) {
  (void)tmC;
  const bool mc = args.multicast && args.tiles_n % 2 == 0 && args.num_tiles >= 2;
  if (!mc) {
    auto kern = cgemm_f16_ileave_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    const int grid = args.num_tiles < num_sms ? args.num_tiles : num_sms;
    kern<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(tmW, tmX, args);
    return cudaGetLastError();
  }
  auto kern = cgemm_f16_ileave_kernel<true>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int pairs = args.num_tiles / 2 < num_sms / 2 ? args.num_tiles / 2 : num_sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, tmW, tmX, args);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace tcbf
