// gemm_f16_ileave_res.cu -- 16-bit-mode beamformer on INTERLEAVED fp16 data with the data
// resident per unit ("a kernel that does not require this transpose";
// fp16 producers), K16 <= 256.
//
// Same arithmetic as gemm_f16_ileave.cu: the interleaved data X[b][k][n] = (x_r, x_i) is the REAL
// matrix Xr[b][k][2n + p] used as stored as the MN-major A operand (real and imaginary part of a
// sample on adjacent TMEM lanes) against the stacked weights [W_r ; W_i] (K-major B), and the
// epilogue pairs adjacent lanes (one shfl.xor 1 and a +-1 FMA):
//     Re[m][n] = D[2n][m] - D[2n+1][BB+m],      Im[m][n] = D[2n][BB+m] + D[2n+1][m].
// Differences from the streaming kernel, all aimed at the radio shape's byte budget:
//   * work unit = (batch entry, 128 samples = 256 real rows); the unit's data (128 KB for K16 =
//     256) is loaded ONCE by TMA into four 64-k-row slots and stays resident while all beam tiles
//     stream past it (the streaming kernel re-reads it from L2 for every beam tile), the slots are
//     refilled by a loader warp as the unit's last beam tile releases them;
//   * beam tile = 64 beams: two M=128, N=128 MMAs per K=16 step (one per 128-row half of the unit),
//     so a 16 KB weight stage serves 128 samples (the streaming kernel's 32 KB stage served 64) and
//     the weight bytes per output byte halve; TMEM holds two 256-column accumulators;
//   * weight stages multicast across CTA pairs walking adjacent units.
// No thread of this kernel issues a global load: the SM's load/store pipeline carries only the
// output line stores (on the fp32-input path those share it with the data loads).
//
// Roles: warp 0 TMA producer (weights), warp 1 MMA issuer, warps 2-9 epilogue (quadrant x half),
// warp 10 data loader (TMA, slot refills).
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BB = 64;                 // beams per tile (stacked N = 128)
constexpr int BS = 128;                // complex samples per unit (two 128-row MMA halves)
constexpr int BK = 64;                 // k-rows per data slot / K per weight stage
constexpr int KMAX = 256;
constexpr int X_SLOTS = KMAX / BK;     // 4
constexpr int X_BOX = 64 * BK * 2;     // one TMA box: 64 real columns x 64 k-rows fp16 (8 KB)
constexpr int X_HALF = 2 * X_BOX;      // one 128-row MMA half of a slot
constexpr int X_SLOT = 2 * X_HALF;     // 32 KB
constexpr int W_TILE = BB * BK * 2;    // one weight plane (8 KB)
constexpr int W_BLK = 2 * W_TILE;      // [W_r ; W_i] of one 64-k block
// Two K blocks per weight stage: the MMA issuer waits and commits once per 16 MMAs.  Every wait or
// commit between MMA issues idles the tensor pipe for a few hundred cycles
// (tools/probes/mma_pattern_probe.cu), against ~630 cycles of tensor work per block at N = 128.
constexpr int W_SBLK = 2;
constexpr int W_STAGE = W_SBLK * W_BLK;
constexpr int W_STAGES = 3;
constexpr int EPI_WARPS = 8;
constexpr int LOADER_WARP = 2 + EPI_WARPS;
constexpr int NUM_THREADS = (LOADER_WARP + 1) * 32;
constexpr int OFF_W = X_SLOTS * X_SLOT;
constexpr int BAR_OFFSET = OFF_W + W_STAGES * W_STAGE;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
static_assert(SMEM_BYTES <= 232448, "smem budget");

__device__ __forceinline__ uint64_t desc_w(const void* tile, uint32_t k_byte_off) {
  uint32_t addr = smem_u32(tile) + k_byte_off;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// MN-major data half: two 64-column boxes X_BOX apart (LBO), 8 k-rows per 1024 B (SBO)
__device__ __forceinline__ uint64_t desc_x(const void* half, uint32_t k_row) {
  uint32_t addr = smem_u32(half) + k_row * 128u;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((uint32_t)X_BOX >> 4) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

// MC: CTA pairs take adjacent units (same batch entry, tiles_n even) and walk the same (beam tile,
// K block) sequence: each CTA loads one weight plane and multicasts it into both.
template <bool MC>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_ileave_res_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                                GemmF16Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = smem;
  uint8_t* sW = smem + OFF_W;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* wempty = wfull + W_STAGES;
  uint64_t* xfull = wempty + W_STAGES;
  uint64_t* xempty = xfull + X_SLOTS;
  uint64_t* tfull = xempty + X_SLOTS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = args.num_kb;  // K16 / 64 <= 4
  const int tiles_m = args.tiles_m, tiles_n = args.tiles_n;  // 64-beam tiles, 128-sample units per batch
  const int num_units = args.B * tiles_n;
  const int rank = MC ? (int)cluster_ctarank() : 0;
  const int u_first = MC ? 2 * (int)(blockIdx.x >> 1) + rank : (int)blockIdx.x;
  const int u_step = MC ? 2 * (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < W_STAGES; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], MC ? 2 : 1);
    }
    for (int s = 0; s < X_SLOTS; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
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
  if (MC) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer: weight stages
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = u_first; u < num_units; u += u_step) {
        const int b = u / tiles_n;
        for (int mt = 0; mt < tiles_m; ++mt) {
          for (int kb0 = 0; kb0 < num_kb; kb0 += W_SBLK) {
            const int nb = min(W_SBLK, num_kb - kb0);
            mbar_wait(&wempty[stage], phase ^ 1);
            uint8_t* st = sW + stage * W_STAGE;
            mbar_arrive_expect_tx(&wfull[stage], nb * W_BLK);
            for (int j = 0; j < nb; ++j) {
              const int kb = kb0 + j;
              if (MC) {
                tma_load_3d_mc(st + j * W_BLK + rank * W_TILE, &tmW, &wfull[stage], kb * BK, mt * BB, 2 * b + rank);
              } else {
                tma_load_3d(st + j * W_BLK, &tmW, &wfull[stage], kb * BK, mt * BB, 2 * b);
                tma_load_3d(st + j * W_BLK + W_TILE, &tmW, &wfull[stage], kb * BK, mt * BB, 2 * b + 1);
              }
            }
            if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (converged warp,
    // one elected lane issues: descriptors stay in uniform registers)
    // kind::f16: fp16 A (MN-major, bit 15) and B (K-major), fp32 D, M = 128, N = 2 BB
    constexpr uint32_t IDESC = (1u << 4) | (1u << 15) | ((uint32_t)((2 * BB) >> 3) << 17) | ((128u >> 4) << 24);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0, ui = 0;
    for (int u = u_first; u < num_units; u += u_step, ++ui) {
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int abuf = it & 1;
        mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + abuf * 4 * BB;  // two halves of 2 BB columns
        for (int kb0 = 0; kb0 < num_kb; kb0 += W_SBLK) {
          const int nb = min(W_SBLK, num_kb - kb0);
          if (mt == 0) {  // the unit's data slots have landed
            mbar_wait(&xfull[kb0], ui & 1);
            if (nb > 1) mbar_wait(&xfull[kb0 + 1], ui & 1);
          }
          mbar_wait(&wfull[stage], phase);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int j = 0; j < W_SBLK; ++j) {
              if (j >= nb) break;
              const int kb = kb0 + j;
              const uint64_t w0 = desc_w(sW + stage * W_STAGE + j * W_BLK, 0);
              const uint64_t x0 = desc_x(sX + kb * X_SLOT, 0), x1 = desc_x(sX + kb * X_SLOT + X_HALF, 0);
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {  // K advance: +32 bytes = +2 in the address field
                const uint32_t acc = (kb | kk) ? 1u : 0u;
                if (TCBF_ABLATE(args, 2)) continue;
                mma_f16_ss(d, x0 + (uint64_t)(kk * 128), w0 + (uint64_t)(kk * 2), IDESC, acc);          // samples 0..63
                mma_f16_ss(d + 2 * BB, x1 + (uint64_t)(kk * 128), w0 + (uint64_t)(kk * 2), IDESC, acc); // 64..127
              }
              if (mt == tiles_m - 1) mma_commit(&xempty[kb]);  // last reader of this data slot
            }
            if (MC) mma_commit_mc(&wempty[stage]);
            else mma_commit(&wempty[stage]);
          }
          __syncwarp();
          if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit(&tfull[abuf]);
        __syncwarp();
      }
    }
  } else if (warp < LOADER_WARP) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;                 // TMEM lane quadrant: real rows 32q..32q+31 of a half
    const int h = (warp - 2) >> 2;          // half of the unit: samples 64h..64h+63
    const int p = lane & 1;                 // 0: real row (even lane), 1: imaginary row (odd lane)
    const float sgn = p ? 1.0f : -1.0f;     // Re = D_r[2n] - D_i[2n+1], Im = D_r[2n+1] + D_i[2n]
    const size_t N = (size_t)args.N;
    const int M = args.M;
    int it = 0;
    for (int u = u_first; u < num_units; u += u_step) {
      const int b = u / tiles_n;
      const int n = (u - b * tiles_n) * BS + h * 64 + q * 16 + (lane >> 1);  // this lane's sample
      const bool n_ok = n < args.N;
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int abuf = it & 1;
        mbar_wait(&tfull[abuf], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 4 * BB + h * 2 * BB;
        uint32_t vr[2][32], vi[2][32];
        tmem_ld_32x32b_x32(tbase, vr[0]);         // D[row][m]       (W_r columns), beams 0..31
        tmem_ld_32x32b_x32(tbase + BB, vi[0]);    // D[row][BB + m]  (W_i columns)
        tmem_ld_32x32b_x32(tbase + 32, vr[1]);    // beams 32..63
        tmem_ld_32x32b_x32(tbase + BB + 32, vi[1]);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[abuf]);  // the accumulator buffer may be reused
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int m0 = mt * BB + c * 32;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float other = __shfl_xor_sync(0xffffffffu, __uint_as_float(vi[c][j]), 1);
            vr[c][j] = __float_as_uint(fmaf(sgn, other, __uint_as_float(vr[c][j])));
          }
          if (TCBF_ABLATE(args, 1)) continue;
          if (n_ok) {
            float* dst = args.out + ((size_t)(2 * b + p) * M + m0) * N + n;
            if (m0 + 32 <= M) {
#pragma unroll
              for (int j = 0; j < 32; ++j) dst[(size_t)j * N] = __uint_as_float(vr[c][j]);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (m0 + j < M) dst[(size_t)j * N] = __uint_as_float(vr[c][j]);
            }
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ data loader: unit slots by TMA
    if (lane == 0) {
      int ui = 0;
      for (int u = u_first; u < num_units; u += u_step, ++ui) {
        const int b = u / tiles_n;
        const int c0 = (u - b * tiles_n) * 2 * BS;  // first real column of the unit
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&xempty[kb], (ui & 1) ^ 1);  // the previous unit's last tile released it
          uint8_t* sx = sX + kb * X_SLOT;
          mbar_arrive_expect_tx(&xfull[kb], X_SLOT);
#pragma unroll
          for (int c = 0; c < 4; ++c)  // 4 boxes of 64 real columns (zero fill past 2N / K)
            tma_load_3d(sx + c * X_BOX, &tmX, &xfull[kb], c0 + c * 64, kb * BK, b);
        }
      }
    }
  }

  tc_fence_before();
  if (MC) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace

bool gemm_f16_ileave_res_supported(int64_t K16) { return K16 <= KMAX; }
int gemm_f16_ileave_res_beams() { return BB; }
int gemm_f16_ileave_res_samples() { return BS; }

// args: tiles_m = 64-beam tiles, tiles_n = 128-sample units per batch entry, num_kb = K16 / 64;
// tmW: packed weights, box {64 K, 64 beams}; tmX: fp16 data as [B][K][2N], box {64 columns, 64 k}
// (both 128-byte swizzle)
cudaError_t launch_gemm_f16_ileave_res(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmF16Args& args,
                                       int num_sms, cudaStream_t stream) {
  const int units = args.B * args.tiles_n;
  const bool mc = args.multicast && args.tiles_n % 2 == 0 && units >= 2;
  if (!mc) {
    auto kern = cgemm_f16_ileave_res_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    const int grid = units < num_sms ? units : num_sms;
    kern<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(tmW, tmX, args);
    return cudaGetLastError();
  }
  auto kern = cgemm_f16_ileave_res_kernel<true>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int pairs = units / 2 < num_sms / 2 ? units / 2 : num_sms / 2;
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
