// gemm_f16_conv.cu -- 16-bit-mode beamformer GEMM streaming the fp32 data (pack fused, long K).
//
// For plans whose weights fit one 128-row tile (M <= 128, e.g. the small-beam M=32 sweep of
// BASELINE config 5), every data element enters exactly one tile, so converting it on the fly
// costs no re-reads: the separate tcbf_pack(DATA) pass (read 8 B + write 4 B + re-read 4 B per
// element) collapses to one 8-byte read.  Same arithmetic and bit-identical results as
// tcbf_pack + tcbf_beamform (fp16 RNE, four real sub-GEMMs per K step).
//
//   warp 0      TMA producer: packed weight tiles A_r, A_i (K-major, 64-byte swizzle, BK = 32)
//   warp 1      single-thread tcgen05.mma issuer (M=128, N=128, K=16; TMEM double-buffered)
//   warps 2-5   epilogue (cooperative 128-row TMA-store boxes)
//   warps 6-13  converters in two groups of 4 warps taking alternate K blocks: coalesced 128-bit
//               fp32 loads (prefetched before waiting for the stage) -> cvt.rn.f16 -> swizzled
//               MN-major B_r, B_i tiles in the stage buffer
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BM = 128, BN = 128, BK = 32;
constexpr int STAGES = 6;
constexpr int EPI_WARPS = 4;
constexpr int CONV_GROUPS = 2, GROUP_WARPS = 4;
constexpr int NUM_THREADS = (2 + EPI_WARPS + CONV_GROUPS * GROUP_WARPS) * 32;
constexpr int A_BYTES = BM * BK * 2;   // 8 KB per plane
constexpr int B_BYTES = BN * BK * 2;   // 8 KB per plane (2 MN blocks of 64 columns x 32 k-rows)
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int EPI_BYTES = 2 * 16384;
constexpr int BAR_OFFSET = STAGES * STAGE_BYTES + EPI_BYTES;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
constexpr int ITEMS = BK * (BN / 8) / (GROUP_WARPS * 32);  // 16-byte output chunks per thread per K block
static_assert(SMEM_BYTES <= 232448, "smem budget");
static_assert(ITEMS == 4, "converter mapping");

__device__ __forceinline__ uint64_t desc_a64(const void* tile, uint32_t k_byte_off) {
  uint32_t addr = smem_u32(tile) + k_byte_off;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(512u >> 4) << 32;  // 8 rows x 64 B
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)4u << 61;           // SWIZZLE_64B
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
__device__ __forceinline__ uint32_t h2u(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int LAYOUT, bool VEC>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_conv_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmC,
                          GemmF16Args args, const float* __restrict__ xsrc, int K) {
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
  const int num_kb = args.num_kb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1 + GROUP_WARPS);  // TMA (A bytes) + the converter group of this block
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmA);
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
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x) {
        int b, mt, nt;
        tile_coords(t, args.tiles_m, args.tiles_n, args.group_m, b, mt, nt);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], 2 * A_BYTES);
          tma_load_3d(st, &tmA, &full_bar[stage], kb * BK, mt * BM, 2 * b);
          tma_load_3d(st + A_BYTES, &tmA, &full_bar[stage], kb * BK, mt * BM, 2 * b + 1);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC = (1u << 4) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      constexpr uint32_t IDESC_NEG = IDESC | (1u << 13);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x, ++it) {
        const int abuf = it & 1;
        mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_re = tmem_base + abuf * 2 * BN;
        const uint32_t d_im = d_re + BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          uint8_t* st = smem + stage * STAGE_BYTES;
          uint8_t* sAr = st;
          uint8_t* sAi = st + A_BYTES;
          uint8_t* sBr = st + 2 * A_BYTES;
          uint8_t* sBi = sBr + B_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ar = desc_a64(sAr, kk * 32), ai = desc_a64(sAi, kk * 32);
            const uint64_t br = desc_b_mn(sBr, kk * 16), bi = desc_b_mn(sBi, kk * 16);
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            mma_f16_ss(d_re, ar, br, IDESC, acc);
            mma_f16_ss(d_re, ai, bi, IDESC_NEG, 1u);
            mma_f16_ss(d_im, ar, bi, IDESC, acc);
            mma_f16_ss(d_im, ai, br, IDESC, 1u);
          }
          mma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[abuf]);
      }
    }
  } else if (warp < 2 + EPI_WARPS) {
    const int q = warp & 3;
    constexpr int CHUNKS = BN / 32;
    int sbuf = 0;
    int it = 0;
    for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x, ++it) {
      int b, mt, nt;
      tile_coords(t, args.tiles_m, args.tiles_n, args.group_m, b, mt, nt);
      const int m0 = mt * BM, n0 = nt * BN;
      const int abuf = it & 1;
      mbar_wait(&tfull[abuf], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 2 * BN;
      uint32_t v[2][32];
      tmem_ld_32x32b_x32(tbase, v[0]);
#pragma unroll
      for (int ch = 0; ch < 2 * CHUNKS; ++ch) {
        const int part = ch / CHUNKS;
        const int c = ch % CHUNKS;
        tmem_wait_ld();
        if (ch + 1 < 2 * CHUNKS) {
          tmem_ld_32x32b_x32(tbase + (ch + 1) * 32, v[(ch + 1) & 1]);
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[abuf]);
        }
        const uint32_t* vv = v[ch & 1];
        uint8_t* buf = epi_base + sbuf * 16384;
        if (threadIdx.x == 64) bulk_wait_group_read<1>();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int row = q * 32 + lane;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int pos = j ^ (row & 7);
          *reinterpret_cast<uint4*>(buf + row * 128 + pos * 16) =
              make_uint4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]);
        }
        fence_proxy_async_smem();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          tma_store_3d(&tmC, buf, n0 + c * 32, m0, 2 * b + part);
          bulk_commit_group();
        }
        sbuf ^= 1;
      }
    }
    if (threadIdx.x == 64) bulk_wait_group<0>();
  } else {
    // ------------------------------------------------------------ converters (two groups, alternate K blocks)
    const int cw = warp - (2 + EPI_WARPS);
    const int grp = cw / GROUP_WARPS;
    const int ct = (cw % GROUP_WARPS) * 32 + lane;  // 0..127 within the group
    constexpr int NT = GROUP_WARPS * 32;
    const int N = args.N;
    int gk = 0;  // global K-block counter of this CTA (selects group and stage)
    for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x) {
      int b, mt, nt;
      tile_coords(t, args.tiles_m, args.tiles_n, args.group_m, b, mt, nt);
      (void)mt;
      const int n0 = nt * BN;
      for (int kb = 0; kb < num_kb; ++kb, ++gk) {
        if ((gk % CONV_GROUPS) != grp) continue;
        const int stage = gk % STAGES;
        const uint32_t phase = (gk / STAGES) & 1;
        float re[ITEMS][8], im[ITEMS][8];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int item = ct + i * NT;
          const int kr = item / (BN / 8), cc = item % (BN / 8);
          const int k = kb * BK + kr, n = n0 + cc * 8;
          if (VEC && LAYOUT == 0 && k < K && n + 8 <= N) {
            const float4* p = reinterpret_cast<const float4*>(xsrc + (((size_t)b * K + k) * N + n) * 2);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 f = __ldg(p + j);
              re[i][2 * j] = f.x; im[i][2 * j] = f.y; re[i][2 * j + 1] = f.z; im[i][2 * j + 1] = f.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float a = 0.f, c = 0.f;
              if (k < K && n + j < N) {
                if (LAYOUT == 0) {
                  const float2 f = __ldg(reinterpret_cast<const float2*>(xsrc) + ((size_t)b * K + k) * N + n + j);
                  a = f.x; c = f.y;
                } else {
                  a = __ldg(xsrc + (((size_t)b * 2 + 0) * K + k) * N + n + j);
                  c = __ldg(xsrc + (((size_t)b * 2 + 1) * K + k) * N + n + j);
                }
              }
              re[i][j] = a; im[i][j] = c;
            }
          }
        }
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sB = smem + stage * STAGE_BYTES + 2 * A_BYTES;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int item = ct + i * NT;
          const int kr = item / (BN / 8), cc = item % (BN / 8);
          const int off = (cc >> 3) * (BK * 128) + kr * 128 + (((cc & 7) ^ (kr & 7)) << 4);
          *reinterpret_cast<uint4*>(sB + off) = make_uint4(h2u(re[i][0], re[i][1]), h2u(re[i][2], re[i][3]),
                                                           h2u(re[i][4], re[i][5]), h2u(re[i][6], re[i][7]));
          *reinterpret_cast<uint4*>(sB + B_BYTES + off) = make_uint4(
              h2u(im[i][0], im[i][1]), h2u(im[i][2], im[i][3]), h2u(im[i][4], im[i][5]), h2u(im[i][6], im[i][7]));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_bar[stage]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

template <int LAYOUT, bool VEC>
cudaError_t launch_conv(const CUtensorMap& tmA, const CUtensorMap& tmC, const GemmF16Args& a, const float* x, int K,
                        int num_sms, cudaStream_t s) {
  auto kern = cgemm_f16_conv_kernel<LAYOUT, VEC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int grid = a.num_tiles < num_sms ? a.num_tiles : num_sms;
  kern<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(tmA, tmC, a, x, K);
  return cudaGetLastError();
}

}  // namespace

int gemm_f16_conv_block_k() { return BK; }

cudaError_t launch_gemm_f16_conv(const CUtensorMap& tmA, const CUtensorMap& tmC, const GemmF16Args& args,
                                 const float* x_src, int layout, int K, int num_sms, cudaStream_t stream) {
  const bool vec = layout == 0 && (args.N % 8 == 0) && (reinterpret_cast<uintptr_t>(x_src) % 16 == 0);
  if (layout == 0)
    return vec ? launch_conv<0, true>(tmA, tmC, args, x_src, K, num_sms, stream)
               : launch_conv<0, false>(tmA, tmC, args, x_src, K, num_sms, stream);
  return launch_conv<1, false>(tmA, tmC, args, x_src, K, num_sms, stream);
}

}  // namespace tcbf
