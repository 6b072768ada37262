// gemm_f16_conv.cu -- 16-bit-mode beamformer GEMM streaming the fp32 data (pack fused, long K).
//
// For plans whose weights fit one 128-row tile (M <= 128, e.g. the small-beam M=32 sweep of
// BASELINE config 5), every data element enters exactly one tile, so converting it on the fly
// costs no re-reads: the separate tcbf_pack(DATA) pass (read 8 B + write 4 B + re-read 4 B per
// element) collapses to one 8-byte read.  Same arithmetic as tcbf_pack + tcbf_beamform (fp16 RNE,
// four real sub-GEMMs per K step); bit-identical to it when splits == 1.
//
//   warp 0      TMA producer of the raw fp32 data tiles (32 k-rows x 128 columns, interleaved or
//               planar, zero-filled out of bounds) into a 4-deep raw ring
//   warp 1      single-thread tcgen05.mma issuer (M=128, N=128, K=16; TMEM double-buffered)
//   warps 2-5   epilogue (cooperative 128-row TMA boxes: store, or reduce-add for split-K)
//   warps 6-13  converters: raw smem tile -> cvt.rn.f16 -> swizzled MN-major B_r, B_i tiles
//   warp 14     TMA producer of the packed weight tiles A_r, A_i (K-major, 64-byte swizzle)
//
// Work unit = (batch, 128-column tile, K split).  Few column tiles (e.g. 128 tiles on 148 SMs)
// are split along K so every SM streams; partial sums are combined with fp32 TMA reduce-add into
// the zeroed output (the host issues the memset).
#include <algorithm>
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BM = 128, BN = 128, BK = 32;
constexpr int STAGES = 2;      // A + converted B stages
constexpr int RAW_STAGES = 4;  // raw fp32 data stages
constexpr int EPI_WARPS = 4;
constexpr int CONV_WARPS = 8;
constexpr int WARP_A = 2 + EPI_WARPS + CONV_WARPS;
constexpr int NUM_THREADS = (WARP_A + 1) * 32;
constexpr int A_BYTES = BM * BK * 2;   // 8 KB per plane
constexpr int B_BYTES = BN * BK * 2;   // 8 KB per plane (2 MN blocks of 64 columns x 32 k-rows)
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int RAW_BYTES = BK * BN * 8; // 32 KB: 32 k-rows x 128 complex fp32
constexpr int EPI_BYTES = 2 * 16384;
constexpr int RAW_OFFSET = STAGES * STAGE_BYTES;
constexpr int EPI_OFFSET = RAW_OFFSET + RAW_STAGES * RAW_BYTES;
constexpr int BAR_OFFSET = EPI_OFFSET + EPI_BYTES;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
static_assert(SMEM_BYTES <= 232448, "smem budget");
static_assert(BK % CONV_WARPS == 0, "converter rows");

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
// byte offset of column n (even) of k-row kr inside one MN-major 128-byte-swizzled B plane
__device__ __forceinline__ int b_off(int kr, int n) {
  const int blk = n >> 6, c = n & 63;
  return blk * (BK * 128) + kr * 128 + ((((c >> 3) ^ (kr & 7))) << 4) + (c & 7) * 2;
}

struct Unit {
  int b, nt, kb0, kb1;
};
__device__ __forceinline__ Unit unit_of(int u, const GemmF16Args& a) {
  Unit r;
  const int t = u / a.splits, s = u - t * a.splits;
  r.b = t / a.tiles_n;
  r.nt = t - r.b * a.tiles_n;
  r.kb0 = s * a.kb_per_split;
  r.kb1 = min(a.num_kb, r.kb0 + a.kb_per_split);
  return r;
}

template <int LAYOUT>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_conv_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
                          const __grid_constant__ CUtensorMap tmC, GemmF16Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* raw_base = smem + RAW_OFFSET;
  uint8_t* epi_base = smem + EPI_OFFSET;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* rfull = empty_bar + STAGES;
  uint64_t* rempty = rfull + RAW_STAGES;
  uint64_t* tfull = rempty + RAW_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_units = args.num_tiles * args.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1 + CONV_WARPS);  // TMA (A bytes) + every converter warp
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < RAW_STAGES; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], CONV_WARPS);
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
    // ------------------------------------------------------------ raw data producer
    if (lane == 0) {
      int rs = 0;
      uint32_t rph = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        const Unit w = unit_of(u, args);
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&rempty[rs], rph ^ 1);
          uint8_t* dst = raw_base + rs * RAW_BYTES;
          mbar_arrive_expect_tx(&rfull[rs], RAW_BYTES);
          if (LAYOUT == 0) {
            tma_load_3d(dst, &tmX, &rfull[rs], w.nt * 2 * BN, kb * BK, w.b);
          } else {
            tma_load_3d(dst, &tmX, &rfull[rs], w.nt * BN, kb * BK, 2 * w.b);
            tma_load_3d(dst + RAW_BYTES / 2, &tmX, &rfull[rs], w.nt * BN, kb * BK, 2 * w.b + 1);
          }
          if (++rs == RAW_STAGES) { rs = 0; rph ^= 1; }
        }
      }
    }
  } else if (warp == WARP_A) {
    // ------------------------------------------------------------ weight producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        const Unit w = unit_of(u, args);
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], 2 * A_BYTES);
          tma_load_3d(st, &tmA, &full_bar[stage], kb * BK, 0, 2 * w.b);
          tma_load_3d(st + A_BYTES, &tmA, &full_bar[stage], kb * BK, 0, 2 * w.b + 1);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (converged warp, one
    // elected lane issues: descriptors stay in uniform registers)
    {
      constexpr uint32_t IDESC = (1u << 4) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      constexpr uint32_t IDESC_NEG = IDESC | (1u << 13);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++it) {
        const Unit w = unit_of(u, args);
        const int abuf = it & 1;
        mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_re = tmem_base + abuf * 2 * BN;
        const uint32_t d_im = d_re + BN;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint8_t* st = smem + stage * STAGE_BYTES;
          // K advance per MMA: 32 bytes of the K-major A (+2), 16 k-rows of the MN-major B (+128)
          const uint64_t ar0 = desc_a64(st, 0), ai0 = desc_a64(st + A_BYTES, 0);
          const uint64_t br0 = desc_b_mn(st + 2 * A_BYTES, 0), bi0 = desc_b_mn(st + 2 * A_BYTES + B_BYTES, 0);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t ar = ar0 + (uint64_t)(2 * kk), ai = ai0 + (uint64_t)(2 * kk);
              const uint64_t br = br0 + (uint64_t)(128 * kk), bi = bi0 + (uint64_t)(128 * kk);
              const uint32_t acc = (kb != w.kb0 || kk) ? 1u : 0u;
              mma_f16_ss(d_re, ar, br, IDESC, acc);
              mma_f16_ss(d_re, ai, bi, IDESC_NEG, 1u);
              mma_f16_ss(d_im, ar, bi, IDESC, acc);
              mma_f16_ss(d_im, ai, br, IDESC, 1u);
            }
            mma_commit(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit(&tfull[abuf]);
        __syncwarp();
      }
    }
  } else if (warp < 2 + EPI_WARPS) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    constexpr int CHUNKS = BN / 32;
    const bool reduce = args.splits > 1;
    int sbuf = 0;
    int it = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++it) {
      const Unit w = unit_of(u, args);
      const int n0 = w.nt * BN;
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
          if (reduce) tma_reduce_add_3d(&tmC, buf, n0 + c * 32, 0, 2 * w.b + part);
          else tma_store_3d(&tmC, buf, n0 + c * 32, 0, 2 * w.b + part);
          bulk_commit_group();
        }
        sbuf ^= 1;
      }
    }
    if (threadIdx.x == 64) bulk_wait_group<0>();
  } else {
    // ------------------------------------------------------------ converters
    // Each warp converts BK / CONV_WARPS k-rows of every K block.  Interleaved rows are 128
    // complex = 64 float4: lane l reads float4 l and 32 + l (conflict-free), i.e. columns
    // (2l, 2l+1) and (64+2l, 65+2l), and writes them as 4-byte fp16 pairs into MN blocks 0 and 1.
    // Planar rows are 128 floats per plane: lane l reads float4 l of each plane (columns 4l..4l+3).
    const int cw = warp - (2 + EPI_WARPS);
    int stage = 0, rs = 0;
    uint32_t phase = 0, rph = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      const Unit w = unit_of(u, args);
      for (int kb = w.kb0; kb < w.kb1; ++kb) {
        mbar_wait(&rfull[rs], rph);
        const uint8_t* raw = raw_base + rs * RAW_BYTES;
        constexpr int ROWS = BK / CONV_WARPS;
        float4 f[ROWS][2];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          const int kr = cw * ROWS + r;
          if (LAYOUT == 0) {
            const float4* row = reinterpret_cast<const float4*>(raw + kr * (BN * 8));
            f[r][0] = row[lane];
            f[r][1] = row[32 + lane];
          } else {
            f[r][0] = reinterpret_cast<const float4*>(raw + kr * (BN * 4))[lane];
            f[r][1] = reinterpret_cast<const float4*>(raw + RAW_BYTES / 2 + kr * (BN * 4))[lane];
          }
        }
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sB = smem + stage * STAGE_BYTES + 2 * A_BYTES;
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          const int kr = cw * ROWS + r;
          if (LAYOUT == 0) {
            const int o0 = b_off(kr, 2 * lane), o1 = b_off(kr, 64 + 2 * lane);
            *reinterpret_cast<uint32_t*>(sB + o0) = h2u(f[r][0].x, f[r][0].z);
            *reinterpret_cast<uint32_t*>(sB + B_BYTES + o0) = h2u(f[r][0].y, f[r][0].w);
            *reinterpret_cast<uint32_t*>(sB + o1) = h2u(f[r][1].x, f[r][1].z);
            *reinterpret_cast<uint32_t*>(sB + B_BYTES + o1) = h2u(f[r][1].y, f[r][1].w);
          } else {
            const int o = b_off(kr, 4 * lane);
            *reinterpret_cast<uint2*>(sB + o) = make_uint2(h2u(f[r][0].x, f[r][0].y), h2u(f[r][0].z, f[r][0].w));
            *reinterpret_cast<uint2*>(sB + B_BYTES + o) =
                make_uint2(h2u(f[r][1].x, f[r][1].y), h2u(f[r][1].z, f[r][1].w));
          }
        }
        // the raw slot is released only after its values were consumed by the conversion (an
        // arrive straight after the shared loads let the next TMA overwrite loads still in flight)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&full_bar[stage]);
          mbar_arrive(&rempty[rs]);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        if (++rs == RAW_STAGES) { rs = 0; rph ^= 1; }
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

template <int LAYOUT>
cudaError_t launch_conv(const CUtensorMap& tmA, const CUtensorMap& tmX, const CUtensorMap& tmC,
                        const GemmF16Args& a, int num_sms, cudaStream_t s) {
  auto kern = cgemm_f16_conv_kernel<LAYOUT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int units = a.num_tiles * a.splits;
  const int grid = units < num_sms ? units : num_sms;
  kern<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(tmA, tmX, tmC, a);
  return cudaGetLastError();
}

}  // namespace

int gemm_f16_conv_block_k() { return BK; }

int gemm_f16_conv_splits(int tiles, int num_kb, int num_sms) {
  // Only when the column tiles leave many SMs idle (measured: from ~100 tiles on, the whole-GPU
  // HBM stream is already saturated and the memset + reduce-add traffic of a split costs 5-15%).
  // Then the smallest split that gives ~85% of the SMs a unit (measured on M=32: 64 tiles -> 2,
  // 32 tiles -> 4; finer balancing loses to the per-unit pipeline ramp), keeping >= 16 K blocks
  // per split so the partial-tile epilogue is amortised.
  if (tiles <= 0 || num_sms <= 0 || tiles * 5 >= num_sms * 3) return 1;
  int s = (num_sms * 85 / 100 + tiles - 1) / tiles;
  s = std::min(s, std::min(16, num_kb / 16));
  return std::max(s, 1);
}

cudaError_t launch_gemm_f16_conv(const CUtensorMap& tmA, const CUtensorMap& tmX, const CUtensorMap& tmC,
                                 const GemmF16Args& args, int layout, int num_sms, cudaStream_t stream) {
  if (layout == 0) return launch_conv<0>(tmA, tmX, tmC, args, num_sms, stream);
  return launch_conv<1>(tmA, tmX, tmC, args, num_sms, stream);
}

}  // namespace tcbf
