// PARKED (round 2): the round-1 beam-major fused fp16 kernel (fp32 data converted into an smem-
// resident operand, TMEM -> smem -> TMA-store epilogue).  Measured slower than the sample-major
// kernels that replaced it (profiles/r02/tuning.md: 0.733 vs 0.689 ms sustained on radio fp16).
// To try it: copy into csrc/ and wire its launch in plan.cu as before (git history).
// gemm_f16_fused.cu -- 16-bit-mode beamformer GEMM that consumes the fp32 data directly
// (the data pack of PAPER.md:107 fused into the GEMM; the direction of the paper's future work
// "a matrix-matrix multiplication kernel that does not require this transpose").
//
// Same arithmetic as gemm_f16_sm100.cu (fp16 RNE inputs, four real sub-GEMMs per K step with
// the negate-A descriptor bit, fp32 accumulation in TMEM -- PAPER.md:143-159), for short K
// (round_up(K, 64) <= 256, e.g. the LOFAR-shaped radio workload):
//
//   * work unit = (batch entry, 128-column data block); the unit's data X[b][0:K][n0:n0+128]
//     is converted ONCE by 8 converter warps (coalesced 128-bit fp32 loads -> cvt.rn.f16 ->
//     swizzled MN-major fp16 planes) into a shared-memory-resident B operand;
//   * every 128-row weight tile of the unit then streams only the packed weights (TMA,
//     2-stage ring) against the resident B; the MMA and epilogue are as in the 1-CTA kernel;
//   * B is split into 64-row K blocks with their own full/empty mbarriers, so the conversion of
//     the next unit's K block starts as soon as the last MMA of the current unit has read it.
//
// Bit-identical to tcbf_pack(DATA) + tcbf_beamform (same rounding, same MMA order).
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 64;
constexpr int KMAX = 256;                 // resident K rows (K16 <= 256)
constexpr int EPI_WARPS = 4;
constexpr int CONV_WARPS = 8;
constexpr int NUM_THREADS = (2 + EPI_WARPS + CONV_WARPS) * 32;
constexpr int A_BYTES = BM * BK * 2;      // one plane of one A stage
constexpr int A_STAGE_BYTES = 2 * A_BYTES;
constexpr int B_PLANE_BYTES = 2 * KMAX * 128;  // 2 column blocks x KMAX rows x 128 B
constexpr int OFF_B = 0;
constexpr int OFF_A = 2 * B_PLANE_BYTES;
// Epilogue: TMA stores staged through 32 KB of swizzled smem boxes, beside 2 weight stages.  (A
// DIRECT variant -- 256-bit st.global from registers, a third weight stage in the freed smem -- was
// bit-identical and measured 15% slower; dropped.)
constexpr int A_STAGES = 2;
constexpr int EPI_BYTES = EPI_WARPS * 2 * 4096;
constexpr int OFF_EPI = OFF_A + A_STAGES * A_STAGE_BYTES;
constexpr int BAR_OFFSET = OFF_EPI + EPI_BYTES;
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
// resident MN-major B: column block j at j * KMAX * 128 B (LBO), 8 k-rows per 1024 B (SBO)
__device__ __forceinline__ uint64_t desc_b_res(const void* plane, uint32_t k_row) {
  uint32_t addr = smem_u32(plane) + k_row * 128u;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((KMAX * 128u) >> 4) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}


__device__ __forceinline__ uint32_t h2u(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}


// MC: CTA pairs (clusters of 2) take adjacent units of the same batch entry, so their weight
// tiles are identical: each CTA TMA-loads one of the two weight planes and multicasts it to both
// (half the L2 -> SM weight traffic); both MMA issuers release a stage in both CTAs.
template <int LAYOUT, bool VEC, bool MC>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmC,
                           GemmF16Args args, const float* __restrict__ xsrc, int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem + OFF_B;  // [2 planes][2 column blocks][KMAX rows][128 B]
  uint8_t* sA = smem + OFF_A;
  uint8_t* epi_base = smem + OFF_EPI;
  uint64_t* afull = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* aempty = afull + A_STAGES;
  uint64_t* bfull = aempty + A_STAGES;    // [KMAX / BK]
  uint64_t* bempty = bfull + KMAX / BK;   // [KMAX / BK]
  uint64_t* tfull = bempty + KMAX / BK;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = args.num_kb;  // K16 / 64 <= 4
  const int tiles_m = args.tiles_m, tiles_n = args.tiles_n;
  const int num_units = args.B * tiles_n;
  // unit walk: single CTAs stride over all units; pairs take units (2p + rank) (tiles_n even)
  const int rank = MC ? (int)cluster_ctarank() : 0;
  const int u_first = MC ? 2 * (int)(blockIdx.x >> 1) + rank : (int)blockIdx.x;
  const int u_step = MC ? 2 * (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < A_STAGES; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], MC ? 2 : 1);
    }
    for (int s = 0; s < KMAX / BK; ++s) {
      mbar_init(&bfull[s], CONV_WARPS);
      mbar_init(&bempty[s], 1);
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
  if (MC) cluster_sync(); else __syncthreads();  // peers signal this CTA's barriers
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer: weight tiles
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = u_first; u < num_units; u += u_step) {
        const int b = u / tiles_n;
        for (int mt = 0; mt < tiles_m; ++mt) {
          for (int kb = 0; kb < num_kb; ++kb) {
            mbar_wait(&aempty[stage], phase ^ 1);
            uint8_t* st = sA + stage * A_STAGE_BYTES;
            if ((TCBF_ABLATE(args, 4)) && mt > 0) {  // ablation: weight tiles loaded once per unit (wrong values)
              mbar_arrive(&afull[stage]);
            } else {
              mbar_arrive_expect_tx(&afull[stage], A_STAGE_BYTES);
              if (MC) {
                tma_load_3d_mc(st + rank * A_BYTES, &tmA, &afull[stage], kb * BK, mt * BM, 2 * b + rank);
              } else {
                tma_load_3d(st, &tmA, &afull[stage], kb * BK, mt * BM, 2 * b);
                tma_load_3d(st + A_BYTES, &tmA, &afull[stage], kb * BK, mt * BM, 2 * b + 1);
              }
            }
            if (++stage == A_STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = (1u << 4) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      constexpr uint32_t IDESC_NEG = IDESC | (1u << 13);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0, ui = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++ui) {
        const uint32_t bphase = ui & 1;
        for (int mt = 0; mt < tiles_m; ++mt, ++it) {
          const int abuf = it & 1;
          mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
          tc_fence_after();
          stamp(args.trace, 4 * it);
          const uint32_t d_re = tmem_base + abuf * 2 * BN;
          const uint32_t d_im = d_re + BN;
          for (int kb = 0; kb < num_kb; ++kb) {
            if (mt == 0 && kb == 0) stamp(args.trace, 512 + 4 * ui);
            if (mt == 0) mbar_wait(&bfull[kb], bphase);  // resident B block converted
            if (mt == 0 && kb == 0) stamp(args.trace, 512 + 4 * ui + 1);
            mbar_wait(&afull[stage], phase);
            tc_fence_after();
            uint8_t* st = sA + stage * A_STAGE_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t krow = kb * BK + kk * 16;
              const uint64_t ar = desc_a128(st, kk * 32), ai = desc_a128(st + A_BYTES, kk * 32);
              const uint64_t br = desc_b_res(sB, krow), bi = desc_b_res(sB + B_PLANE_BYTES, krow);
              const uint32_t acc = (kb | kk) ? 1u : 0u;
              if (TCBF_ABLATE(args, 2)) continue;
              mma_f16_ss(d_re, ar, br, IDESC, acc);
              mma_f16_ss(d_re, ai, bi, IDESC_NEG, 1u);
              mma_f16_ss(d_im, ar, bi, IDESC, acc);
              mma_f16_ss(d_im, ai, br, IDESC, 1u);
            }
            if (MC) mma_commit_mc(&aempty[stage]);  // the stage is free in both CTAs
            else mma_commit(&aempty[stage]);
            if (mt == tiles_m - 1) mma_commit(&bempty[kb]);  // last reader of this B block
            if (++stage == A_STAGES) { stage = 0; phase ^= 1; }
          }
          mma_commit(&tfull[abuf]);
          stamp(args.trace, 4 * it + 1);
        }
      }
    }
  } else if (warp < 2 + EPI_WARPS) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    constexpr int CHUNKS = BN / 32;
    int sbuf = 0;
    int it = 0;
    for (int u = u_first; u < num_units; u += u_step) {
      const int b = u / tiles_n;
      const int n0 = (u - b * tiles_n) * BN;
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int m0 = mt * BM;
        const int abuf = it & 1;
        mbar_wait(&tfull[abuf], (it >> 1) & 1);
        tc_fence_after();
        if (threadIdx.x == 64) stamp(args.trace, 4 * it + 2);
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
          if (TCBF_ABLATE(args, 1)) continue;
          // cooperative staging: the 4 epilogue warps fill one 128-row x 32-column box (16 KB),
          // one thread issues a single TMA store per chunk
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
        if (threadIdx.x == 64) stamp(args.trace, 4 * it + 3);
      }
    }
    if (threadIdx.x == 64) bulk_wait_group<0>();
  } else {
    // ------------------------------------------------------------ converters: fp32 data -> resident B
    const int ct = threadIdx.x - (2 + EPI_WARPS) * 32;  // 0..255
    constexpr int NT = CONV_WARPS * 32;
    constexpr int ITEMS = BK * (BN / 8) / NT;           // 16-byte output chunks per thread per K block
    const int N = args.N;
    int ui = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++ui) {
      const int b = u / tiles_n;
      const int n0 = (u - b * tiles_n) * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        float re[ITEMS][8], im[ITEMS][8];
        // loads first (all in flight), then wait for the block to be free, then convert + store
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
        if (ct == 0 && kb == 0) stamp(args.trace, 512 + 4 * ui + 2);
        mbar_wait(&bempty[kb], (ui & 1) ^ 1);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int item = ct + i * NT;
          const int kr = item / (BN / 8), cc = item % (BN / 8);
          const int k = kb * BK + kr;
          const int off = (cc >> 3) * (KMAX * 128) + k * 128 + (((cc & 7) ^ (k & 7)) << 4);
          *reinterpret_cast<uint4*>(sB + off) = make_uint4(h2u(re[i][0], re[i][1]), h2u(re[i][2], re[i][3]),
                                                           h2u(re[i][4], re[i][5]), h2u(re[i][6], re[i][7]));
          *reinterpret_cast<uint4*>(sB + B_PLANE_BYTES + off) = make_uint4(
              h2u(im[i][0], im[i][1]), h2u(im[i][2], im[i][3]), h2u(im[i][4], im[i][5]), h2u(im[i][6], im[i][7]));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bfull[kb]);
        if (ct == 0 && kb == 0) stamp(args.trace, 512 + 4 * ui + 3);
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

template <int LAYOUT, bool VEC, bool MC>
cudaError_t launch_fused(const CUtensorMap& tmA, const CUtensorMap& tmC, const GemmF16Args& a, const float* x,
                         int K, int num_sms, cudaStream_t s) {
  auto kern = cgemm_f16_fused_kernel<LAYOUT, VEC, MC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int units = a.B * a.tiles_n;
  if (!MC) {
    const int grid = units < num_sms ? units : num_sms;
    kern<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(tmA, tmC, a, x, K);
    return cudaGetLastError();
  }
  const int pairs = units / 2 < num_sms / 2 ? units / 2 : num_sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, tmA, tmC, a, x, K);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int LAYOUT, bool VEC>
cudaError_t launch_fused_sel(const CUtensorMap& tmA, const CUtensorMap& tmC, const GemmF16Args& a, const float* x,
                             int K, bool multicast, int num_sms, cudaStream_t s) {
  // weight multicast across CTA pairs needs pairs of units of one batch entry (tiles_n even)
  const bool mc = multicast && a.tiles_n % 2 == 0 && a.B * a.tiles_n >= 2;
  return mc ? launch_fused<LAYOUT, VEC, true>(tmA, tmC, a, x, K, num_sms, s)
            : launch_fused<LAYOUT, VEC, false>(tmA, tmC, a, x, K, num_sms, s);
}

}  // namespace

bool gemm_f16_fused_supported(int64_t K16, int64_t N) { return K16 <= KMAX && N % 4 == 0; }

cudaError_t launch_gemm_f16_fused(const CUtensorMap& tmA, const CUtensorMap& tmC, const GemmF16Args& args,
                                  const float* x_src, int layout, int K, bool multicast, int num_sms,
                                  cudaStream_t stream) {
  const bool vec = layout == 0 && (args.N % 8 == 0) && (reinterpret_cast<uintptr_t>(x_src) % 16 == 0);
  if (layout == 0)
    return vec ? launch_fused_sel<0, true>(tmA, tmC, args, x_src, K, multicast, num_sms, stream)
               : launch_fused_sel<0, false>(tmA, tmC, args, x_src, K, multicast, num_sms, stream);
  return launch_fused_sel<1, false>(tmA, tmC, args, x_src, K, multicast, num_sms, stream);
}

}  // namespace tcbf
