// gemm_f16_fused2.cu -- fp32-input 16-bit-mode beamformer GEMM on CTA pairs (tcgen05 cta_group::2)
// for short K (round_up(K, 64) <= 256: the LOFAR-shaped radio workload).
//
// Same arithmetic as gemm_f16_fused.cu / tcbf_pack + tcbf_beamform (fp16 RNE inputs, four real
// sub-GEMMs per K step with the negate-A bit, fp32 accumulation), bit-identical.
// Measured on the single-CTA fused kernel (dev timeline, tools/trace_fused.py): the tile loop is
// bound by shared-memory traffic -- the MMA operand reads (8 KB per 128x128x16 step) dominate,
// then the TMA weight writes and the epilogue staging.  A CTA pair issues M=256 MMAs whose data
// operand is split between the two SMs, so each SM reads 6 KB per 128x128x16 instead of 8 KB,
// and each CTA keeps only ITS HALF of the unit's converted data resident -- 64 KB, small enough
// to double-buffer, so converting the next unit overlaps the current unit's MMAs completely.
//
//   unit      = (batch entry, 128 data columns); pair tile = 256 weight rows x 128 columns
//   warp 0    TMA producer: own 128 weight rows per K block, completion on the leader's barrier
//   warp 1    MMA issuer (leader CTA): tcgen05.mma.cta_group::2 M=256 N=128 K=16, commits
//             multicast to both CTAs (weight stage free, accumulators ready, data block free)
//   warps 2-5 epilogue: own 128 rows x 128 columns from TMEM, cooperative 128-row TMA stores
//   warps 6-13 converters: own 64 columns of the unit, fp32 -> fp16 RNE -> swizzled MN-major
//             resident planes (double-buffered by unit), arrivals on the leader's barrier
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BN = 128;                   // unit columns (MMA N); each CTA holds 64
constexpr int BH = BN / 2;
constexpr int BK = 64;
constexpr int KMAX = 256;
constexpr int NKB = KMAX / BK;
constexpr int A_STAGES = 2;
constexpr int EPI_WARPS = 4;
constexpr int CONV_WARPS = 8;
constexpr int NUM_THREADS = (2 + EPI_WARPS + CONV_WARPS) * 32;
constexpr int A_BYTES = 128 * BK * 2;          // one plane of one A stage (own 128 rows)
constexpr int A_STAGE_BYTES = 2 * A_BYTES;
constexpr int B_PLANE_BYTES = KMAX * 128;      // one 64-column block x KMAX rows x 128 B
constexpr int B_BUF_BYTES = 2 * B_PLANE_BYTES; // re, im
constexpr int EPI_BYTES = 2 * 16384;
constexpr int OFF_B = 0;
constexpr int OFF_A = 2 * B_BUF_BYTES;
constexpr int OFF_EPI = OFF_A + A_STAGES * A_STAGE_BYTES;
constexpr int BAR_OFFSET = OFF_EPI + EPI_BYTES;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
static_assert(SMEM_BYTES <= 232448, "smem budget");

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_3d_2sm(void* smem_dst, const CUtensorMap* map, uint32_t leader_bar,
                                                int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void mma_f16_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_2sm_mc(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t desc_a128(const void* tile, uint32_t k_byte_off) {
  uint32_t addr = smem_u32(tile) + k_byte_off;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// resident MN-major data half: one 64-column block, 8 k-rows per 1024 B (SBO)
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

template <int LAYOUT, bool VEC>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_fused2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmC,
                            GemmF16Args args, const float* __restrict__ xsrc, int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem + OFF_B;  // [2 buffers][re, im][KMAX rows][128 B]
  uint8_t* sA = smem + OFF_A;
  uint8_t* epi_base = smem + OFF_EPI;
  uint64_t* afull = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* aempty = afull + A_STAGES;
  uint64_t* bfull = aempty + A_STAGES;  // [2][NKB] (leader's are used)
  uint64_t* bempty = bfull + 2 * NKB;   // [2][NKB]
  uint64_t* tfull = bempty + 2 * NKB;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int num_kb = args.num_kb;  // K16 / 64 <= 4
  const int tiles_m = args.tiles_m;  // 256-row pair tiles
  const int tiles_n = args.tiles_n;
  const int num_units = args.B * tiles_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < A_STAGES; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < 2 * NKB; ++s) {
      mbar_init(&bfull[s], 2 * CONV_WARPS);
      mbar_init(&bempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmC);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < num_units; u += npairs) {
        const int b = u / tiles_n;
        for (int mt = 0; mt < tiles_m; ++mt) {
          const int m0 = mt * 256 + (int)rank * 128;
          for (int kb = 0; kb < num_kb; ++kb) {
            mbar_wait(&aempty[stage], phase ^ 1);
            const uint32_t lbar = mapa_shared(&afull[stage], 0);
            if (leader) mbar_arrive_expect_tx(&afull[stage], 2 * A_STAGE_BYTES);
            uint8_t* st = sA + stage * A_STAGE_BYTES;
            tma_load_3d_2sm(st, &tmA, lbar, kb * BK, m0, 2 * b);
            tma_load_3d_2sm(st + A_BYTES, &tmA, lbar, kb * BK, m0, 2 * b + 1);
            if (++stage == A_STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    if (leader && lane == 0) {
      constexpr uint32_t IDESC = (1u << 4) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) | ((256u >> 4) << 24);
      constexpr uint32_t IDESC_NEG = IDESC | (1u << 13);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0, ui = 0;
      for (int u = pair; u < num_units; u += npairs, ++ui) {
        const int bb = ui & 1;
        const uint32_t bphase = (ui >> 1) & 1;
        uint8_t* sBr = sB + bb * B_BUF_BYTES;
        uint8_t* sBi = sBr + B_PLANE_BYTES;
        for (int mt = 0; mt < tiles_m; ++mt, ++it) {
          const int abuf = it & 1;
          mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_re = tmem_base + abuf * 2 * BN;
          const uint32_t d_im = d_re + BN;
          for (int kb = 0; kb < num_kb; ++kb) {
            if (mt == 0) mbar_wait(&bfull[bb * NKB + kb], bphase);  // both halves converted
            mbar_wait(&afull[stage], phase);
            tc_fence_after();
            uint8_t* st = sA + stage * A_STAGE_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t krow = kb * BK + kk * 16;
              const uint64_t ar = desc_a128(st, kk * 32), ai = desc_a128(st + A_BYTES, kk * 32);
              const uint64_t br = desc_b_res(sBr, krow), bi = desc_b_res(sBi, krow);
              const uint32_t acc = (kb | kk) ? 1u : 0u;
              if (args.debug & 2) continue;
              mma_f16_2sm(d_re, ar, br, IDESC, acc);
              mma_f16_2sm(d_re, ai, bi, IDESC_NEG, 1u);
              mma_f16_2sm(d_im, ar, bi, IDESC, acc);
              mma_f16_2sm(d_im, ai, br, IDESC, 1u);
            }
            mma_commit_2sm_mc(&aempty[stage]);
            if (mt == tiles_m - 1) mma_commit_2sm_mc(&bempty[bb * NKB + kb]);  // last reader
            if (++stage == A_STAGES) { stage = 0; phase ^= 1; }
          }
          mma_commit_2sm_mc(&tfull[abuf]);
        }
      }
    }
  } else if (warp < 2 + EPI_WARPS) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    constexpr int CHUNKS = BN / 32;
    int sbuf = 0;
    int it = 0;
    const uint32_t tempty_leader[2] = {mapa_shared(&tempty[0], 0), mapa_shared(&tempty[1], 0)};
    for (int u = pair; u < num_units; u += npairs) {
      const int b = u / tiles_n;
      const int n0 = (u - b * tiles_n) * BN;
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int m0 = mt * 256 + (int)rank * 128;
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
            if (lane == 0) mbar_arrive_cluster(tempty_leader[abuf]);
          }
          const uint32_t* vv = v[ch & 1];
          if (args.debug & 1) continue;
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
    }
    if (threadIdx.x == 64) bulk_wait_group<0>();
  } else {
    // ------------------------------------------------------------ converters: own 64 columns
    const int ct = threadIdx.x - (2 + EPI_WARPS) * 32;  // 0..255
    constexpr int NT = CONV_WARPS * 32;
    constexpr int ITEMS = BK * (BH / 8) / NT;           // 16-byte output chunks per thread per K block
    static_assert(ITEMS == 2, "converter mapping");
    const int N = args.N;
    uint32_t bfull_leader[2 * NKB];
#pragma unroll
    for (int s = 0; s < 2 * NKB; ++s) bfull_leader[s] = mapa_shared(&bfull[s], 0);
    int ui = 0;
    for (int u = pair; u < num_units; u += npairs, ++ui) {
      const int b = u / tiles_n;
      const int n0 = (u - b * tiles_n) * BN + (int)rank * BH;
      const int bb = ui & 1;
      uint8_t* sBr = sB + bb * B_BUF_BYTES;
      for (int kb = 0; kb < num_kb; ++kb) {
        float re[ITEMS][8], im[ITEMS][8];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int item = ct + i * NT;
          const int kr = item / (BH / 8), cc = item % (BH / 8);
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
        mbar_wait(&bempty[bb * NKB + kb], ((ui >> 1) & 1) ^ 1);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int item = ct + i * NT;
          const int kr = item / (BH / 8), cc = item % (BH / 8);
          const int k = kb * BK + kr;
          const int off = k * 128 + ((cc ^ (k & 7)) << 4);
          *reinterpret_cast<uint4*>(sBr + off) = make_uint4(h2u(re[i][0], re[i][1]), h2u(re[i][2], re[i][3]),
                                                            h2u(re[i][4], re[i][5]), h2u(re[i][6], re[i][7]));
          *reinterpret_cast<uint4*>(sBr + B_PLANE_BYTES + off) = make_uint4(
              h2u(im[i][0], im[i][1]), h2u(im[i][2], im[i][3]), h2u(im[i][4], im[i][5]), h2u(im[i][6], im[i][7]));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(bfull_leader[bb * NKB + kb]);
      }
    }
  }

  tc_fence_before();
  cluster_sync();  // no CTA of the pair may free TMEM / exit while its peer still signals it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512u) : "memory");
  }
}

template <int LAYOUT, bool VEC>
cudaError_t launch_fused2(const CUtensorMap& tmA, const CUtensorMap& tmC, const GemmF16Args& a, const float* x,
                          int K, int num_sms, cudaStream_t s) {
  auto kern = cgemm_f16_fused2_kernel<LAYOUT, VEC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int units = a.B * a.tiles_n;
  const int pairs = units < num_sms / 2 ? units : num_sms / 2;
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

}  // namespace

cudaError_t launch_gemm_f16_fused2(const CUtensorMap& tmA, const CUtensorMap& tmC, const GemmF16Args& args,
                                   const float* x_src, int layout, int K, int num_sms, cudaStream_t stream) {
  const bool vec = layout == 0 && (args.N % 8 == 0) && (reinterpret_cast<uintptr_t>(x_src) % 16 == 0);
  if (layout == 0)
    return vec ? launch_fused2<0, true>(tmA, tmC, args, x_src, K, num_sms, stream)
               : launch_fused2<0, false>(tmA, tmC, args, x_src, K, num_sms, stream);
  return launch_fused2<1, false>(tmA, tmC, args, x_src, K, num_sms, stream);
}

}  // namespace tcbf
