// gemm_f16_2cta.cu -- 16-bit-mode complex beamformer GEMM with CTA pairs (tcgen05 cta_group::2).
//
// Same arithmetic as gemm_f16_sm100.cu (four real sub-GEMMs per K step, the
// Im(a)Im(b) product negated through the instruction descriptor), but each 2-CTA cluster computes
// a 256 x BN complex tile with one M=256 MMA stream:
//   * CTA r of the pair TMA-loads its own 128 weight rows (A_r, A_i) and its half of the BN data
//     columns (B_r, B_i), signalling the leader's full barrier (cp.async.bulk.tensor.cta_group::2);
//   * the leader's single MMA thread issues tcgen05.mma.cta_group::2 (M=256, N=BN, K=16); the
//     tensor cores of the pair exchange the B halves, so each SM loads and serves only half of B
//     per MMA (less TMA, L2 and shared-memory traffic -- and power -- per useful flop);
//   * commits are multicast to both CTAs' barriers; each CTA drains its own TMEM (its 128 rows x
//     BN) in the epilogue and arrives remotely on the leader's TMEM-empty barrier.
// BN = 128 keeps two accumulator sets in TMEM (store-bound radio shapes, epilogue overlapped);
// BN = 256 fills TMEM with one set (compute-bound shapes, epilogue negligible).
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BK = 64;
constexpr int EPI_WARPS = 4;

template <int BN, int STAGES>
struct Cfg2 {
  static constexpr int A_BYTES = 128 * BK * 2;        // per plane, own 128 rows
  static constexpr int BH = BN / 2;                   // data columns held by this CTA
  static constexpr int B_BYTES = BH * BK * 2;         // per plane
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int ACC_BUFS = (4 * BN <= 512) ? 2 : 1;
  static constexpr int TMEM_COLS = 2 * BN * ACC_BUFS;
  static constexpr int EPI_BYTES = EPI_WARPS * 2 * 4096;
  static constexpr int BAR_OFFSET = STAGES * STAGE_BYTES + EPI_BYTES;
  static constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
  static constexpr int NUM_THREADS = (2 + EPI_WARPS) * 32;
  static_assert(TMEM_COLS == 256 || TMEM_COLS == 512, "TMEM allocation");
  static_assert(SMEM_BYTES <= 232448, "smem budget");
  static_assert(BH % 64 == 0, "B half must be whole 64-column blocks");
};

// shared::cluster address of the same variable in CTA `rank` of the cluster
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
__device__ __forceinline__ uint64_t desc_b_mn(const void* tile, uint32_t k_row) {
  uint32_t addr = smem_u32(tile) + k_row * 128u;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((BK * 128u) >> 4) << 16;  // LBO: next 64-column block
  d |= (uint64_t)(1024u >> 4) << 32;        // SBO: next 8 k-rows
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(Cfg2<BN, STAGES>::NUM_THREADS, 1)
    cgemm_f16_2cta_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmC, GemmF16Args args) {
  using Cfg = Cfg2<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_base = smem + STAGES * Cfg::STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFFSET);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2 * EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)Cfg::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  // Barriers initialised and TMEM allocated in both CTAs.  (compute-sanitizer racecheck reports
  // the PEER CTA's cta_group::2 alloc -- which writes the address into both CTAs' tmem_slot --
  // against the read below: a tool limitation, the cluster barrier orders them; profiles/r02.)
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int tiles_n = args.tiles_n;
  // tiles_m counts 256-row pair tiles

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < args.num_tiles; t += npairs) {
        int b, mt, nt;
        tile_coords(t, args.tiles_m, tiles_n, args.group_m, b, mt, nt);
        const int m0 = mt * 256 + (int)rank * 128;
        const int n0 = nt * BN + (int)rank * Cfg::BH;
        for (int kb = 0; kb < args.num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          const uint32_t lbar = mapa_shared(&full_bar[stage], 0);
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::STAGE_BYTES);
          uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
          tma_load_3d_2sm(st, &tmA, lbar, kb * BK, m0, 2 * b);
          tma_load_3d_2sm(st + Cfg::A_BYTES, &tmA, lbar, kb * BK, m0, 2 * b + 1);
          uint8_t* sb = st + 2 * Cfg::A_BYTES;
#pragma unroll
          for (int j = 0; j < Cfg::BH / 64; ++j) {
            tma_load_3d_2sm(sb + j * BK * 128, &tmB, lbar, n0 + 64 * j, kb * BK, 2 * b);
            tma_load_3d_2sm(sb + Cfg::B_BYTES + j * BK * 128, &tmB, lbar, n0 + 64 * j, kb * BK, 2 * b + 1);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA only;
    // converged warp, one elected lane issues: descriptors stay in uniform registers)
    if (leader) {
      constexpr uint32_t IDESC = (1u << 4) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) | ((256u >> 4) << 24);
      constexpr uint32_t IDESC_NEG = IDESC | (1u << 13);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = pair; t < args.num_tiles; t += npairs, ++it) {
        const int abuf = Cfg::ACC_BUFS == 2 ? (it & 1) : 0;
        const uint32_t aphase = Cfg::ACC_BUFS == 2 ? ((it >> 1) & 1) : (it & 1);
        mbar_wait(&tempty_bar[abuf], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_re = tmem_base + abuf * 2 * BN;
        const uint32_t d_im = d_re + BN;
        for (int kb = 0; kb < args.num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
          // K advance per MMA: 16 K = 32 bytes of the K-major A (+2 in the address field), 16
          // k-rows = 2048 bytes of the MN-major B (+128)
          const uint64_t ar0 = desc_a128(st, 0), ai0 = desc_a128(st + Cfg::A_BYTES, 0);
          const uint64_t br0 = desc_b_mn(st + 2 * Cfg::A_BYTES, 0);
          const uint64_t bi0 = desc_b_mn(st + 2 * Cfg::A_BYTES + Cfg::B_BYTES, 0);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t ar = ar0 + (uint64_t)(2 * kk), ai = ai0 + (uint64_t)(2 * kk);
              const uint64_t br = br0 + (uint64_t)(128 * kk), bi = bi0 + (uint64_t)(128 * kk);
              const uint32_t acc = (kb | kk) ? 1u : 0u;
              if (TCBF_ABLATE(args, 2)) continue;
              mma_f16_2sm(d_re, ar, br, IDESC, acc);
              mma_f16_2sm(d_re, ai, bi, IDESC_NEG, 1u);
              mma_f16_2sm(d_im, ar, bi, IDESC, acc);
              mma_f16_2sm(d_im, ai, br, IDESC, 1u);
            }
            mma_commit_2sm_mc(&empty_bar[stage]);  // frees the stage in both CTAs
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit_2sm_mc(&tfull_bar[abuf]);  // accumulators ready in both CTAs
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    const int ew = warp - 2;
    constexpr int CHUNKS = BN / 32;
    uint8_t* stg = epi_base + ew * 8192;
    int sbuf = 0;
    int it = 0;
    const uint32_t tempty_leader[2] = {mapa_shared(&tempty_bar[0], 0), mapa_shared(&tempty_bar[1], 0)};
    for (int t = pair; t < args.num_tiles; t += npairs, ++it) {
      int b, mt, nt;
      tile_coords(t, args.tiles_m, tiles_n, args.group_m, b, mt, nt);
      const int m0 = mt * 256 + (int)rank * 128;
      const int n0 = nt * BN;
      const int abuf = Cfg::ACC_BUFS == 2 ? (it & 1) : 0;
      const uint32_t aphase = Cfg::ACC_BUFS == 2 ? ((it >> 1) & 1) : (it & 1);
      mbar_wait(&tfull_bar[abuf], aphase);
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
        if (TCBF_ABLATE(args, 1)) continue;
        const uint32_t* vv = v[ch & 1];
        if (lane == 0) bulk_wait_group_read<1>();
        __syncwarp();
        uint8_t* buf = stg + sbuf * 4096;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int pos = j ^ (lane & 7);
          *reinterpret_cast<uint4*>(buf + lane * 128 + pos * 16) =
              make_uint4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&tmC, buf, n0 + c * 32, m0 + q * 32, 2 * b + part);
          bulk_commit_group();
        }
        sbuf ^= 1;
      }
    }
    if (lane == 0) bulk_wait_group<0>();
    __syncwarp();
  }

  tc_fence_before();
  cluster_sync();  // no CTA of the pair may free TMEM / exit while its peer still signals it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)Cfg::TMEM_COLS)
                 : "memory");
  }
}

template <int BN, int STAGES>
cudaError_t launch2(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const GemmF16Args& g,
                    int num_sms, cudaStream_t s) {
  using Cfg = Cfg2<BN, STAGES>;
  auto kern = cgemm_f16_2cta_kernel<BN, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  int pairs = g.num_tiles < num_sms / 2 ? g.num_tiles : num_sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(Cfg::NUM_THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, a, b, c, g);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemm_f16_2cta(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                                 const GemmF16Args& args, int block_n, int num_sms, cudaStream_t stream) {
  return block_n == 256 ? launch2<256, 3>(tmA, tmB, tmC, args, num_sms, stream)
                        : launch2<128, 4>(tmA, tmB, tmC, args, num_sms, stream);
}

}  // namespace tcbf
