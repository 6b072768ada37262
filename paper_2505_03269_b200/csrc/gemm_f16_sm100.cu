// gemm_f16_sm100.cu -- 16-bit-mode complex beamformer GEMM on the sm_100a tensor cores.
//
// C[b] = W[b] . X[b] over complex numbers (Eq. 3), fp16 inputs, fp32
// accumulation and output (Table I "float16 / float32").  The complex
// product is formed as four real sub-GEMMs inside one kernel (Sec. III-B):
//     D_r += A_r B_r ;  D_r += (-A_i) B_i ;  D_i += A_r B_i ;  D_i += A_i B_r
// where the paper's "negate Im(b) in registers" becomes the negate-A bit of the tcgen05
// instruction descriptor (exact; reading R7).
//
// B200 design (not the paper's WMMA design, PAPER.md:416 lists this as future work):
//   * persistent CTAs (grid = #SMs), static batch-major tile schedule (PAPER.md:101 batch);
//   * warp 0: TMA producer filling a STAGES-deep smem ring (A_r, A_i K-major boxes and B_r, B_i
//     MN-major boxes, 128-byte swizzle), mbarrier full/empty pipeline (replaces the paper's
//     cp.async multi-buffer);
//   * warp 1: one thread issues tcgen05.mma (M=128, N=BN, K=16) into TMEM; TMEM holds two
//     accumulator sets (D_r, D_i) so the epilogue of tile i overlaps the mainloop of i+1;
//   * warps 2..2+EPI_WARPS-1: epilogue, tcgen05.ld -> registers -> swizzled smem -> TMA bulk
//     store of the fp32 planar output (the dominant HBM traffic for the radio shapes).  With 8
//     epilogue warps two warps share each TMEM lane quadrant and split the columns.
// The data operand is consumed MN-major ([K][N], N contiguous), so tcbf_pack(DATA) is a pure
// streaming conversion without the transpose of the paper's design.
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BM = 128;

template <int BN, int BK, int STAGES, int EPI_WARPS, int EPI>
struct F16Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int EPI_BUFS = 2;
  // EPI: 0 = swizzled smem staging + TMA bulk store (N % 4 == 0), 2 = masked scalar stores (any N).
  // (Measured and dropped: direct 256-bit st.global from registers, smem-staged coalesced
  // st.global, cooperative 128-row TMA boxes -- all slower than EPI 0.)
  static_assert(EPI == 0 || EPI == 2, "epilogue kind");
  static constexpr int EPI_BYTES = EPI == 0 ? EPI_WARPS * EPI_BUFS * 4096 : 0;
  static constexpr int TMEM_COLS = 4 * BN;  // 2 buffers x (D_r, D_i)
  static constexpr int BAR_OFFSET = STAGES * STAGE_BYTES + EPI_BYTES;
  static constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
  static constexpr int NUM_THREADS = (2 + EPI_WARPS) * 32;
  static_assert(TMEM_COLS == 256 || TMEM_COLS == 512, "TMEM allocation must be a power of two");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(BK == 32 || BK == 64, "BK");
  static_assert(BN % 64 == 0, "MN-major B operand is loaded in 64-column blocks");
};

// K-major A operand, swizzle width = BK*2 bytes (64 B -> SWIZZLE_64B, 128 B -> SWIZZLE_128B).
template <int BK>
__device__ __forceinline__ uint64_t desc_a(const void* tile, uint32_t k_byte_off) {
  uint32_t addr = smem_u32(tile) + k_byte_off;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;                               // LBO (unused, swizzled K-major)
  d |= (uint64_t)((8u * BK * 2) >> 4) << 32;             // SBO: 8 rows of BK*2 bytes
  d |= (uint64_t)1u << 46;                               // version
  d |= (uint64_t)(BK == 64 ? 2u : 4u) << 61;             // SWIZZLE_128B / SWIZZLE_64B
  return d;
}
// MN-major B operand: 64-element (128 B) MN blocks of BK k-rows each, 128-byte swizzle.
// LBO = distance between MN blocks (BK rows x 128 B), SBO = 8 k-rows (1024 B).
template <int BK>
__device__ __forceinline__ uint64_t desc_b_mn(const void* tile, uint32_t k_row) {
  uint32_t addr = smem_u32(tile) + k_row * 128u;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((BK * 128u) >> 4) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_f16_mn(uint32_t M, uint32_t N, bool negate_a) {
  return (1u << 4) | ((negate_a ? 1u : 0u) << 13) | (0u << 15) /* A K-major */ | (1u << 16) /* B MN-major */ |
         ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <int BN, int BK, int STAGES, int EPI_WARPS, int EPI>
__global__ void __launch_bounds__(F16Cfg<BN, BK, STAGES, EPI_WARPS, EPI>::NUM_THREADS, 1)
    cgemm_f16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, GemmF16Args args) {
  using Cfg = F16Cfg<BN, BK, STAGES, EPI_WARPS, EPI>;
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

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (EPI == 0) tma_prefetch_desc(&tmC);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
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
        const int m0 = mt * BM;
        const int n0 = nt * BN;
        for (int kb = 0; kb < args.num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
          tma_load_3d(st, &tmA, &full_bar[stage], kb * BK, m0, 2 * b);
          tma_load_3d(st + Cfg::A_BYTES, &tmA, &full_bar[stage], kb * BK, m0, 2 * b + 1);
          uint8_t* sb = st + 2 * Cfg::A_BYTES;
#pragma unroll
          for (int j = 0; j < BN / 64; ++j) {
            tma_load_3d(sb + j * BK * 128, &tmB, &full_bar[stage], n0 + 64 * j, kb * BK, 2 * b);
            tma_load_3d(sb + Cfg::B_BYTES + j * BK * 128, &tmB, &full_bar[stage], n0 + 64 * j, kb * BK, 2 * b + 1);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (converged warp, one
    // elected lane issues: descriptors stay in uniform registers)
    {
      constexpr uint32_t IDESC = idesc_f16_mn(BM, BN, false);
      constexpr uint32_t IDESC_NEG = idesc_f16_mn(BM, BN, true);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x, ++it) {
        const int abuf = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(&tempty_bar[abuf], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_re = tmem_base + abuf * 2 * BN;
        const uint32_t d_im = d_re + BN;
        for (int kb = 0; kb < args.num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
          // K advance per MMA: 32 bytes of the K-major A (+2), 16 k-rows of the MN-major B (+128)
          const uint64_t ar0 = desc_a<BK>(st, 0), ai0 = desc_a<BK>(st + Cfg::A_BYTES, 0);
          const uint64_t br0 = desc_b_mn<BK>(st + 2 * Cfg::A_BYTES, 0);
          const uint64_t bi0 = desc_b_mn<BK>(st + 2 * Cfg::A_BYTES + Cfg::B_BYTES, 0);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t ar = ar0 + (uint64_t)(2 * kk), ai = ai0 + (uint64_t)(2 * kk);
              const uint64_t br = br0 + (uint64_t)(128 * kk), bi = bi0 + (uint64_t)(128 * kk);
              const uint32_t acc = (kb | kk) ? 1u : 0u;
              if (TCBF_ABLATE(args, 2)) continue;
              mma_f16_ss(d_re, ar, br, IDESC, acc);     // Re += Re(a) Re(b)
              mma_f16_ss(d_re, ai, bi, IDESC_NEG, 1u);  // Re += -Im(a) Im(b)
              mma_f16_ss(d_im, ar, bi, IDESC, acc);     // Im += Re(a) Im(b)
              mma_f16_ss(d_im, ai, br, IDESC, 1u);      // Im += Im(a) Re(b)
            }
            mma_commit(&empty_bar[stage]);  // frees the smem slot when these MMAs retire
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit(&tfull_bar[abuf]);  // accumulator ready for the epilogue
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;               // TMEM lane quadrant this warp may access
    const int ew = warp - 2;              // private staging buffers
    const int half = ew / 4;              // which columns of the quadrant (8 warps: 2 halves)
    constexpr int SPLIT = EPI_WARPS / 4;  // 1 or 2 warps per quadrant
    constexpr int CHUNKS = BN / 32;
    constexpr int MY_CHUNKS = 2 * CHUNKS / SPLIT;
    uint8_t* stg = epi_base + ew * (Cfg::EPI_BUFS * 4096);
    int sbuf = 0;
    int it = 0;
    for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x, ++it) {
      int b, mt, nt;
      tile_coords(t, args.tiles_m, args.tiles_n, args.group_m, b, mt, nt);
      const int m0 = mt * BM;
      const int n0 = nt * BN;
      const int abuf = it & 1;
      mbar_wait(&tfull_bar[abuf], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 2 * BN;
      uint32_t v[2][32];
      // chunk i of this warp: global chunk ch = i * SPLIT + half (interleaved column split)
      tmem_ld_32x32b_x32(tbase + (0 * SPLIT + half) * 32, v[0]);
#pragma unroll
      for (int i = 0; i < MY_CHUNKS; ++i) {
        const int ch = i * SPLIT + half;
        const int part = ch / CHUNKS;  // 0 = Re, 1 = Im
        const int c = ch % CHUNKS;
        tmem_wait_ld();
        if (i + 1 < MY_CHUNKS) {
          tmem_ld_32x32b_x32(tbase + ((i + 1) * SPLIT + half) * 32, v[(i + 1) & 1]);
        } else {  // all TMEM reads of this tile issued and complete: release the buffer
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[abuf]);
        }
        const uint32_t* vv = v[i & 1];
        if (TCBF_ABLATE(args, 1)) continue;
        if constexpr (EPI == 0) {
          if (lane == 0) bulk_wait_group_read<Cfg::EPI_BUFS - 1>();
          __syncwarp();
          uint8_t* buf = stg + sbuf * 4096;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int pos = j ^ (lane & 7);  // 128-byte swizzle, matches the tensor map
            *reinterpret_cast<uint4*>(buf + lane * 128 + pos * 16) =
                make_uint4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmC, buf, n0 + c * 32, m0 + q * 32, 2 * b + part);
            bulk_commit_group();
          }
          sbuf = (sbuf + 1 == Cfg::EPI_BUFS) ? 0 : sbuf + 1;
        } else {
          const int m = m0 + q * 32 + lane;
          if (m < args.M) {
            float* row = args.out + ((size_t)(2 * b + part) * args.M + m) * (size_t)args.N;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = n0 + c * 32 + j;
              if (n < args.N) row[n] = __uint_as_float(vv[j]);
            }
          }
        }
      }
    }
    if constexpr (EPI == 0) {
      if (lane == 0) bulk_wait_group<0>();
      __syncwarp();
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

template <int BN, int BK, int STAGES, int EPI_WARPS, int EPI>
cudaError_t launch_impl(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                        const GemmF16Args& args, int num_sms, cudaStream_t stream) {
  using Cfg = F16Cfg<BN, BK, STAGES, EPI_WARPS, EPI>;
  auto kern = cgemm_f16_kernel<BN, BK, STAGES, EPI_WARPS, EPI>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  int grid = args.num_tiles < num_sms ? args.num_tiles : num_sms;
  kern<<<grid, Cfg::NUM_THREADS, Cfg::SMEM_BYTES, stream>>>(tmA, tmB, tmC, args);
  return cudaGetLastError();
}

cudaError_t dispatch(int variant, int epi, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                     const GemmF16Args& g, int sms, cudaStream_t s) {
  if (epi == 2) {  // N % 8 != 0: masked stores
    return variant == F16_V_N64 ? launch_impl<64, 64, 4, 4, 2>(a, b, c, g, sms, s)
                                : launch_impl<128, 64, 3, 4, 2>(a, b, c, g, sms, s);
  }
  switch (variant) {
    case F16_V_N64:       return launch_impl<64, 64, 4, 4, 0>(a, b, c, g, sms, s);
    case F16_V_K32_S4_E8: return launch_impl<128, 32, 4, 8, 0>(a, b, c, g, sms, s);
    default:              return launch_impl<128, 64, 3, 4, 0>(a, b, c, g, sms, s);
  }
}

}  // namespace

int gemm_f16_block_n(int variant) {
  return variant == F16_V_N64 ? 64 : (variant == F16_V_2CTA_N256 ? 256 : 128);
}

cudaError_t launch_gemm_f16(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                            const GemmF16Args& args, int variant, int epi, int num_sms,
                            cudaStream_t stream) {
  return dispatch(variant, epi, tmA, tmB, tmC, args, num_sms, stream);
}

int gemm_f16_block_k(int variant) {
  return variant == F16_V_K32_S4_E8 ? 32 : 64;
}

}  // namespace tcbf
