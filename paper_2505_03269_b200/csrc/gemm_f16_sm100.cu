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
//   * warp 0: TMA producer filling a STAGES-deep smem ring (A_r, A_i, B_r, B_i tiles,
//     128-byte swizzle), mbarrier full/empty pipeline (replaces the paper's cp.async
//     multi-buffer);
//   * warp 1: one thread issues tcgen05.mma (M=128, N=BN, K=16) into TMEM; TMEM holds two
//     accumulator sets (D_r, D_i) so the epilogue of tile i overlaps the mainloop of i+1;
//   * warps 2-5: epilogue, tcgen05.ld -> registers -> swizzled smem -> TMA bulk store of
//     the fp32 planar output (the dominant HBM traffic for the radio shapes).
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // fp16 elements per 128-byte swizzle row
constexpr int NUM_THREADS = 192;

template <int BN, int STAGES, bool TMA_STORE>
struct F16Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int EPI_BYTES = TMA_STORE ? 4 * 2 * 4096 : 0;
  static constexpr int TMEM_COLS = 4 * BN;  // 2 buffers x (D_r, D_i)
  static constexpr int BAR_OFFSET = STAGES * STAGE_BYTES + EPI_BYTES;
  static constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
  static_assert(TMEM_COLS == 256 || TMEM_COLS == 512, "TMEM allocation must be a power of two");
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};

template <int BN, int STAGES, bool TMA_STORE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, GemmF16Args args) {
  using Cfg = F16Cfg<BN, STAGES, TMA_STORE>;
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
      mbar_init(&tempty_bar[s], 4);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (TMA_STORE) tma_prefetch_desc(&tmC);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int tiles_per_batch = args.tiles_m * args.tiles_n;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x) {
        const int b = t / tiles_per_batch;
        const int r = t - b * tiles_per_batch;
        const int m0 = (r / args.tiles_n) * BM;
        const int n0 = (r % args.tiles_n) * BN;
        for (int kb = 0; kb < args.num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
          tma_load_3d(st, &tmA, &full_bar[stage], kb * BK, m0, 2 * b);
          tma_load_3d(st + Cfg::A_BYTES, &tmA, &full_bar[stage], kb * BK, m0, 2 * b + 1);
          tma_load_3d(st + 2 * Cfg::A_BYTES, &tmB, &full_bar[stage], kb * BK, n0, 2 * b);
          tma_load_3d(st + 2 * Cfg::A_BYTES + Cfg::B_BYTES, &tmB, &full_bar[stage], kb * BK, n0, 2 * b + 1);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC = idesc_f16(BM, BN, false);
      constexpr uint32_t IDESC_NEG = idesc_f16(BM, BN, true);
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
          uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sAr = st;
          uint8_t* sAi = st + Cfg::A_BYTES;
          uint8_t* sBr = st + 2 * Cfg::A_BYTES;
          uint8_t* sBi = sBr + Cfg::B_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint32_t off = kk * 32;
            const uint64_t ar = smem_desc_k128(sAr, off), ai = smem_desc_k128(sAi, off);
            const uint64_t br = smem_desc_k128(sBr, off), bi = smem_desc_k128(sBi, off);
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            mma_f16_ss(d_re, ar, br, IDESC, acc);     // Re += Re(a) Re(b)
            mma_f16_ss(d_re, ai, bi, IDESC_NEG, 1u);  // Re += -Im(a) Im(b)
            mma_f16_ss(d_im, ar, bi, IDESC, acc);     // Im += Re(a) Im(b)
            mma_f16_ss(d_im, ai, br, IDESC, 1u);      // Im += Im(a) Re(b)
          }
          mma_commit(&empty_bar[stage]);  // frees the smem slot when these MMAs retire
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull_bar[abuf]);  // accumulator ready for the epilogue
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;        // TMEM lane quadrant this warp may access
    const int ew = warp - 2;       // private staging buffers
    uint8_t* stg = epi_base + ew * 8192;
    int sbuf = 0;
    int it = 0;
    for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x, ++it) {
      const int b = t / tiles_per_batch;
      const int r = t - b * tiles_per_batch;
      const int m0 = (r / args.tiles_n) * BM;
      const int n0 = (r % args.tiles_n) * BN;
      const int abuf = it & 1;
      mbar_wait(&tfull_bar[abuf], (it >> 1) & 1);
      tc_fence_after();
      constexpr int CHUNKS = BN / 32;
#pragma unroll 1
      for (int ch = 0; ch < 2 * CHUNKS; ++ch) {
        const int part = ch / CHUNKS;  // 0 = Re, 1 = Im
        const int c = ch % CHUNKS;
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 2 * BN + part * BN + c * 32, v);
        tmem_wait_ld();
        if (ch == 2 * CHUNKS - 1) {  // all TMEM reads of this tile done: release the buffer
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[abuf]);
        }
        if constexpr (TMA_STORE) {
          if (lane == 0) bulk_wait_group_read<1>();
          __syncwarp();
          uint8_t* buf = stg + sbuf * 4096;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int pos = j ^ (lane & 7);  // 128-byte swizzle, matches the tensor map
            *reinterpret_cast<uint4*>(buf + lane * 128 + pos * 16) =
                make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmC, buf, n0 + c * 32, m0 + q * 32, 2 * b + part);
            bulk_commit_group();
          }
          sbuf ^= 1;
        } else {
          const int m = m0 + q * 32 + lane;
          if (m < args.M) {
            float* row = args.out + ((size_t)(2 * b + part) * args.M + m) * (size_t)args.N;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = n0 + c * 32 + j;
              if (n < args.N) row[n] = __uint_as_float(v[j]);
            }
          }
        }
      }
    }
    if constexpr (TMA_STORE) {
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

template <int BN, int STAGES, bool TMA_STORE>
cudaError_t launch_impl(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                        const GemmF16Args& args, int num_sms, cudaStream_t stream) {
  using Cfg = F16Cfg<BN, STAGES, TMA_STORE>;
  auto kern = cgemm_f16_kernel<BN, STAGES, TMA_STORE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  int grid = args.num_tiles < num_sms ? args.num_tiles : num_sms;
  kern<<<grid, NUM_THREADS, Cfg::SMEM_BYTES, stream>>>(tmA, tmB, tmC, args);
  return cudaGetLastError();
}

}  // namespace

int gemm_f16_block_n(int variant) { return variant == 64 ? 64 : 128; }

cudaError_t launch_gemm_f16(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                            const GemmF16Args& args, int block_n, bool tma_store, int num_sms,
                            cudaStream_t stream) {
  if (block_n == 64) {
    return tma_store ? launch_impl<64, 4, true>(tmA, tmB, tmC, args, num_sms, stream)
                     : launch_impl<64, 4, false>(tmA, tmB, tmC, args, num_sms, stream);
  }
  return tma_store ? launch_impl<128, 3, true>(tmA, tmB, tmC, args, num_sms, stream)
                   : launch_impl<128, 3, false>(tmA, tmB, tmC, args, num_sms, stream);
}

}  // namespace tcbf
