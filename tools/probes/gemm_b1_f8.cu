// gemm_b1_f8.cu -- 1-bit-mode complex beamformer GEMM on the tensor cores with +-1 fp8 operands.
//
// The 1-bit encoding (bit 1 = +1, bit 0 = -1, one bit per component; Fig. 1
// PAPER.md:209-210) is expanded IN SHARED MEMORY straight to the values +-1 in fp8 e4m3
// (0x38 = +1.0, 0xB8 = -1.0) by bit-plane masking: byte i of plane j holds bit (8i + j) of the
// word -- a fixed permutation of the 32 K-elements of a word, applied identically to both
// operands, so every dot product is unchanged.  tcgen05.mma.kind::f8f6f4 then forms the complex
// product exactly as the paper's five steps, with the Im(a)Im(b) product
// negated through the instruction descriptor (the paper's "Im(b) = -Im(b) in local registers"):
//     D_r += A_r B_r ;  D_r += (-A_i) B_i ;  D_i += A_r B_i ;  D_i += A_i B_r
// Products are +-1 and every partial sum is an integer of magnitude <= 2 K_tot < 2^24, so the
// fp32 accumulation is exact (K_tot <= 2^23; larger K uses the int8 kernel).
// Padding bits are 0 and therefore expand to -1 in both operands: they add
// (-1)(-1) - (-1)(-1) = 0 to Re and 2 per padded position to Im, so
//     Re = D_r,   Im = D_i - 2 K_pad      (K_pad = 32 Kw - K: the paper's Eq. 5 Im correction).
//
// Roles (persistent CTA per SM, 416 threads):
//   warp 0      TMEM allocator + single-thread MMA issuer (4 MMAs per K=32 step)
//   warps 1-4   epilogue: tcgen05.ld, fp32 -> int32, Im - 2 K_pad, TMA store of int32
//   warps 5-8   expanders for A_r, A_i (one weight row per thread)
//   warps 9-12  expanders for B_r, B_i (one data column per thread)
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int KB_WORDS = 4;            // 128 bits per K block -> 128 expanded bytes per row
constexpr int TILE_BYTES = 128 * 128;  // one expanded operand tile (rows x 128 B)
constexpr int STAGES = 3;
constexpr int STAGE_BYTES = 4 * TILE_BYTES;  // A_r, A_i, B_r, B_i
constexpr int EPI_BYTES = 4 * 2 * 4096;      // per epilogue warp: two 32-row x 32-column int32 boxes
constexpr int BAR_OFFSET = STAGES * STAGE_BYTES + EPI_BYTES;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
constexpr int NUM_THREADS = 13 * 32;
constexpr int EXPANDER_WARPS = 8;
constexpr uint32_t TMEM_COLS = 512;  // 2 buffers x (D_r, D_i) x 128 columns
static_assert(SMEM_BYTES <= 232448, "smem budget");

// plane j of word w as four e4m3 bytes: +1.0 (0x38) for a set bit, -1.0 (0xB8) for a clear bit
template <int J>
__device__ __forceinline__ uint32_t plane_pm1(uint32_t w) {
  const uint32_t t = (J <= 7) ? (w << (7 - J)) : w;
  return (t & 0x80808080u) ^ 0xB8B8B8B8u;
}

__device__ __forceinline__ void expand_word(uint8_t* row_base, int row, int q, uint32_t w) {
  const uint4 c0 = make_uint4(plane_pm1<0>(w), plane_pm1<1>(w), plane_pm1<2>(w), plane_pm1<3>(w));
  const uint4 c1 = make_uint4(plane_pm1<4>(w), plane_pm1<5>(w), plane_pm1<6>(w), plane_pm1<7>(w));
  const int sw = row & 7;  // 128-byte swizzle of the K-major UMMA operand
  *reinterpret_cast<uint4*>(row_base + (((2 * q) ^ sw) << 4)) = c0;
  *reinterpret_cast<uint4*>(row_base + (((2 * q + 1) ^ sw) << 4)) = c1;
}

__device__ __forceinline__ void mma_f8_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <bool TMA_STORE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_b1_f8_kernel(const __grid_constant__ CUtensorMap tmC, GemmB1Args p, int tiles_m, int tiles_n,
                       int num_tiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_base = smem + STAGES * STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = p.Kw / KB_WORDS;
  const int two_kpad = 2 * (32 * p.Kw - p.K);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], EXPANDER_WARPS);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);
    }
    fence_barrier_init();
    if (TMA_STORE) tma_prefetch_desc(&tmC);
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // kind::f8f6f4: A, B e4m3 (format 0), D fp32, both K-major, M = 128, N = BN
      constexpr uint32_t IDESC = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)(BM >> 4) << 24);
      constexpr uint32_t IDESC_NEG = IDESC | (1u << 13);  // negate A
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int abuf = it & 1;
        mbar_wait(&tempty_bar[abuf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_re = tmem_base + abuf * 2 * BN;
        const uint32_t d_im = d_re + BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          uint8_t* st = smem + stage * STAGE_BYTES;
          uint8_t* sAr = st;
          uint8_t* sAi = st + TILE_BYTES;
          uint8_t* sBr = st + 2 * TILE_BYTES;
          uint8_t* sBi = st + 3 * TILE_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // K = 32 elements (bytes) per MMA
            const uint32_t off = kk * 32;
            const uint64_t ar = smem_desc_k128(sAr, off), ai = smem_desc_k128(sAi, off);
            const uint64_t br = smem_desc_k128(sBr, off), bi = smem_desc_k128(sBi, off);
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            if (p.debug & 2) continue;
            mma_f8_ss(d_re, ar, br, IDESC, acc);      // Re += Re(a) Re(b)
            mma_f8_ss(d_re, ai, bi, IDESC_NEG, 1u);   // Re += -Im(a) Im(b)
            mma_f8_ss(d_im, ar, bi, IDESC, acc);      // Im += Re(a) Im(b)
            mma_f8_ss(d_im, ai, br, IDESC, 1u);       // Im += Im(a) Re(b)
          }
          mma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull_bar[abuf]);
      }
    }
  } else if (warp <= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    constexpr int CHUNKS = BN / 32;
    int sbuf = 0;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      int b, mt, nt;
      tile_coords(t, tiles_m, tiles_n, p.group_m, b, mt, nt);
      const int m0 = mt * BM;
      const int n0 = nt * BN;
      const int abuf = it & 1;
      mbar_wait(&tfull_bar[abuf], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 2 * BN;
      uint32_t vbuf[2][32];
      tmem_ld_32x32b_x32(tbase, vbuf[0]);
#pragma unroll
      for (int ch = 0; ch < 2 * CHUNKS; ++ch) {
        const int part = ch / CHUNKS;
        const int c = ch % CHUNKS;
        tmem_wait_ld();
        if (ch + 1 < 2 * CHUNKS) {
          tmem_ld_32x32b_x32(tbase + (ch + 1) * 32, vbuf[(ch + 1) & 1]);
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[abuf]);
        }
        uint32_t* v = vbuf[ch & 1];
        const int corr = part == 0 ? 0 : two_kpad;
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (uint32_t)(__float2int_rn(__uint_as_float(v[j])) - corr);
        if (p.debug & 1) continue;
        if constexpr (TMA_STORE) {  // per-warp 32-row boxes, 2 staging buffers per warp
          uint8_t* buf = epi_base + ((warp - 1) * 2 + sbuf) * 4096;
          if (lane == 0) bulk_wait_group_read<1>();
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int pos = j ^ (lane & 7);
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
          if (m < p.M) {
            int32_t* rowp = p.out + ((size_t)(2 * b + part) * p.M + m) * (size_t)p.N;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = n0 + c * 32 + j;
              if (n < p.N) rowp[n] = (int32_t)v[j];
            }
          }
        }
      }
    }
    if constexpr (TMA_STORE) {
      if (lane == 0) bulk_wait_group<0>();
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ expanders
    const int e = threadIdx.x - 5 * 32;  // 0..255
    const bool a_side = e < 128;
    const int row = a_side ? e : e - 128;
    int stage = 0;
    uint32_t phase = 0;
    const uint4 zero = make_uint4(0, 0, 0, 0);
    auto row_ptrs = [&](int t, const uint4*& pr, const uint4*& pi) {
      int b, mt, nt;
      tile_coords(t, tiles_m, tiles_n, p.group_m, b, mt, nt);
      pr = pi = nullptr;
      if (a_side) {
        const int m = mt * BM + row;
        if (m < p.M) {
          pr = reinterpret_cast<const uint4*>(p.w + ((size_t)(2 * b) * p.M + m) * p.Kw);
          pi = reinterpret_cast<const uint4*>(p.w + ((size_t)(2 * b + 1) * p.M + m) * p.Kw);
        }
      } else {
        const int n = nt * BN + row;
        if (n < p.N) {
          pr = reinterpret_cast<const uint4*>(p.x + ((size_t)(2 * b) * p.N + n) * p.Kw);
          pi = reinterpret_cast<const uint4*>(p.x + ((size_t)(2 * b + 1) * p.N + n) * p.Kw);
        }
      }
    };
    const uint4* src_r;
    const uint4* src_i;
    row_ptrs(blockIdx.x, src_r, src_i);
    uint4 nr = (blockIdx.x < (unsigned)num_tiles && src_r) ? __ldg(src_r) : zero;
    uint4 ni = (blockIdx.x < (unsigned)num_tiles && src_i) ? __ldg(src_i) : zero;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const bool valid = src_r != nullptr;
      const uint4* next_r = nullptr;
      const uint4* next_i = nullptr;
      const int tn = t + gridDim.x;
      if (tn < num_tiles) row_ptrs(tn, next_r, next_i);
      for (int kb = 0; kb < num_kb; ++kb) {
        const uint4 wr = nr, wi = ni;
        if (kb + 1 < num_kb) {
          nr = valid ? __ldg(src_r + kb + 1) : zero;
          ni = valid ? __ldg(src_i + kb + 1) : zero;
        } else {  // first K block of this thread's next tile
          nr = next_r ? __ldg(next_r) : zero;
          ni = next_i ? __ldg(next_i) : zero;
        }
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* st = smem + stage * STAGE_BYTES;
        if (!(p.debug & 4)) {
          uint8_t* dr = st + (a_side ? 0 : 2 * TILE_BYTES) + row * 128;
          uint8_t* di = dr + TILE_BYTES;
          expand_word(dr, row, 0, wr.x); expand_word(dr, row, 1, wr.y);
          expand_word(dr, row, 2, wr.z); expand_word(dr, row, 3, wr.w);
          expand_word(di, row, 0, wi.x); expand_word(di, row, 1, wi.y);
          expand_word(di, row, 2, wi.z); expand_word(di, row, 3, wi.w);
        }
        fence_proxy_async_smem();  // each thread's generic-proxy smem writes -> async proxy
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_bar[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      src_r = next_r;
      src_i = next_i;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

template <bool TMA_STORE>
cudaError_t launch_f8(const CUtensorMap& tmC, const GemmB1Args& a, int num_sms, cudaStream_t stream) {
  auto kern = cgemm_b1_f8_kernel<TMA_STORE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  const long long nt = (long long)tiles_m * tiles_n * a.B;
  if (nt > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int grid = (int)(nt < num_sms ? nt : num_sms);
  kern<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(tmC, a, tiles_m, tiles_n, (int)nt);
  return cudaGetLastError();
}

}  // namespace

// fp32 accumulation of +-1 products is exact while every partial sum stays below 2^24
bool gemm_b1_f8_supported(int64_t Kw) { return 32 * Kw <= (int64_t(1) << 23); }

cudaError_t launch_gemm_b1_f8(const CUtensorMap& tmC, const GemmB1Args& args, bool tma_store, int num_sms,
                              cudaStream_t stream) {
  return tma_store ? launch_f8<true>(tmC, args, num_sms, stream) : launch_f8<false>(tmC, args, num_sms, stream);
}

}  // namespace tcbf
