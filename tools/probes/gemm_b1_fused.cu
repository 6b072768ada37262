// gemm_b1_fused.cu -- 1-bit-mode beamformer GEMM consuming the fp32 data directly (the 1-bit
// quantise-and-pack of PAPER.md:107 fused into the GEMM; short K, Kw <= 16 words = K <= 512).
//
// Work unit = (batch entry, 128 data columns).  8 converter warps read the unit's fp32 data once
// (warp-coalesced 256-byte row segments), apply the sign rule (bit = value >= 0, PAPER.md:170-172,
// reading R4) and keep the unit's packed words -- 2 planes x 128 columns x Kw words, LSB-first
// (R3), padding bits 0 -- resident in shared memory, double-buffered so the next
// unit converts while the current one computes.  The GEMM itself is the int8 AND-form kernel of
// gemm_b1_tc.cu (bytes {0,2} by bit-plane masking, tcgen05.mma.kind::i8, single-AND correction
// R1b), here with 64-bit K blocks (64-byte swizzle) so the resident words fit beside the stages.
// Bit-identical to tcbf_pack(DATA) + tcbf_beamform.
//
//   warp 0       TMEM allocator + single-thread MMA issuer
//   warps 1-4    epilogue (row term + column term, TMA store of int32)
//   warps 5-8    weight-row expanders (packed weights from global memory)
//   warps 9-12   data-column expanders (resident words from shared memory)
//   warps 13-16  converters, one data column per thread (fp32 -> resident words + column terms)
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BM = 128, BN = 128;
constexpr int KBW = 4;                    // words per K block (128 bits -> 128-byte expanded rows)
constexpr int ROWB = 128;
constexpr int TILE = 128 * ROWB;          // 16 KB
constexpr int STAGES = 2;
constexpr int STAGE_BYTES = 5 * TILE;     // A_r, A_i, B_r, B_i, ~B_i
constexpr int KWMAX = 16;
constexpr int BITS_BYTES = 2 * BN * KWMAX * 4;    // one unit: [2 planes][128 cols][KWMAX words]
constexpr int EPI_BYTES = 4 * 1 * 4096;   // one staging box per epilogue warp (smem budget)
constexpr int OFF_BITS = STAGES * STAGE_BYTES;
constexpr int OFF_EPI = OFF_BITS + 2 * BITS_BYTES;
constexpr int OFF_CT = OFF_EPI + EPI_BYTES;       // column terms [2 units][re, im][128]
constexpr int OFF_RT = OFF_CT + 2 * 2 * 128 * 4;   // row terms [2 tiles][128]
constexpr int BAR_OFFSET = OFF_RT + 2 * 128 * 4;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
constexpr int NUM_THREADS = 17 * 32;
constexpr uint32_t TMEM_COLS = 512;
static_assert(SMEM_BYTES <= 232448, "smem budget");

__device__ __forceinline__ uint4 planes_lo(uint32_t w) {
  const uint32_t m = 0x02020202u;
  return make_uint4((w << 1) & m, w & m, (w >> 1) & m, (w >> 2) & m);
}
__device__ __forceinline__ uint4 planes_hi(uint32_t w) {
  const uint32_t m = 0x02020202u;
  return make_uint4((w >> 3) & m, (w >> 4) & m, (w >> 5) & m, (w >> 6) & m);
}
// word q (0..3) of a 128-bit K block into a 128-byte row, 128-byte swizzle (chunk ^= row & 7)
__device__ __forceinline__ void expand64(uint8_t* row_base, int row, int q, uint32_t w) {
  const int sw = row & 7;
  *reinterpret_cast<uint4*>(row_base + (((2 * q) ^ sw) << 4)) = planes_lo(w);
  *reinterpret_cast<uint4*>(row_base + (((2 * q + 1) ^ sw) << 4)) = planes_hi(w);
}
__device__ __forceinline__ void expand64_pair(uint8_t* base, uint8_t* base_c, int row, int q, uint32_t w) {
  const uint32_t m = 0x02020202u;
  const uint4 c0 = planes_lo(w), c1 = planes_hi(w);
  const int sw = row & 7;
  const int p0 = ((2 * q) ^ sw) << 4, p1 = ((2 * q + 1) ^ sw) << 4;
  *reinterpret_cast<uint4*>(base + p0) = c0;
  *reinterpret_cast<uint4*>(base + p1) = c1;
  *reinterpret_cast<uint4*>(base_c + p0) = make_uint4(c0.x ^ m, c0.y ^ m, c0.z ^ m, c0.w ^ m);
  *reinterpret_cast<uint4*>(base_c + p1) = make_uint4(c1.x ^ m, c1.y ^ m, c1.z ^ m, c1.w ^ m);
}
__device__ __forceinline__ uint64_t desc_k64(const void* tile, uint32_t k_byte_off) {
  uint32_t addr = smem_u32(tile) + k_byte_off;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(512u >> 4) << 32;  // 8 rows x 64 B
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)4u << 61;           // SWIZZLE_64B
  return d;
}

template <int LAYOUT, bool VEC>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_b1_fused_kernel(const __grid_constant__ CUtensorMap tmC, GemmB1Args p, const float* __restrict__ xsrc,
                          int tiles_m, int tiles_n) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint32_t* bits = reinterpret_cast<uint32_t*>(smem + OFF_BITS);  // [2][2 planes][KWMAX][128] (conflict-free)
  uint8_t* epi_base = smem + OFF_EPI;
  int* cterm = reinterpret_cast<int*>(smem + OFF_CT);   // [2][2][128]
  int* rterm = reinterpret_cast<int*>(smem + OFF_RT);   // [2][128]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull = empty_bar + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + 2;
  uint64_t* bfull = sempty + 2;
  uint64_t* bempty = bfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int Kw = p.Kw;
  const int num_kb = Kw / KBW;
  const int num_units = p.B * tiles_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 8);   // 4 weight-row + 4 data-column expander warps
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
      mbar_init(&sfull[s], 4);      // row terms of a tile
      mbar_init(&sempty[s], 4);
      mbar_init(&bfull[s], 4);      // converted unit (words + column terms): 4 converter warps
      mbar_init(&bempty[s], 8);     // 4 data-column expander warps + 4 epilogue warps
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmC);
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
      constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        for (int mt = 0; mt < tiles_m; ++mt, ++it) {
          const int abuf = it & 1;
          mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_re = tmem_base + abuf * 2 * BN;
          const uint32_t d_im = d_re + BN;
          for (int kb = 0; kb < num_kb; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            uint8_t* st = smem + stage * STAGE_BYTES;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // four K = 32-byte MMA steps per 128-byte row
              const uint32_t off = kk * 32;
              const uint64_t ar = smem_desc_k128(st, off), ai = smem_desc_k128(st + TILE, off);
              const uint64_t br = smem_desc_k128(st + 2 * TILE, off), bi = smem_desc_k128(st + 3 * TILE, off);
              const uint64_t bc = smem_desc_k128(st + 4 * TILE, off);
              const uint32_t acc = (kb | kk) ? 1u : 0u;
              mma_i8_ss(d_re, ar, br, IDESC, acc);  // P(A_r & B_r)
              mma_i8_ss(d_re, ai, bc, IDESC, 1u);   // P(A_i & ~B_i)
              mma_i8_ss(d_im, ar, bi, IDESC, acc);  // P(A_r & B_i)
              mma_i8_ss(d_im, ai, br, IDESC, 1u);   // P(A_i & B_r)
            }
            mma_commit(&empty_bar[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          mma_commit(&tfull[abuf]);
        }
      }
    }
  } else if (warp <= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    uint8_t* stg = epi_base + (warp - 1) * 4096;
    int it = 0, ui = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++ui) {
      const int b = u / tiles_n;
      const int n0 = (u - b * tiles_n) * BN;
      const int bb = ui & 1;
      mbar_wait(&bfull[bb], (ui >> 1) & 1);  // this unit's column terms
      const int* ct_re = cterm + (bb * 2 + 0) * 128;
      const int* ct_im = cterm + (bb * 2 + 1) * 128;
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int m0 = mt * BM;
        const int cb = it & 1;
        mbar_wait(&sfull[cb], (it >> 1) & 1);
        const int rt = rterm[cb * 128 + q * 32 + lane];
        const int abuf = it & 1;
        mbar_wait(&tfull[abuf], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 2 * BN;
        uint32_t vbuf[2][32];
        tmem_ld_32x32b_x32(tbase, vbuf[0]);
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          const int part_ = ch / 4;
          const int c = ch % 4;
          tmem_wait_ld();
          if (ch + 1 < 8) {
            tmem_ld_32x32b_x32(tbase + (ch + 1) * 32, vbuf[(ch + 1) & 1]);
          } else {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              mbar_arrive(&tempty[abuf]);
              mbar_arrive(&sempty[cb]);
            }
          }
          uint32_t* v = vbuf[ch & 1];
          const int* ctp = (part_ == 0 ? ct_re : ct_im) + c * 32;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int4 t4 = *reinterpret_cast<const int4*>(ctp + 4 * j);
            v[4 * j + 0] = (uint32_t)((int)v[4 * j + 0] + t4.x + rt);
            v[4 * j + 1] = (uint32_t)((int)v[4 * j + 1] + t4.y + rt);
            v[4 * j + 2] = (uint32_t)((int)v[4 * j + 2] + t4.z + rt);
            v[4 * j + 3] = (uint32_t)((int)v[4 * j + 3] + t4.w + rt);
          }
          if (lane == 0) bulk_wait_group_read<0>();
          __syncwarp();
          uint8_t* buf = stg;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int pos = j ^ (lane & 7);
            *reinterpret_cast<uint4*>(buf + lane * 128 + pos * 16) =
                make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmC, buf, n0 + c * 32, m0 + q * 32, 2 * b + part_);
            bulk_commit_group();
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bempty[bb]);  // column terms of this unit consumed
    }
    if (lane == 0) bulk_wait_group<0>();
    __syncwarp();
  } else if (warp <= 12) {
    // ------------------------------------------------------------ expanders
    const bool a_side = warp <= 8;
    const int row = (warp - (a_side ? 5 : 9)) * 32 + lane;  // weight row / data column in the tile
    int stage = 0;
    uint32_t phase = 0;
    int it = 0, ui = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++ui) {
      const int b = u / tiles_n;
      const int bb = ui & 1;
      const uint32_t* wr_src = bits + (bb * 2 + 0) * KWMAX * BN + row;
      const uint32_t* wi_src = bits + (bb * 2 + 1) * KWMAX * BN + row;
      if (!a_side) mbar_wait(&bfull[bb], (ui >> 1) & 1);
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const uint4* gr = nullptr;
        const uint4* gi = nullptr;
        const int m = mt * BM + row;
        if (a_side && m < p.M) {
          gr = reinterpret_cast<const uint4*>(p.w + ((size_t)(2 * b) * p.M + m) * Kw);
          gi = reinterpret_cast<const uint4*>(p.w + ((size_t)(2 * b + 1) * p.M + m) * Kw);
        }
        int pc = 0;
        const uint4 z4 = make_uint4(0, 0, 0, 0);
        uint4 nr = gr ? __ldg(gr) : z4;
        uint4 ni = gi ? __ldg(gi) : z4;
        for (int kb = 0; kb < num_kb; ++kb) {
          uint4 wr, wi;
          if (a_side) {
            wr = nr; wi = ni;
            if (kb + 1 < num_kb) {
              nr = gr ? __ldg(gr + kb + 1) : z4;
              ni = gi ? __ldg(gi + kb + 1) : z4;
            }
            pc += __popc(wr.x) + __popc(wr.y) + __popc(wr.z) + __popc(wr.w) + __popc(wi.x) + __popc(wi.y) +
                  __popc(wi.z) + __popc(wi.w);
          } else {
            const int w0 = kb * KBW;
            wr = make_uint4(wr_src[w0 * BN], wr_src[(w0 + 1) * BN], wr_src[(w0 + 2) * BN], wr_src[(w0 + 3) * BN]);
            wi = make_uint4(wi_src[w0 * BN], wi_src[(w0 + 1) * BN], wi_src[(w0 + 2) * BN], wi_src[(w0 + 3) * BN]);
          }
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          if (a_side) {
            uint8_t* ar = st + row * ROWB;
            uint8_t* ai = st + TILE + row * ROWB;
            expand64(ar, row, 0, wr.x); expand64(ar, row, 1, wr.y);
            expand64(ar, row, 2, wr.z); expand64(ar, row, 3, wr.w);
            expand64(ai, row, 0, wi.x); expand64(ai, row, 1, wi.y);
            expand64(ai, row, 2, wi.z); expand64(ai, row, 3, wi.w);
          } else {
            uint8_t* br = st + 2 * TILE + row * ROWB;
            uint8_t* bi = st + 3 * TILE + row * ROWB;
            uint8_t* bc = st + 4 * TILE + row * ROWB;
            expand64(br, row, 0, wr.x); expand64(br, row, 1, wr.y);
            expand64(br, row, 2, wr.z); expand64(br, row, 3, wr.w);
            expand64_pair(bi, bc, row, 0, wi.x); expand64_pair(bi, bc, row, 1, wi.y);
            expand64_pair(bi, bc, row, 2, wi.z); expand64_pair(bi, bc, row, 3, wi.w);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (a_side) {  // row term of this tile, R1b
          const int cb = it & 1;
          mbar_wait(&sempty[cb], ((it >> 1) & 1) ^ 1);
          rterm[cb * 128 + row] = -2 * pc;
          __syncwarp();
          if (lane == 0) mbar_arrive(&sfull[cb]);
        }
      }
      if (!a_side) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&bempty[bb]);  // resident words of this unit no longer needed
      }
    }
  } else {
    // ------------------------------------------------------------ converters
    const int col = threadIdx.x - 13 * 32;  // 0..127
    const int N = p.N, K = p.K;
    int ui = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++ui) {
      const int b = u / tiles_n;
      const int n = (u - b * tiles_n) * BN + col;
      const int bb = ui & 1;
      mbar_wait(&bempty[bb], ((ui >> 1) & 1) ^ 1);
      uint32_t* dr = bits + (bb * 2 + 0) * KWMAX * BN + col;
      uint32_t* di = bits + (bb * 2 + 1) * KWMAX * BN + col;
      int pr = 0, pi = 0;
      for (int w = 0; w < Kw; ++w) {
        uint32_t br = 0, bi = 0;
        const int k0 = w * 32;
        if (n < N && k0 < K) {
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {  // 16 loads in flight per batch
            float2 v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int k = k0 + 16 * h2 + j;
              if (k < K) {
                if (LAYOUT == 0) {
                  v[j] = __ldg(reinterpret_cast<const float2*>(xsrc) + ((size_t)b * K + k) * N + n);
                } else {
                  v[j] = make_float2(__ldg(xsrc + (((size_t)b * 2 + 0) * K + k) * N + n),
                                     __ldg(xsrc + (((size_t)b * 2 + 1) * K + k) * N + n));
                }
              } else {
                v[j] = make_float2(-1.f, -1.f);  // padding -> bit 0
              }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              br |= (v[j].x >= 0.f ? 1u : 0u) << (16 * h2 + j);  // NaN -> 0
              bi |= (v[j].y >= 0.f ? 1u : 0u) << (16 * h2 + j);
            }
          }
        }
        dr[w * BN] = br;
        di[w * BN] = bi;
        pr += __popc(br);
        pi += __popc(bi);
      }
      cterm[(bb * 2 + 0) * 128 + col] = 2 * (pi - pr);          // 2 (|B_i| - |B_r|)
      cterm[(bb * 2 + 1) * 128 + col] = 2 * K - 2 * (pr + pi);  // 2K - 2 (|B_r| + |B_i|)
      __syncwarp();
      if (lane == 0) mbar_arrive(&bfull[bb]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

template <int LAYOUT, bool VEC>
cudaError_t launch_b1f(const CUtensorMap& tmC, const GemmB1Args& a, const float* x, int num_sms, cudaStream_t s) {
  auto kern = cgemm_b1_fused_kernel<LAYOUT, VEC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  const long long units = (long long)tiles_n * a.B;
  if (units * tiles_m > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int grid = (int)(units < num_sms ? units : num_sms);
  kern<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(tmC, a, x, tiles_m, tiles_n);
  return cudaGetLastError();
}

}  // namespace

bool gemm_b1_fused_supported(int64_t Kw, int64_t N) { return Kw <= KWMAX && N % 4 == 0; }

cudaError_t launch_gemm_b1_fused(const CUtensorMap& tmC, const GemmB1Args& args, const float* x_src, int layout,
                                 int num_sms, cudaStream_t stream) {
  if (layout == 0) return launch_b1f<0, false>(tmC, args, x_src, num_sms, stream);
  return launch_b1f<1, false>(tmC, args, x_src, num_sms, stream);
}

}  // namespace tcbf
