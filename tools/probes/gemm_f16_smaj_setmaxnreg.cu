// PARKED dev probe (not built): the sample-major kernel with 20 warps, setmaxnreg (converters 128
// registers, producer/MMA 32) and a 3-deep register pipeline of 32-row blocks per converter.
// Bit-identical; measured 0.69 vs 0.63 ms (the unit-switch stall stayed ~7.6 us).

// gemm_f16_smaj.cu -- sample-major fused 16-bit beamformer: fp32 data in, fp32 beams out, with
// the SAMPLES on the 128-row MMA dimension and the beams on N.
//
// Same arithmetic as the other 16-bit kernels (fp16 RNE inputs, exact products, fp32 accumulation
// in TMEM, four real sub-products per K step -- PAPER.md:143-159), computed transposed:
//     D^T[n][m] = sum_k X[k][n] W[m][k]
// with the data X (converted once per unit from fp32 by converter warps) as the MN-major A operand
// and the weights as the K-major B operand, stacked [W_r ; W_i]:
//     [Re | Im] += X_r [W_r ; W_i]^T          (one M=128, N=256 MMA)
//     Re        += (-X_i) W_i^T               (N=128, negate-A bit: the paper's negation step)
//     Im        += X_i W_r^T                  (N=128)
// Per K step that is 28 KB of operand reads per 128x128 complex tile instead of the 32 KB of four
// N=128 MMAs, and no third (negated) operand plane is needed.
//
// Why transposed: the radio shapes are bound by the 8 bytes/complex output stream.
// With samples on TMEM lanes, `tcgen05.ld 32x32b` gives thread t of a warp the sample n0+t, so one
// warp store of register j writes 32 CONSECUTIVE floats (one full 128-byte line) of beam row m+j:
// the output leaves the SM as fully coalesced line writes straight from registers -- no smem
// staging, no TMA store engine (measured capped near 6.0 TB/s on these patterns), any N.
//
// Work unit = (batch entry b, 128 samples); the unit's data stays resident in smem (K16 <= 256,
// eight 32-k-row slots) while every 128-beam weight tile streams through a 3-stage TMA ring; TMEM
// holds two 256-column accumulators so the epilogue of one tile overlaps the MMAs of the next.
//
// Unit switch (the TCBF_TRACE timeline, tools/trace_smaj.py).  A unit's slots are read by every
// beam tile, so the next unit's data can only enter them once the last tile has released them;
// the converters then pay a global-load latency per block that the output-store stream stretches
// to 3-5 us.  With one block of loads in flight per thread that stalled the MMAs ~8 us per switch
// (~15% of the kernel).  The converter warps therefore get the registers the producer / MMA warps
// do not need (setmaxnreg: 128 per thread instead of 96) and keep the loads of the next THREE
// 32-row blocks in flight, so most of the next unit is already in registers when its slots free.
//
// Roles (20 warps, warpgroup-aligned for setmaxnreg): warps 0-7 epilogue (tcgen05.ld -> coalesced
// st.global), warps 8-15 converters (fp32 -> fp16 MN-major slots), warp 16 TMA producer (weights),
// warp 17 MMA issuer (converged warp, elected lane), warps 18-19 idle.
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BS = 128;                    // samples per tile (MMA M)
constexpr int BB = 128;                    // beams per tile (stacked N = 256)
constexpr int BK = 32;                     // k-rows per data slot
constexpr int WK = 64;                     // K per weight stage (128-byte rows)
constexpr int KMAX = 256;                  // resident K rows (K16 <= 256)
constexpr int W_TILE = BB * WK * 2;        // one weight plane of one stage (16 KB)
constexpr int W_STAGE = 2 * W_TILE;        // [W_r ; W_i]
constexpr int W_STAGES = 3;
constexpr int X_SLOTS = KMAX / BK;         // 8
constexpr int X_HALF = BK * 128;           // 64 samples of one plane: 32 k-rows x 128 B
constexpr int X_PLANE = 2 * X_HALF;        // 128 samples of one plane
constexpr int X_SLOT = 2 * X_PLANE;        // [X_r | X_i] = 16 KB
constexpr int OFF_W = X_SLOTS * X_SLOT;
constexpr int BAR_OFFSET = OFF_W + W_STAGES * W_STAGE;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
static_assert(SMEM_BYTES <= 232448, "smem budget");

constexpr int EPI_WARPS = 8;
constexpr int CONV_WARP0 = 8;
constexpr int CONV_WARPS = 8;
constexpr int PRODUCER_WARP = 16;
constexpr int MMA_WARP = 17;
constexpr int NUM_THREADS = 20 * 32;
// register budget after setmaxnreg (the CTA pool = the 640 x 96 launch allocation): epilogue
// 8 x 32 x 96 + converters 8 x 32 x 128 + producer / MMA / idle 4 x 32 x 32 = 61440
constexpr int CONV_REGS = 128;
constexpr int LOW_REGS = 32;
constexpr int CONV_DEPTH = 3;              // 32-row blocks of fp32 loads in flight per converter thread

// K-major weights (B operand): 128-byte swizzle, 8-row groups 1024 B apart; the W_i tile follows
// the W_r tile directly, so one descriptor spans the stacked N = 256 operand
__device__ __forceinline__ uint64_t desc_w(const void* tile, uint32_t k_byte_off) {
  uint32_t addr = smem_u32(tile) + k_byte_off;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// resident MN-major data (A operand): 64-sample half j at j * X_HALF (LBO), 8 k-rows per
// 1024 B (SBO), 128-byte swizzle
__device__ __forceinline__ uint64_t desc_x(const void* plane, uint32_t k_row) {
  uint32_t addr = smem_u32(plane) + k_row * 128u;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((uint32_t)X_HALF >> 4) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// kind::f16: fp16 A/B, fp32 D, A MN-major (bit 15), B K-major, M = 128
__host__ __device__ constexpr uint32_t idesc_smaj(uint32_t N, bool negate_a) {
  return (1u << 4) | ((negate_a ? 1u : 0u) << 13) | (1u << 15) | ((N >> 3) << 17) | ((uint32_t)(BS >> 4) << 24);
}

__device__ __forceinline__ uint32_t h2u(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <uint32_t R>
__device__ __forceinline__ void regs_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R)); }
template <uint32_t R>
__device__ __forceinline__ void regs_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R)); }

// converter work per 32-k-row block: 32 rows x 16 chunks of 8 samples over 256 threads
constexpr int CONV_THREADS = CONV_WARPS * 32;
constexpr int ITEMS = BK * (BS / 8) / CONV_THREADS;  // 2
struct XRegs {
  float re[ITEMS][8], im[ITEMS][8];
};

// CL = 2: CTA pairs (clusters of 2) take adjacent units of the same batch entry and walk the same
// (beam tile, K block) sequence, so their weight stages are identical: each CTA TMA-loads half of
// the stage (two 64-row boxes) and multicasts it into both (half the L2 -> SM weight reads); a
// stage is refilled only when the MMAs of both CTAs have retired (empty count 2, multicast commit).
template <int LAYOUT, bool VEC, int CL>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_smaj_kernel(const __grid_constant__ CUtensorMap tmW, GemmF16Args args, const float* __restrict__ xsrc,
                          int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = smem;          // [X_SLOTS][2 planes][2 sample halves][BK rows][128 B]
  uint8_t* sW = smem + OFF_W;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* wempty = wfull + W_STAGES;
  uint64_t* xfull = wempty + W_STAGES;   // [X_SLOTS]
  uint64_t* xempty = xfull + X_SLOTS;    // [X_SLOTS]
  uint64_t* tfull = xempty + X_SLOTS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = args.K16 / BK;  // data slots per unit (<= 8, even)
  const int tiles_m = args.tiles_m, tiles_n = args.tiles_n;  // beam tiles, sample tiles (units per batch)
  const int num_units = args.B * tiles_n;
  // unit walk: single CTAs stride over all units; pairs take units (2c + rank) (tiles_n even)
  constexpr bool MC = CL > 1;
  constexpr uint16_t CL_MASK = (uint16_t)((1u << CL) - 1u);
  const int rank = MC ? (int)cluster_ctarank() : 0;
  const int u_first = MC ? CL * (int)(blockIdx.x / CL) + rank : (int)blockIdx.x;
  const int u_step = MC ? CL * (int)(gridDim.x / CL) : (int)gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < W_STAGES; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], CL);
    }
    for (int s = 0; s < X_SLOTS; ++s) {
      mbar_init(&xfull[s], CONV_WARPS);
      mbar_init(&xempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmW);
  }
  if (warp == MMA_WARP) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  if (MC) cluster_sync(); else __syncthreads();  // peers signal this CTA's barriers
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp >= PRODUCER_WARP) {
    regs_dec<LOW_REGS>();
    if (warp == PRODUCER_WARP) {
      // ---------------------------------------------------------- TMA producer: weight tiles
      if (lane == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int u = u_first; u < num_units; u += u_step) {
          const int b = u / tiles_n;
          for (int mt = 0; mt < tiles_m; ++mt) {
            for (int kw = 0; kw < num_kb / 2; ++kw) {  // 64-K weight stages
              mbar_wait(&wempty[stage], phase ^ 1);
              uint8_t* st = sW + stage * W_STAGE;
              if (TCBF_ABLATE(args, 8) && mt > 0) {  // ablation: weights once per unit (wrong values)
                mbar_arrive(&wfull[stage]);
              } else {
                mbar_arrive_expect_tx(&wfull[stage], W_STAGE);
                // the stage = 4 boxes of 64 beam rows (plane = box >> 1, rows 64 (box & 1)); CTA
                // `rank` of a cluster of CL loads boxes rank * 4/CL .. and multicasts them
#pragma unroll
                for (int bx = rank * (4 / CL); bx < (rank + 1) * (4 / CL); ++bx) {
                  uint8_t* dst = st + (bx >> 1) * W_TILE + (bx & 1) * (W_TILE / 2);
                  if (MC)
                    tma_load_3d_mc(dst, &tmW, &wfull[stage], kw * WK, mt * BB + (bx & 1) * 64, 2 * b + (bx >> 1),
                                   CL_MASK);
                  else
                    tma_load_3d(dst, &tmW, &wfull[stage], kw * WK, mt * BB + (bx & 1) * 64, 2 * b + (bx >> 1));
                }
              }
              if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    } else if (warp == MMA_WARP) {
      // ---------------------------------------------------------- MMA issuer (converged warp, one
      // elected lane issues: descriptors stay in uniform registers)
      constexpr uint32_t I256 = idesc_smaj(2 * BB, false);
      constexpr uint32_t I128 = idesc_smaj(BB, false);
      constexpr uint32_t I128_NEG = idesc_smaj(BB, true);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0, ui = 0;
      for (int u = u_first; u < num_units; u += u_step, ++ui) {
        const int g0 = ui * num_kb;  // ring index of the unit's first data block
        for (int mt = 0; mt < tiles_m; ++mt, ++it) {
          const int abuf = it & 1;
          const unsigned long long tw0 = args.trace ? gtimer() : 0;  // dev timeline (tools/trace_smaj.py)
          mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
          tc_fence_after();
          unsigned long long wwait = 0, xwait = 0;
          if (args.trace && lane == 0) {
            stamp(args.trace, 4 * it);
            stamp_val(args.trace, 512 + 4 * it + 3, gtimer() - tw0);
          }
          const uint32_t d_re = tmem_base + abuf * 2 * BB;  // [Re | Im]: 256 columns
          const uint32_t d_im = d_re + BB;
          for (int kw = 0; kw < num_kb / 2; ++kw) {  // one 64-K weight stage = two data slots
            const unsigned long long a1 = args.trace ? gtimer() : 0;
            mbar_wait(&wfull[stage], phase);
            if (args.trace) wwait += gtimer() - a1;
            tc_fence_after();
            const uint8_t* st = sW + stage * W_STAGE;
            const uint64_t wri0 = desc_w(st, 0);           // [W_r ; W_i], N = 256 (W_r alone: N = 128)
            const uint64_t wi0 = desc_w(st + W_TILE, 0);   // W_i, N = 128
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int g = g0 + 2 * kw + h;
              const int xs = g % X_SLOTS;
              if (mt == 0) {  // the data block has been converted into its slot
                const unsigned long long a0 = args.trace ? gtimer() : 0;
                mbar_wait(&xfull[xs], (g / X_SLOTS) & 1);
                tc_fence_after();
                if (args.trace) xwait += gtimer() - a0;
              }
              const uint8_t* sx = sX + xs * X_SLOT;
              const uint64_t xr0 = desc_x(sx, 0), xi0 = desc_x(sx + X_PLANE, 0);
              if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk) {
                  // K advance: 16 k-rows of the MN-major data = 2048 B (+128 in the address field),
                  // 16 K of the K-major weights = 32 B (+2)
                  const uint64_t xr = xr0 + (uint64_t)(128 * kk), xi = xi0 + (uint64_t)(128 * kk);
                  const uint32_t wo = 2 * (h * (BK / 16) + kk);
                  const uint64_t w_ri = wri0 + wo, w_i = wi0 + wo;
                  const uint32_t acc = (kw | h | kk) ? 1u : 0u;
                  if (TCBF_ABLATE(args, 2)) continue;
                  mma_f16_ss(d_re, xr, w_ri, I256, acc);      // [Re | Im] += X_r [W_r ; W_i]^T
                  mma_f16_ss(d_re, xi, w_i, I128_NEG, 1u);    // Re += -X_i W_i^T
                  mma_f16_ss(d_im, xi, w_ri, I128, 1u);       // Im += X_i W_r^T
                }
                if (mt == tiles_m - 1) mma_commit(&xempty[xs]);  // last reader of this data block
              }
              __syncwarp();
            }
            if (elect_one()) {
              if (MC) mma_commit_mc(&wempty[stage], CL_MASK);  // the stage is free in both CTAs
              else mma_commit(&wempty[stage]);
            }
            __syncwarp();
            if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
          }
          if (elect_one()) mma_commit(&tfull[abuf]);
          __syncwarp();
          if (args.trace && lane == 0) {
            stamp(args.trace, 4 * it + 1);
            stamp_val(args.trace, 512 + 4 * it, wwait);
            stamp_val(args.trace, 512 + 4 * it + 1, xwait);
          }
        }
      }
    }
  } else if (warp < CONV_WARP0) {
    // ------------------------------------------------------------ epilogue: coalesced line stores
    const int q = warp & 3;                 // TMEM lane quadrant = samples 32q..32q+31 of the tile
    const int half = warp >> 2;             // half 0 stores Re, half 1 Im
    constexpr int MY_CHUNKS = 4;            // 32-column chunks of this warp's 128 accumulator columns
    const size_t N = (size_t)args.N;
    const int M = args.M;
    int it = 0;
    for (int u = u_first; u < num_units; u += u_step) {
      const int b = u / tiles_n;
      const int n = (u - b * tiles_n) * BS + q * 32 + lane;  // this thread's sample
      const bool n_ok = n < args.N;
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int abuf = it & 1;
        mbar_wait(&tfull[abuf], (it >> 1) & 1);
        tc_fence_after();
        if (threadIdx.x == 0) stamp(args.trace, 4 * it + 2);
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 2 * BB + half * BB;
        uint32_t v[2][32];
        tmem_ld_32x32b_x32(tbase, v[0]);
#pragma unroll
        for (int i = 0; i < MY_CHUNKS; ++i) {
          const int m0 = mt * BB + i * 32;
          tmem_wait_ld();
          if (i + 1 < MY_CHUNKS) {
            tmem_ld_32x32b_x32(tbase + (i + 1) * 32, v[(i + 1) & 1]);
          } else {  // all TMEM reads of this tile issued and complete: release the buffer
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[abuf]);
          }
          const uint32_t* vv = v[i & 1];
          if (TCBF_ABLATE(args, 1)) continue;
          if (n_ok) {
            float* dst = args.out + ((size_t)(2 * b + half) * M + m0) * N + n;
            if (m0 + 32 <= M) {
#pragma unroll
              for (int j = 0; j < 32; ++j) dst[(size_t)j * N] = __uint_as_float(vv[j]);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (m0 + j < M) dst[(size_t)j * N] = __uint_as_float(vv[j]);
            }
          }
        }
        if (args.trace && lane == 0) {
          if (warp == 0) stamp(args.trace, 4 * it + 3);
          if (warp == EPI_WARPS - 1) stamp(args.trace, 512 + 4 * it + 2);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ converters: fp32 data -> resident A
    regs_inc<CONV_REGS>();
    const int ct = threadIdx.x - CONV_WARP0 * 32;  // 0..255
    const int N = args.N;
    const int my_units = u_first < num_units ? (num_units - 1 - u_first) / u_step + 1 : 0;
    const int total = my_units * num_kb;  // this CTA's data blocks, in ring order
    // block g of this CTA -> registers (zeros past the end, out-of-range k or n)
    auto load_block = [&](int g, XRegs& rg) {
      const int ui = g / num_kb, kb = g - ui * num_kb;
      const int u = u_first + ui * u_step;
      const int b = u / tiles_n;
      const int n0 = (u - b * tiles_n) * BS;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int item = ct + i * CONV_THREADS;
        const int kr = item / (BS / 8), cc = item % (BS / 8);
        const int k = kb * BK + kr, n = n0 + cc * 8;
        if (g >= total || TCBF_ABLATE(args, 4)) {  // past the end / ablation: no data reads
#pragma unroll
          for (int j = 0; j < 8; ++j) rg.re[i][j] = rg.im[i][j] = 0.f;
        } else if (VEC && LAYOUT == 0 && k < K && n + 8 <= N) {
          const float4* p = reinterpret_cast<const float4*>(xsrc + (((size_t)b * K + k) * N + n) * 2);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 f = __ldg(p + j);
            rg.re[i][2 * j] = f.x; rg.im[i][2 * j] = f.y; rg.re[i][2 * j + 1] = f.z; rg.im[i][2 * j + 1] = f.w;
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
            rg.re[i][j] = a; rg.im[i][j] = c;
          }
        }
      }
    };
    // block g (in registers) -> its ring slot, once the MMAs have released the slot
    auto store_block = [&](int g, const XRegs& rg) {
      if (g >= total) return;
      const int xs = g % X_SLOTS;
      mbar_wait(&xempty[xs], ((g / X_SLOTS) & 1) ^ 1);
      uint8_t* sx = sX + xs * X_SLOT;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int item = ct + i * CONV_THREADS;
        const int kr = item / (BS / 8), cc = item % (BS / 8);
        const int off = (cc >> 3) * X_HALF + kr * 128 + (((cc & 7) ^ (kr & 7)) << 4);
        *reinterpret_cast<uint4*>(sx + off) = make_uint4(h2u(rg.re[i][0], rg.re[i][1]), h2u(rg.re[i][2], rg.re[i][3]),
                                                         h2u(rg.re[i][4], rg.re[i][5]), h2u(rg.re[i][6], rg.re[i][7]));
        *reinterpret_cast<uint4*>(sx + X_PLANE + off) =
            make_uint4(h2u(rg.im[i][0], rg.im[i][1]), h2u(rg.im[i][2], rg.im[i][3]), h2u(rg.im[i][4], rg.im[i][5]),
                       h2u(rg.im[i][6], rg.im[i][7]));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&xfull[xs]);
    };
    // CONV_DEPTH blocks of loads in flight ahead of the one being stored; the ring of register
    // buffers is unrolled so every buffer index is static
    XRegs r[CONV_DEPTH];
#pragma unroll
    for (int d = 0; d < CONV_DEPTH; ++d) load_block(d, r[d]);
    for (int g = 0; g < total; g += CONV_DEPTH) {
#pragma unroll
      for (int d = 0; d < CONV_DEPTH; ++d) {
        store_block(g + d, r[d]);
        load_block(g + d + CONV_DEPTH, r[d]);
      }
    }
  }

  tc_fence_before();
  if (MC) cluster_sync(); else __syncthreads();  // no CTA exits while its peer may still signal it
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

template <int LAYOUT, bool VEC, int CL>
cudaError_t launch_smaj(const CUtensorMap& tmW, const GemmF16Args& a, const float* x, int K, int num_sms,
                        cudaStream_t s) {
  auto kern = cgemm_f16_smaj_kernel<LAYOUT, VEC, CL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int units = a.B * a.tiles_n;
  if (CL == 1) {
    const int grid = units < num_sms ? units : num_sms;
    kern<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(tmW, a, x, K);
    return cudaGetLastError();
  }
  const int clusters = units / CL < num_sms / CL ? units / CL : num_sms / CL;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL * clusters);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, tmW, a, x, K);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int CL>
cudaError_t launch_smaj_layout(const CUtensorMap& tmW, const GemmF16Args& args, const float* x_src, int layout,
                               int K, int num_sms, cudaStream_t stream) {
  const bool vec = layout == 0 && (args.N % 8 == 0) && (reinterpret_cast<uintptr_t>(x_src) % 16 == 0);
  if (layout == 0)
    return vec ? launch_smaj<0, true, CL>(tmW, args, x_src, K, num_sms, stream)
               : launch_smaj<0, false, CL>(tmW, args, x_src, K, num_sms, stream);
  return launch_smaj<1, false, CL>(tmW, args, x_src, K, num_sms, stream);
}

}  // namespace

bool gemm_f16_smaj_supported(int64_t K16) { return K16 <= KMAX; }

// args: tiles_m = beam tiles (128), tiles_n = sample tiles (128), K16 = padded K (multiple of 64);
// weights tensor map: box {64 K, 64 beam rows} per plane, 128-byte swizzle.  cluster = weight-
// multicast cluster size (2 = CTA pairs when tiles_n is even, else 1).
cudaError_t launch_gemm_f16_smaj(const CUtensorMap& tmW, const GemmF16Args& args, const float* x_src, int layout,
                                 int K, int cluster, int num_sms, cudaStream_t stream) {
  // (clusters of 4 were measured 1.5x slower on radio fp16 -- 0.99 vs 0.67 ms: co-scheduling 4-CTA
  // clusters and lock-stepping them costs more than the halved L2 weight reads save -- so the
  // kernel is built for pairs only)
  const int units = args.B * args.tiles_n;
  if (cluster >= 2 && args.tiles_n % 2 == 0 && units >= 2)
    return launch_smaj_layout<2>(tmW, args, x_src, layout, K, num_sms, stream);
  return launch_smaj_layout<1>(tmW, args, x_src, layout, K, num_sms, stream);
}

}  // namespace tcbf
