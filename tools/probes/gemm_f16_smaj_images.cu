// PARKED dev probe (not built): sample-major fused kernel with fp16 slot images staged in a per-CTA
// global scratch and TMA bulk-copied into the slots at the unit switch.  Bit-identical; measured
// slower (659 vs 607 us burst on radio fp16): the switch stall disappears but the extra scratch
// stores slow the epilogue.  Needs GemmF16Args::xscratch to build.

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
// Unit switch (measured with the TCBF_TRACE timeline, tools/trace_smaj.py).  A unit's slots are
// read by every beam tile, so the next unit's data can only enter them once the last tile has
// released them.  When the converters loaded fp32 straight into the slots, every block of the
// switch paid a global-load latency that the heavy output-store stream stretched to 3-7 us (the
// loads queue behind the epilogue's stores in the SM's memory pipeline), an MMA stall of ~7 us per
// switch, ~15% of the kernel.  So the conversion is decoupled from the switch: during unit u the
// converters turn unit u+1's fp32 data into fp16 slot IMAGES in a per-CTA global scratch (latency
// no longer matters, there is a whole unit of time), and at the switch a loader warp moves each
// 16 KB image into its slot with one TMA bulk copy the moment the slot frees (all eight in flight,
// served from L2, no LSU queue).  Extra traffic: 2 x 128 KB of L2 per unit, no extra HBM bytes
// while the scratch stays in L2 (checked with ncu dram bytes).
//
// Roles: warp 0 TMA producer (weights), warp 1 MMA issuer, warps 2..2+EPI_WARPS-1 epilogue
// (tcgen05.ld -> coalesced st.global), then 8 converter warps (fp32 -> fp16 slot images in the
// scratch), then the slot loader warp (scratch -> smem slots, TMA bulk copies).
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
constexpr int CONV_WARPS = 8;
constexpr int W_TILE = BB * WK * 2;        // one weight plane of one stage (16 KB)
constexpr int W_STAGE = 2 * W_TILE;        // [W_r ; W_i]
constexpr int W_STAGES = 3;
constexpr int X_SLOTS = KMAX / BK;         // a unit's blocks
constexpr int X_HALF = BK * 128;           // 64 samples of one plane: 32 k-rows x 128 B
constexpr int X_PLANE = 2 * X_HALF;        // 128 samples of one plane
constexpr int X_SLOT = 2 * X_PLANE;        // [X_r | X_i] = 16 KB
constexpr int OFF_X = 0;
constexpr int OFF_W = X_SLOTS * X_SLOT;
constexpr int BAR_OFFSET = OFF_W + W_STAGES * W_STAGE;
constexpr int BAR_BYTES = (2 * W_STAGES + 2 * X_SLOTS + 5) * 8 + 16;  // mbarriers + TMEM address slot
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + BAR_BYTES;
static_assert(SMEM_BYTES <= 232448, "smem budget");

template <int EPI_WARPS>
struct SCfg {
  static constexpr int CONV0 = 2 + EPI_WARPS;
  static constexpr int LOADER = CONV0 + CONV_WARPS;
  static constexpr int NUM_THREADS = (LOADER + 1) * 32;
};

// K-major weights (B operand): 128-byte rows of 64 K, 128-byte swizzle, 8-row groups 1024 B
// apart; the W_i tile follows the W_r tile directly, so one descriptor spans the stacked N = 256
// operand.  (32-K stages with a 64-byte swizzle were measured ~15% slower per MMA tile.)
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

// converter work per 32-k-row block: 32 rows x 16 chunks of 8 samples over 256 threads
constexpr int CONV_THREADS = CONV_WARPS * 32;
constexpr int ITEMS = BK * (BS / 8) / CONV_THREADS;  // 2
struct XRegs {
  float re[ITEMS][8], im[ITEMS][8];
};

// MC: CTA pairs (clusters of 2) take adjacent units of the same batch entry and walk the same
// (beam tile, K block) sequence, so their weight stages are identical: each CTA TMA-loads one of
// the two planes and multicasts it into both (half the L2 -> SM weight traffic); a stage is
// refilled only when the MMAs of BOTH CTAs have retired (empty barrier count 2, multicast commit).
template <int LAYOUT, bool VEC, int EPI_WARPS, bool MC>
__global__ void __launch_bounds__(SCfg<EPI_WARPS>::NUM_THREADS, 1)
    cgemm_f16_smaj_kernel(const __grid_constant__ CUtensorMap tmW, GemmF16Args args, const float* __restrict__ xsrc,
                          int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = smem + OFF_X;  // [X_SLOTS][2 planes][2 sample halves][BK rows][128 B]
  uint8_t* sW = smem + OFF_W;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* wempty = wfull + W_STAGES;
  uint64_t* xfull = wempty + W_STAGES;   // [X_SLOTS]: slot image landed (TMA transaction count)
  uint64_t* xempty = xfull + X_SLOTS;    // [X_SLOTS]: last MMA reader of the slot retired
  uint64_t* tfull = xempty + X_SLOTS;
  uint64_t* tempty = tfull + 2;
  uint64_t* sready = tempty + 2;         // the converters finished an occurrence's scratch images
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sready + 1);
  // this CTA's scratch: one unit's slot images (X_SLOTS x 16 KB), written by the converters
  uint8_t* scratch = args.xscratch + (size_t)blockIdx.x * X_SLOTS * X_SLOT;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = args.K16 / BK;  // <= 8, even
  const int tiles_m = args.tiles_m, tiles_n = args.tiles_n;  // beam tiles, sample tiles (units per batch)
  const int num_units = args.B * tiles_n;
  // unit walk: single CTAs stride over all units; pairs take units (2p + rank) (units even)
  const int rank = MC ? (int)cluster_ctarank() : 0;
  const int u_first = MC ? 2 * (int)(blockIdx.x >> 1) + rank : (int)blockIdx.x;
  const int u_step = MC ? 2 * (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int my_units = u_first < num_units ? (num_units - 1 - u_first) / u_step + 1 : 0;
  // Staggered walk (TCBF_DEBUG bit 32 turns it off): every CTA (pair) starts its first unit at
  // beam tile r and finishes that unit's tiles 0..r-1 at the very end (its data converted a second
  // time), so the CTAs' unit switches are spread over the unit period rather than synchronised.
  // Occurrence i of the walk: unit occ_unit(i), beam tiles [occ_mt0(i), occ_mt1(i)).
  const int r = (tiles_m > 1 && my_units > 0 && !TCBF_ABLATE(args, 32))
                    ? (int)((MC ? (blockIdx.x >> 1) : blockIdx.x) % tiles_m) : 0;
  const int n_occ = my_units + (r > 0 ? 1 : 0);
  auto occ_unit = [&](int i) { return u_first + (i < my_units ? i : 0) * u_step; };
  auto occ_mt0 = [&](int i) { return i == 0 ? r : 0; };
  auto occ_mt1 = [&](int i) { return i == my_units ? r : tiles_m; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < W_STAGES; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], MC ? 2 : 1);
    }
    for (int s = 0; s < X_SLOTS; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPI_WARPS);
    }
    mbar_init(sready, CONV_WARPS);
    fence_barrier_init();
    tma_prefetch_desc(&tmW);
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
      for (int i = 0; i < n_occ; ++i) {
        const int b = occ_unit(i) / tiles_n;
        for (int mt = occ_mt0(i); mt < occ_mt1(i); ++mt) {
          for (int kw = 0; kw < num_kb / 2; ++kw) {  // 64-K weight stages
            mbar_wait(&wempty[stage], phase ^ 1);
            uint8_t* st = sW + stage * W_STAGE;
            if (TCBF_ABLATE(args, 8) && mt > occ_mt0(i)) {  // ablation: weights once per unit (wrong values)
              mbar_arrive(&wfull[stage]);
            } else {
              mbar_arrive_expect_tx(&wfull[stage], W_STAGE);
              if (MC) {
                tma_load_3d_mc(st + rank * W_TILE, &tmW, &wfull[stage], kw * WK, mt * BB, 2 * b + rank);
              } else {
                tma_load_3d(st, &tmW, &wfull[stage], kw * WK, mt * BB, 2 * b);
                tma_load_3d(st + W_TILE, &tmW, &wfull[stage], kw * WK, mt * BB, 2 * b + 1);
              }
            }
            if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t I256 = idesc_smaj(2 * BB, false);
      constexpr uint32_t I128 = idesc_smaj(BB, false);
      constexpr uint32_t I128_NEG = idesc_smaj(BB, true);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int i = 0; i < n_occ; ++i) {
        const int g0 = i * num_kb;  // ring index of the occurrence's first data block
        const int mt0 = occ_mt0(i), mt1 = occ_mt1(i);
        for (int mt = mt0; mt < mt1; ++mt, ++it) {
          const int abuf = it & 1;
          const unsigned long long tw0 = args.trace ? gtimer() : 0;
          mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
          tc_fence_after();
          unsigned long long wwait = 0, xwait = 0;
          if (args.trace) {
            stamp(args.trace, 4 * it);
            stamp_val(args.trace, 512 + 4 * it + 3, gtimer() - tw0);
          }
          const uint32_t d_re = tmem_base + abuf * 2 * BB;  // [Re | Im]: 256 columns
          const uint32_t d_im = d_re + BB;
          for (int kw = 0; kw < num_kb / 2; ++kw) {  // one 64-K weight stage = two data slots
            if (args.trace) {
              const unsigned long long a1 = gtimer();
              mbar_wait(&wfull[stage], phase);
              wwait += gtimer() - a1;
            }
            mbar_wait(&wfull[stage], phase);
            tc_fence_after();
            const uint8_t* st = sW + stage * W_STAGE;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int g = g0 + 2 * kw + h;
              const int xs = g % X_SLOTS;
              if (mt == mt0) {  // the slot image has landed
                const unsigned long long a0 = args.trace ? gtimer() : 0;
                mbar_wait(&xfull[xs], (g / X_SLOTS) & 1);
                tc_fence_after();
                if (args.trace) xwait += gtimer() - a0;
              }
              const uint8_t* sx = sX + xs * X_SLOT;
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                const uint32_t kw_off = (h * BK + kk * 16) * 2;       // byte offset in the 128-byte weight row
                const uint64_t xr = desc_x(sx, kk * 16), xi = desc_x(sx + X_PLANE, kk * 16);
                const uint64_t w_ri = desc_w(st, kw_off);            // [W_r ; W_i], N = 256
                const uint64_t w_i = desc_w(st + W_TILE, kw_off);    // W_i, N = 128
                const uint64_t w_r = w_ri;                           // W_r, N = 128
                const uint32_t acc = (kw | h | kk) ? 1u : 0u;
                if (TCBF_ABLATE(args, 2)) continue;
                mma_f16_ss(d_re, xr, w_ri, I256, acc);      // [Re | Im] += X_r [W_r ; W_i]^T
                mma_f16_ss(d_re, xi, w_i, I128_NEG, 1u);    // Re += -X_i W_i^T
                mma_f16_ss(d_im, xi, w_r, I128, 1u);        // Im += X_i W_r^T
              }
              if (mt == mt1 - 1) mma_commit(&xempty[xs]);  // last reader of this data block
            }
            if (MC) mma_commit_mc(&wempty[stage]);  // the stage is free in both CTAs
            else mma_commit(&wempty[stage]);
            if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
          }
          mma_commit(&tfull[abuf]);
          if (args.trace) {
            stamp(args.trace, 4 * it + 1);
            stamp_val(args.trace, 512 + 4 * it, wwait);
            stamp_val(args.trace, 512 + 4 * it + 1, xwait);
          }
        }
      }
    }
  } else if (warp < 2 + EPI_WARPS) {
    // ------------------------------------------------------------ epilogue: coalesced line stores
    const int q = warp & 3;                 // TMEM lane quadrant = samples 32q..32q+31 of the tile
    const int half = (warp - 2) / 4;        // 8 warps: half 0 stores Re, half 1 Im
    constexpr int SPLIT = EPI_WARPS / 4;
    constexpr int MY_CHUNKS = 8 / SPLIT;    // 32-column chunks of the 256 accumulator columns
    const size_t N = (size_t)args.N;
    const int M = args.M;
    int it = 0;
    for (int i = 0; i < n_occ; ++i) {
      const int u = occ_unit(i);
      const int b = u / tiles_n;
      const int n = (u - b * tiles_n) * BS + q * 32 + lane;  // this thread's sample
      const bool n_ok = n < args.N;
      for (int mt = occ_mt0(i); mt < occ_mt1(i); ++mt, ++it) {
        const int abuf = it & 1;
        mbar_wait(&tfull[abuf], (it >> 1) & 1);
        tc_fence_after();
        if (threadIdx.x == 64) stamp(args.trace, 4 * it + 2);
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 2 * BB + half * (8 / SPLIT) * 32;
        uint32_t v[2][32];
        tmem_ld_32x32b_x32(tbase, v[0]);
#pragma unroll
        for (int c = 0; c < MY_CHUNKS; ++c) {
          const int ch = half * MY_CHUNKS + c;  // 0..3 Re, 4..7 Im
          const int part = ch >> 2;
          const int m0 = mt * BB + (ch & 3) * 32;
          tmem_wait_ld();
          if (c + 1 < MY_CHUNKS) {
            tmem_ld_32x32b_x32(tbase + (c + 1) * 32, v[(c + 1) & 1]);
          } else {  // all TMEM reads of this tile issued and complete: release the buffer
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[abuf]);
          }
          const uint32_t* vv = v[c & 1];
          if (TCBF_ABLATE(args, 1)) continue;
          if (n_ok) {
            float* dst = args.out + ((size_t)(2 * b + part) * M + m0) * N + n;
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
          if (warp == 2) stamp(args.trace, 4 * it + 3);
          if (warp == 1 + EPI_WARPS) stamp(args.trace, 512 + 4 * it + 2);
        }
      }
    }
  } else if (warp < SCfg<EPI_WARPS>::LOADER) {
    // ------------------------------------------------------------ converters: fp32 data -> scratch images
    const int ct = threadIdx.x - SCfg<EPI_WARPS>::CONV0 * 32;  // 0..255
    const int N = args.N;
    const int total = n_occ * num_kb;  // this CTA's data blocks, in walk order
    // block g of this CTA -> registers (zeros past the end, out-of-range k or n)
    auto load_block = [&](int g, XRegs& rg) {
      const int oi = g / num_kb, kb = g - oi * num_kb;
      const int u = occ_unit(oi);
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
    // block g (in registers) -> its fp16 slot image in the scratch (the exact smem layout)
    auto store_block = [&](int g, const XRegs& rg) {
      uint8_t* img = scratch + (g % num_kb) * X_SLOT;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int item = ct + i * CONV_THREADS;
        const int kr = item / (BS / 8), cc = item % (BS / 8);
        const int off = (cc >> 3) * X_HALF + kr * 128 + (((cc & 7) ^ (kr & 7)) << 4);
        *reinterpret_cast<uint4*>(img + off) = make_uint4(h2u(rg.re[i][0], rg.re[i][1]), h2u(rg.re[i][2], rg.re[i][3]),
                                                          h2u(rg.re[i][4], rg.re[i][5]), h2u(rg.re[i][6], rg.re[i][7]));
        *reinterpret_cast<uint4*>(img + X_PLANE + off) =
            make_uint4(h2u(rg.im[i][0], rg.im[i][1]), h2u(rg.im[i][2], rg.im[i][3]), h2u(rg.im[i][4], rg.im[i][5]),
                       h2u(rg.im[i][6], rg.im[i][7]));
      }
    };
    // the scratch holds one occurrence: its images may be rewritten once the previous occurrence's
    // images have all landed in smem; after the last block the loader is told they are ready
    auto begin_occ = [&](int oi) {
      if (oi == 0) return;
      for (int kb = 0; kb < num_kb; ++kb) {
        const int g = (oi - 1) * num_kb + kb;
        mbar_wait(&xfull[g % X_SLOTS], (g / X_SLOTS) & 1);
      }
    };
    auto end_occ = [&]() {
      __threadfence();             // the images are in L2 before the loader's TMA reads them
      fence_proxy_async_global();  // generic-proxy writes -> async-proxy (bulk copy) reads
      __syncwarp();
      if (lane == 0) mbar_arrive(sready);
    };
    // two blocks in flight ahead of the one being stored (register double buffer, unrolled by 2
    // so both buffers stay in registers); num_kb is even, so an occurrence starts on an even g
    XRegs ra, rb;
    load_block(0, ra);
    load_block(1, rb);
    for (int g = 0; g < total; g += 2) {
      if (g % num_kb == 0) begin_occ(g / num_kb);
      store_block(g, ra);
      load_block(g + 2, ra);
      store_block(g + 1, rb);
      load_block(g + 3, rb);
      if ((g + 2) % num_kb == 0) end_occ();
    }
  } else {
    // ------------------------------------------------------------ slot loader: scratch images -> smem slots
    if (lane == 0) {
      for (int i = 0; i < n_occ; ++i) {
        mbar_wait(sready, i & 1);
        for (int kb = 0; kb < num_kb; ++kb) {
          const int g = i * num_kb + kb, xs = g % X_SLOTS;
          mbar_wait(&xempty[xs], ((g / X_SLOTS) & 1) ^ 1);
          mbar_arrive_expect_tx(&xfull[xs], X_SLOT);
          bulk_load_g2s(sX + xs * X_SLOT, scratch + kb * X_SLOT, X_SLOT, &xfull[xs]);
        }
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

template <int LAYOUT, bool VEC, int EPI_WARPS, bool MC>
cudaError_t launch_smaj(const CUtensorMap& tmW, const GemmF16Args& a, const float* x, int K, int num_sms,
                        cudaStream_t s) {
  auto kern = cgemm_f16_smaj_kernel<LAYOUT, VEC, EPI_WARPS, MC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int units = a.B * a.tiles_n;
  if (!MC) {
    const int grid = units < num_sms ? units : num_sms;
    kern<<<grid, SCfg<EPI_WARPS>::NUM_THREADS, SMEM_BYTES, s>>>(tmW, a, x, K);
    return cudaGetLastError();
  }
  const int pairs = units / 2 < num_sms / 2 ? units / 2 : num_sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(SCfg<EPI_WARPS>::NUM_THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, tmW, a, x, K);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int EPI_WARPS, bool MC>
cudaError_t launch_smaj_layout(const CUtensorMap& tmW, const GemmF16Args& args, const float* x_src, int layout,
                               int K, int num_sms, cudaStream_t stream) {
  const bool vec = layout == 0 && (args.N % 8 == 0) && (reinterpret_cast<uintptr_t>(x_src) % 16 == 0);
  if (layout == 0)
    return vec ? launch_smaj<0, true, EPI_WARPS, MC>(tmW, args, x_src, K, num_sms, stream)
               : launch_smaj<0, false, EPI_WARPS, MC>(tmW, args, x_src, K, num_sms, stream);
  return launch_smaj<1, false, EPI_WARPS, MC>(tmW, args, x_src, K, num_sms, stream);
}

}  // namespace

bool gemm_f16_smaj_supported(int64_t K16) { return K16 <= KMAX; }
size_t gemm_f16_smaj_scratch_bytes(int num_sms) { return (size_t)num_sms * X_SLOTS * X_SLOT; }

// args: tiles_m = beam tiles (128), tiles_n = sample tiles (128), K16 = padded K (multiple of 64),
// xscratch = gemm_f16_smaj_scratch_bytes(num_sms) bytes of device memory (one unit of fp16 slot
// images per CTA); weights tensor map: box {64 K, 128 beams} per plane, 128-byte swizzle
cudaError_t launch_gemm_f16_smaj(const CUtensorMap& tmW, const GemmF16Args& args, const float* x_src, int layout,
                                 int K, int epi_warps, bool multicast, int num_sms, cudaStream_t stream) {
  if (args.xscratch == nullptr) return cudaErrorInvalidValue;
  // weight multicast across CTA pairs needs pairs of units of one batch entry (tiles_n even)
  const bool mc = multicast && args.tiles_n % 2 == 0 && args.B * args.tiles_n >= 2;
  if (epi_warps == 4)
    return mc ? launch_smaj_layout<4, true>(tmW, args, x_src, layout, K, num_sms, stream)
              : launch_smaj_layout<4, false>(tmW, args, x_src, layout, K, num_sms, stream);
  return mc ? launch_smaj_layout<8, true>(tmW, args, x_src, layout, K, num_sms, stream)
            : launch_smaj_layout<8, false>(tmW, args, x_src, layout, K, num_sms, stream);
}

}  // namespace tcbf
