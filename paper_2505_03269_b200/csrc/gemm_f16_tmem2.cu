// gemm_f16_tmem2.cu -- the data-in-TMEM radio kernel (gemm_f16_tmem.cu) with 32-beam tiles, so
// that half of the NEXT unit's data fits in tensor memory too: K16 = 256 only.
//
// Same arithmetic and roles as gemm_f16_tmem.cu (see there).  TMEM: three 128-column data regions
// (each two 64-K blocks: X_r 64 columns, X_i 64) and two 64-column accumulators [Re 32 | Im 32].
// The running unit occupies two regions (blocks 0-1 in `lo`, 2-3 in `hi`); the converters write
// the next unit's blocks 0-1 straight into the third region (tcgen05.st) and stage only blocks 2-3
// in shared memory (64 KB instead of 128), copied into the running unit's `lo` region once its last
// beam tile has read it.  Regions rotate (lo, hi, free) -> (free, lo, hi).  The 64 KB of staging
// this frees go to the weight ring: 128 KB, 16 K blocks of 32 beams, two tiles ahead, where the
// 64-beam kernel's 64 KB ring starved the MMA issuer (~0.6 us of waiting per tile).  Per K step:
// [Re | Im] += X_r [W_r ; W_i]^T (N = 64) and two N = 32 MMAs (Re += X_i (-W_i)^T, Im += X_i W_r^T):
// peaks.cu kind 14 runs that pattern at the full fp16 rate.
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int UN = 128;                     // samples per unit (MMA M, TMEM lanes)
constexpr int BNB = 32;                     // beams per tile
constexpr int BK = 64;                      // K per data block / per 128-byte weight row
constexpr int KMAX = 256;                   // K16 (four 64-K blocks)
constexpr int W_PLANE = BNB * BK * 2;       // 4 KB: 32 beams x 128 B
constexpr int W_ATOM = 2 * W_PLANE;         // [W_r ; W_i] for one K block (the stacked N=64 operand)
constexpr int EPI_WARPS = 8;
constexpr int CONV_WARPS = 8;
constexpr int CONV0 = 2 + EPI_WARPS;
constexpr int RAW_WARP = CONV0 + CONV_WARPS;
constexpr int SYNC_WARP = RAW_WARP + 1;  // waits on the MMA issuer's barriers for it
constexpr int NUM_THREADS = (SYNC_WARP + 1) * 32;
constexpr int NB_STAGE0 = 2;             // named barriers 2.. : weight stage s ready (sync warp -> MMA warp)
constexpr int RAW_ROWS = 16;                     // k-rows per raw data box (two 8-row halves)
constexpr int RAW_BYTES = RAW_ROWS * UN * 8;     // 16 rows x 128 complex samples: 16 KB
constexpr int RAW_SLOTS = 2;
constexpr int STG_BLOCK = 2 * 8 * UN * 16;      // staged fp16 of one 64-K block: [plane][k group of 8][sample] x 16 B
constexpr int OFF_STG = 0;
constexpr int STG_BLOCKS = 2;                   // blocks 2-3 of the next unit
constexpr int OFF_W = STG_BLOCKS * STG_BLOCK;    // 64 KB of staging
constexpr int W_BYTES = 224 * 1024 - OFF_W - RAW_SLOTS * RAW_BYTES;  // weight ring: the rest (128 KB)
constexpr int OFF_RAW = OFF_W + W_BYTES;
constexpr int BAR_OFFSET = OFF_RAW + RAW_SLOTS * RAW_BYTES;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 512;
constexpr uint32_t REG_COLS = 128;           // data regions at 0, 128, 256: block j X_r at 32 j, X_i at 64 + 32 j
constexpr uint32_t ACC_COL = 384;            // accumulators [384,448), [448,512)
// region of the unit with per-CTA index ui: blocks 0-1 (lo) and 2-3 (hi); rotation (lo, hi, free)
__device__ __forceinline__ uint32_t reg_lo(int ui) { return (uint32_t)((3 - ui % 3) % 3); }
__device__ __forceinline__ uint32_t reg_hi(int ui) { return (uint32_t)((3 - (ui + 2) % 3) % 3); }
static_assert(SMEM_BYTES <= 232448, "smem budget");
static_assert(NB_STAGE0 + W_BYTES / (2 * W_ATOM) <= 16, "named barriers: one per weight stage");

// D[tmem] (+)= A[tmem] . B[smem]^T, kind::f16
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x4(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// K-major weights (B operand): 128-byte swizzle, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t desc_w(const void* tile) {
  uint64_t d = (uint64_t)((smem_u32(tile) >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// kind::f16: fp16 A/B, fp32 D, A from TMEM, B K-major, M = 128; bit 14 negates B
__host__ __device__ constexpr uint32_t idesc_t(uint32_t N, bool negate_b) {
  return (1u << 4) | ((negate_b ? 1u : 0u) << 14) | ((N >> 3) << 17) | ((uint32_t)(UN >> 4) << 24);
}

__device__ __forceinline__ uint32_t h2u(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// LAYOUT: 0 interleaved fp32 source [B][K][N] x (re, im), 1 planar [B][2][K][N], 2 interleaved fp16
// [B][K][N] x (re, im) (tcbf_beamform_f16i: NEXT-1, no rounding on the way in); WKB: K blocks per
// weight stage (64 KB of weight ring: 4 / WKB stages)
// CL = 2: CTA pairs (clusters) take adjacent units of one batch entry and walk the same weight
// stages; each CTA TMA-loads one plane of a stage and multicasts it into both (half the L2 -> SM
// weight reads), a stage is refilled once the MMAs of both CTAs have retired it
template <int LAYOUT, int WKB, int CL>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_tmem2_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                          GemmF16Args args) {
  constexpr int W_STAGE = WKB * W_ATOM;
  constexpr int W_STAGES = W_BYTES / W_STAGE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sStg = smem + OFF_STG;
  uint8_t* sW = smem + OFF_W;
  uint8_t* sRaw = smem + OFF_RAW;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* wempty = wfull + W_STAGES;
  uint64_t* xfull = wempty + W_STAGES;   // [unit parity][block]: the unit's block is in TMEM
  uint64_t* xempty = xfull + 8;          // [unit parity][block]: the unit's last tile has read it
  uint64_t* tfull = xempty + 8;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;          // [RAW_SLOTS]: raw fp32 box landed
  uint64_t* rempty = rfull + RAW_SLOTS;  // [RAW_SLOTS]: converters have read it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty + RAW_SLOTS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr bool MC = CL > 1;
  const int rank = MC ? (int)cluster_ctarank() : 0;
  const int u_first = MC ? CL * (int)(blockIdx.x / CL) + rank : (int)blockIdx.x;
  const int u_step = MC ? CL * (int)(gridDim.x / CL) : (int)gridDim.x;
  const int num_kb = args.num_kb;    // K16 / 64 <= 4
  const int num_ws = (num_kb + WKB - 1) / WKB;  // weight stages per tile
  const int tiles_m = args.tiles_m;  // 64-beam tiles
  const int tiles_n = args.tiles_n;  // 128-sample units per batch entry
  const int num_units = args.B * tiles_n;
  const int M = args.M, N = args.N;
  const int nraw = args.K16 / RAW_ROWS;  // raw boxes per unit

  if (threadIdx.x == 0) {
    for (int s = 0; s < W_STAGES; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], CL);
    }
    for (int s = 0; s < 8; ++s) {
      mbar_init(&xfull[s], CONV_WARPS);  // every converter warp writes part of each block
      mbar_init(&xempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPI_WARPS);
    }
    for (int s = 0; s < RAW_SLOTS; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], CONV_WARPS);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  if (MC) cluster_sync(); else __syncthreads();  // the peer signals this CTA's barriers
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer: weight stages of
    // WKB K blocks, each block's [W_r ; W_i] contiguous (the stacked N = 64 operand)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = u_first; u < num_units; u += u_step) {
        const int b = u / tiles_n;
        for (int mt = 0; mt < tiles_m; ++mt) {
          for (int ws = 0; ws < num_ws; ++ws) {
            mbar_wait(&wempty[stage], phase ^ 1);
            uint8_t* st = sW + stage * W_STAGE;
            const int nkb = (num_kb - ws * WKB) < WKB ? (num_kb - ws * WKB) : WKB;
            if (TCBF_ABLATE(args, 8) && mt > 0) {  // ablation: weights once per unit (wrong values)
              mbar_arrive(&wfull[stage]);
              if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
              continue;
            }
            mbar_arrive_expect_tx(&wfull[stage], nkb * W_ATOM);
            for (int j = 0; j < nkb; ++j) {
              const int kb = ws * WKB + j;
              if (MC) {  // this CTA's plane of the pair's shared stage, into both CTAs
                tma_load_3d_mc(st + j * W_ATOM + rank * W_PLANE, &tmW, &wfull[stage], kb * BK, mt * BNB,
                               2 * b + rank, (uint16_t)((1u << CL) - 1u));
                continue;
              }
              tma_load_3d(st + j * W_ATOM, &tmW, &wfull[stage], kb * BK, mt * BNB, 2 * b);
              tma_load_3d(st + j * W_ATOM + W_PLANE, &tmW, &wfull[stage], kb * BK, mt * BNB, 2 * b + 1);
            }
            if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (converged warp, one
    // elected lane issues)
    constexpr uint32_t IWW = idesc_t(2 * BNB, false);
    constexpr uint32_t IW = idesc_t(BNB, false);
    constexpr uint32_t IW_NEGB = idesc_t(BNB, true);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0, ui = 0;
    for (int u = u_first; u < num_units; u += u_step, ++ui) {
      const uint32_t reg0 = tmem_base + reg_lo(ui) * REG_COLS, reg1 = tmem_base + reg_hi(ui) * REG_COLS;
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int abuf = it & 1;
        unsigned long long* const trace = it < 128 ? args.trace : nullptr;  // dev timeline (tools/trace_smaj.py)
        const unsigned long long tw0 = trace ? gtimer() : 0;
        unsigned long long wwait = 0, xwait = 0;
        if (trace && lane == 0) {
          stamp(trace, 4 * it);
          stamp_val(trace, 512 + 4 * it + 3, gtimer() - tw0);
        }
        const uint32_t d_re = tmem_base + ACC_COL + abuf * 2 * BNB;  // [Re | Im]: 64 columns
        const uint32_t d_im = d_re + BNB;
        for (int ws = 0; ws < num_ws; ++ws) {
          const int nkb = (num_kb - ws * WKB) < WKB ? (num_kb - ws * WKB) : WKB;
          // one named-barrier sync per stage: the sync warp has seen this stage's weights, and for a
          // tile's first stage the free accumulator buffer and (first tile of a unit) the data blocks
          // in TMEM (an mbarrier wait in this issue stream costs the tensor pipe a ~300-cycle bubble
          // even when the barrier is complete)
          const unsigned long long a0 = trace ? gtimer() : 0;
          asm volatile("bar.sync %0, 64;" ::"r"(NB_STAGE0 + stage) : "memory");
          tc_fence_after();  // the accumulator released by the epilogue, the data written by tcgen05.st
          if (trace) wwait += gtimer() - a0;
          const uint8_t* st = sW + stage * W_STAGE;
          const uint64_t w0 = desc_w(st);
          if (elect_one()) {
            for (int j = 0; j < nkb; ++j) {
              const int kb = ws * WKB + j;
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                // 16 K: 8 TMEM columns of the data, 32 B of the K-major weights (+2)
                const uint32_t xr = (kb < 2 ? reg0 : reg1) + (uint32_t)((kb & 1) * 32 + kk * 8);
                const uint32_t xi = xr + 64;
                const uint64_t wri = w0 + (uint64_t)((j * W_ATOM) >> 4) + (uint64_t)(2 * kk);  // [W_r ; W_i]
                const uint64_t wi = wri + (uint64_t)(W_PLANE >> 4);                               // W_i
                const uint32_t acc = (kb | kk) ? 1u : 0u;
                if (TCBF_ABLATE(args, 2)) continue;
                mma_f16_ts(d_re, xr, wri, IWW, acc);     // [Re | Im] += X_r [W_r ; W_i]^T
                mma_f16_ts(d_re, xi, wi, IW_NEGB, 1u);   // Re += X_i (-W_i)^T
                mma_f16_ts(d_im, xi, wri, IW, 1u);       // Im += X_i W_r^T
              }
            }
            if (MC) mma_commit_mc(&wempty[stage], (uint16_t)((1u << CL) - 1u));  // free in both CTAs
            else mma_commit(&wempty[stage]);
            if (mt == tiles_m - 1)
              for (int j = 0; j < nkb; ++j) mma_commit(&xempty[(ui & 1) * 4 + ws * WKB + j]);  // last reader
          }
          __syncwarp();
          if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit(&tfull[abuf]);
        __syncwarp();
        if (trace && lane == 0) {
          stamp(trace, 4 * it + 1);
          stamp_val(trace, 512 + 4 * it, wwait);
          stamp_val(trace, 512 + 4 * it + 1, xwait);
        }
      }
    }
  } else if (warp < CONV0) {
    // ------------------------------------------------------------ epilogue: coalesced line stores
    const int q = warp & 3;           // TMEM lane quadrant = samples 32q..32q+31 of the unit
    const int half = (warp - 2) / 4;  // half 0 stores Re, half 1 Im
    int it = 0;
    for (int u = u_first; u < num_units; u += u_step) {
      const int b = u / tiles_n;
      const int n = (u - b * tiles_n) * UN + q * 32 + lane;  // this thread's sample
      const bool n_ok = n < N;
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int abuf = it & 1;
        mbar_wait(&tfull[abuf], (it >> 1) & 1);
        tc_fence_after();
        unsigned long long* const trace = it < 128 ? args.trace : nullptr;
        if (threadIdx.x == 64) stamp(trace, 4 * it + 2);
        const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + ACC_COL + abuf * 2 * BNB + half * BNB;
        uint32_t v[32];
        const bool no_ld = TCBF_ABLATE(args, 16);  // ablation: no TMEM reads (stores of garbage)
        if (!no_ld) {
          tmem_ld_32x32b_x32(tb, v);
          tmem_wait_ld();
        }
        tc_fence_before();  // all TMEM reads of this tile complete: release the buffer
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[abuf]);
        const int mb = mt * BNB;
        if (n_ok && !TCBF_ABLATE(args, 1)) {
          float* col = args.out + ((size_t)(2 * b + half) * M + mb) * (size_t)N + n;
          if (mb + 32 <= M) {
#pragma unroll
            for (int j = 0; j < 32; ++j) col[(size_t)j * N] = __uint_as_float(v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (mb + j < M) col[(size_t)j * N] = __uint_as_float(v[j]);
          }
        }
        if (trace && lane == 0) {
          if (warp == 2) stamp(trace, 4 * it + 3);
          if (warp == 1 + EPI_WARPS) stamp(trace, 512 + 4 * it + 2);
        }
      }
    }
  } else if (warp < RAW_WARP) {
    // ------------------------------------------------------------ converters: a unit's raw fp32
    // boxes -> fp16 while the previous unit runs in TMEM: blocks 0-1 straight into the free TMEM
    // region, blocks 2-3 into the staging, copied into the previous unit's `lo` region once its
    // last tile has read it.  Thread (quadrant q, lane) converts sample s = 32 q + lane (the TMEM
    // lane its warp may access) and k groups 2 r + ch of each box r
    const int q = warp & 3;
    const int s = q * 32 + lane;
    const int ch = (warp - CONV0) >> 2;     // conversion: 8-row half of each box; copy: K half of a block
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
    uint4* const stg = reinterpret_cast<uint4*>(sStg);  // [kb - 2][plane][k group of 8][sample]
    int rs = 0;
    uint32_t rphase = 0;
    int ui = 0;
    for (int u = u_first; u < num_units; u += u_step, ++ui) {
      // the free region is the `hi` region of unit ui - 2: wait for its blocks 2-3 to be read
      if (ui >= 2) {
        const int up = ui - 2;
        mbar_wait(&xempty[(up & 1) * 4 + 2], (up >> 1) & 1);
        mbar_wait(&xempty[(up & 1) * 4 + 3], (up >> 1) & 1);
        tc_fence_after();
      }
      const uint32_t lo = lane_base + reg_lo(ui) * REG_COLS, hi = lane_base + reg_hi(ui) * REG_COLS;
      // 1) convert: box r holds k-rows 16 r ..; this thread's 8 rows = k group 2 r + ch
      for (int r = 0; r < nraw; ++r) {
        mbar_wait(&rfull[rs], rphase);
        uint4 pre, pim;  // this thread's 8 k-values of X_r and X_i as fp16
        if (LAYOUT == 2) {  // fp16 (re, im) pairs: de-interleave with byte permutes, no rounding
          const uint32_t* raw = reinterpret_cast<const uint32_t*>(sRaw + rs * RAW_BYTES);
          uint32_t v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = raw[(ch * 8 + j) * UN + s];
          pre = make_uint4(__byte_perm(v[0], v[1], 0x5410), __byte_perm(v[2], v[3], 0x5410),
                           __byte_perm(v[4], v[5], 0x5410), __byte_perm(v[6], v[7], 0x5410));
          pim = make_uint4(__byte_perm(v[0], v[1], 0x7632), __byte_perm(v[2], v[3], 0x7632),
                           __byte_perm(v[4], v[5], 0x7632), __byte_perm(v[6], v[7], 0x7632));
        } else {
          const float* raw = reinterpret_cast<const float*>(sRaw + rs * RAW_BYTES);
          float re[8], im[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int row = ch * 8 + j;
            if (LAYOUT == 0) {
              const float2 f = reinterpret_cast<const float2*>(raw)[row * UN + s];
              re[j] = f.x; im[j] = f.y;
            } else {
              re[j] = raw[row * UN + s];
              im[j] = raw[(RAW_ROWS + row) * UN + s];
            }
          }
          pre = make_uint4(h2u(re[0], re[1]), h2u(re[2], re[3]), h2u(re[4], re[5]), h2u(re[6], re[7]));
          pim = make_uint4(h2u(im[0], im[1]), h2u(im[2], im[3]), h2u(im[4], im[5]), h2u(im[6], im[7]));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&rempty[rs]);
        if (++rs == RAW_SLOTS) { rs = 0; rphase ^= 1; }
        if (TCBF_ABLATE(args, 4)) pre = pim = make_uint4(0u, 0u, 0u, 0u);  // ablation: data ignored (timing)
        const int g = 2 * r + ch;  // global k group (8 rows)
        const int kb = g >> 3;
        if (kb < 2) {  // 4 columns (8 k-values) of X_r and of X_i in the free region
          const uint32_t ta = lo + (uint32_t)((kb & 1) * 32 + (g & 7) * 4);
          const uint32_t vr[4] = {pre.x, pre.y, pre.z, pre.w}, vi[4] = {pim.x, pim.y, pim.z, pim.w};
          tmem_st_32x32b_x4(ta, vr);
          tmem_st_32x32b_x4(ta + 64, vi);
          if ((r & 3) == 3) {  // the block's last box: this warp's part of it is written
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&xfull[(ui & 1) * 4 + kb]);
          }
        } else {
          stg[(((kb - 2) * 2 + 0) * 8 + (g & 7)) * UN + s] = pre;
          stg[(((kb - 2) * 2 + 1) * 8 + (g & 7)) * UN + s] = pim;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(CONV_WARPS * 32) : "memory");  // staging complete
      // 2) at the switch: blocks 2-3 into the previous unit's `lo` region once its last tile read it
      if (ui >= 1) {
        const int up = ui - 1;
        mbar_wait(&xempty[(up & 1) * 4 + 0], (up >> 1) & 1);
        mbar_wait(&xempty[(up & 1) * 4 + 1], (up >> 1) & 1);
        tc_fence_after();
      }
      for (int kb = 2; kb < 4; ++kb) {
        uint32_t pr[16], pi[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint4 r4 = stg[(((kb - 2) * 2 + 0) * 8 + 4 * ch + c) * UN + s];
          const uint4 i4 = stg[(((kb - 2) * 2 + 1) * 8 + 4 * ch + c) * UN + s];
          pr[4 * c] = r4.x; pr[4 * c + 1] = r4.y; pr[4 * c + 2] = r4.z; pr[4 * c + 3] = r4.w;
          pi[4 * c] = i4.x; pi[4 * c + 1] = i4.y; pi[4 * c + 2] = i4.z; pi[4 * c + 3] = i4.w;
        }
        const uint32_t ta = hi + (uint32_t)((kb & 1) * 32 + ch * 16);
        tmem_st_32x32b_x16(ta, pr);
        tmem_st_32x32b_x16(ta + 64, pi);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&xfull[(ui & 1) * 4 + kb]);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(CONV_WARPS * 32) : "memory");  // staging read: reusable
    }
  } else if (warp == SYNC_WARP) {
    // ------------------------------------------------------------ sync warp: the MMA issuer's mbarrier
    // waits (each a bubble in its tensor-pipe issue stream), passed on by one named barrier per stage
    int stage = 0;
    uint32_t phase = 0;
    int it = 0, ui = 0;
    for (int u = u_first; u < num_units; u += u_step, ++ui) {
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        for (int ws = 0; ws < num_ws; ++ws) {
          const int nkb = (num_kb - ws * WKB) < WKB ? (num_kb - ws * WKB) : WKB;
          if (ws == 0) mbar_wait(&tempty[it & 1], ((it >> 1) & 1) ^ 1);
          if (mt == 0)
            for (int j = 0; j < nkb; ++j) mbar_wait(&xfull[(ui & 1) * 4 + ws * WKB + j], (ui >> 1) & 1);
          mbar_wait(&wfull[stage], phase);
          asm volatile("bar.arrive %0, 64;" ::"r"(NB_STAGE0 + stage) : "memory");
          if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ TMA producer: raw fp32 data boxes
    // (16 k-rows x 128 samples; rows >= K and samples >= N are zero-filled)
    if (lane == 0) {
      int rs = 0;
      uint32_t rphase = 0;
      for (int u = u_first; u < num_units; u += u_step) {
        const int b = u / tiles_n;
        const int n0 = (u - b * tiles_n) * UN;
        for (int r = 0; r < nraw; ++r) {
          mbar_wait(&rempty[rs], rphase ^ 1);
          uint8_t* dst = sRaw + rs * RAW_BYTES;
          mbar_arrive_expect_tx(&rfull[rs], LAYOUT == 2 ? RAW_BYTES / 2 : RAW_BYTES);
          if (LAYOUT == 2) {  // fp16 (re, im) pairs as 32-bit elements {N, K, B}
            tma_load_3d(dst, &tmX, &rfull[rs], n0, r * RAW_ROWS, b);
          } else if (LAYOUT == 0) {
            tma_load_3d(dst, &tmX, &rfull[rs], 2 * n0, r * RAW_ROWS, b);
          } else {
            tma_load_3d(dst, &tmX, &rfull[rs], n0, r * RAW_ROWS, 2 * b);
            tma_load_3d(dst + RAW_BYTES / 2, &tmX, &rfull[rs], n0, r * RAW_ROWS, 2 * b + 1);
          }
          if (++rs == RAW_SLOTS) { rs = 0; rphase ^= 1; }
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

}  // namespace

bool gemm_f16_tmem2_supported(int64_t K16) { return K16 == KMAX; }
int gemm_f16_tmem2_beams() { return BNB; }

// args: tiles_m = 32-beam tiles, tiles_n = 128-sample units per batch entry, num_kb = 4;
// weights tensor map: box {64 K, 32 beam rows} per plane, 128-byte swizzle; data tensor map as
// gemm_f16_tmem.cu
template <int LAYOUT, int WKB, int CL>
cudaError_t launch_tmem2(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmF16Args& args, int num_sms,
                         cudaStream_t stream) {
  auto kern = cgemm_f16_tmem2_kernel<LAYOUT, WKB, CL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int units = args.B * args.tiles_n;
  int grid = units < num_sms ? units : num_sms;
  if (CL == 1) {
    kern<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(tmW, tmX, args);
    return cudaGetLastError();
  }
  grid = grid / CL * CL;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, tmW, tmX, args);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// cluster 2 (weight multicast) needs an even number of units per batch entry and at least two;
// WKB 2 (8 stages of 32 beams x 128 K) or 4
cudaError_t launch_gemm_f16_tmem2(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmF16Args& args,
                                  int layout, int wkb, int cluster, int num_sms, cudaStream_t stream) {
  if (args.num_kb != 4) return cudaErrorInvalidValue;
  const bool pair = cluster >= 2 && args.tiles_n % 2 == 0 && args.B * args.tiles_n >= 2;
#define TCBF_TMEM2_LAUNCH(L, W) \
  return pair ? launch_tmem2<L, W, 2>(tmW, tmX, args, num_sms, stream) : launch_tmem2<L, W, 1>(tmW, tmX, args, num_sms, stream)
  if (layout == 0) {
    if (wkb == 4) TCBF_TMEM2_LAUNCH(0, 4);
    TCBF_TMEM2_LAUNCH(0, 2);
  }
  if (layout == 2) {
    if (wkb == 4) TCBF_TMEM2_LAUNCH(2, 4);
    TCBF_TMEM2_LAUNCH(2, 2);
  }
  if (wkb == 4) TCBF_TMEM2_LAUNCH(1, 4);
  TCBF_TMEM2_LAUNCH(1, 2);
#undef TCBF_TMEM2_LAUNCH
}

}  // namespace tcbf
