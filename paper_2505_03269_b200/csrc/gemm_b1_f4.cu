// gemm_b1_f4.cu -- 1-bit-mode complex beamformer GEMM on the fp4 tensor cores (kind::mxf4).
//
// The 1-bit encoding (bit 1 = +1, bit 0 = -1, one bit per component; Fig. 1
// PAPER.md:209-210) is expanded IN SHARED MEMORY to the values +-1 in fp4 e2m1 (0x2 = +1.0,
// 0xA = -1.0), two K elements per byte: nibble i of output word j holds bit (4i + j) of a
// packed word -- a fixed permutation of the 32 K-elements of a word, applied identically to both
// operands, so every dot product is unchanged.  tcgen05.mma.kind::mxf4.block_scale with unit
// block scales (UE8M0 127 = 2^0, written once into TMEM) then forms the products; one MMA of
// N = 256 covers both accumulators [D_r | D_i] against two stacked data tiles:
//     [D_r | D_i] += A_r [B_r ; B_i]          [D_r | D_i] += A_i [-B_i ; B_r]
// i.e. the paper's five steps with Im(b) negated during expansion (the
// block-scaled kinds have no negate bit).  Products are +-1 and every partial sum is an integer
// of magnitude <= 2 K_tot < 2^24, so the fp32 accumulation is exact (K_tot <= 2^23).
// Padding bits are 0 and expand to -1 in both operands: they add 0 to Re and 2 per
// padded position to Im, so Re = D_r, Im = D_i - 2 K_pad (the paper's Eq. 5 Im correction).
//
// Against the int8 kernel this halves both the expanded bytes written and the operand bytes the
// MMAs read per useful op, and runs at the fp4 rate (2x int8).
//
// Data movement per 256-bit K block of a 128 x 128 tile:
//   TMA      packed words of A_r, A_i, B_r, B_i (4 x 128 rows x 32 B, zero-filled out of range)
//            -> 2-deep packed ring (measured: per-thread look-ahead loads were L1-miss bound)
//   expand   each thread its row: 32 B per plane -> 128 B of nibbles, 128-byte swizzle, into the
//            2-deep expanded ring (A_r, A_i, -B_i, B_r, B_i tiles of 16 KB)
//   MMA      8 x (M=128, N=256, K=64) per K block
// TMEM (512 columns): one accumulator tile [D_r | D_i] (256 columns) + the scale factors (columns
// of 0x7F bytes -- every byte the MMA may read as a scale is 2^0, whatever its layout).
// With a single accumulator buffer the next tile's MMAs wait for the 8 epilogue warps' TMEM reads.
//
// Default (ATMEM): the expanded WEIGHT tiles A_r, A_i are written by their expander threads
// straight into TMEM (tcgen05.st, lane = weight row, 8 nibbles per column, logical K order) and
// the MMAs read A from TMEM (columns 256 + 64 s, three stages), scale factors in 448..511.  The
// kernel is shared-memory-bandwidth bound (expansion writes + MMA operand reads):
// moving A out of smem removes 2 of the 5 expanded tiles and a third of the MMA operand reads, and
// the freed 64 KB hold a third stage (square 8192^3: 0.82 -> 0.70 ms).
//
// Roles (persistent CTA per SM, 576 threads):
//   warp 0      TMEM allocator + single-thread MMA issuer
//   warps 1-8   epilogue: tcgen05.ld, fp32 -> int32, Im - 2 K_pad, TMA store of int32 (32 x 16 boxes)
//   warps 9-12  expanders for A_r, A_i (one weight row per thread)
//   warps 13-16 expanders for B_r, B_i, -B_i (one data column per thread)
//   warp 17     TMA producer of the packed words
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int KBW = 8;                 // 256 bits per K block -> 128 bytes of nibbles per row
constexpr int TILE_BYTES = 128 * 128;  // one expanded operand tile (rows x 128 B)
constexpr int STAGES = 2;
constexpr int ATMEM_STAGES = 3;  // the smem the TMEM-resident weights free holds a third stage
constexpr int STAGE_BYTES = 5 * TILE_BYTES;  // A_r, A_i, -B_i, B_r, B_i
constexpr int PLANE_BYTES = 128 * KBW * 4;   // packed words of one plane: 128 rows x 32 B
constexpr int P_STAGE_BYTES = 4 * PLANE_BYTES;  // A_r, A_i, B_r, B_i
constexpr int EPI_WARPS = 8;
constexpr int EXP_WARP0 = 1 + EPI_WARPS;
constexpr int EXPANDER_WARPS = 8;
constexpr int PRODUCER_WARP = EXP_WARP0 + EXPANDER_WARPS;
constexpr int NUM_THREADS = (PRODUCER_WARP + 1) * 32;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t SF_COL = 256;  // scale factors: columns 256..511

// Two ways to bring the packed words in, sharing everything else:
//   TMA_WORDS  a TMA producer fills a 2-deep ring of packed tiles (long K: measured 1.07 -> 0.81 ms
//              on 8192^3); the output is staged in 32-row x 16-column boxes (2 per warp, 32 KB)
//   otherwise  each expander thread loads its row's words two K blocks ahead (short K, store-bound
//              radio shape: the 64 KB of 32 x 32 output boxes it leaves room for measured faster)
// ATMEM: the expanded weights (A_r, A_i) go to TENSOR memory (tcgen05.st from the expander
// registers) and the MMAs read A from TMEM; only the three data tiles stay in shared memory
// (~30% less smem traffic per K block).  TMEM: [D_r | D_i] 0..255, A stages 256 + 64 s, scale
// factors in the remaining columns.
// Short K (register look-ahead words, the store-bound radio shape): the epilogue stages a warp's
// WHOLE 32 x 128 output block (four 32 x 32 boxes, 16 KB) before one wait per tile, so the single
// TMEM accumulator is released as soon as it is read, not after each box's TMA store has drained;
// the 128 KB of staging this needs leaves room for two expanded stages (enough for K <= 1024).
template <bool TMA_WORDS, bool ATMEM = false>
struct Cfg {
  static constexpr int STAGE = ATMEM ? 3 * TILE_BYTES : STAGE_BYTES;  // smem bytes per stage
  static constexpr int NST = ATMEM ? (TMA_WORDS ? ATMEM_STAGES : 2) : STAGES;  // expanded-operand stages
  static constexpr int BOFF = ATMEM ? 0 : 2 * TILE_BYTES;             // -B_i, B_r, B_i tiles
  static constexpr uint32_t A_COL = 256;
  static constexpr uint32_t SFC = ATMEM ? A_COL + 64 * NST : SF_COL;
  static constexpr uint32_t SFB_OFF = ATMEM ? 32 : 128;
  static constexpr int P_STAGES = TMA_WORDS ? 2 : 0;
  static constexpr int BOX_COLS = TMA_WORDS ? 16 : 32;
  static constexpr int EPI_BOX = 32 * BOX_COLS * 4;
  static constexpr int EPI_BOXES = TMA_WORDS ? 2 : BN / BOX_COLS;  // per warp: double buffer / whole row
  static constexpr int EPI_BYTES = EPI_WARPS * EPI_BOXES * EPI_BOX;
  static constexpr int P_OFFSET = NST * STAGE;
  static constexpr int EPI_OFFSET = P_OFFSET + P_STAGES * P_STAGE_BYTES;
  static constexpr int BAR_OFFSET = EPI_OFFSET + EPI_BYTES;
  static constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
  static_assert(SMEM_BYTES <= 232448, "smem budget");
};
constexpr int REG_PF = 2;  // K blocks of register look-ahead (measured: 2 > 1 > 3, 4)

// output word j (4 per packed word) of the +-1 e2m1 expansion: nibble i <- bit (4i + j)
template <int J>
__device__ __forceinline__ uint32_t nib_pm1(uint32_t w) {
  return ((w << (3 - J)) & 0x88888888u) ^ 0xAAAAAAAAu;  // bit 1 -> 0x2 (+1), bit 0 -> 0xA (-1)
}
template <int J>
__device__ __forceinline__ uint32_t nib_neg(uint32_t w) {
  return ((w << (3 - J)) & 0x88888888u) ^ 0x22222222u;  // bit 1 -> 0xA (-1), bit 0 -> 0x2 (+1)
}

__device__ __forceinline__ void put(uint8_t* row_base, int row, int q, uint4 v) {
  *reinterpret_cast<uint4*>(row_base + ((q ^ (row & 7)) << 4)) = v;  // 128-byte swizzle
}
__device__ __forceinline__ void expand(uint8_t* row_base, int row, const uint4& lo, const uint4& hi) {
  const uint32_t w[KBW] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
  for (int q = 0; q < KBW; ++q)
    put(row_base, row, q, make_uint4(nib_pm1<0>(w[q]), nib_pm1<1>(w[q]), nib_pm1<2>(w[q]), nib_pm1<3>(w[q])));
}
__device__ __forceinline__ void expand_pair(uint8_t* pos_base, uint8_t* neg_base, int row, const uint4& lo,
                                            const uint4& hi) {
  const uint32_t w[KBW] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
  for (int q = 0; q < KBW; ++q) {
    put(pos_base, row, q, make_uint4(nib_pm1<0>(w[q]), nib_pm1<1>(w[q]), nib_pm1<2>(w[q]), nib_pm1<3>(w[q])));
    put(neg_base, row, q, make_uint4(nib_neg<0>(w[q]), nib_neg<1>(w[q]), nib_neg<2>(w[q]), nib_neg<3>(w[q])));
  }
}

__device__ __forceinline__ void mma_mxf4(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
      : "memory");
}

__device__ __forceinline__ void tmem_st_32x32b_x32_same(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
      "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
      "r"(v)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void mma_mxf4_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                            uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%6], p;\n\t}" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
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
// the 32 e2m1 words of one row's 256-bit K block in logical (unswizzled) order -> TMEM columns,
// in two 16-column halves (keeps 16 instead of 32 expanded words live: the 576-thread CTA gets
// 96 registers per thread)
__device__ __forceinline__ void expand_tmem(uint32_t taddr, const uint4& lo, const uint4& hi) {
  const uint32_t w[KBW] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t v[16];
#pragma unroll
    for (int q = 0; q < KBW / 2; ++q) {
      v[4 * q] = nib_pm1<0>(w[4 * h + q]);
      v[4 * q + 1] = nib_pm1<1>(w[4 * h + q]);
      v[4 * q + 2] = nib_pm1<2>(w[4 * h + q]);
      v[4 * q + 3] = nib_pm1<3>(w[4 * h + q]);
    }
    tmem_st_32x32b_x16(taddr + 16 * h, v);
  }
}

template <bool TMA_STORE, bool TMA_WORDS, bool ATMEM>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_b1_f4_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                       const __grid_constant__ CUtensorMap tmC, GemmB1Args p, int tiles_m, int tiles_n,
                       int num_tiles) {
  using C = Cfg<TMA_WORDS, ATMEM>;
  constexpr int P_STAGES = C::P_STAGES > 0 ? C::P_STAGES : 1;  // barrier slots (unused without TMA words)
  constexpr int EPI_BOX = C::EPI_BOX, BOX_COLS = C::BOX_COLS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* packed = smem + C::P_OFFSET;
  uint8_t* epi_base = smem + C::EPI_OFFSET;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::BAR_OFFSET);
  uint64_t* empty_bar = full_bar + C::NST;
  uint64_t* pfull = empty_bar + C::NST;
  uint64_t* pempty = pfull + P_STAGES;
  uint64_t* tfull_bar = pempty + P_STAGES;
  uint64_t* tempty_bar = tfull_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = p.Kw / KBW;
  const int two_kpad = 2 * (32 * p.Kw - p.K);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(&full_bar[s], EXPANDER_WARPS);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(&pfull[s], 1);
      mbar_init(&pempty[s], EXPANDER_WARPS);
    }
    mbar_init(tfull_bar, 1);
    mbar_init(tempty_bar, EPI_WARPS);
    fence_barrier_init();
    if (TMA_WORDS) {
      tma_prefetch_desc(&tmW);
      tma_prefetch_desc(&tmX);
    }
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
  if (warp >= 1 && warp <= 4) {  // unit block scales: every byte of columns 256..511 = 0x7F
    const uint32_t lanes = (uint32_t)((warp & 3) * 32) << 16;
#pragma unroll
    for (uint32_t c = C::SFC; c < TMEM_COLS; c += 32) tmem_st_32x32b_x32_same(tmem_base + lanes + c, 0x7F7F7F7Fu);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer (converged warp, one
    // elected lane issues: descriptors stay in uniform registers)
    // kind::mxf4 block32: A, B e2m1 (format 1), UE8M0 scales, fp32 D, K-major, M = 128, N = 256
    constexpr uint32_t IDESC = (1u << 7) | (1u << 10) | ((uint32_t)((2 * BN) >> 3) << 17) | (1u << 23) |
                               ((uint32_t)(BM >> 4) << 24);
    const uint32_t sfa = tmem_base + C::SFC, sfb = tmem_base + C::SFC + C::SFB_OFF;
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      mbar_wait(tempty_bar, (it & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base;  // [D_r | D_i]
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        const uint8_t* st = smem + stage * C::STAGE;
        const uint8_t* sBn = st + C::BOFF;  // -B_i, B_r, B_i: consecutive 128-row tiles
        // K advance per MMA: 64 nibbles = 32 bytes = +2 in the descriptor address field
        const uint64_t ar0 = smem_desc_k128(st, 0), ai0 = smem_desc_k128(st + TILE_BYTES, 0);
        const uint64_t b_ri0 = smem_desc_k128(sBn + TILE_BYTES, 0);  // [B_r; B_i]
        const uint64_t b_nr0 = smem_desc_k128(sBn, 0);               // [-B_i; B_r]
        const uint32_t ta = tmem_base + C::A_COL + 64 * stage;      // ATMEM: A_r columns, A_i at +32
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < KBW / 2; ++kk) {  // K = 64 elements (32 bytes) per MMA
            const uint64_t b_ri = b_ri0 + (uint64_t)(2 * kk), b_nr = b_nr0 + (uint64_t)(2 * kk);
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            if (TCBF_ABLATE(p, 2)) continue;
            if constexpr (ATMEM) {  // K = 64 nibbles = 8 TMEM columns per MMA
              mma_mxf4_ts(d, ta + kk * 8, b_ri, IDESC, sfa, sfb, acc);
              mma_mxf4_ts(d, ta + 32 + kk * 8, b_nr, IDESC, sfa, sfb, 1u);
            } else {
              mma_mxf4(d, ar0 + (uint64_t)(2 * kk), b_ri, IDESC, sfa, sfb, acc);  // [Re(a)Re(b) | Re(a)Im(b)]
              mma_mxf4(d, ai0 + (uint64_t)(2 * kk), b_nr, IDESC, sfa, sfb, 1u);   // [-Im(a)Im(b) | Im(a)Re(b)]
            }
          }
          mma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == C::NST) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) mma_commit(tfull_bar);
      __syncwarp();
    }
  } else if (warp <= EPI_WARPS) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int part = (warp - 1) >> 2;  // 0: Re (columns 0..127), 1: Im (128..255)
    uint8_t* bufs = epi_base + (warp - 1) * C::EPI_BOXES * EPI_BOX;
    int sbuf = 0;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      int b, mt, nt;
      tile_coords(t, tiles_m, tiles_n, p.group_m, b, mt, nt);
      const int m0 = mt * BM;
      const int n0 = nt * BN;
      mbar_wait(tfull_bar, it & 1);
      tc_fence_after();
      constexpr bool WHOLE = TMA_STORE && !TMA_WORDS;  // stage the whole row block, one wait per tile
      if constexpr (WHOLE) {
        if (lane == 0) bulk_wait_group_read<0>();  // the previous tile's boxes have been read out
        __syncwarp();
      }
      // ablation (TCBF_DEBUG bit 3; timing only, wrong values): release TMEM before reading it.
      // Measured upper bound of any early-release epilogue: +3-5% (square 8192^3 0.82 -> 0.79 ms)
      if ((TCBF_ABLATE(p, 8)) && lane == 0) mbar_arrive(tempty_bar);
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + part * BN;
      const int corr = part == 0 ? 0 : two_kpad;
      // 16-column TMEM loads, two in flight (32 live registers instead of 64: the 576-thread CTA
      // has 96 registers per thread and the 32-column version spilled)
      constexpr int CW = 16;
      constexpr int NCH = BN / CW;
      uint32_t vbuf[2][CW];
      tmem_ld_32x32b_x16(tbase, vbuf[0]);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        tmem_wait_ld();
        if (c + 1 < NCH) {
          tmem_ld_32x32b_x16(tbase + (c + 1) * CW, vbuf[(c + 1) & 1]);
        } else {  // all TMEM reads of this warp done: the next tile's MMAs may start
          tc_fence_before();
          __syncwarp();
          if (lane == 0 && !(TCBF_ABLATE(p, 8))) mbar_arrive(tempty_bar);
        }
        uint32_t* vv = vbuf[c & 1];
#pragma unroll
        for (int j = 0; j < CW; ++j) vv[j] = (uint32_t)(__float2int_rn(__uint_as_float(vv[j])) - corr);
        if (TCBF_ABLATE(p, 1)) continue;
        if constexpr (WHOLE) {  // chunk c -> box c * CW / BOX_COLS of this warp's row block
          const int off = (c * CW) % BOX_COLS;
          uint8_t* buf = bufs + ((c * CW) / BOX_COLS) * EPI_BOX;
#pragma unroll
          for (int j = 0; j < CW / 4; ++j) {  // 16-byte chunks, 128-byte swizzle
            const int jj = off / 4 + j;
            *reinterpret_cast<uint4*>(buf + lane * (BOX_COLS * 4) + ((jj ^ (lane & 7)) * 16)) =
                make_uint4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]);
          }
          if (c == NCH - 1) {  // all boxes staged: one TMA store each
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
#pragma unroll
              for (int x = 0; x < C::EPI_BOXES; ++x) tma_store_3d(&tmC, bufs + x * EPI_BOX, n0 + x * BOX_COLS, m0 + q * 32, 2 * b + part);
              bulk_commit_group();
            }
          }
        } else if constexpr (TMA_STORE) {  // 32-row boxes of BOX_COLS columns, double-buffered per warp
          const int off = (c * CW) % BOX_COLS;  // column of this chunk inside its box
          uint8_t* buf = bufs + sbuf * EPI_BOX;
          if (off == 0) {
            if (lane == 0) bulk_wait_group_read<1>();
            __syncwarp();
          }
#pragma unroll
          for (int j = 0; j < CW / 4; ++j) {  // 16-byte chunks, 64- or 128-byte swizzle
            const int jj = off / 4 + j;
            const int pos = BOX_COLS == 16 ? (jj ^ ((lane >> 1) & 3)) : (jj ^ (lane & 7));
            *reinterpret_cast<uint4*>(buf + lane * (BOX_COLS * 4) + pos * 16) =
                make_uint4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]);
          }
          if (off + CW == BOX_COLS) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(&tmC, buf, n0 + c * CW + CW - BOX_COLS, m0 + q * 32, 2 * b + part);
              bulk_commit_group();
            }
            sbuf ^= 1;
          }
        } else {
          const int m = m0 + q * 32 + lane;
          if (m < p.M) {
            int32_t* rowp = p.out + ((size_t)(2 * b + part) * p.M + m) * (size_t)p.N;
#pragma unroll
            for (int j = 0; j < CW; ++j) {
              const int n = n0 + c * CW + j;
              if (n < p.N) rowp[n] = (int32_t)vv[j];
            }
          }
        }
      }
    }
    if constexpr (TMA_STORE) {
      if (lane == 0) bulk_wait_group<0>();
      __syncwarp();
    }
  } else if (warp < PRODUCER_WARP) {
    // ------------------------------------------------------------ expanders
    const int e = threadIdx.x - EXP_WARP0 * 32;  // 0..255
    const bool a_side = e < 128;
    // ATMEM: an A-side warp may only write its TMEM lane quarter (warp % 4)
    const int row = a_side ? (ATMEM ? 32 * (warp & 3) + lane : e) : e - 128;
    int stage = 0, ps = 0;
    uint32_t phase = 0, pph = 0;
    auto expand_block = [&](const uint4& r0, const uint4& r1, const uint4& i0, const uint4& i1) {
      mbar_wait(&empty_bar[stage], phase ^ 1);
      uint8_t* st = smem + stage * C::STAGE;
      if (!(TCBF_ABLATE(p, 4))) {
        if (a_side) {
          if constexpr (ATMEM) {
            tc_fence_after();
            const uint32_t ta = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + C::A_COL + 64 * stage;
            expand_tmem(ta, r0, r1);
            expand_tmem(ta + 32, i0, i1);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
          } else {
            expand(st + row * 128, row, r0, r1);
            expand(st + TILE_BYTES + row * 128, row, i0, i1);
          }
        } else {
          expand(st + C::BOFF + TILE_BYTES + row * 128, row, r0, r1);
          expand_pair(st + C::BOFF + 2 * TILE_BYTES + row * 128, st + C::BOFF + row * 128, row, i0, i1);
        }
      } else {
        asm volatile("" ::"r"(r0.x), "r"(r1.x), "r"(i0.x), "r"(i1.x));
      }
      fence_proxy_async_smem();  // each thread's generic-proxy smem writes -> async proxy
      __syncwarp();
    };
    if constexpr (TMA_WORDS) {
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&pfull[ps], pph);
          const uint8_t* pk = packed + ps * P_STAGE_BYTES + (a_side ? 0 : 2 * PLANE_BYTES) + row * (KBW * 4);
          const uint4 r0 = *reinterpret_cast<const uint4*>(pk);
          const uint4 r1 = *reinterpret_cast<const uint4*>(pk + 16);
          const uint4 i0 = *reinterpret_cast<const uint4*>(pk + PLANE_BYTES);
          const uint4 i1 = *reinterpret_cast<const uint4*>(pk + PLANE_BYTES + 16);
          expand_block(r0, r1, i0, i1);
          if (lane == 0) {
            mbar_arrive(&full_bar[stage]);
            mbar_arrive(&pempty[ps]);  // the words were consumed by the expansion above
          }
          if (++stage == C::NST) { stage = 0; phase ^= 1; }
          if (++ps == C::P_STAGES) { ps = 0; pph ^= 1; }
        }
      }
    } else {
      // The thread's K blocks over all its tiles form one flat stream; word loads run REG_PF
      // blocks ahead of the expansion in a register ring.
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
      int lt = blockIdx.x, lkb = 0;  // load cursor (tile, K block)
      const uint4* lr = nullptr;
      const uint4* li = nullptr;
      if (lt < num_tiles) row_ptrs(lt, lr, li);
      auto load_next = [&](uint4 (&d)[4]) {
        const bool ok = lr != nullptr;
        d[0] = ok ? __ldg(lr + 2 * lkb) : zero;
        d[1] = ok ? __ldg(lr + 2 * lkb + 1) : zero;
        d[2] = ok ? __ldg(li + 2 * lkb) : zero;
        d[3] = ok ? __ldg(li + 2 * lkb + 1) : zero;
        if (++lkb == num_kb) {
          lkb = 0;
          lt += gridDim.x;
          lr = li = nullptr;
          if (lt < num_tiles) row_ptrs(lt, lr, li);
        }
      };
      uint4 ring[REG_PF][4];
#pragma unroll
      for (int u = 0; u < REG_PF; ++u) load_next(ring[u]);
      const int my_tiles =
          blockIdx.x < (unsigned)num_tiles ? (num_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
      const int total = my_tiles * num_kb;
      for (int base = 0; base < total; base += REG_PF) {
#pragma unroll
        for (int u = 0; u < REG_PF; ++u) {
          if (base + u >= total) break;
          const uint4 r0 = ring[u][0], r1 = ring[u][1], i0 = ring[u][2], i1 = ring[u][3];
          load_next(ring[u]);
          expand_block(r0, r1, i0, i1);
          if (lane == 0) mbar_arrive(&full_bar[stage]);
          if (++stage == C::NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ TMA producer of packed words
    if (TMA_WORDS && lane == 0) {
      int ps = 0;
      uint32_t pph = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int b, mt, nt;
        tile_coords(t, tiles_m, tiles_n, p.group_m, b, mt, nt);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&pempty[ps], pph ^ 1);
          uint8_t* dst = packed + ps * P_STAGE_BYTES;
          mbar_arrive_expect_tx(&pfull[ps], P_STAGE_BYTES);
          tma_load_3d(dst, &tmW, &pfull[ps], kb * KBW, mt * BM, 2 * b);
          tma_load_3d(dst + PLANE_BYTES, &tmW, &pfull[ps], kb * KBW, mt * BM, 2 * b + 1);
          tma_load_3d(dst + 2 * PLANE_BYTES, &tmX, &pfull[ps], kb * KBW, nt * BN, 2 * b);
          tma_load_3d(dst + 3 * PLANE_BYTES, &tmX, &pfull[ps], kb * KBW, nt * BN, 2 * b + 1);
          if (++ps == C::P_STAGES) { ps = 0; pph ^= 1; }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

template <bool TMA_STORE, bool TMA_WORDS, bool ATMEM>
cudaError_t launch_f4(const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmC, const GemmB1Args& a,
                      int num_sms, cudaStream_t stream) {
  auto kern = cgemm_b1_f4_kernel<TMA_STORE, TMA_WORDS, ATMEM>;
  constexpr int SMEM_BYTES = Cfg<TMA_WORDS, ATMEM>::SMEM_BYTES;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  const long long nt = (long long)tiles_m * tiles_n * a.B;
  if (nt > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int grid = (int)(nt < num_sms ? nt : num_sms);
  kern<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(tmW, tmX, tmC, a, tiles_m, tiles_n, (int)nt);
  return cudaGetLastError();
}

}  // namespace

// fp32 accumulation of +-1 products is exact while every partial sum stays below 2^24; the
// expansion works on 256-bit K blocks (Kw is a multiple of 8 words by the packed layout)
bool gemm_b1_f4_supported(int64_t Kw) { return Kw % KBW == 0 && 32 * Kw <= (int64_t(1) << 23); }
int gemm_b1_f4_block_words() { return KBW; }
bool gemm_b1_f4_tma_words(int64_t Kw) { return Kw / KBW > 4; }  // K > 1024: TMA-fed words
int gemm_b1_f4_store_box_cols(int64_t Kw) { return gemm_b1_f4_tma_words(Kw) ? 16 : 32; }

cudaError_t launch_gemm_b1_f4(const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmC,
                              const GemmB1Args& args, bool tma_store, int num_sms, cudaStream_t stream) {
  // weights in TMEM (measured against smem-resident weights: square 8192^3 0.816 -> 0.700 ms,
  // 16384^3 6.34 -> 5.49 ms, radio 1.600 -> 1.572 ms; the smem-weights instantiation was dropped)
  if (gemm_b1_f4_tma_words(args.Kw))
    return tma_store ? launch_f4<true, true, true>(tmW, tmX, tmC, args, num_sms, stream)
                     : launch_f4<false, true, true>(tmW, tmX, tmC, args, num_sms, stream);
  return tma_store ? launch_f4<true, false, true>(tmW, tmX, tmC, args, num_sms, stream)
                   : launch_f4<false, false, true>(tmW, tmX, tmC, args, num_sms, stream);
}

}  // namespace tcbf
