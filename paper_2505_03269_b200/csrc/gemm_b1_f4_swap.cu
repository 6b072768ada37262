// gemm_b1_f4_swap.cu -- 1-bit-mode beamformer GEMM for few beams (M <= 64) on the fp4 tensor
// cores, with the operand roles swapped.
//
// Same arithmetic as gemm_b1_f4.cu (+-1 e2m1 nibbles from the packed sign bits, kind::mxf4 with
// unit block scales, exact fp32 accumulation, Im - 2 K_pad),
// but the 128-row MMA dimension runs over the DATA columns and the beams form the MMA N
// dimension, so a 32-beam plan does not pad its weights to 128 MMA rows (4x the tensor work) --
// the small-beam sweep of BASELINE config 5.  With lanes = samples n and columns = beams m:
//     [D_r^T | D_i^T] += X_r [W_r ; W_i]^T      [D_r^T | D_i^T] += X_i [-W_i ; W_r]^T
// (the weights' stacked tiles -W_i, W_r, W_i are expanded once per K block; N = 2 TM).
//
// This shape is a stream of packed data words (N x K bits) against a few weight rows: per
// 256-bit K block a tile reads 8 KB of packed data and does little MMA work (8 MMAs of N = 64 for
// 32 beams, ~36 cycles each at the tensor rate), so what bounds it is the packed stream and the
// latency of every hand-off around the MMA issuer:
//   * packed words arrive by TMA in stages of FOUR K blocks (128-byte rows, 128-byte swizzle so
//     the expanders' row reads are bank-conflict free), three stages deep (~120 KB in flight);
//   * the expanded DATA goes to TENSOR memory (tcgen05.st, lane = sample, the layout the MMA reads
//     A from), so shared memory only holds the small weight tiles; two groups of data-expander
//     warps take alternate K blocks, each expanding its block in registers before the stage frees;
//   * for 32 beams a stage holds TWO K blocks (one wait and one commit per 16 MMAs): a wait or
//     commit between MMA issues idles the tensor pipe (tools/probes/mma_pattern_probe.cu, one per
//     8 of these MMAs: ~70 cycles each instead of ~38), so the accumulator is single-buffered to
//     make room in TMEM (these shapes run one tile per CTA).
// Measured (N = K = 16384, 32 beams, 128 tiles): 44.5 us before the converged-warp MMA issue, 30.8
// after it, 28.8 with the two expander groups and two-block stages.  Left on the table: the packed
// word stream alone reaches ~4.7 TB/s on 128 SMs (tools/probes/tma_read_probe.cu: K-contiguous
// rows 2 KB apart read 128 B at a time; longer runs, L2 prefetch runs, deeper rings and 147
// shorter tiles were each measured no faster), the full pipeline ~2.5 TB/s.
//
// Tile = 128 samples x TM beams (TM = 32 or 64).  TMEM: accumulators (2 TM columns each), the
// expanded-data stages (64 columns per K block: X_r 32 + X_i 32), unit scale factors in the
// remaining columns.  The epilogue writes the transposed accumulator back as [m][n] rows: each
// lane holds one sample n, so a warp's 32 lanes write 128 contiguous bytes of one beam row.
//
// Roles (persistent CTA per SM):
//   warp 0        TMEM allocator + MMA issuer (converged warp, one elected lane issues)
//   warps 1-4     epilogue (TMEM lane quarters), 32 x 32 TMA store boxes
//   warps 5-12    data expanders, two groups of four taking alternate K blocks (one sample per
//                 thread, its TMEM lane), tcgen05.st
//   warps 13-16   weight expanders (-W_i, W_r, W_i into 128-byte-swizzled smem tiles)
//   warp 17       TMA producer of the packed words
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int TN = 128;   // samples per tile (MMA M)
constexpr int KBW = 8;    // 256-bit K blocks -> 128-byte rows of nibbles
constexpr int PKB = 4;    // K blocks per packed TMA stage (128-byte rows of words)
constexpr int EPI_WARPS = 4;
constexpr int XEXP_WARPS = 4;   // per group (one warp per TMEM lane quarter)
constexpr int XEXP_GROUPS = 2;  // groups take alternate K blocks (one group is latency-bound)
constexpr int WEXP_WARPS = 4;
constexpr uint32_t TMEM_COLS = 512;

template <int TM>
struct SwapCfg {
  // Expanded stages (data in TMEM, weights in smem) of SBLK K blocks each: the MMA issuer waits,
  // and commits, once per stage.  Every cycle of latency between MMA issues idles the tensor pipe
  // (tools/probes/mma_pattern_probe.cu: with one wait + commit per 8 of these small-N MMAs they
  // ran at ~70 cycles each, with one per 16 at ~51, back to back at ~38), so stages are two K
  // blocks and the accumulator is single-buffered to make room for them in TMEM (one tile per CTA
  // on the wave-limited shapes this kernel serves; the epilogue frees TMEM right after its loads).
  static constexpr int SBLK = TM == 32 ? 2 : 1;  // (TM = 64: N = 128 MMAs, twice the work per wait,
  static constexpr int NST = 3;                   //  and a two-block stage would not fit the registers
  static constexpr int ACC_BUFS = TM == 32 ? 1 : 2;  //  of the weight expanders: measured 37.2 vs 39.1 us)
  static constexpr int W_TILE = TM * 128;                 // one expanded weight tile
  static constexpr int BLK_BYTES = 3 * W_TILE;             // -W_i, W_r, W_i of one K block
  static constexpr int STAGE_BYTES = SBLK * BLK_BYTES;
  static constexpr int P_PLANE_X = TN * PKB * KBW * 4;     // packed words: 128 rows x 128 B
  static constexpr int P_PLANE_W = TM * PKB * KBW * 4;
  static constexpr int P_STAGE_BYTES = 2 * P_PLANE_X + 2 * P_PLANE_W;
  // (a fourth 40 KB packed stage in place of a weight stage and an epilogue buffer: measured equal)
  static constexpr int P_STAGES = TM == 32 ? 3 : 2;
  static constexpr int EPI_BUFS = 2;
  static constexpr int EPI_BYTES = EPI_WARPS * EPI_BUFS * 4096;
  static constexpr int P_OFFSET = NST * STAGE_BYTES;
  static constexpr int EPI_OFFSET = P_OFFSET + P_STAGES * P_STAGE_BYTES;
  static constexpr int BAR_OFFSET = EPI_OFFSET + EPI_BYTES;
  static constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
  static constexpr int EXP_WARP0 = 1 + EPI_WARPS;
  static constexpr int WEXP_WARP0 = EXP_WARP0 + XEXP_GROUPS * XEXP_WARPS;
  static constexpr int PRODUCER_WARP = WEXP_WARP0 + WEXP_WARPS;
  static constexpr int NUM_THREADS = (PRODUCER_WARP + 1) * 32;
  // TMEM columns: accumulators [0, ACC_BUFS * 2 TM), data stages (64 columns per K block: X_r 32,
  // X_i 32), scale factors
  static constexpr uint32_t X_COL = ACC_BUFS * 2 * TM;
  static constexpr uint32_t SF_COL = X_COL + 64 * SBLK * NST;
  static constexpr int W_TPR = 128 / TM;                  // weight-expander threads per weight row
  static constexpr int W_WPT = KBW / W_TPR;               // words per thread per K block
  static_assert(SMEM_BYTES <= 232448, "smem budget");
  static_assert(SF_COL + 64 <= TMEM_COLS, "TMEM budget");
  static_assert(W_TILE % 1024 == 0, "stacked weight tiles must stay on swizzle-atom boundaries");
};

template <int J>
__device__ __forceinline__ uint32_t nib_pm1(uint32_t w) {
  return ((w << (3 - J)) & 0x88888888u) ^ 0xAAAAAAAAu;  // bit 1 -> 0x2 (+1), bit 0 -> 0xA (-1)
}
template <int J>
__device__ __forceinline__ uint32_t nib_neg(uint32_t w) {
  return ((w << (3 - J)) & 0x88888888u) ^ 0x22222222u;  // bit 1 -> 0xA (-1), bit 0 -> 0x2 (+1)
}
__device__ __forceinline__ uint4 pm1(uint32_t w) {
  return make_uint4(nib_pm1<0>(w), nib_pm1<1>(w), nib_pm1<2>(w), nib_pm1<3>(w));
}
__device__ __forceinline__ uint4 neg(uint32_t w) {
  return make_uint4(nib_neg<0>(w), nib_neg<1>(w), nib_neg<2>(w), nib_neg<3>(w));
}
// words 4h..4h+3 of K block j of a row in a packed stage (128-byte rows, 128-byte TMA swizzle)
__device__ __forceinline__ uint4 packed_chunk(const uint8_t* plane, int row, int j, int h) {
  return *reinterpret_cast<const uint4*>(plane + row * 128 + (((2 * j + h) ^ (row & 7)) << 4));
}
// word q of K block j of a row in a packed stage
__device__ __forceinline__ uint32_t packed_word(const uint8_t* plane, int row, int j, int q) {
  const int chunk = (2 * j + (q >> 2)) ^ (row & 7);
  return *reinterpret_cast<const uint32_t*>(plane + row * 128 + chunk * 16 + (q & 3) * 4);
}
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
__device__ __forceinline__ void tmem_st_same(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
      "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
      "r"(v)
      : "memory");
}
// one row's 256-bit K block (8 words) as e2m1 +-1 nibbles for 32 TMEM columns of its lane, in
// logical K order (output word 4q + j <- nib_pm1<j>(word q): the same permutation the smem
// expansion of the weights applies, so every dot product is unchanged)
__device__ __forceinline__ void expand_words(uint32_t (&v)[32], const uint32_t (&w)[KBW]) {
#pragma unroll
  for (int q = 0; q < KBW; ++q) {
    v[4 * q] = nib_pm1<0>(w[q]);
    v[4 * q + 1] = nib_pm1<1>(w[q]);
    v[4 * q + 2] = nib_pm1<2>(w[q]);
    v[4 * q + 3] = nib_pm1<3>(w[q]);
  }
}
__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
      "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
      "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

// tile t -> (batch, sample tile, beam tile); beam tiles innermost (the weights stay in L2)
__device__ __forceinline__ void swap_coords(int t, int tiles_m, int tiles_n, int& b, int& nt, int& mt) {
  const int per_b = tiles_m * tiles_n;
  b = t / per_b;
  const int r = t - b * per_b;
  nt = r / tiles_m;
  mt = r - nt * tiles_m;
}

template <int TM, bool TMA_STORE>
__global__ void __launch_bounds__(SwapCfg<TM>::NUM_THREADS, 1)
    cgemm_b1_f4_swap_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                            const __grid_constant__ CUtensorMap tmC, GemmB1Args p, int tiles_m, int tiles_n,
                            int num_tiles) {
  using C = SwapCfg<TM>;
  constexpr int P_STAGES = C::P_STAGES;
  constexpr int NST = C::NST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* packed = smem + C::P_OFFSET;
  uint8_t* epi_base = smem + C::EPI_OFFSET;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::BAR_OFFSET);
  uint64_t* empty_bar = full_bar + NST;
  uint64_t* pfull = empty_bar + NST;
  uint64_t* pempty = pfull + P_STAGES;
  uint64_t* tfull = pempty + P_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = p.Kw / KBW;
  const int two_kpad = 2 * (32 * p.Kw - p.K);

  // a tile's K blocks in stages of SBLK; a ragged last stage is padded with virtual blocks (the
  // expanders arrive for them without writing, the issuer skips their MMAs)
  const int num_st = (num_kb + C::SBLK - 1) / C::SBLK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full_bar[s], C::SBLK * (XEXP_WARPS + WEXP_WARPS));
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(&pfull[s], 1);
      mbar_init(&pempty[s], XEXP_GROUPS * XEXP_WARPS + WEXP_WARPS);
    }
    for (int s = 0; s < C::ACC_BUFS; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
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
  if (warp >= 1 && warp <= EPI_WARPS) {  // unit block scales: every byte of the scale columns = 0x7F
    const uint32_t lanes = (uint32_t)((warp & 3) * 32) << 16;
#pragma unroll
    for (uint32_t c = C::SF_COL; c < TMEM_COLS; c += 32) tmem_st_same(tmem_base + lanes + c, 0x7F7F7F7Fu);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer (converged warp, one
    // elected lane issues: descriptors stay in uniform registers -- issuing from `lane == 0` cost an
    // elect/broadcast loop per instruction, ~2.4x the small-N MMA's own time)
    // kind::mxf4 block32: e2m1 A/B, UE8M0 scales, fp32 D, K-major, M = 128 samples, N = 2 TM
    constexpr uint32_t IDESC = (1u << 7) | (1u << 10) | ((uint32_t)((2 * TM) >> 3) << 17) | (1u << 23) |
                               ((uint32_t)(TN >> 4) << 24);
    const uint32_t sfa = tmem_base + C::SF_COL, sfb = tmem_base + C::SF_COL + 32;
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      const int abuf = it % C::ACC_BUFS;
      mbar_wait(&tempty[abuf], ((it / C::ACC_BUFS) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + abuf * 2 * TM;  // [D_r^T | D_i^T]
      for (int st = 0; st < num_st; ++st) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (it == 0 && st < 64 && lane == 0) stamp(p.trace, st);  // dev timeline: MMA got stage st
        const int nb = min(C::SBLK, num_kb - st * C::SBLK);
        if (elect_one()) {
#pragma unroll
          for (int j = 0; j < C::SBLK; ++j) {
            if (j >= nb) break;
            const uint8_t* sWn = smem + stage * C::STAGE_BYTES + j * C::BLK_BYTES;  // -W_i, W_r, W_i
            const uint64_t w_nr = smem_desc_k128(sWn, 0);                           // [-W_i; W_r]
            const uint64_t w_ri = smem_desc_k128(sWn + C::W_TILE, 0);                 // [W_r; W_i]
            const uint32_t xa = tmem_base + C::X_COL + 64 * (stage * C::SBLK + j);  // X_r, X_i at +32
#pragma unroll
            for (int kk = 0; kk < KBW / 2; ++kk) {  // K = 64 elements = 32 bytes (+2 in the descriptor) = 8 TMEM columns
              const uint32_t acc = (st | j | kk) ? 1u : 0u;
              if (TCBF_ABLATE(p, 2)) continue;
              mma_mxf4_ts(d, xa + kk * 8, w_ri + (uint64_t)(2 * kk), IDESC, sfa, sfb, acc);
              mma_mxf4_ts(d, xa + 32 + kk * 8, w_nr + (uint64_t)(2 * kk), IDESC, sfa, sfb, 1u);
            }
          }
          mma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == NST) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) mma_commit(&tfull[abuf]);
      __syncwarp();
      if (it == 0 && lane == 0) stamp(p.trace, 1000);
    }
  } else if (warp <= EPI_WARPS) {
    // ------------------------------------------------------------ epilogue (lane = sample)
    const int q = warp & 3;
    uint8_t* bufs = epi_base + (warp - 1) * C::EPI_BUFS * 4096;
    int sbuf = 0;
    int it = 0;
    constexpr int CHUNKS = 2 * TM / 32;  // 32-beam column chunks: Re parts, then Im parts
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      int b, nt, mt;
      swap_coords(t, tiles_m, tiles_n, b, nt, mt);
      const int n = nt * TN + q * 32 + lane;
      const int abuf = it % C::ACC_BUFS;
      mbar_wait(&tfull[abuf], (it / C::ACC_BUFS) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 2 * TM;
      uint32_t vbuf[2][32];
      tmem_ld_32x32b_x32(tbase, vbuf[0]);
#pragma unroll
      for (int c = 0; c < CHUNKS; ++c) {
        const int part = c / (TM / 32);
        const int m0 = mt * TM + (c % (TM / 32)) * 32;
        tmem_wait_ld();
        if (c + 1 < CHUNKS) {
          tmem_ld_32x32b_x32(tbase + (c + 1) * 32, vbuf[(c + 1) & 1]);
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[abuf]);
        }
        uint32_t* vv = vbuf[c & 1];
        const int corr = part == 0 ? 0 : two_kpad;
#pragma unroll
        for (int j = 0; j < 32; ++j) vv[j] = (uint32_t)(__float2int_rn(__uint_as_float(vv[j])) - corr);
        if (TCBF_ABLATE(p, 1)) continue;
        if constexpr (TMA_STORE) {  // box of 32 beams x 32 samples, row = beam (128 B)
          uint8_t* buf = bufs + sbuf * 4096;
          if (lane == 0) bulk_wait_group_read<C::EPI_BUFS - 1>();
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 32; ++j) *reinterpret_cast<uint32_t*>(buf + j * 128 + lane * 4) = vv[j];
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmC, buf, nt * TN + q * 32, m0, 2 * b + part);
            bulk_commit_group();
          }
          if (++sbuf == C::EPI_BUFS) sbuf = 0;
        } else if (n < p.N) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int m = m0 + j;
            if (m < p.M) p.out[((size_t)(2 * b + part) * p.M + m) * (size_t)p.N + n] = (int32_t)vv[j];
          }
        }
      }
    }
    if constexpr (TMA_STORE) {
      if (lane == 0) bulk_wait_group<0>();
      __syncwarp();
    }
  } else if (warp < C::WEXP_WARP0) {
    // ------------------------------------------------------------ data expanders -> TMEM (lane = sample)
    // the groups take alternate K blocks (a virtual block past K only arrives)
    const int row = 32 * (warp & 3) + lane;  // a warp may only write its TMEM lane quarter
    const uint32_t lanes = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t grp = (uint32_t)((warp - C::EXP_WARP0) / XEXP_WARPS);
    const bool tw = p.trace && (warp - C::EXP_WARP0) % XEXP_WARPS == 0 && lane == 0 && blockIdx.x == 0;
    int stage = 0, pos = 0, ps = 0, it = 0;
    uint32_t phase = 0, pph = 0, blk = 0;  // blk: blocks seen so far, virtual ones included
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      for (int kb0 = 0; kb0 < C::SBLK * num_st; kb0 += PKB) {  // (kb0 < num_kb always: PKB % SBLK == 0)
        mbar_wait(&pfull[ps], pph);
        if (tw && grp == 0 && it == 0 && kb0 < 512) stamp(p.trace, 128 + kb0 / PKB);
        const uint8_t* pk = packed + ps * C::P_STAGE_BYTES;
#pragma unroll
        for (int j = 0; j < PKB; ++j) {
          const int kb = kb0 + j;
          if (kb >= C::SBLK * num_st) break;
          if (blk++ % XEXP_GROUPS == grp) {
            const bool tr = tw && it == 0 && kb < 128;
            if (kb < num_kb) {
              const uint4 r0 = packed_chunk(pk, row, j, 0), r1 = packed_chunk(pk, row, j, 1);
              const uint4 i0 = packed_chunk(pk + C::P_PLANE_X, row, j, 0), i1 = packed_chunk(pk + C::P_PLANE_X, row, j, 1);
              const uint32_t wr[KBW] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
              const uint32_t wi[KBW] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
              uint32_t vr[32], vi[32];  // expanded before the stage is free: only the stores wait
              expand_words(vr, wr);
              expand_words(vi, wi);
              mbar_wait(&empty_bar[stage], phase ^ 1);
              if (tr) stamp(p.trace, 256 + kb);
              tc_fence_after();
              const uint32_t ta = tmem_base + lanes + C::X_COL + 64 * (stage * C::SBLK + pos);
              if (!(TCBF_ABLATE(p, 4))) {
                tmem_st_x32(ta, vr);
                tmem_st_x32(ta + 32, vi);
              } else {
                asm volatile("" ::"r"(vr[0]), "r"(vi[0]));
              }
              asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
              tc_fence_before();
            } else {
              mbar_wait(&empty_bar[stage], phase ^ 1);  // a virtual block's arrival must count toward this use
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full_bar[stage]);
            if (tr) stamp(p.trace, 384 + kb);
          }
          if (++pos == C::SBLK) {
            pos = 0;
            if (++stage == NST) { stage = 0; phase ^= 1; }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&pempty[ps]);
        if (++ps == P_STAGES) { ps = 0; pph ^= 1; }
      }
    }
  } else if (warp < C::PRODUCER_WARP) {
    // ------------------------------------------------------------ weight expanders -> smem (-W_i, W_r, W_i)
    const int e = threadIdx.x - C::WEXP_WARP0 * 32;  // 0..127
    const int row = e / C::W_TPR;
    const int q0 = (e % C::W_TPR) * C::W_WPT;        // first word of the K block this thread expands
    int stage = 0, ps = 0, it = 0;
    uint32_t phase = 0, pph = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      for (int kb0 = 0; kb0 < C::SBLK * num_st; kb0 += PKB) {
        mbar_wait(&pfull[ps], pph);  // (kb0 < num_kb always: PKB % SBLK == 0)
        const uint8_t* pw = packed + ps * C::P_STAGE_BYTES + 2 * C::P_PLANE_X;
        for (int j0 = 0; j0 < PKB; j0 += C::SBLK) {
          if (kb0 + j0 >= C::SBLK * num_st) break;
          // per block: load, (first block of the stage) wait, store, proxy fence, arrive (one wait and
          // fence for the whole stage with its blocks expanded in registers measured 7% slower)
          bool waited = false;
#pragma unroll
          for (int jj = 0; jj < C::SBLK; ++jj) {
            const int j = j0 + jj;
            if (kb0 + j < num_kb) {
              uint32_t wr[C::W_WPT], wi[C::W_WPT];
#pragma unroll
              for (int qq = 0; qq < C::W_WPT; ++qq) {
                wr[qq] = packed_word(pw, row, j, q0 + qq);
                wi[qq] = packed_word(pw + C::P_PLANE_W, row, j, q0 + qq);
              }
              if (!waited) mbar_wait(&empty_bar[stage], phase ^ 1);
              waited = true;
              uint8_t* wn = smem + stage * C::STAGE_BYTES + jj * C::BLK_BYTES;  // -W_i, W_r, W_i
              if (!(TCBF_ABLATE(p, 4))) {
#pragma unroll
                for (int qq = 0; qq < C::W_WPT; ++qq) {
                  const int pos = ((q0 + qq) ^ (row & 7)) << 4;  // 128-byte swizzle of the 16-byte chunk
                  *reinterpret_cast<uint4*>(wn + row * 128 + pos) = neg(wi[qq]);
                  *reinterpret_cast<uint4*>(wn + C::W_TILE + row * 128 + pos) = pm1(wr[qq]);
                  *reinterpret_cast<uint4*>(wn + 2 * C::W_TILE + row * 128 + pos) = pm1(wi[qq]);
                }
              }
              fence_proxy_async_smem();
            } else if (!waited) {
              mbar_wait(&empty_bar[stage], phase ^ 1);  // a virtual block's arrival counts toward this use
              waited = true;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full_bar[stage]);
          }
          if (p.trace && warp == C::WEXP_WARP0 && lane == 0 && blockIdx.x == 0 && it == 0 && kb0 + j0 < 128)
            stamp(p.trace, 640 + (kb0 + j0) / C::SBLK);
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&pempty[ps]);
        if (++ps == P_STAGES) { ps = 0; pph ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ TMA producer of packed words
    if (lane == 0) {
      int ps = 0;
      uint32_t pph = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int b, nt, mt;
        swap_coords(t, tiles_m, tiles_n, b, nt, mt);
        for (int kb0 = 0; kb0 < num_kb; kb0 += PKB) {
          mbar_wait(&pempty[ps], pph ^ 1);
          if (t == (int)blockIdx.x && kb0 < 128) stamp(p.trace, 512 + kb0 / PKB);
          uint8_t* dst = packed + ps * C::P_STAGE_BYTES;
          mbar_arrive_expect_tx(&pfull[ps], C::P_STAGE_BYTES);  // words past Kw are zero-filled
          tma_load_3d(dst, &tmX, &pfull[ps], kb0 * KBW, nt * TN, 2 * b);
          tma_load_3d(dst + C::P_PLANE_X, &tmX, &pfull[ps], kb0 * KBW, nt * TN, 2 * b + 1);
          tma_load_3d(dst + 2 * C::P_PLANE_X, &tmW, &pfull[ps], kb0 * KBW, mt * TM, 2 * b);
          tma_load_3d(dst + 2 * C::P_PLANE_X + C::P_PLANE_W, &tmW, &pfull[ps], kb0 * KBW, mt * TM, 2 * b + 1);
          if (++ps == P_STAGES) { ps = 0; pph ^= 1; }
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

template <int TM, bool TMA_STORE>
cudaError_t launch_swap(const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmC, const GemmB1Args& a,
                        int num_sms, cudaStream_t stream) {
  using C = SwapCfg<TM>;
  auto kern = cgemm_b1_f4_swap_kernel<TM, TMA_STORE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles_m = (a.M + TM - 1) / TM, tiles_n = (a.N + TN - 1) / TN;
  const long long nt = (long long)tiles_m * tiles_n * a.B;
  if (nt > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int grid = (int)(nt < num_sms ? nt : num_sms);
  kern<<<grid, C::NUM_THREADS, C::SMEM_BYTES, stream>>>(tmW, tmX, tmC, a, tiles_m, tiles_n, (int)nt);
  return cudaGetLastError();
}

}  // namespace

int gemm_b1_f4_swap_beams(int64_t M) { return M <= 32 ? 32 : (M <= 64 ? 64 : 0); }
int gemm_b1_f4_swap_box_words() { return PKB * KBW; }

// tensor maps: packed words [2B][rows][Kw] u32, box {32 words, 128 samples} (data) and
// {32 words, TM beams} (weights), 128-byte swizzle, zero fill past Kw
cudaError_t launch_gemm_b1_f4_swap(const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmC,
                                   const GemmB1Args& args, int beams, bool tma_store, int num_sms, cudaStream_t stream) {
  // beams per tile as the plan chose it (the weight tensor map's box was built for it)
  if (beams == 32)
    return tma_store ? launch_swap<32, true>(tmW, tmX, tmC, args, num_sms, stream)
                     : launch_swap<32, false>(tmW, tmX, tmC, args, num_sms, stream);
  return tma_store ? launch_swap<64, true>(tmW, tmX, tmC, args, num_sms, stream)
                   : launch_swap<64, false>(tmW, tmX, tmC, args, num_sms, stream);
}

}  // namespace tcbf
