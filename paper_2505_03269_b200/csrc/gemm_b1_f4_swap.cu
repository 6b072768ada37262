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
// 256-bit K block a tile reads 8 KB of packed data and does little MMA work, so what bounds it
// is how many packed bytes each SM keeps in flight and how cheaply they are expanded.
//   * packed words arrive by TMA in stages of FOUR K blocks (128-byte rows, 128-byte swizzle so
//     the expanders' row reads are bank-conflict free), three stages deep: ~120 KB in flight per
//     SM (was one K block of 32-byte row segments, four deep: 40 KB, latency-bound at ~1360
//     cycles per K block, 0.22 of the HBM roof);
//   * the expanded DATA tiles go to TENSOR memory (tcgen05.st, lane = sample, the layout the MMA
//     reads A from), so shared memory only holds the small weight tiles;
//   * the weight expansion is spread over four warps (several threads per weight row).
//
// Tile = 128 samples x TM beams (TM = 32 or 64).  TMEM: two accumulator buffers of 2 TM columns
// (the epilogue of one tile overlaps the next tile's MMAs), three expanded-data stages of 64
// columns (X_r 32 + X_i 32), unit scale factors in the remaining columns.  The epilogue writes the
// transposed accumulator back as [m][n] rows: each lane holds one sample n, so a warp's 32 lanes
// write 128 contiguous bytes of one beam row.
//
// Roles (persistent CTA per SM):
//   warp 0        TMEM allocator + single-thread MMA issuer
//   warps 1-4     epilogue (TMEM lane quarters), 32 x 32 TMA store boxes
//   warps 5-8     data expanders (one sample per thread, its TMEM lane), tcgen05.st
//   warps 9-12    weight expanders (-W_i, W_r, W_i into 128-byte-swizzled smem tiles)
//   warp 13       TMA producer of the packed words
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
constexpr int XEXP_WARPS = 4;
constexpr int WEXP_WARPS = 4;
constexpr uint32_t TMEM_COLS = 512;

template <int TM>
struct SwapCfg {
  // expanded stages (data in TMEM, weights in smem): as many as TMEM holds beside the accumulators
  // and the scale factors (the MMAs of a stage complete ~2.5 stages after their issue)
  static constexpr int NST = TM == 32 ? 5 : 3;
  static constexpr int W_TILE = TM * 128;                 // one expanded weight tile
  static constexpr int STAGE_BYTES = 3 * W_TILE;           // -W_i, W_r, W_i
  static constexpr int P_PLANE_X = TN * PKB * KBW * 4;     // packed words: 128 rows x 128 B
  static constexpr int P_PLANE_W = TM * PKB * KBW * 4;
  static constexpr int P_STAGE_BYTES = 2 * P_PLANE_X + 2 * P_PLANE_W;
  static constexpr int P_STAGES = TM == 32 ? 3 : 2;
  static constexpr int EPI_BYTES = EPI_WARPS * 2 * 4096;
  static constexpr int P_OFFSET = NST * STAGE_BYTES;
  static constexpr int EPI_OFFSET = P_OFFSET + P_STAGES * P_STAGE_BYTES;
  static constexpr int BAR_OFFSET = EPI_OFFSET + EPI_BYTES;
  static constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
  static constexpr int EXP_WARP0 = 1 + EPI_WARPS;
  static constexpr int WEXP_WARP0 = EXP_WARP0 + XEXP_WARPS;
  static constexpr int PRODUCER_WARP = WEXP_WARP0 + WEXP_WARPS;
  static constexpr int NUM_THREADS = (PRODUCER_WARP + 1) * 32;
  // TMEM columns: accumulators [0, 4 TM), data stages, scale factors
  static constexpr uint32_t X_COL = 4 * TM;
  static constexpr uint32_t SF_COL = X_COL + 64 * NST;
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
__device__ __forceinline__ void tmem_st_x16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
// one row's 256-bit K block (8 words) as e2m1 +-1 nibbles into 32 TMEM columns of its lane, in
// logical K order (output word 4q + j <- nib_pm1<j>(word q): the same permutation the smem
// expansion of the weights applies, so every dot product is unchanged)
__device__ __forceinline__ void expand_tmem(uint32_t taddr, const uint32_t (&w)[KBW]) {
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
    tmem_st_x16(taddr + 16 * h, v);
  }
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

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full_bar[s], XEXP_WARPS + WEXP_WARPS);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(&pfull[s], 1);
      mbar_init(&pempty[s], XEXP_WARPS + WEXP_WARPS);
    }
    for (int s = 0; s < 2; ++s) {
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
      const int abuf = it & 1;
      mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + abuf * 2 * TM;  // [D_r^T | D_i^T]
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (it == 0 && kb < 128 && lane == 0) stamp(p.trace, kb);  // dev timeline: MMA got stage kb
        const uint8_t* sWn = smem + stage * C::STAGE_BYTES;  // -W_i, W_r, W_i: consecutive TM-row tiles
        const uint64_t w_nr = smem_desc_k128(sWn, 0);            // [-W_i; W_r]
        const uint64_t w_ri = smem_desc_k128(sWn + C::W_TILE, 0);  // [W_r; W_i]
        const uint32_t xa = tmem_base + C::X_COL + 64 * stage;  // X_r columns, X_i at +32
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < KBW / 2; ++kk) {  // K = 64 elements = 32 bytes (+2 in the descriptor) = 8 TMEM columns
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            if (TCBF_ABLATE(p, 2)) continue;
            mma_mxf4_ts(d, xa + kk * 8, w_ri + (uint64_t)(2 * kk), IDESC, sfa, sfb, acc);
            mma_mxf4_ts(d, xa + 32 + kk * 8, w_nr + (uint64_t)(2 * kk), IDESC, sfa, sfb, 1u);
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
    uint8_t* bufs = epi_base + (warp - 1) * 2 * 4096;
    int sbuf = 0;
    int it = 0;
    constexpr int CHUNKS = 2 * TM / 32;  // 32-beam column chunks: Re parts, then Im parts
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      int b, nt, mt;
      swap_coords(t, tiles_m, tiles_n, b, nt, mt);
      const int n = nt * TN + q * 32 + lane;
      const int abuf = it & 1;
      mbar_wait(&tfull[abuf], (it >> 1) & 1);
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
          if (lane == 0) bulk_wait_group_read<1>();
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 32; ++j) *reinterpret_cast<uint32_t*>(buf + j * 128 + lane * 4) = vv[j];
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&tmC, buf, nt * TN + q * 32, m0, 2 * b + part);
            bulk_commit_group();
          }
          sbuf ^= 1;
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
    const int row = 32 * (warp & 3) + lane;  // a warp may only write its TMEM lane quarter
    const uint32_t lanes = (uint32_t)(32 * (warp & 3)) << 16;
    int stage = 0, ps = 0;
    uint32_t phase = 0, pph = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      for (int kb0 = 0; kb0 < num_kb; kb0 += PKB) {
        mbar_wait(&pfull[ps], pph);
        const bool tr = p.trace && warp == C::EXP_WARP0 && lane == 0 && t == (int)blockIdx.x && kb0 < 128;
        if (tr) stamp(p.trace, 128 + kb0 / PKB);
        const uint8_t* pk = packed + ps * C::P_STAGE_BYTES;
        const int nj = min(PKB, num_kb - kb0);
        for (int j = 0; j < nj; ++j) {
          const uint4 r0 = packed_chunk(pk, row, j, 0), r1 = packed_chunk(pk, row, j, 1);
          const uint4 i0 = packed_chunk(pk + C::P_PLANE_X, row, j, 0), i1 = packed_chunk(pk + C::P_PLANE_X, row, j, 1);
          const uint32_t wr[KBW] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
          const uint32_t wi[KBW] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z, i1.w};
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (tr) stamp(p.trace, 256 + kb0 + j);
          tc_fence_after();
          const uint32_t ta = tmem_base + lanes + C::X_COL + 64 * stage;
          if (!(TCBF_ABLATE(p, 4))) {
            expand_tmem(ta, wr);
            expand_tmem(ta + 32, wi);
          } else {
            asm volatile("" ::"r"(wr[0]), "r"(wi[0]));
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full_bar[stage]);
          if (tr) stamp(p.trace, 384 + kb0 + j);
          if (++stage == NST) { stage = 0; phase ^= 1; }
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
    int stage = 0, ps = 0;
    uint32_t phase = 0, pph = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      for (int kb0 = 0; kb0 < num_kb; kb0 += PKB) {
        mbar_wait(&pfull[ps], pph);
        const uint8_t* pw = packed + ps * C::P_STAGE_BYTES + 2 * C::P_PLANE_X;
        const int nj = min(PKB, num_kb - kb0);
        for (int j = 0; j < nj; ++j) {
          uint32_t wr[C::W_WPT], wi[C::W_WPT];
#pragma unroll
          for (int qq = 0; qq < C::W_WPT; ++qq) {
            wr[qq] = packed_word(pw, row, j, q0 + qq);
            wi[qq] = packed_word(pw + C::P_PLANE_W, row, j, q0 + qq);
          }
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* wn = smem + stage * C::STAGE_BYTES;  // -W_i
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
          __syncwarp();
          if (lane == 0) mbar_arrive(&full_bar[stage]);
          if (p.trace && warp == C::WEXP_WARP0 && lane == 0 && t == (int)blockIdx.x && kb0 + j < 128)
            stamp(p.trace, 640 + kb0 + j);
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
