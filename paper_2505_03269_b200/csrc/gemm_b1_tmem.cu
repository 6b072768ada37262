// gemm_b1_tmem.cu -- 1-bit-mode beamformer GEMM, sample-major, with each 128-sample unit's
// expanded data resident in TENSOR memory (short K: Kw <= 24 words, K <= 768 bits).
//
// Same arithmetic as gemm_b1_f4.cu / gemm_b1_f4_swap.cu (+-1 e2m1 nibbles from the packed sign
// bits, tcgen05.mma kind::mxf4 with unit block scales, exact fp32 accumulation, Re = D_r,
// Im = D_i - 2 K_pad), transposed like the swapped kernel:
// lanes = samples n, columns = beams m,
//     [D_r^T | D_i^T] += X_r [W_r ; W_i]^T      [D_r^T | D_i^T] += X_i [-W_i ; W_r]^T
// (N = 128: 64 beams per tile).  Why ("1-bit resident-data kernel"): the radio
// 1-bit shape is bound by its 8.6 GB int32 output.  The beam-major fp4 kernel writes it through
// smem staging and TMA store boxes (stores alone 4.7 TB/s), while the fp16 radio kernels'
// sample-major epilogue writes one full 128-byte line of a beam row per warp store, straight
// from TMEM.  The swapped kernel already runs this orientation but re-loads and re-expands the
// data for every beam tile; here a unit's data is expanded ONCE into TMEM (X_r, X_i: 64 columns
// per 256-bit K block) and read by all of the unit's beam tiles, while the next unit's packed
// words land in smem by TMA and are expanded into TMEM block by block as the last beam tile
// releases each block.  The weights (tiny: 8 KB of packed words per 64-beam tile at K = 512)
// come by TMA per tile and are expanded into [-W_i | W_r | W_i] smem tiles one tile ahead.
//
// TMEM: two accumulators [Re 64 | Im 64] (0..255), data blocks at 256 + 64 kb, unit scale
// factors 448..511.  Roles: warp 0 TMA producer (packed weights), warp 1 MMA issuer, warps 2..9
// epilogue (line stores), warps 10..13 data expanders (thread = sample = TMEM lane), warps
// 14..17 weight expanders, warp 18 TMA producer (packed data), warp 19 sync warp (the MMA
// issuer's mbarrier waits, handed on by named barriers).
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int UN = 128;                    // samples per unit (MMA M, TMEM lanes)
constexpr int TM = 64;                     // beams per tile (MMA N = 2 TM)
constexpr int KBW = 8;                     // words per 256-bit K block
constexpr int NKB_MAX = 3;                 // K blocks resident in TMEM (Kw <= 24)
constexpr int KW_MAX = NKB_MAX * KBW;
constexpr int EPI_WARPS = 8;
constexpr int DEXP_WARPS = 4;
constexpr int WEXP_WARPS = 4;
constexpr int EPI0 = 2;
constexpr int DEXP0 = EPI0 + EPI_WARPS;
constexpr int WEXP0 = DEXP0 + DEXP_WARPS;
constexpr int DPROD_WARP = WEXP0 + WEXP_WARPS;
constexpr int SYNC_WARP = DPROD_WARP + 1;
constexpr int NUM_THREADS = (SYNC_WARP + 1) * 32;
constexpr int W_TILE = TM * 128;           // one expanded weight tile: 64 rows x 128 B (one K block)
constexpr int W_BLK = 3 * W_TILE;          // -W_i, W_r, W_i of one K block (24 KB)
constexpr int W_STAGE = NKB_MAX * W_BLK;   // a tile's expanded weights (72 KB)
constexpr int W_STAGES = 2;
constexpr int PW_PLANE = TM * KW_MAX * 4;  // packed weight words of one plane (box {Kw, 64})
constexpr int PW_STAGE = 2 * PW_PLANE;
constexpr int PW_STAGES = 3;
constexpr int PX_PLANE = UN * KW_MAX * 4;  // packed data words of one plane (box {Kw, 128})
constexpr int OFF_W = 0;
constexpr int OFF_PW = OFF_W + W_STAGES * W_STAGE;
constexpr int OFF_PX = OFF_PW + PW_STAGES * PW_STAGE;
constexpr int BAR_OFFSET = OFF_PX + 2 * PX_PLANE;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
constexpr uint32_t ACC_COL = 0;            // [Re | Im] x 2 buffers
constexpr uint32_t X_COL = 256;            // data: K block kb at 256 + 64 kb (X_r 32, X_i 32)
constexpr uint32_t SF_COL = X_COL + 64 * NKB_MAX;
constexpr int NB_STAGE0 = 2;               // named barriers 2, 3: weight stage s ready
static_assert(SMEM_BYTES <= 232448, "smem budget");
static_assert(SF_COL + 64 <= 512, "TMEM budget");
static_assert(W_TILE % 1024 == 0, "stacked weight tiles stay on swizzle-atom boundaries");

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

// args.M, N, K, Kw, B as in GemmB1Args; tiles_m = 64-beam tiles, tiles_n = 128-sample units
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_b1_tmem_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                         GemmB1Args p, int tiles_m, int tiles_n) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem + OFF_W;
  uint8_t* sPW = smem + OFF_PW;
  uint8_t* sPX = smem + OFF_PX;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);  // expanded weight stage ready
  uint64_t* wempty = wfull + W_STAGES;       // its MMAs retired
  uint64_t* pwfull = wempty + W_STAGES;      // packed weight words landed
  uint64_t* pwempty = pwfull + PW_STAGES;    // expanded
  uint64_t* xfull = pwempty + PW_STAGES;     // [NKB_MAX]: the unit's data block in TMEM
  uint64_t* xempty = xfull + NKB_MAX;        // [NKB_MAX]: the unit's last tile has read it
  uint64_t* dfull = xempty + NKB_MAX;        // the next unit's packed words landed
  uint64_t* dempty = dfull + 1;              // expanded (the staging is free)
  uint64_t* tfull = dempty + 1;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int Kw = p.Kw;
  const int nkb = Kw / KBW;
  const int num_units = p.B * tiles_n;
  const int two_kpad = 2 * (32 * Kw - p.K);

  if (threadIdx.x == 0) {
    for (int s = 0; s < W_STAGES; ++s) {
      mbar_init(&wfull[s], WEXP_WARPS);
      mbar_init(&wempty[s], 1);
    }
    for (int s = 0; s < PW_STAGES; ++s) {
      mbar_init(&pwfull[s], 1);
      mbar_init(&pwempty[s], WEXP_WARPS);
    }
    for (int s = 0; s < NKB_MAX; ++s) {
      mbar_init(&xfull[s], DEXP_WARPS);
      mbar_init(&xempty[s], 1);
    }
    mbar_init(dfull, 1);
    mbar_init(dempty, DEXP_WARPS);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp >= EPI0 && warp < EPI0 + 4) {  // unit block scales: every byte of the scale columns = 0x7F
    const uint32_t lanes = (uint32_t)((warp & 3) * 32) << 16;
#pragma unroll
    for (uint32_t c = SF_COL; c < 512; c += 32) tmem_st_same(tmem_base + lanes + c, 0x7F7F7F7Fu);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer: packed weight words
    // of each tile (64 rows x Kw words per plane; rows >= M zero-filled = -1, masked at the store)
    if (lane == 0) {
      int ps = 0;
      uint32_t pph = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        const int b = u / tiles_n;
        for (int mt = 0; mt < tiles_m; ++mt) {
          mbar_wait(&pwempty[ps], pph ^ 1);
          uint8_t* dst = sPW + ps * PW_STAGE;
          mbar_arrive_expect_tx(&pwfull[ps], 2 * TM * Kw * 4);
          tma_load_3d(dst, &tmW, &pwfull[ps], 0, mt * TM, 2 * b);
          tma_load_3d(dst + PW_PLANE, &tmW, &pwfull[ps], 0, mt * TM, 2 * b + 1);
          if (++ps == PW_STAGES) { ps = 0; pph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (converged warp)
    // kind::mxf4 block32: e2m1 A (TMEM) / B (smem, K-major), UE8M0 scales, fp32 D, M = 128, N = 128
    constexpr uint32_t IDESC = (1u << 7) | (1u << 10) | ((uint32_t)((2 * TM) >> 3) << 17) | (1u << 23) |
                               ((uint32_t)(UN >> 4) << 24);
    const uint32_t sfa = tmem_base + SF_COL, sfb = tmem_base + SF_COL + 32;
    int stage = 0, it = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int abuf = it & 1;
        const uint32_t d = tmem_base + ACC_COL + abuf * 2 * TM;  // [D_r^T | D_i^T]
        // one named-barrier sync per tile: the sync warp has seen the expanded weights, the free
        // accumulator and (first tile of a unit) the unit's data blocks in TMEM
        asm volatile("bar.sync %0, 64;" ::"r"(NB_STAGE0 + stage) : "memory");
        tc_fence_after();
        const uint8_t* st = sW + stage * W_STAGE;
        if (elect_one()) {
          for (int kb = 0; kb < nkb; ++kb) {
            const uint64_t w_nr = smem_desc_k128(st + kb * W_BLK, 0);           // [-W_i ; W_r]
            const uint64_t w_ri = smem_desc_k128(st + kb * W_BLK + W_TILE, 0);  // [W_r ; W_i]
            const uint32_t xa = tmem_base + X_COL + 64 * kb;                    // X_r, X_i at +32
#pragma unroll
            for (int kk = 0; kk < KBW / 2; ++kk) {  // K = 64 elements = 8 TMEM columns = 32 B (+2)
              const uint32_t acc = (kb | kk) ? 1u : 0u;
              if (TCBF_ABLATE(p, 2)) continue;
              mma_mxf4_ts(d, xa + kk * 8, w_ri + (uint64_t)(2 * kk), IDESC, sfa, sfb, acc);
              mma_mxf4_ts(d, xa + 32 + kk * 8, w_nr + (uint64_t)(2 * kk), IDESC, sfa, sfb, 1u);
            }
          }
          mma_commit(&wempty[stage]);
          if (mt == tiles_m - 1)
            for (int kb = 0; kb < nkb; ++kb) mma_commit(&xempty[kb]);  // last reader of the data
          mma_commit(&tfull[abuf]);
        }
        __syncwarp();
        if (++stage == W_STAGES) stage = 0;
      }
    }
  } else if (warp < DEXP0) {
    // ------------------------------------------------------------ epilogue: int32 line stores
    const int q = warp & 3;              // TMEM lane quadrant = samples 32q..32q+31 of the unit
    const int half = (warp - EPI0) / 4;  // half 0 stores Re, half 1 Im
    const int M = p.M;
    const size_t N = (size_t)p.N;
    const int corr = half ? two_kpad : 0;
    int it = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      const int b = u / tiles_n;
      const int n = (u - b * tiles_n) * UN + q * 32 + lane;  // this thread's sample
      const bool n_ok = n < p.N;
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int abuf = it & 1;
        mbar_wait(&tfull[abuf], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + ACC_COL + abuf * 2 * TM + half * TM;
        uint32_t v[2][32];
        tmem_ld_32x32b_x32(tb, v[0]);
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          tmem_wait_ld();
          if (ch == 0) {
            tmem_ld_32x32b_x32(tb + 32, v[1]);
          } else {  // all TMEM reads of this tile complete: release the buffer
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[abuf]);
          }
          if (TCBF_ABLATE(p, 1)) continue;
          const int m0 = mt * TM + ch * 32;
          if (n_ok) {
            int32_t* col = p.out + ((size_t)(2 * b + half) * M + m0) * N + n;
            if (m0 + 32 <= M) {
#pragma unroll
              for (int j = 0; j < 32; ++j) col[(size_t)j * N] = __float2int_rn(__uint_as_float(v[ch][j])) - corr;
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (m0 + j < M) col[(size_t)j * N] = __float2int_rn(__uint_as_float(v[ch][j])) - corr;
            }
          }
        }
      }
    }
  } else if (warp < WEXP0) {
    // ------------------------------------------------------------ data expanders: thread = sample =
    // TMEM lane; at each unit switch the staged packed words -> +-1 nibbles -> TMEM, block by block
    // as the previous unit's last tile releases it
    const int q = warp & 3;
    const int s = q * 32 + lane;
    const uint32_t lanes = (uint32_t)(q * 32) << 16;
    int ui = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++ui) {
      mbar_wait(dfull, ui & 1);
      for (int kb = 0; kb < nkb; ++kb) {
        uint32_t vr[32], vi[32];
        {
          uint32_t wr[KBW], wi[KBW];
          const uint32_t* rr = reinterpret_cast<const uint32_t*>(sPX) + s * Kw + kb * KBW;
          const uint32_t* ri = reinterpret_cast<const uint32_t*>(sPX + PX_PLANE) + s * Kw + kb * KBW;
#pragma unroll
          for (int w = 0; w < KBW; ++w) { wr[w] = rr[w]; wi[w] = ri[w]; }
          // output word 4w + j <- nib_pm1<j>(word w): the permutation the weight expansion applies
#pragma unroll
          for (int w = 0; w < KBW; ++w) {
            vr[4 * w] = nib_pm1<0>(wr[w]); vr[4 * w + 1] = nib_pm1<1>(wr[w]);
            vr[4 * w + 2] = nib_pm1<2>(wr[w]); vr[4 * w + 3] = nib_pm1<3>(wr[w]);
            vi[4 * w] = nib_pm1<0>(wi[w]); vi[4 * w + 1] = nib_pm1<1>(wi[w]);
            vi[4 * w + 2] = nib_pm1<2>(wi[w]); vi[4 * w + 3] = nib_pm1<3>(wi[w]);
          }
        }
        if (kb == nkb - 1) {  // all words of the unit read: the staging may take the next unit
          __syncwarp();
          if (lane == 0) mbar_arrive(dempty);
        }
        mbar_wait(&xempty[kb], (ui & 1) ^ 1);
        tc_fence_after();
        const uint32_t ta = tmem_base + lanes + X_COL + 64 * kb;
        tmem_st_x32(ta, vr);
        tmem_st_x32(ta + 32, vi);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&xfull[kb]);
      }
    }
  } else if (warp < DPROD_WARP) {
    // ------------------------------------------------------------ weight expanders: a tile's packed
    // words -> [-W_i | W_r | W_i] 128-byte-swizzled tiles, one tile ahead of the MMAs
    const int e = threadIdx.x - WEXP0 * 32;  // 0..127
    const int row = e >> 1;                  // weight row of the tile
    const int h = e & 1;                     // 16-byte chunks 4h..4h+3 of each 128-byte row
    int ps = 0, stage = 0;
    uint32_t pph = 0, wph = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      for (int mt = 0; mt < tiles_m; ++mt) {
        mbar_wait(&pwfull[ps], pph);
        const uint32_t* pr = reinterpret_cast<const uint32_t*>(sPW + ps * PW_STAGE) + row * Kw;
        const uint32_t* pi = reinterpret_cast<const uint32_t*>(sPW + ps * PW_STAGE + PW_PLANE) + row * Kw;
        mbar_wait(&wempty[stage], wph ^ 1);
        uint8_t* wn = sW + stage * W_STAGE;
        for (int kb = 0; kb < nkb; ++kb) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int w = 4 * h + c;  // word of the K block = 16-byte chunk of the expanded row
            const uint32_t wr = pr[kb * KBW + w], wi = pi[kb * KBW + w];
            const int pos = (w ^ (row & 7)) << 4;  // 128-byte swizzle
            uint8_t* blk = wn + kb * W_BLK + row * 128 + pos;
            if (!(TCBF_ABLATE(p, 4))) {
              *reinterpret_cast<uint4*>(blk) = neg(wi);
              *reinterpret_cast<uint4*>(blk + W_TILE) = pm1(wr);
              *reinterpret_cast<uint4*>(blk + 2 * W_TILE) = pm1(wi);
            }
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&wfull[stage]);
          mbar_arrive(&pwempty[ps]);
        }
        if (++ps == PW_STAGES) { ps = 0; pph ^= 1; }
        if (++stage == W_STAGES) { stage = 0; wph ^= 1; }
      }
    }
  } else if (warp == DPROD_WARP) {
    // ------------------------------------------------------------ TMA producer: packed data words of
    // the next unit (128 samples x Kw words per plane; samples >= N zero-filled)
    if (lane == 0) {
      int ui = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++ui) {
        const int b = u / tiles_n;
        const int n0 = (u - b * tiles_n) * UN;
        mbar_wait(dempty, (ui & 1) ^ 1);
        mbar_arrive_expect_tx(dfull, 2 * UN * Kw * 4);
        tma_load_3d(sPX, &tmX, dfull, 0, n0, 2 * b);
        tma_load_3d(sPX + PX_PLANE, &tmX, dfull, 0, n0, 2 * b + 1);
      }
    }
  } else {
    // ------------------------------------------------------------ sync warp: the MMA issuer's waits
    int stage = 0, it = 0, ui = 0;
    uint32_t wph = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++ui) {
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        mbar_wait(&tempty[it & 1], ((it >> 1) & 1) ^ 1);
        if (mt == 0)
          for (int kb = 0; kb < nkb; ++kb) mbar_wait(&xfull[kb], ui & 1);
        mbar_wait(&wfull[stage], wph);
        asm volatile("bar.arrive %0, 64;" ::"r"(NB_STAGE0 + stage) : "memory");
        if (++stage == W_STAGES) { stage = 0; wph ^= 1; }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace

bool gemm_b1_tmem_supported(int64_t Kw) { return Kw % KBW == 0 && Kw <= KW_MAX; }
int gemm_b1_tmem_beams() { return TM; }

// weights tensor map: {Kw words, M rows, 2B planes} uint32, box {Kw, 64}; data map: {Kw, N, 2B},
// box {Kw, 128}; no swizzle
cudaError_t launch_gemm_b1_tmem(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmB1Args& a, int num_sms,
                                cudaStream_t stream) {
  auto kern = cgemm_b1_tmem_kernel;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles_m = (a.M + TM - 1) / TM, tiles_n = (a.N + UN - 1) / UN;
  const long long units = (long long)tiles_n * a.B;
  if (units * tiles_m > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int grid = (int)(units < num_sms ? units : num_sms);
  kern<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(tmW, tmX, a, tiles_m, tiles_n);
  return cudaGetLastError();
}

}  // namespace tcbf
