// PARKED EXPERIMENT (not built into libtcbf.so): bit-identical to pack + beamform but
// measured 1.17 ms against 0.69 ms for gemm_f16_fused.cu on radio fp16 -- the loader warps' plain
// global loads (one K block of register look-ahead, 80 registers per thread at 672 threads) cannot
// keep the TMEM weight ring fed: with MMAs and stores skipped it still takes 0.72 ms.
//
// gemm_f16_fusedw.cu -- the fused fp32-data 16-bit beamformer kernel (gemm_f16_fused.cu) with the
// WEIGHTS in tensor memory: the design that took the fp4 1-bit kernel from 0.79 to 0.92 of its roof,
// applied to the short-K radio shape (PAPER.md:143-159 arithmetic, PAPER.md:414 fused pack).
//
//   * unit = (batch entry, 128 data columns); the unit's data is converted once by 8 converter
//     warps into a shared-memory-resident MN-major fp16 B operand (as in gemm_f16_fused.cu);
//   * 8 loader warps read the packed fp16 weights of the current 128-beam tile with plain global
//     loads (thread = weight row, one plane per warp pair) and write them with tcgen05.st into a
//     4-deep TMEM ring of 64-K stages (A_r 32 columns | A_i 32 columns); the MMAs take A from TMEM,
//     so shared memory carries only the B operand reads, the conversion and the epilogue staging;
//   * TMEM: one accumulator buffer [D_re | D_im] (columns 0..255) + the weight ring (256..511);
//     the epilogue drains TMEM through a 6-box (96 KB) smem staging ring into TMA stores, so the
//     next tile's MMAs wait only for the TMEM reads.
// Bit-identical to pack + beamform (same products, negation on the B operand, same K order).
// Opt-in (TCBF_F16_FUSED=4) until measured faster.
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 64;
constexpr int KMAX = 256;
constexpr int W_STAGES = 4;               // TMEM weight ring (64 columns each)
constexpr int EPI_WARPS = 4;
constexpr int CONV_WARPS = 8;
constexpr int LOAD_WARPS = 8;
constexpr int NUM_THREADS = (1 + EPI_WARPS + CONV_WARPS + LOAD_WARPS) * 32;
constexpr int B_PLANE_BYTES = 2 * KMAX * 128;
constexpr int NBOX = 6;                   // epilogue staging boxes (128 rows x 32 columns fp32)
constexpr int OFF_B = 0;
constexpr int OFF_EPI = 2 * B_PLANE_BYTES;
constexpr int BAR_OFFSET = OFF_EPI + NBOX * 16384;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
constexpr uint32_t W_COL = 256;
static_assert(SMEM_BYTES <= 232448, "smem budget");

__device__ __forceinline__ uint64_t desc_b_res(const void* plane, uint32_t k_row) {
  uint32_t addr = smem_u32(plane) + k_row * 128u;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((KMAX * 128u) >> 4) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_st_u4x8(uint32_t taddr, const uint4 (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(v[0].x), "r"(v[0].y), "r"(v[0].z), "r"(v[0].w), "r"(v[1].x), "r"(v[1].y), "r"(v[1].z), "r"(v[1].w),
      "r"(v[2].x), "r"(v[2].y), "r"(v[2].z), "r"(v[2].w), "r"(v[3].x), "r"(v[3].y), "r"(v[3].z), "r"(v[3].w),
      "r"(v[4].x), "r"(v[4].y), "r"(v[4].z), "r"(v[4].w), "r"(v[5].x), "r"(v[5].y), "r"(v[5].z), "r"(v[5].w),
      "r"(v[6].x), "r"(v[6].y), "r"(v[6].z), "r"(v[6].w), "r"(v[7].x), "r"(v[7].y), "r"(v[7].z), "r"(v[7].w)
      : "memory");
}
__device__ __forceinline__ uint32_t h2u(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int LAYOUT, bool VEC>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_fusedw_kernel(const __grid_constant__ CUtensorMap tmC, GemmF16Args args, const uint16_t* __restrict__ wp,
                            const float* __restrict__ xsrc, int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem + OFF_B;
  uint8_t* epi_base = smem + OFF_EPI;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* wempty = wfull + W_STAGES;
  uint64_t* bfull = wempty + W_STAGES;
  uint64_t* bempty = bfull + KMAX / BK;
  uint64_t* tfull = bempty + KMAX / BK;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = args.num_kb;
  const int tiles_m = args.tiles_m, tiles_n = args.tiles_n;
  const int num_units = args.B * tiles_n;
  const int M = args.M, K16 = args.K16;

  if (threadIdx.x == 0) {
    for (int s = 0; s < W_STAGES; ++s) {
      mbar_init(&wfull[s], LOAD_WARPS);
      mbar_init(&wempty[s], 1);
    }
    for (int s = 0; s < KMAX / BK; ++s) {
      mbar_init(&bfull[s], CONV_WARPS);
      mbar_init(&bempty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, EPI_WARPS);
    fence_barrier_init();
    tma_prefetch_desc(&tmC);
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // kind::f16, F32 D, A from TMEM, B MN-major (bit 16), N = 128, M = 128; A_i.B_i negates B
      constexpr uint32_t IDESC = (1u << 4) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      constexpr uint32_t IDESC_NEGB = IDESC | (1u << 14);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0, ui = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++ui) {
        const uint32_t bphase = ui & 1;
        for (int mt = 0; mt < tiles_m; ++mt, ++it) {
          mbar_wait(tempty, (it & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_re = tmem_base, d_im = tmem_base + BN;
          for (int kb = 0; kb < num_kb; ++kb) {
            if (mt == 0) mbar_wait(&bfull[kb], bphase);
            mbar_wait(&wfull[stage], phase);
            tc_fence_after();
            const uint32_t wa = tmem_base + W_COL + 64 * stage;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t krow = kb * BK + kk * 16;
              const uint32_t ar = wa + kk * 8, ai = wa + 32 + kk * 8;
              const uint64_t br = desc_b_res(sB, krow), bi = desc_b_res(sB + B_PLANE_BYTES, krow);
              const uint32_t acc = (kb | kk) ? 1u : 0u;
              if (args.debug & 2) continue;
              mma_f16_ts(d_re, ar, br, IDESC, acc);
              mma_f16_ts(d_re, ai, bi, IDESC_NEGB, 1u);
              mma_f16_ts(d_im, ar, bi, IDESC, acc);
              mma_f16_ts(d_im, ai, br, IDESC, 1u);
            }
            mma_commit(&wempty[stage]);
            if (mt == tiles_m - 1) mma_commit(&bempty[kb]);
            if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
          }
          mma_commit(tfull);
        }
      }
    }
  } else if (warp <= EPI_WARPS) {
    // ------------------------------------------------------------ epilogue: TMEM -> 6-box smem ring -> TMA
    const int q = warp & 3;
    int box = 0;
    int it = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      const int b = u / tiles_n;
      const int n0 = (u - b * tiles_n) * BN;
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int m0 = mt * BM;
        mbar_wait(tfull, it & 1);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16);
        uint32_t v[2][32];
        tmem_ld_32x32b_x32(tbase, v[0]);
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {  // (Re, 4 chunks of 32 columns), (Im, 4 chunks)
          tmem_wait_ld();
          if (ch + 1 < 8) {
            tmem_ld_32x32b_x32(tbase + (ch + 1) * 32, v[(ch + 1) & 1]);
          } else {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty);  // TMEM drained: the next tile's MMAs may start
          }
          const uint32_t* vv = v[ch & 1];
          if (args.debug & 1) continue;
          uint8_t* buf = epi_base + box * 16384;
          if (threadIdx.x == 32) bulk_wait_group_read<NBOX - 1>();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          const int row = q * 32 + lane;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int pos = j ^ (row & 7);
            *reinterpret_cast<uint4*>(buf + row * 128 + pos * 16) =
                make_uint4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]);
          }
          fence_proxy_async_smem();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (threadIdx.x == 32) {
            tma_store_3d(&tmC, buf, n0 + (ch & 3) * 32, m0, 2 * b + (ch >> 2));
            bulk_commit_group();
          }
          box = box + 1 == NBOX ? 0 : box + 1;
        }
      }
    }
    if (threadIdx.x == 32) bulk_wait_group<0>();
  } else if (warp <= EPI_WARPS + CONV_WARPS) {
    // ------------------------------------------------------------ converters: fp32 data -> resident B
    const int ct = threadIdx.x - (1 + EPI_WARPS) * 32;  // 0..255
    constexpr int NT = CONV_WARPS * 32;
    constexpr int ITEMS = BK * (BN / 8) / NT;
    const int N = args.N;
    int ui = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++ui) {
      const int b = u / tiles_n;
      const int n0 = (u - b * tiles_n) * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        float re[ITEMS][8], im[ITEMS][8];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int item = ct + i * NT;
          const int kr = item / (BN / 8), cc = item % (BN / 8);
          const int k = kb * BK + kr, n = n0 + cc * 8;
          if (VEC && LAYOUT == 0 && k < K && n + 8 <= N) {
            const float4* p = reinterpret_cast<const float4*>(xsrc + (((size_t)b * K + k) * N + n) * 2);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 f = __ldg(p + j);
              re[i][2 * j] = f.x; im[i][2 * j] = f.y; re[i][2 * j + 1] = f.z; im[i][2 * j + 1] = f.w;
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
              re[i][j] = a; im[i][j] = c;
            }
          }
        }
        mbar_wait(&bempty[kb], (ui & 1) ^ 1);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int item = ct + i * NT;
          const int kr = item / (BN / 8), cc = item % (BN / 8);
          const int k = kb * BK + kr;
          const int off = (cc >> 3) * (KMAX * 128) + k * 128 + (((cc & 7) ^ (k & 7)) << 4);
          *reinterpret_cast<uint4*>(sB + off) = make_uint4(h2u(re[i][0], re[i][1]), h2u(re[i][2], re[i][3]),
                                                           h2u(re[i][4], re[i][5]), h2u(re[i][6], re[i][7]));
          *reinterpret_cast<uint4*>(sB + B_PLANE_BYTES + off) = make_uint4(
              h2u(im[i][0], im[i][1]), h2u(im[i][2], im[i][3]), h2u(im[i][4], im[i][5]), h2u(im[i][6], im[i][7]));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bfull[kb]);
      }
    }
  } else {
    // ------------------------------------------------------------ loaders: packed weights -> TMEM ring
    // warp w writes TMEM lanes 32 (w % 4) ..; warps 13-16 load plane Re, 17-20 plane Im
    const int lw = warp - (1 + EPI_WARPS + CONV_WARPS);  // 0..7
    const int plane = lw >> 2;
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int stage = 0;
    uint32_t phase = 0;
    // flat stream of (unit, tile, K block) with one K block of look-ahead in registers
    int lu = blockIdx.x, lmt = 0, lkb = 0;
    auto load = [&](uint4 (&d)[8]) {
      const uint4 zero = make_uint4(0, 0, 0, 0);
      if (lu < num_units) {
        const int b = lu / tiles_n;
        const int m = lmt * BM + row;
        if (m < M) {
          const uint4* src = reinterpret_cast<const uint4*>(wp + (((size_t)b * 2 + plane) * M + m) * K16 + lkb * BK);
#pragma unroll
          for (int j = 0; j < 8; ++j) d[j] = __ldg(src + j);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) d[j] = zero;
        }
      }
      if (++lkb == num_kb) {
        lkb = 0;
        if (++lmt == tiles_m) { lmt = 0; lu += gridDim.x; }
      }
    };
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16) + W_COL + 32 * plane;
    auto put = [&](const uint4 (&d)[8]) {
      mbar_wait(&wempty[stage], phase ^ 1);
      tc_fence_after();
      tmem_st_u4x8(lane_base + 64 * stage, d);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&wfull[stage]);
      if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
    };
    uint4 ra[8], rb[8];  // ping-pong: the next K block's loads are in flight while one is stored
    load(ra);
    const int my_units = blockIdx.x < (unsigned)num_units ? (num_units - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int total = my_units * tiles_m * num_kb;
    for (int s = 0; s < total; s += 2) {
      load(rb);
      put(ra);
      if (s + 1 >= total) break;
      load(ra);
      put(rb);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

template <int LAYOUT, bool VEC>
cudaError_t launch_w(const CUtensorMap& tmC, const GemmF16Args& a, const uint16_t* w, const float* x, int K,
                     int num_sms, cudaStream_t s) {
  auto kern = cgemm_f16_fusedw_kernel<LAYOUT, VEC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int units = a.B * a.tiles_n;
  const int grid = units < num_sms ? units : num_sms;
  kern<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(tmC, a, w, x, K);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemm_f16_fusedw(const CUtensorMap& tmC, const GemmF16Args& args, const void* w_packed,
                                   const float* x_src, int layout, int K, int num_sms, cudaStream_t stream) {
  const uint16_t* w = static_cast<const uint16_t*>(w_packed);
  const bool vec = layout == 0 && (args.N % 8 == 0) && (reinterpret_cast<uintptr_t>(x_src) % 16 == 0);
  if (layout == 0)
    return vec ? launch_w<0, true>(tmC, args, w, x_src, K, num_sms, stream)
               : launch_w<0, false>(tmC, args, w, x_src, K, num_sms, stream);
  return launch_w<1, false>(tmC, args, w, x_src, K, num_sms, stream);
}

}  // namespace tcbf
