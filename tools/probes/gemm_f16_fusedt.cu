// PARKED EXPERIMENT (not built into libtcbf.so; kept for the record): measured 0.76-0.80 ms
// against 0.685 ms for gemm_f16_fused.cu on radio fp16 -- the M=128 N=64 MMAs that TMEM capacity forces
// (256 data columns + 2 x 128 accumulator columns) run at 1412 TFLOP/s against 1893 for N=128
// (peaks.cu kinds 6 / 7), and the MMA path alone took 0.65 ms instead of 0.44.  Numerically correct
// (equal to pack + beamform to rounding), not bit-identical.  To try it: copy into csrc/ and wire a
// launch in plan.cu as gemm_f16_fused.cu is.
//
// gemm_f16_fusedt.cu -- 16-bit-mode beamformer GEMM from fp32 data with the DATA operand resident in
// TENSOR MEMORY (the transposed form of gemm_f16_fused.cu; the data pack of PAPER.md:107 fused
// into the GEMM).
//
// Same arithmetic (fp16 RNE inputs, four real sub-GEMMs per K step, fp32 accumulation in TMEM --
// PAPER.md:143-159), computed as the transposed product  C^T[b] = X[b]^T W[b]^T  so that the
// operand reused by every tile of a work unit can live in TMEM:
//
//   * work unit = (batch entry, 128 samples); the converter warps turn the unit's fp32 data
//     X[b][0:K][n0:n0+128] into fp16 ONCE and write it straight from registers into TMEM with
//     tcgen05.st (lane = sample, two K elements per 32-bit column, planes X_r / X_i), where it is
//     the A operand of every MMA of the unit (tcgen05.mma with A in TMEM);
//   * the weights stream through a TMA ring as the B operand (64 beams x 64 K per stage and
//     plane, K-major, 128-byte swizzle): the only shared-memory operand traffic left is the
//     weight tile (2 KB per M=128 N=64 K=16 MMA instead of 8 KB for A and B from smem);
//   * accumulators: D_re | D_im, 64 beams each, double-buffered (2 x 128 columns beside the 256
//     columns of resident data);
//   * epilogue: TMEM lane = sample, so after tcgen05.ld a warp holds 32 consecutive samples of a
//     beam row -- plain coalesced 128-byte st.global per beam, no shared-memory staging.
//
// Per 128-sample unit this moves ~3 MB through shared memory instead of ~7 MB.
// K16 <= 256 (the resident data uses 2 x 128 TMEM columns).  Bit-identical to pack + beamform:
// the same products are summed in the same K order into fp32.
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int UN = 128;        // samples per unit (MMA M)
constexpr int BNB = 64;        // beams per tile (MMA N)
constexpr int BK = 64;         // K per weight stage / per converted data block
constexpr int KMAX = 256;      // resident K
constexpr int W_STAGES = 8;
constexpr int W_PLANE = BNB * BK * 2;      // 8 KB: 64 beams x 128 B
constexpr int W_STAGE = 2 * W_PLANE;       // W_r, W_i
constexpr int EPI_WARPS = 4;
constexpr int CONV_WARPS = 8;
constexpr int NUM_THREADS = (2 + EPI_WARPS + CONV_WARPS) * 32;
constexpr int BAR_OFFSET = W_STAGES * W_STAGE;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 512;
constexpr uint32_t X_COL = 0;              // X_r^T columns [0,128), X_i^T [128,256)
constexpr uint32_t ACC_COL = 256;          // accumulator buffers: [256,384), [384,512)
static_assert(SMEM_BYTES <= 232448, "smem budget");

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
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t h2u(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int LAYOUT>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_fusedt_kernel(const __grid_constant__ CUtensorMap tmW, GemmF16Args args, const float* __restrict__ xsrc,
                            int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* wempty = wfull + W_STAGES;
  uint64_t* xfull = wempty + W_STAGES;   // [KMAX / BK]
  uint64_t* xempty = xfull + KMAX / BK;  // [KMAX / BK]
  uint64_t* tfull = xempty + KMAX / BK;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = args.num_kb;            // K16 / 64 <= 4
  const int tiles_m = args.tiles_m;          // beam tiles of 64
  const int tiles_n = args.tiles_n;          // sample units of 128
  const int num_units = args.B * tiles_n;
  const int M = args.M, N = args.N;

  if (threadIdx.x == 0) {
    for (int s = 0; s < W_STAGES; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);
    }
    for (int s = 0; s < KMAX / BK; ++s) {
      mbar_init(&xfull[s], CONV_WARPS / 4 * 4);  // every converter warp writes part of each block
      mbar_init(&xempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmW);
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer: weight tiles
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        const int b = u / tiles_n;
        for (int mt = 0; mt < tiles_m; ++mt) {
          for (int kb = 0; kb < num_kb; ++kb) {
            mbar_wait(&wempty[stage], phase ^ 1);
            uint8_t* st = smem + stage * W_STAGE;
            mbar_arrive_expect_tx(&wfull[stage], W_STAGE);
            tma_load_3d(st, &tmW, &wfull[stage], kb * BK, mt * BNB, 2 * b);
            tma_load_3d(st + W_PLANE, &tmW, &wfull[stage], kb * BK, mt * BNB, 2 * b + 1);
            if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // kind::f16: D F32, A/B F16, A from TMEM (K-major), B K-major, N = 64, M = 128;
      // the X_i . W_i product negates B (bit 14)
      constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BNB >> 3) << 17) | ((uint32_t)(UN >> 4) << 24);
      constexpr uint32_t IDESC_NEGB = IDESC | (1u << 14);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0, ui = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++ui) {
        const uint32_t xphase = ui & 1;
        for (int mt = 0; mt < tiles_m; ++mt, ++it) {
          const int abuf = it & 1;
          mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_re = tmem_base + ACC_COL + abuf * 2 * BNB;
          const uint32_t d_im = d_re + BNB;
          for (int kb = 0; kb < num_kb; ++kb) {
            if (mt == 0) mbar_wait(&xfull[kb], xphase);  // the unit's data block is in TMEM
            mbar_wait(&wfull[stage], phase);
            tc_fence_after();
            uint8_t* st = smem + stage * W_STAGE;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t xc = X_COL + (uint32_t)(kb * BK + kk * 16) / 2;  // 2 fp16 per column
              const uint32_t xr = tmem_base + xc, xi = tmem_base + xc + KMAX / 2;
              const uint64_t wr = smem_desc_k128(st, kk * 32), wi = smem_desc_k128(st + W_PLANE, kk * 32);
              const uint32_t acc = (kb | kk) ? 1u : 0u;
              if (args.debug & 2) continue;
              mma_f16_ts(d_re, xr, wr, IDESC, acc);
              mma_f16_ts(d_re, xi, wi, IDESC_NEGB, 1u);
              mma_f16_ts(d_im, xr, wi, IDESC, acc);
              mma_f16_ts(d_im, xi, wr, IDESC, 1u);
            }
            mma_commit(&wempty[stage]);
            if (mt == tiles_m - 1) mma_commit(&xempty[kb]);  // last reader of this data block
            if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
          }
          mma_commit(&tfull[abuf]);
        }
      }
    }
  } else if (warp < 2 + EPI_WARPS) {
    // ------------------------------------------------------------ epilogue: coalesced stores
    const int q = warp & 3;  // TMEM lane quarter = samples 32q .. 32q+31 of the unit
    int it = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      const int b = u / tiles_n;
      const int n = (u - b * tiles_n) * UN + q * 32 + lane;  // this thread's sample
      const bool n_ok = n < N;
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int abuf = it & 1;
        mbar_wait(&tfull[abuf], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + ACC_COL + abuf * 2 * BNB;
        uint32_t v[2][32];
        tmem_ld_32x32b_x32(tb, v[0]);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {  // (Re, beams 0-31), (Re, 32-63), (Im, 0-31), (Im, 32-63)
          tmem_wait_ld();
          if (ch + 1 < 4) {
            tmem_ld_32x32b_x32(tb + (ch + 1) * 32, v[(ch + 1) & 1]);
          } else {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[abuf]);
          }
          if (args.debug & 1) continue;
          const int part = ch >> 1;
          const int mb = mt * BNB + (ch & 1) * 32;
          float* col = args.out + ((size_t)(2 * b + part) * M + mb) * (size_t)N + n;
          const uint32_t* vv = v[ch & 1];
          if (n_ok) {
            if (mb + 32 <= M) {
#pragma unroll
              for (int j = 0; j < 32; ++j) col[(size_t)j * N] = __uint_as_float(vv[j]);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (mb + j < M) col[(size_t)j * N] = __uint_as_float(vv[j]);
            }
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ converters: fp32 data -> TMEM
    // warp w may access TMEM lanes 32 (w % 4) ..; two warps per lane quarter split each 64-K block
    // into halves: thread = one sample, 32 K rows -> 16 columns of X_r and 16 of X_i
    const int cw = warp - (2 + EPI_WARPS);  // 0..7
    const int q = warp & 3;
    const int half = cw >> 2;               // K rows [32 half, 32 half + 32) of each block
    int ui = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++ui) {
      const int b = u / tiles_n;
      const int n = (u - b * tiles_n) * UN + q * 32 + lane;
      const bool n_ok = n < N;
      for (int kb = 0; kb < num_kb; ++kb) {
        const int k0 = kb * BK + half * 32;
        float re[32], im[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {  // loads first (all in flight), coalesced across the warp
          const int k = k0 + j;
          float a = 0.f, c = 0.f;
          if (n_ok && k < K) {
            if (LAYOUT == 0) {
              const float2 f = __ldg(reinterpret_cast<const float2*>(xsrc) + ((size_t)b * K + k) * N + n);
              a = f.x; c = f.y;
            } else {
              a = __ldg(xsrc + (((size_t)b * 2 + 0) * K + k) * N + n);
              c = __ldg(xsrc + (((size_t)b * 2 + 1) * K + k) * N + n);
            }
          }
          re[j] = a; im[j] = c;
        }
        mbar_wait(&xempty[kb], (ui & 1) ^ 1);
        tc_fence_after();
        uint32_t pr[16], pi[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          pr[j] = h2u(re[2 * j], re[2 * j + 1]);
          pi[j] = h2u(im[2 * j], im[2 * j + 1]);
        }
        const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + X_COL + (uint32_t)k0 / 2;
        tmem_st_32x32b_x16(ta, pr);
        tmem_st_32x32b_x16(ta + KMAX / 2, pi);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&xfull[kb]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace

int gemm_f16_fusedt_block_n() { return BNB; }

cudaError_t launch_gemm_f16_fusedt(const CUtensorMap& tmW, const GemmF16Args& args, const float* x_src, int layout,
                                   int K, int num_sms, cudaStream_t stream) {
  auto kern = layout == 0 ? cgemm_f16_fusedt_kernel<0> : cgemm_f16_fusedt_kernel<1>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int units = args.B * args.tiles_n;
  const int grid = units < num_sms ? units : num_sms;
  kern<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(tmW, args, x_src, K);
  return cudaGetLastError();
}

}  // namespace tcbf
