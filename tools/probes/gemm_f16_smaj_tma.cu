// PARKED dev probe (not built): the sample-major kernel with the fp32 data staged by TMA (no
// converter global loads; 2 weight stages to make room for a 2 x 16 KB raw ring; 10 converted
// blocks held in registers via setmaxnreg).  Bit-identical; measured 0.72 vs 0.66 ms (300
// launches) and 0.67 vs 0.61 ms (100): the lost weight stage costs more than the LSU relief gains.

// gemm_f16_smaj_tma.cu -- the sample-major fused 16-bit beamformer (gemm_f16_smaj.cu) with the
// fp32 data brought in by TMA instead of by the converter threads' global loads.
//
// Same arithmetic and operand layout as gemm_f16_smaj.cu (fp16 RNE inputs, exact products, fp32
// accumulation in TMEM; [Re | Im] += X_r [W_r ; W_i]^T, Re += (-X_i) W_i^T, Im += X_i W_r^T with
// the samples on the 128 TMEM lanes -- PAPER.md:143-159) and the same epilogue (coalesced line
// stores straight from TMEM).  What changes is how the data reaches the resident operand.
//
// Measured on the load-in-the-converter kernel: the SM's load/store pipeline
// carries the 2.15 GB of output line stores AND the 0.54 GB of fp32 data loads, loads queue behind
// stores (3-7 us per 32 KB block at a unit switch, an ~8 us MMA stall per switch), and with no data
// loads at all the same kernel runs 0.47 instead of 0.62-0.66 ms.  Here a producer warp streams
// the raw fp32 rows (16 k-rows x 128 samples = 16 KB per block, interleaved complex, zero fill past
// K / N) with TMA into a 2-deep staging ring -- the LSU carries only the output stores -- and the
// converter warps turn each staged block into fp16 REGISTERS (8 per thread per block) right away,
// freeing the staging for the next TMA, and write them into the resident slots when the last beam
// tile of the previous unit has released them.  Ten blocks held in registers (setmaxnreg: the
// converters get 128 registers, the producer / MMA warps 32) plus the two staged ones cover 3/4
// of the next unit before the switch; the last quarter streams in while the unit's first tile runs.
//
// smem: resident data 128 KB (4 K blocks of 64 rows, both planes), weights 2 x 32 KB, raw staging
// 2 x 16 KB.  Requirements (checked by the caller): interleaved fp32 source, N even, 16-byte
// aligned base (TMA strides), K16 <= 256.
//
// Roles (20 warps, warpgroup-aligned for setmaxnreg): warps 0-7 epilogue, 8-15 converters,
// 16 weight producer, 17 MMA issuer, 18 raw-data producer, 19 idle.
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
constexpr int BK = 64;                     // k-rows per resident slot / K per weight stage
constexpr int KMAX = 256;
constexpr int W_TILE = BB * BK * 2;        // 16 KB
constexpr int W_STAGE = 2 * W_TILE;        // [W_r ; W_i]
constexpr int W_STAGES = 2;
constexpr int X_PLANE = 2 * KMAX * 128;    // 2 blocks of 64 samples x KMAX k-rows x 128 B
constexpr int RB = 16;                     // k-rows per raw staging block
constexpr int RAW_BYTES = RB * BS * 8;     // 16 KB of interleaved fp32
constexpr int RAW_STAGES = 2;
constexpr int OFF_W = 2 * X_PLANE;
constexpr int OFF_RAW = OFF_W + W_STAGES * W_STAGE;
constexpr int BAR_OFFSET = OFF_RAW + RAW_STAGES * RAW_BYTES;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
static_assert(SMEM_BYTES <= 232448, "smem budget");

constexpr int EPI_WARPS = 8;
constexpr int CONV_WARP0 = 8;
constexpr int CONV_WARPS = 8;
constexpr int WPROD_WARP = 16;
constexpr int MMA_WARP = 17;
constexpr int RPROD_WARP = 18;
constexpr int NUM_THREADS = 20 * 32;
// CTA register pool = the 640 x 96 launch allocation: epilogue 8 x 32 x 96 + converters
// 8 x 32 x 128 + producers / MMA / idle 4 x 32 x 32 = 61440
constexpr int CONV_REGS = 128;
constexpr int LOW_REGS = 32;
constexpr int HOLD = 10;                   // converted blocks held in registers per converter thread

__device__ __forceinline__ uint64_t desc_w(const void* tile, uint32_t k_byte_off) {
  uint32_t addr = smem_u32(tile) + k_byte_off;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__device__ __forceinline__ uint64_t desc_x(const void* plane, uint32_t k_row) {
  uint32_t addr = smem_u32(plane) + k_row * 128u;
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((KMAX * 128u) >> 4) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
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

// A converter warp's share of one 16-row raw block: two k-rows; lane t holds complex samples
// (2t, 2t+1) and (64 + 2t, 65 + 2t) of each, as four fp16 pairs per row: [row][re/im][half]
struct Held {
  uint32_t v[2][2][2];
};

template <int CL>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_f16_smaj_tma_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                              GemmF16Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sX = smem;                // [2 planes][2 sample blocks][KMAX rows][128 B]
  uint8_t* sW = smem + OFF_W;
  uint8_t* sRaw = smem + OFF_RAW;    // [RAW_STAGES][RB rows][128 complex fp32]
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* wempty = wfull + W_STAGES;
  uint64_t* xfull = wempty + W_STAGES;   // [KMAX / BK]
  uint64_t* xempty = xfull + KMAX / BK;
  uint64_t* rfull = xempty + KMAX / BK;  // [RAW_STAGES]
  uint64_t* rempty = rfull + RAW_STAGES;
  uint64_t* tfull = rempty + RAW_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = args.num_kb;              // K16 / 64 <= 4
  const int rpu = args.K16 / RB;               // raw blocks per unit
  const int tiles_m = args.tiles_m, tiles_n = args.tiles_n;
  const int num_units = args.B * tiles_n;
  constexpr bool MC = CL > 1;
  constexpr uint16_t CL_MASK = (uint16_t)((1u << CL) - 1u);
  const int rank = MC ? (int)cluster_ctarank() : 0;
  const int u_first = MC ? CL * (int)(blockIdx.x / CL) + rank : (int)blockIdx.x;
  const int u_step = MC ? CL * (int)(gridDim.x / CL) : (int)gridDim.x;
  const int my_units = u_first < num_units ? (num_units - 1 - u_first) / u_step + 1 : 0;
  const int total = my_units * rpu;            // this CTA's raw blocks, in order

  if (threadIdx.x == 0) {
    for (int s = 0; s < W_STAGES; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], CL);
    }
    for (int s = 0; s < KMAX / BK; ++s) {
      mbar_init(&xfull[s], CONV_WARPS);
      mbar_init(&xempty[s], 1);
    }
    for (int s = 0; s < RAW_STAGES; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], CONV_WARPS);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
  }
  if (warp == MMA_WARP) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  if (MC) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp >= WPROD_WARP) {
    regs_dec<LOW_REGS>();
    if (warp == WPROD_WARP) {
      // ---------------------------------------------------------- TMA producer: weight stages
      if (lane == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int u = u_first; u < num_units; u += u_step) {
          const int b = u / tiles_n;
          for (int mt = 0; mt < tiles_m; ++mt) {
            for (int kb = 0; kb < num_kb; ++kb) {
              mbar_wait(&wempty[stage], phase ^ 1);
              uint8_t* st = sW + stage * W_STAGE;
              mbar_arrive_expect_tx(&wfull[stage], W_STAGE);
#pragma unroll
              for (int bx = rank * (4 / CL); bx < (rank + 1) * (4 / CL); ++bx) {
                uint8_t* dst = st + (bx >> 1) * W_TILE + (bx & 1) * (W_TILE / 2);
                if (MC)
                  tma_load_3d_mc(dst, &tmW, &wfull[stage], kb * BK, mt * BB + (bx & 1) * 64, 2 * b + (bx >> 1),
                                 CL_MASK);
                else
                  tma_load_3d(dst, &tmW, &wfull[stage], kb * BK, mt * BB + (bx & 1) * 64, 2 * b + (bx >> 1));
              }
              if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    } else if (warp == RPROD_WARP) {
      // ---------------------------------------------------------- TMA producer: raw fp32 data rows
      if (lane == 0) {
        for (int r = 0; r < total; ++r) {
          const int s = r % RAW_STAGES;
          mbar_wait(&rempty[s], ((r / RAW_STAGES) & 1) ^ 1);
          const int ui = r / rpu, rb = r - ui * rpu;
          const int u = u_first + ui * u_step;
          const int b = u / tiles_n, n0 = (u - b * tiles_n) * BS;
          mbar_arrive_expect_tx(&rfull[s], RAW_BYTES);
          // interleaved [B][K][2N] fp32: 256 floats (128 complex) x 16 k-rows, zero fill past K / 2N
          tma_load_3d(sRaw + s * RAW_BYTES, &tmX, &rfull[s], 2 * n0, rb * RB, b);
        }
      }
    } else if (warp == MMA_WARP) {
      // ---------------------------------------------------------- MMA issuer (converged warp)
      constexpr uint32_t I256 = idesc_smaj(2 * BB, false);
      constexpr uint32_t I128 = idesc_smaj(BB, false);
      constexpr uint32_t I128_NEG = idesc_smaj(BB, true);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0, ui = 0;
      for (int u = u_first; u < num_units; u += u_step, ++ui) {
        for (int mt = 0; mt < tiles_m; ++mt, ++it) {
          const int abuf = it & 1;
          mbar_wait(&tempty[abuf], ((it >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_re = tmem_base + abuf * 2 * BB;
          const uint32_t d_im = d_re + BB;
          for (int kb = 0; kb < num_kb; ++kb) {
            if (mt == 0) mbar_wait(&xfull[kb], ui & 1);  // the unit's data block is in its slot
            mbar_wait(&wfull[stage], phase);
            tc_fence_after();
            const uint8_t* st = sW + stage * W_STAGE;
            const uint64_t xr0 = desc_x(sX, kb * BK), xi0 = desc_x(sX + X_PLANE, kb * BK);
            const uint64_t wri0 = desc_w(st, 0), wi0 = desc_w(st + W_TILE, 0);
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                const uint64_t xr = xr0 + (uint64_t)(128 * kk), xi = xi0 + (uint64_t)(128 * kk);
                const uint64_t w_ri = wri0 + (uint64_t)(2 * kk), w_i = wi0 + (uint64_t)(2 * kk);
                const uint32_t acc = (kb | kk) ? 1u : 0u;
                if (TCBF_ABLATE(args, 2)) continue;
                mma_f16_ss(d_re, xr, w_ri, I256, acc);      // [Re | Im] += X_r [W_r ; W_i]^T
                mma_f16_ss(d_re, xi, w_i, I128_NEG, 1u);    // Re += -X_i W_i^T
                mma_f16_ss(d_im, xi, w_ri, I128, 1u);       // Im += X_i W_r^T
              }
              if (MC) mma_commit_mc(&wempty[stage], CL_MASK);
              else mma_commit(&wempty[stage]);
              if (mt == tiles_m - 1) mma_commit(&xempty[kb]);  // last reader of this data block
            }
            __syncwarp();
            if (++stage == W_STAGES) { stage = 0; phase ^= 1; }
          }
          if (elect_one()) mma_commit(&tfull[abuf]);
          __syncwarp();
        }
      }
    }
  } else if (warp < CONV_WARP0) {
    // ------------------------------------------------------------ epilogue: coalesced line stores
    const int q = warp & 3;
    const int half = warp >> 2;  // 0: Re, 1: Im
    const size_t N = (size_t)args.N;
    const int M = args.M;
    int it = 0;
    for (int u = u_first; u < num_units; u += u_step) {
      const int b = u / tiles_n;
      const int n = (u - b * tiles_n) * BS + q * 32 + lane;
      const bool n_ok = n < args.N;
      for (int mt = 0; mt < tiles_m; ++mt, ++it) {
        const int abuf = it & 1;
        mbar_wait(&tfull[abuf], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 2 * BB + half * BB;
        uint32_t v[2][32];
        tmem_ld_32x32b_x32(tbase, v[0]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int m0 = mt * BB + i * 32;
          tmem_wait_ld();
          if (i + 1 < 4) {
            tmem_ld_32x32b_x32(tbase + (i + 1) * 32, v[(i + 1) & 1]);
          } else {
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
      }
    }
  } else {
    // ------------------------------------------------------------ converters: staged fp32 -> fp16
    regs_inc<CONV_REGS>();
    const int cw = warp - CONV_WARP0;  // rows 2cw, 2cw+1 of every raw block
    // raw block r (TMA-staged) -> this thread's four fp16 pairs per row; frees the staging
    auto convert = [&](int r, Held& h) {
      const int s = r % RAW_STAGES;
      mbar_wait(&rfull[s], (r / RAW_STAGES) & 1);
      const uint8_t* raw = sRaw + s * RAW_BYTES;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float4* row = reinterpret_cast<const float4*>(raw + (2 * cw + j) * (BS * 8));
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {  // samples 64 hh + 2 lane, +1 (consecutive 16 B per lane)
          const float4 f = TCBF_ABLATE(args, 4) ? make_float4(0.f, 0.f, 0.f, 0.f) : row[hh * 32 + lane];
          h.v[j][0][hh] = h2u(f.x, f.z);  // re(2t), re(2t+1)
          h.v[j][1][hh] = h2u(f.y, f.w);  // im(2t), im(2t+1)
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&rempty[s]);
    };
    // held block r -> the resident slot of its K block (waiting for the slot on the first block)
    auto store = [&](int r, const Held& h) {
      const int ui = r / rpu, rb = r - ui * rpu;
      const int kb = (rb * RB) / BK;
      if ((rb * RB) % BK == 0) mbar_wait(&xempty[kb], (ui & 1) ^ 1);  // slot released by the last tile
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int k = rb * RB + 2 * cw + j;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {  // 64-sample block hh: sample 2 lane, 128-byte swizzle
          const int off = hh * (KMAX * 128) + k * 128 + ((((2 * lane) >> 3) ^ (k & 7)) << 4) + ((2 * lane) & 7) * 2;
          *reinterpret_cast<uint32_t*>(sX + off) = h.v[j][0][hh];
          *reinterpret_cast<uint32_t*>(sX + X_PLANE + off) = h.v[j][1][hh];
        }
      }
      if ((rb * RB + RB) % BK == 0) {  // last raw block of the slot: the slot is complete
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&xfull[kb]);
      }
    };
    // HOLD converted blocks in flight in registers (the ring is unrolled: static indices)
    Held hold[HOLD];
    for (int r0 = 0; r0 < total + HOLD; r0 += HOLD) {
#pragma unroll
      for (int i = 0; i < HOLD; ++i) {
        const int r = r0 + i;
        if (r >= HOLD && r - HOLD < total) store(r - HOLD, hold[i]);
        if (r < total) convert(r, hold[i]);
      }
    }
  }

  tc_fence_before();
  if (MC) cluster_sync(); else __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

template <int CL>
cudaError_t launch_smaj_tma(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmF16Args& a, int num_sms,
                            cudaStream_t s) {
  auto kern = cgemm_f16_smaj_tma_kernel<CL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int units = a.B * a.tiles_n;
  if (CL == 1) {
    const int grid = units < num_sms ? units : num_sms;
    kern<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(tmW, tmX, a);
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
  e = cudaLaunchKernelEx(&cfg, kern, tmW, tmX, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

// the TMA-staged variant applies to an interleaved source with N even and a 16-byte aligned base
// (the raw rows are 8N bytes apart) and K16 <= 256
bool gemm_f16_smaj_tma_supported(int64_t K16, int64_t N, int layout, const void* x_src) {
  return K16 <= KMAX && layout == 0 && (N % 2) == 0 && (reinterpret_cast<uintptr_t>(x_src) % 16) == 0;
}
int gemm_f16_smaj_tma_raw_rows() { return RB; }

// args as launch_gemm_f16_smaj (num_kb = K16 / 64); tmW: box {64 K, 64 beam rows} per plane,
// 128-byte swizzle; tmX: the interleaved fp32 source as [B][K][2N] floats, box {256, 16}, no swizzle
cudaError_t launch_gemm_f16_smaj_tma(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmF16Args& args,
                                     int cluster, int num_sms, cudaStream_t stream) {
  const int units = args.B * args.tiles_n;
  if (cluster >= 2 && args.tiles_n % 2 == 0 && units >= 2) return launch_smaj_tma<2>(tmW, tmX, args, num_sms, stream);
  return launch_smaj_tma<1>(tmW, tmX, args, num_sms, stream);
}

}  // namespace tcbf
