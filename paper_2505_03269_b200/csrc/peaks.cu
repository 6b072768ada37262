// peaks.cu -- register/shared-memory-only peak micro-benchmarks for the 1-bit and 16-bit
// beamformer arithmetic on sm_100a: the analogue of the paper's cudapeak measurements
// (Table I), which establish the tensor-core ceilings the
// roofline is drawn against (no datasheet b1 peak exists for B200).
//
// No global-memory traffic inside the timed loops.  Measured kinds (enum tcbf_peak_kind):
//   0  mma.sync m16n8k256 .b1 .and.popc  (the paper's sm_90 AND form)
//   1  mma.sync m16n8k256 .b1 .xor.popc  (the paper's sm_80 XOR form)
//   2  CUDA-core LOP3 XOR + POPC + IADD  (32 binary MACs per instruction triple)
//   3  tcgen05.mma kind::f16   M=128 N=256 K=16, fp32 accumulate (smem operands, TMEM D)
//   4  tcgen05.mma kind::i8    M=128 N=256 K=32, int32 accumulate
//   5  tcgen05.mma kind::mxf4  M=128 N=256 K=64, block32 unit scales, fp32 accumulate
//   6  tcgen05.mma kind::f16   M=128 N=64  K=16, A from TMEM (the data-in-TMEM fused variant)
//   7  tcgen05.mma kind::f16   M=128 N=128 K=16, both operands from smem (the fused kernel's MMA)
//   8  tcgen05.mma kind::mxf4  M=128 N=64  K=64, A from TMEM (the swapped small-M 1-bit kernel, TM=32)
//   9  tcgen05.mma kind::mxf4  M=128 N=64  K=64, both operands from smem
//  10  tcgen05.mma kind::mxf4  M=128 N=128 K=64, A from TMEM (swapped kernel, TM=64)
//  11  tcgen05.mma kind::f16   M=128 N=128 K=16, A from TMEM
//  12  the data-in-TMEM radio kernel's K step: N=128 + N=64 (negate B) + N=64, A from TMEM
//  13  tcgen05.mma kind::f16   M=128 N=32 K=16, A from TMEM
//  14  the same K step for 32-beam tiles: N=64 + 2 x N=32, A from TMEM
// (every tensor kind issued from a converged warp through elect.sync since round 2)
// Ops are counted as 2 per multiply-accumulate (binary MACs for kinds 0-2).  Host entry point:
// tcbf_peak_run (extern "C"), timed with CUDA events around one launch after a warm-up launch.
// This library is a measurement tool: it is not on the beamforming path.
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int B1_CHAINS = 8;  // independent accumulator sets per warp (hides MMA latency)

template <bool XOR>
__global__ void __launch_bounds__(256) peak_b1_mma_kernel(const uint32_t* seed, int iters, int32_t* sink) {
  const uint32_t s = seed[threadIdx.x & 31] ^ blockIdx.x;
  uint32_t a0 = s, a1 = s * 3u, a2 = s * 5u, a3 = s * 7u, b0 = ~s, b1v = s ^ 0x5555u;
  int32_t d[B1_CHAINS][4];
#pragma unroll
  for (int c = 0; c < B1_CHAINS; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < B1_CHAINS; ++c) {
      if (XOR) {
        asm volatile(
            "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.xor.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1v));
      } else {
        asm volatile(
            "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1v));
      }
    }
  }
  int32_t acc = 0;
#pragma unroll
  for (int c = 0; c < B1_CHAINS; ++c) acc += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (acc == 0x7FFFFFFF) sink[0] = acc;  // keeps the loop alive
}

constexpr int POPC_CHAINS = 8;

__global__ void __launch_bounds__(256) peak_popc_kernel(const uint32_t* seed, int iters, int32_t* sink) {
  uint32_t a[POPC_CHAINS];
  int32_t acc[POPC_CHAINS];
#pragma unroll
  for (int c = 0; c < POPC_CHAINS; ++c) {
    a[c] = seed[(threadIdx.x + c) & 31] * (2u * c + 1u);
    acc[c] = 0;
  }
  uint32_t b = seed[0] ^ threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int c = 0; c < POPC_CHAINS; ++c) acc[c] += __popc(a[c] ^ (b + r));
    }
    b += 0x9E3779B9u;  // one IADD per 32 XOR+POPC+IADD triples: the loop is not invariant
  }
  int32_t t = 0;
#pragma unroll
  for (int c = 0; c < POPC_CHAINS; ++c) t += acc[c];
  if (t == 0x7FFFFFFF) sink[0] = t;
}

// ---------------------------------------------------------------- tcgen05 smem-only MMA loop
// A tile 128 rows x 128 B and B tile 256 rows x 128 B, K-major, 128-byte swizzle, filled with a
// hashed bit pattern (finite fp16 / e2m1 / int8 values, so the datapath toggles as on real data).
constexpr int TC_A_BYTES = 128 * 128;
constexpr int TC_B_BYTES = 256 * 128;
constexpr int TC_SMEM = 1024 + TC_A_BYTES + TC_B_BYTES + 64;

__device__ __forceinline__ void mma_mxf4_peak(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t sfa, uint32_t sfb) {
  asm volatile(
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], 1;" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb)
      : "memory");
}
__device__ __forceinline__ void tmem_st_same(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
      "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
      "r"(v)
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void mma_mxf4_ts_peak(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t sfa, uint32_t sfb) {
  asm volatile(
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], 1;" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb)
      : "memory");
}
__device__ __forceinline__ void mma_f16_ts_peak(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc) {
  asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(d_tmem), "r"(a_tmem), "l"(bdesc),
               "r"(idesc)
               : "memory");
}

template <int KIND>  // 3 f16, 4 i8, 5 mxf4, 6 f16 A-in-TMEM N=64, 7 f16 N=128, 8-10 mxf4 N=64/128
__global__ void __launch_bounds__(128, 1) peak_tc_kernel(int iters, int32_t* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + TC_A_BYTES;
  uint64_t* done = reinterpret_cast<uint64_t*>(sB + TC_B_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5;

  // operand fill: fp16 values in [-1, 1) (exponent bits cleared of inf/nan), int8 anything,
  // e2m1 nibbles anything (all finite)
  for (int i = threadIdx.x; i < (TC_A_BYTES + TC_B_BYTES) / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 0x9E3779B9u ^ (blockIdx.x * 0x85EBCA6Bu);
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 13;
    if (KIND == 3 || KIND == 6 || KIND == 7 || KIND >= 11) h &= 0xBBFFBBFFu;  // clear exponent MSB -> |x| < 2 in both halves
    reinterpret_cast<uint32_t*>(smem)[i] = h;
  }
  if (threadIdx.x == 0) {
    mbar_init(done, 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (KIND == 5 || KIND >= 8) {  // unit UE8M0 block scales in columns 256..511
    const uint32_t lanes = (uint32_t)(warp * 32) << 16;
    for (uint32_t c = 256; c < 512; c += 32) tmem_st_same(tmem + lanes + c, 0x7F7F7F7Fu);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  if (warp == 0) {  // converged warp, one elected lane issues (descriptors in uniform registers)
    uint32_t idesc;
    if (KIND == 3) idesc = idesc_f16(128, 256, false);
    else if (KIND == 6) idesc = idesc_f16(128, 64, false);
    else if (KIND == 11 || KIND == 12) idesc = idesc_f16(128, 128, false);
    else if (KIND == 13) idesc = idesc_f16(128, 32, false);
    else if (KIND == 14) idesc = idesc_f16(128, 64, false);
    else if (KIND == 7) idesc = idesc_f16(128, 128, false);
    else if (KIND == 4) idesc = idesc_s8(128, 256);
    else idesc = (1u << 7) | (1u << 10) | (((KIND == 8 || KIND == 9 ? 64u : KIND == 10 ? 128u : 256u) >> 3) << 17) |
                 (1u << 23) | ((128u >> 4) << 24);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {  // 4 x 32 bytes of K per 128-byte row
        const uint64_t ad = smem_desc_k128(sA, kk * 32), bd = smem_desc_k128(sB, kk * 32);
        if (!elect_one()) continue;
        if (KIND == 14) {  // the same K step for 32-beam tiles: N=64 + 2 x N=32
          constexpr uint32_t I32 = idesc_f16(128, 32, false), I32N = idesc_f16(128, 32, false) | (1u << 14);
          const uint64_t bw = smem_desc_k128(sB, kk * 32), bwi = bw + (uint64_t)((32 * 128) >> 4);
          mma_f16_ts_peak(tmem + 256, tmem + kk * 8, bw, idesc);
          mma_f16_ts_peak(tmem + 256, tmem + 128 + kk * 8, bwi, I32N);
          mma_f16_ts_peak(tmem + 256 + 32, tmem + 128 + kk * 8, bw, I32);
          continue;
        }
        if (KIND == 13) { mma_f16_ts_peak(tmem + 256, tmem + kk * 8, bd, idesc); continue; }
        if (KIND == 12) {  // the data-in-TMEM radio kernel's K step: [Re|Im] += X_r [W_r;W_i], Re -= X_i W_i, Im += X_i W_r
          constexpr uint32_t I64 = idesc_f16(128, 64, false), I64N = idesc_f16(128, 64, false) | (1u << 14);
          const uint64_t bw = smem_desc_k128(sB, kk * 32), bwi = bw + (uint64_t)((64 * 128) >> 4);
          mma_f16_ts_peak(tmem + 256, tmem + kk * 8, bw, idesc);
          mma_f16_ts_peak(tmem + 256, tmem + 128 + kk * 8, bwi, I64N);
          mma_f16_ts_peak(tmem + 256 + 64, tmem + 128 + kk * 8, bw, I64);
          continue;
        }
        if (KIND == 3 || KIND == 7) mma_f16_ss(tmem, ad, bd, idesc, 1u);
        else if (KIND == 6 || KIND == 11) mma_f16_ts_peak(tmem + 256, tmem + kk * 8, bd, idesc);  // A: columns 0..31
        else if (KIND == 4) mma_i8_ss(tmem, ad, bd, idesc, 1u);
        else if (KIND == 8 || KIND == 10) mma_mxf4_ts_peak(tmem + 128, tmem + kk * 8, bd, idesc, tmem + 256, tmem + 256 + 128);
        else if (KIND == 9) mma_mxf4_peak(tmem + 128, ad, bd, idesc, tmem + 256, tmem + 256 + 128);
        else mma_mxf4_peak(tmem, ad, bd, idesc, tmem + 256, tmem + 256 + 128);
      }
    }
    if (elect_one()) mma_commit(done);
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();
  if (warp == 0) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(tmem, v);
    tmem_wait_ld();
    if (v[0] == 0x7FFFFFFFu && v[1] == 0x12345u) sink[0] = (int32_t)v[2];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace
}  // namespace tcbf

extern "C" {

// Run peak kind `kind` (0..5, see the header comment) with `iters` loop iterations per warp /
// issuing thread on the current device.  Writes the duration of one timed launch (seconds, CUDA
// events, after one warm-up launch) and the ops it performed (2 per MAC).  Returns 0 on success,
// -1 for an unknown kind or iters <= 0, else the cudaError_t value.
__attribute__((visibility("default"))) int tcbf_peak_run(int kind, int iters, double* seconds, double* ops) {
  using namespace tcbf;
  if (kind < 0 || kind > 14 || iters <= 0 || !seconds || !ops) return -1;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint32_t* seed = nullptr;
  int32_t* sink = nullptr;
  cudaError_t e = cudaMalloc(&seed, 32 * sizeof(uint32_t));
  if (e != cudaSuccess) return (int)e;
  e = cudaMalloc(&sink, sizeof(int32_t));
  if (e != cudaSuccess) { cudaFree(seed); return (int)e; }
  uint32_t hseed[32];
  for (int i = 0; i < 32; ++i) hseed[i] = 0x9E3779B9u * (uint32_t)(i + 1);
  cudaMemcpy(seed, hseed, sizeof(hseed), cudaMemcpyHostToDevice);

  double work = 0.0;
  auto launch = [&]() -> cudaError_t {
    if (kind <= 1) {
      const int blocks = sms * 4, threads = 256;  // 32 warps per SM
      if (kind == 0) peak_b1_mma_kernel<false><<<blocks, threads>>>(seed, iters, sink);
      else peak_b1_mma_kernel<true><<<blocks, threads>>>(seed, iters, sink);
      work = 2.0 * 16 * 8 * 256 * B1_CHAINS * (double)iters * (blocks * threads / 32);
    } else if (kind == 2) {
      const int blocks = sms * 8, threads = 256;
      peak_popc_kernel<<<blocks, threads>>>(seed, iters, sink);
      work = 2.0 * 32 * 4 * POPC_CHAINS * (double)iters * blocks * threads;
    } else {
      auto k = kind == 3 ? peak_tc_kernel<3> : kind == 4 ? peak_tc_kernel<4> : kind == 5 ? peak_tc_kernel<5>
             : kind == 6 ? peak_tc_kernel<6> : kind == 7 ? peak_tc_kernel<7> : kind == 8 ? peak_tc_kernel<8>
             : kind == 9 ? peak_tc_kernel<9> : kind == 10 ? peak_tc_kernel<10> : kind == 11 ? peak_tc_kernel<11> : kind == 12 ? peak_tc_kernel<12>
             : kind == 13 ? peak_tc_kernel<13> : peak_tc_kernel<14>;
      cudaError_t a = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
      if (a != cudaSuccess) return a;
      k<<<sms, 128, TC_SMEM>>>(iters, sink);
      const double kdim = (kind == 3 || kind == 6 || kind == 7 || kind >= 11) ? 16 : kind == 4 ? 32 : 64;
      const double ndim = (kind == 6 || kind == 8 || kind == 9) ? 64 : (kind == 7 || kind == 10 || kind == 11 || kind == 14) ? 128
                         : kind == 13 ? 32 : 256;
      work = 2.0 * 128 * ndim * kdim * 4 * (double)iters * sms;
    }
    return cudaGetLastError();
  };
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  e = launch();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  float ms = 0.f;
  if (e == cudaSuccess) {
    cudaEventRecord(t0);
    e = launch();
    cudaEventRecord(t1);
    if (e == cudaSuccess) e = cudaEventSynchronize(t1);
    if (e == cudaSuccess) cudaEventElapsedTime(&ms, t0, t1);
  }
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(seed);
  cudaFree(sink);
  if (e != cudaSuccess) return (int)e;
  *seconds = ms * 1e-3;
  *ops = work;
  return 0;
}

}  // extern "C"
