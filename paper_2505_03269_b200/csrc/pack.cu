// pack.cu -- the memory-bound operand packing kernels ("For 1-bit precision,
// the input data must be packed, i.e. 32 consecutive 1-bit samples must be stored in a
// single 32-bit integer ... the matrix-matrix multiplication kernel requires that the input
// matrices are tiled in device memory ... a transpose kernel"; real and
// imaginary components separated).
//
//   F16: fp32 -> fp16 round-to-nearest-even (cvt.rn.f16.f32), planar, K-contiguous,
//        K padded with zeros to Kp = round_up(K, 64) (one 128-byte swizzle row).
//   B1 : bit = (value >= 0) (reading R4), LSB-first along K, padding
//        bits 0, Kp = round_up(ceil(K/32), 8) words (256-bit granule).
// Weights [B][M][K] keep their row order; data [B][K][N] is transposed to [B][2][N][Kp]
// so both GEMM operands are K-major (what the tcgen05 smem descriptors and TMA want).
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace tcbf {
namespace {

template <int LAYOUT>
__device__ __forceinline__ float2 load_c(const float* __restrict__ s, int64_t b, int64_t r, int64_t c,
                                         int64_t R, int64_t C) {
  if (LAYOUT == 0) return __ldg(reinterpret_cast<const float2*>(s) + ((b * R + r) * C + c));
  return make_float2(__ldg(s + ((b * 2 + 0) * R + r) * C + c), __ldg(s + ((b * 2 + 1) * R + r) * C + c));
}

__device__ __forceinline__ uint32_t h2u(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// weights: [B][M][K] -> [B][2][M][K16]; one thread per 8 consecutive k.
template <int LAYOUT>
__global__ void pack_f16_rows(const float* __restrict__ src, int64_t B, int64_t M, int64_t K, int64_t K16,
                              uint16_t* __restrict__ dst) {
  const int64_t groups = K16 / 8;
  const int64_t total = B * M * groups;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = i % groups;
    const int64_t bm = i / groups;
    const int64_t m = bm % M;
    const int64_t b = bm / M;
    float re[8], im[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t k = g * 8 + j;
      if (k < K) {
        float2 v = load_c<LAYOUT>(src, b, m, k, M, K);
        re[j] = v.x;
        im[j] = v.y;
      } else {
        re[j] = 0.f;
        im[j] = 0.f;
      }
    }
    uint4 pr = make_uint4(h2u(re[0], re[1]), h2u(re[2], re[3]), h2u(re[4], re[5]), h2u(re[6], re[7]));
    uint4 pi = make_uint4(h2u(im[0], im[1]), h2u(im[2], im[3]), h2u(im[4], im[5]), h2u(im[6], im[7]));
    *reinterpret_cast<uint4*>(dst + ((b * 2 + 0) * M + m) * K16 + g * 8) = pr;
    *reinterpret_cast<uint4*>(dst + ((b * 2 + 1) * M + m) * K16 + g * 8) = pi;
  }
}

// data: [B][K][N] -> [B][2][N][K16]; 64(k) x 32(n) tile through shared memory.
template <int LAYOUT>
__global__ void __launch_bounds__(256) pack_f16_transpose(const float* __restrict__ src, int64_t B, int64_t K,
                                                          int64_t N, int64_t K16, uint16_t* __restrict__ dst) {
  __shared__ __half sre[64][40];
  __shared__ __half sim[64][40];
  const int64_t n0 = (int64_t)blockIdx.x * 32;
  for (int64_t b = blockIdx.z; b < B; b += gridDim.z)
  for (int64_t k0 = (int64_t)blockIdx.y * 64; k0 < K16; k0 += (int64_t)gridDim.y * 64) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int kl = ty + 8 * r;
    const int64_t k = k0 + kl, n = n0 + tx;
    float2 v = make_float2(0.f, 0.f);
    if (k < K && n < N) v = load_c<LAYOUT>(src, b, k, n, K, N);
    sre[kl][tx] = __float2half_rn(v.x);
    sim[kl][tx] = __float2half_rn(v.y);
  }
  __syncthreads();
  const int nl = threadIdx.x >> 3, kg = threadIdx.x & 7;
  const int64_t n = n0 + nl;
  if (n < N) {
    uint32_t wr[4], wi[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __half2 hr = __halves2half2(sre[kg * 8 + 2 * j][nl], sre[kg * 8 + 2 * j + 1][nl]);
      __half2 hi = __halves2half2(sim[kg * 8 + 2 * j][nl], sim[kg * 8 + 2 * j + 1][nl]);
      wr[j] = *reinterpret_cast<uint32_t*>(&hr);
      wi[j] = *reinterpret_cast<uint32_t*>(&hi);
    }
    *reinterpret_cast<uint4*>(dst + ((b * 2 + 0) * N + n) * K16 + k0 + kg * 8) = make_uint4(wr[0], wr[1], wr[2], wr[3]);
    *reinterpret_cast<uint4*>(dst + ((b * 2 + 1) * N + n) * K16 + k0 + kg * 8) = make_uint4(wi[0], wi[1], wi[2], wi[3]);
  }
  __syncthreads();
  }
}

// weights: [B][M][K] -> [B][2][M][Kw]; one warp per output word pair (ballot of 32 signs).
template <int LAYOUT>
__global__ void pack_b1_rows(const float* __restrict__ src, int64_t B, int64_t M, int64_t K, int64_t Kw,
                             uint32_t* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t total = B * M * Kw;
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total; w += warps_total) {
    const int64_t kw = w % Kw;
    const int64_t bm = w / Kw;
    const int64_t m = bm % M;
    const int64_t b = bm / M;
    const int64_t k = kw * 32 + lane;
    bool pr = false, pi = false;
    if (k < K) {
      float2 v = load_c<LAYOUT>(src, b, m, k, M, K);
      pr = v.x >= 0.f;  // NaN -> false -> bit 0
      pi = v.y >= 0.f;
    }
    const uint32_t br = __ballot_sync(0xffffffffu, pr);  // lane j -> bit j (LSB-first)
    const uint32_t bi = __ballot_sync(0xffffffffu, pi);
    if (lane == 0) dst[((b * 2 + 0) * M + m) * Kw + kw] = br;
    if (lane == 1) dst[((b * 2 + 1) * M + m) * Kw + kw] = bi;
  }
}

// data: [B][K][N] -> [B][2][N][Kw]; thread per (n, word), coalesced reads along n.
template <int LAYOUT>
__global__ void __launch_bounds__(256) pack_b1_transpose(const float* __restrict__ src, int64_t B, int64_t K,
                                                         int64_t N, int64_t Kw, uint32_t* __restrict__ dst) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  for (int64_t b = blockIdx.z; b < B; b += gridDim.z)
  for (int64_t kw = blockIdx.y; kw < Kw; kw += gridDim.y) {
  uint32_t br = 0, bi = 0;
  const int64_t kbase = kw * 32;
#pragma unroll 8
  for (int j = 0; j < 32; ++j) {
    const int64_t k = kbase + j;
    if (k < K) {
      float2 v = load_c<LAYOUT>(src, b, k, n, K, N);
      br |= (v.x >= 0.f ? 1u : 0u) << j;
      bi |= (v.y >= 0.f ? 1u : 0u) << j;
    }
  }
  dst[((b * 2 + 0) * N + n) * Kw + kw] = br;
  dst[((b * 2 + 1) * N + n) * Kw + kw] = bi;
  }
}

inline unsigned grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  const int64_t cap = 148LL * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

inline int64_t cap_dim(int64_t v) { return v < 65535 ? (v < 1 ? 1 : v) : 65535; }

}  // namespace

cudaError_t launch_pack_f16(const float* src, int layout, int operand, int64_t B, int64_t R, int64_t C,
                            int64_t K16, uint16_t* dst, cudaStream_t stream) {
  if (operand == 0) {  // weights, R = M, C = K
    const int64_t work = B * R * (K16 / 8);
    if (layout == 0) pack_f16_rows<0><<<grid_for(work, 256), 256, 0, stream>>>(src, B, R, C, K16, dst);
    else pack_f16_rows<1><<<grid_for(work, 256), 256, 0, stream>>>(src, B, R, C, K16, dst);
  } else {  // data, R = K, C = N
    dim3 grid((unsigned)((C + 31) / 32), (unsigned)cap_dim(K16 / 64), (unsigned)cap_dim(B));
    if (layout == 0) pack_f16_transpose<0><<<grid, 256, 0, stream>>>(src, B, R, C, K16, dst);
    else pack_f16_transpose<1><<<grid, 256, 0, stream>>>(src, B, R, C, K16, dst);
  }
  return cudaGetLastError();
}

cudaError_t launch_pack_b1(const float* src, int layout, int operand, int64_t B, int64_t R, int64_t C,
                           int64_t Kw, uint32_t* dst, cudaStream_t stream) {
  if (operand == 0) {
    const int64_t work = B * R * Kw * 32;
    if (layout == 0) pack_b1_rows<0><<<grid_for(work, 256), 256, 0, stream>>>(src, B, R, C, Kw, dst);
    else pack_b1_rows<1><<<grid_for(work, 256), 256, 0, stream>>>(src, B, R, C, Kw, dst);
  } else {
    dim3 grid((unsigned)((C + 255) / 256), (unsigned)cap_dim(Kw), (unsigned)cap_dim(B));
    if (layout == 0) pack_b1_transpose<0><<<grid, 256, 0, stream>>>(src, B, R, C, Kw, dst);
    else pack_b1_transpose<1><<<grid, 256, 0, stream>>>(src, B, R, C, Kw, dst);
  }
  return cudaGetLastError();
}

}  // namespace tcbf
