// pack.cu -- the memory-bound operand packing kernels ("For 1-bit precision,
// the input data must be packed, i.e. 32 consecutive 1-bit samples must be stored in a
// single 32-bit integer ... the matrix-matrix multiplication kernel requires that the input
// matrices are tiled in device memory ... a transpose kernel"; real and
// imaginary components separated).
//
//   F16: fp32 -> fp16 round-to-nearest-even (cvt.rn.f16.f32), planar.  Weights [B][M][K] ->
//        [B][2][M][Kp], K-contiguous, K padded with zeros to Kp = round_up(K, 64) (one 128-byte
//        swizzle row).  Data [B][K][N] -> [B][2][K][Np], N-contiguous, Np = round_up(N, 8):
//        NO transpose -- the GEMMs read the data MN-major (the tcgen05 B-major descriptor bit).
//   B1 : bit = (value >= 0) (reading R4), LSB-first along K, padding
//        bits 0, Kp = round_up(ceil(K/32), 8) words (256-bit granule).
//        Weights keep their row order [B][2][M][Kp]; data [B][K][N] is transposed to
//        [B][2][N][Kp] so the bits of one sample run along K (the paper's transpose kernel).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
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

// [B][R][C] fp32 complex -> [B][2][R][Cp] fp16 planar, zero tail C..Cp-1; one thread per 8
// consecutive elements of a row, rows distributed over blocks (no 64-bit divisions per element).
// Used for the weights (R = M, C = K, Cp = K16: K-major A operand) and for the data (R = K,
// C = N, Cp = Np: the GEMM reads the data MN-major, so no transpose is needed).
template <int LAYOUT, bool VEC>
__global__ void __launch_bounds__(256) pack_f16_rows(const float* __restrict__ src, int64_t rows, int64_t R,
                                                     int64_t C, int64_t Cp, uint16_t* __restrict__ dst) {
  const int groups = (int)(Cp / 8);
  const int rpb = groups >= 256 ? 1 : 256 / groups;  // rows per block pass
  const int lr = threadIdx.x / groups;
  const int g0 = threadIdx.x - lr * groups;
  for (int64_t row0 = (int64_t)blockIdx.x * rpb; row0 < rows; row0 += (int64_t)gridDim.x * rpb) {
    const int64_t row = row0 + lr;
    if (lr >= rpb || row >= rows) continue;
    const int64_t b = row / R, r = row - b * R;
    for (int g = g0; g < groups; g += (groups >= 256 ? 256 : groups)) {
      const int64_t c0 = (int64_t)g * 8;
      float re[8], im[8];
      if (VEC && LAYOUT == 0 && c0 + 8 <= C) {
        const float4* p = reinterpret_cast<const float4*>(src + ((b * R + r) * C + c0) * 2);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float4 v = __ldg(p + j);
          re[2 * j] = v.x; im[2 * j] = v.y; re[2 * j + 1] = v.z; im[2 * j + 1] = v.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (c0 + j < C) {
            float2 v = load_c<LAYOUT>(src, b, r, c0 + j, R, C);
            re[j] = v.x;
            im[j] = v.y;
          } else {
            re[j] = 0.f;
            im[j] = 0.f;
          }
        }
      }
      uint4 pr = make_uint4(h2u(re[0], re[1]), h2u(re[2], re[3]), h2u(re[4], re[5]), h2u(re[6], re[7]));
      uint4 pi = make_uint4(h2u(im[0], im[1]), h2u(im[2], im[3]), h2u(im[4], im[5]), h2u(im[6], im[7]));
      *reinterpret_cast<uint4*>(dst + ((b * 2 + 0) * R + r) * Cp + c0) = pr;
      *reinterpret_cast<uint4*>(dst + ((b * 2 + 1) * R + r) * Cp + c0) = pi;
    }
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

// data: [B][K][N] -> [B][2][N][Kw]; one thread per (column n, chunk of `wpt` words = 32 wpt k):
// the 32 k-rows of a word are read with warp-coalesced 256-byte row segments (consecutive n),
// all 32 loads of a word in flight; the thread's consecutive words of a row merge in L2
// (the packed output is 1/64 of the bytes read).  wpt = 32 on large operands; small ones use
// shorter chunks so that the grid still fills every SM (square 1024^2: 8 CTAs -> 256).
template <int LAYOUT, int wpt>  // compile-time chunk: a runtime trip count measured 1.3-3.5x slower
__global__ void __launch_bounds__(128) pack_b1_transpose(const float* __restrict__ src, int64_t B, int64_t K,
                                                         int64_t N, int64_t Kw, uint32_t* __restrict__ dst) {
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  for (int64_t b = blockIdx.z; b < B; b += gridDim.z)
    for (int64_t w0 = (int64_t)blockIdx.y * wpt; w0 < Kw; w0 += (int64_t)gridDim.y * wpt) {
      uint32_t* dr = dst + ((b * 2 + 0) * N + n) * Kw + w0;
      uint32_t* di = dst + ((b * 2 + 1) * N + n) * Kw + w0;
#pragma unroll 1
      for (int w = 0; w < wpt && w0 + w < Kw; ++w) {
        uint32_t br = 0, bi = 0;
        const int64_t kbase = (w0 + w) * 32;
        if (kbase < K) {
          float2 v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = (kbase + j < K) ? load_c<LAYOUT>(src, b, kbase + j, n, K, N)
                                                           : make_float2(-1.f, -1.f);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            br |= (v[j].x >= 0.f ? 1u : 0u) << j;  // NaN -> 0; rows k >= K -> padding bit 0
            bi |= (v[j].y >= 0.f ? 1u : 0u) << j;
          }
        }
        dr[w] = br;
        di[w] = bi;
      }
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
                            int64_t Cp, uint16_t* dst, cudaStream_t stream) {
  (void)operand;  // weights: R=M, C=K, Cp=K16; data: R=K, C=N, Cp=Np -- the same row conversion
  const int64_t rows = B * R;
  const int64_t groups = Cp / 8;
  const int64_t rpb = groups >= 256 ? 1 : 256 / groups;
  const int64_t blocks = std::min<int64_t>((rows + rpb - 1) / rpb, 148LL * 16);
  const bool vec = (C % 2 == 0) && (reinterpret_cast<uintptr_t>(src) % 16 == 0);
  if (layout == 0) {
    if (vec) pack_f16_rows<0, true><<<(unsigned)blocks, 256, 0, stream>>>(src, rows, R, C, Cp, dst);
    else pack_f16_rows<0, false><<<(unsigned)blocks, 256, 0, stream>>>(src, rows, R, C, Cp, dst);
  } else {
    pack_f16_rows<1, false><<<(unsigned)blocks, 256, 0, stream>>>(src, rows, R, C, Cp, dst);
  }
  return cudaGetLastError();
}

cudaError_t launch_pack_b1(const float* src, int layout, int operand, int64_t B, int64_t R, int64_t C,
                           int64_t Kw, int wpt_override, uint32_t* dst, cudaStream_t stream) {
  if (operand == 0) {
    const int64_t work = B * R * Kw * 32;
    if (layout == 0) pack_b1_rows<0><<<grid_for(work, 256), 256, 0, stream>>>(src, B, R, C, Kw, dst);
    else pack_b1_rows<1><<<grid_for(work, 256), 256, 0, stream>>>(src, B, R, C, Kw, dst);
  } else {
    // words per thread: 32, cut to 8, 2, 1 while fewer (column, chunk) items than four
    // full-occupancy waves (148 SMs x 2048 threads) would be launched.  Measured (us): square 1024^2
    // 41.7 -> 10.6, M=32 N=K=4096 52.6 -> 41, N=K=16384 385 -> 345, radio 1-bit unchanged (644)
    int wpt = 32;
    while (wpt > 1 && B * C * ((Kw + wpt - 1) / wpt) < 4LL * 148 * 2048) wpt = wpt == 32 ? 8 : wpt == 8 ? 2 : 1;
    if (wpt_override > 0) wpt = wpt_override;  // experiments / tests: 32, 8, 2 or 1
    wpt = wpt >= 32 ? 32 : wpt >= 8 ? 8 : wpt >= 2 ? 2 : 1;
    dim3 grid((unsigned)((C + 127) / 128), (unsigned)cap_dim((Kw + wpt - 1) / wpt), (unsigned)cap_dim(B));
#define TCBF_PACK_B1_T(L, W) pack_b1_transpose<L, W><<<grid, 128, 0, stream>>>(src, B, R, C, Kw, dst)
    if (layout == 0) {
      if (wpt == 32) TCBF_PACK_B1_T(0, 32); else if (wpt == 8) TCBF_PACK_B1_T(0, 8);
      else if (wpt == 2) TCBF_PACK_B1_T(0, 2); else TCBF_PACK_B1_T(0, 1);
    } else {
      if (wpt == 32) TCBF_PACK_B1_T(1, 32); else if (wpt == 8) TCBF_PACK_B1_T(1, 8);
      else if (wpt == 2) TCBF_PACK_B1_T(1, 2); else TCBF_PACK_B1_T(1, 1);
    }
#undef TCBF_PACK_B1_T
  }
  return cudaGetLastError();
}

}  // namespace tcbf
