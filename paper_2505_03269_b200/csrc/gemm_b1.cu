// gemm_b1.cu -- 1-bit-mode complex beamformer GEMM, warp-level XOR + __popc on the CUDA cores.
//
// Method (Eq. 4, Eq. 5): with bit 1 = +1, bit 0 = -1,
// a real +-1 dot product over K is K - 2 popc(A xor B).  Our padded operands carry zero
// padding bits in BOTH operands, which contribute nothing to any XOR
// popcount, so the complex result needs no K_pad term at all (reading R1):
//     Re = 2 (popc(A_i ^ B_i) - popc(A_r ^ B_r))
//     Im = 2 K - 2 (popc(A_r ^ B_i) + popc(A_i ^ B_r))
// This is the paper's Eq. 5 with K = K_log + K_pad, rearranged.  XOR is a single LOP3 on
// the CUDA cores (the sm_90 XOR deprecation, concerns only b1 MMA).
//
// Why CUDA cores: on sm_100a the legacy `mma.sync ... .b1 ... .popc` is emulated by
// ptxas with 8 IMMA.16832.U8 + LOP3 masks per m16n8k256 (cuobjdump -sass, profiles/),
// so it is not a native BMMA path (PAPER.md:122 saw the same for XOR on sm_90).
//
// Tiling: 64 x 64 complex outputs per CTA, 256 threads, 4 x 4 outputs per thread,
// K staged through double-buffered shared memory in 8-word (256-bit) chunks stored
// k-major so that each thread reads its 4 rows / 4 columns with one 128-bit LDS.
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"

namespace tcbf {
namespace {

constexpr int TB = 64;  // tile (rows and cols)
constexpr int KC = 8;   // words per K chunk

__global__ void __launch_bounds__(256) cgemm_b1_popc_kernel(GemmB1Args p) {
  __shared__ __align__(16) uint32_t sA[2][2][KC][TB];
  __shared__ __align__(16) uint32_t sB[2][2][KC][TB];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int n0 = blockIdx.x * TB, m0 = blockIdx.y * TB;
  // loader mapping: plane, row, which half of the 8-word chunk
  const int lp = tid >> 7, lrow = (tid >> 1) & 63, lhalf = tid & 1;

  for (int b = blockIdx.z; b < p.B; b += gridDim.z) {
    const uint32_t* Ab = p.w + (size_t)(2 * b + lp) * p.M * p.Kw;
    const uint32_t* Bb = p.x + (size_t)(2 * b + lp) * p.N * p.Kw;
    const bool a_ok = (m0 + lrow) < p.M, b_ok = (n0 + lrow) < p.N;
    const uint4* a_src = reinterpret_cast<const uint4*>(Ab + (size_t)(m0 + lrow) * p.Kw) + lhalf;
    const uint4* b_src = reinterpret_cast<const uint4*>(Bb + (size_t)(n0 + lrow) * p.Kw) + lhalf;

    int s_re[4][4], s_im[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) { s_re[i][j] = 0; s_im[i][j] = 0; }

    const int nchunks = p.Kw / KC;
    uint4 ra = a_ok ? __ldg(a_src) : make_uint4(0, 0, 0, 0);
    uint4 rb = b_ok ? __ldg(b_src) : make_uint4(0, 0, 0, 0);
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1;
      sA[buf][lp][lhalf * 4 + 0][lrow] = ra.x;
      sA[buf][lp][lhalf * 4 + 1][lrow] = ra.y;
      sA[buf][lp][lhalf * 4 + 2][lrow] = ra.z;
      sA[buf][lp][lhalf * 4 + 3][lrow] = ra.w;
      sB[buf][lp][lhalf * 4 + 0][lrow] = rb.x;
      sB[buf][lp][lhalf * 4 + 1][lrow] = rb.y;
      sB[buf][lp][lhalf * 4 + 2][lrow] = rb.z;
      sB[buf][lp][lhalf * 4 + 3][lrow] = rb.w;
      __syncthreads();
      if (c + 1 < nchunks) {  // prefetch the next chunk into registers
        ra = a_ok ? __ldg(a_src + 2 * (c + 1)) : make_uint4(0, 0, 0, 0);
        rb = b_ok ? __ldg(b_src + 2 * (c + 1)) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int kw = 0; kw < KC; ++kw) {
        const uint4 ar = *reinterpret_cast<const uint4*>(&sA[buf][0][kw][ty * 4]);
        const uint4 ai = *reinterpret_cast<const uint4*>(&sA[buf][1][kw][ty * 4]);
        const uint4 br = *reinterpret_cast<const uint4*>(&sB[buf][0][kw][tx * 4]);
        const uint4 bi = *reinterpret_cast<const uint4*>(&sB[buf][1][kw][tx * 4]);
        const uint32_t a_r[4] = {ar.x, ar.y, ar.z, ar.w}, a_i[4] = {ai.x, ai.y, ai.z, ai.w};
        const uint32_t b_r[4] = {br.x, br.y, br.z, br.w}, b_i[4] = {bi.x, bi.y, bi.z, bi.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            s_re[i][j] += __popc(a_i[i] ^ b_i[j]) - __popc(a_r[i] ^ b_r[j]);
            s_im[i][j] += __popc(a_r[i] ^ b_i[j]) + __popc(a_i[i] ^ b_r[j]);
          }
      }
      // the next iteration writes the other buffer; the one after writes this buffer again
      // only after its __syncthreads, so one barrier per chunk suffices.
    }

    // epilogue: exact complex value (PAPER.md:252-259 with the padded-K reading)
    const int twoK = 2 * p.K;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + ty * 4 + i;
      if (m >= p.M) continue;
      int32_t* ore = p.out + ((size_t)(2 * b) * p.M + m) * p.N;
      int32_t* oim = p.out + ((size_t)(2 * b + 1) * p.M + m) * p.N;
      const int n = n0 + tx * 4;
      int vr[4], vi[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        vr[j] = 2 * s_re[i][j];
        vi[j] = twoK - 2 * s_im[i][j];
      }
      if ((p.N & 3) == 0 && n + 3 < p.N) {
        *reinterpret_cast<int4*>(ore + n) = make_int4(vr[0], vr[1], vr[2], vr[3]);
        *reinterpret_cast<int4*>(oim + n) = make_int4(vi[0], vi[1], vi[2], vi[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (n + j < p.N) { ore[n + j] = vr[j]; oim[n + j] = vi[j]; }
      }
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_gemm_b1_popc(const GemmB1Args& args, cudaStream_t stream) {
  dim3 grid((unsigned)((args.N + TB - 1) / TB), (unsigned)((args.M + TB - 1) / TB),
            (unsigned)(args.B < 65535 ? args.B : 65535));
  cgemm_b1_popc_kernel<<<grid, 256, 0, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace tcbf
