// gemm_b1_mma.cu -- 1-bit-mode complex beamformer GEMM on the legacy warp-level binary MMA,
// `mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc` (the paper's 16x8x256 b1
// fragment, and its sm_90 AND form).
//
// Why AND and why single-AND: on sm_100a ptxas lowers both b1 forms to a subroutine of
// MOVM.U4TO8 + IMMA.16832.U8 (emulated; profiles/r01/peaks.json): register-only peaks 413 TeraOps/s
// for .and.popc against 181 for .xor.popc and 292 for CUDA-core LOP3+POPC, so AND is the faster
// legacy form.  The paper's AND emulation of XOR needs 8 b1 MMAs per complex K slice
// (PAPER.md:265-272); with per-row / per-column popcounts the same exact result needs only 4
// (reading R1b, with u = (a+1)/2 in {0,1}):
//   Re = 4[P(A_r & B_r) + P(A_i & ~B_i)] - 2|A_r| - 2|A_i| - 2|B_r| + 2|B_i|
//   Im = 4[P(A_r & B_i) + P(A_i & B_r)]  - 2(|A_r| + |A_i| + |B_r| + |B_i|) + 2K
// ~B_i is complemented in registers as the paper complements Im(b); padding bits
// are 0 in both operands, so A_i's zero padding masks the complemented padding of
// B_i and every popcount covers exactly the logical K.
//
// Tiling: CTA 128 beams x 64 samples, 8 warps (4 x 2) of 32 x 32 outputs = 2 m16 x 4 n8 fragments,
// two int32 accumulator sets (Re, Im).  Packed words stream through a 2-stage cp.async ring of
// 32-word (1024-bit) K chunks; rows are padded to 36 words so the fragment loads (row = lane/4,
// word = lane%4) hit 32 distinct banks.  Row/column popcounts are accumulated from the same smem
// chunks by the CUDA cores.  Selected with TCBF_B1_KERNEL=bmma (a measured variant, not the default).
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"

namespace tcbf {
namespace {

constexpr int TM = 128, TN = 64;
constexpr int KC = 32;           // words per stage
constexpr int RS = KC + 4;       // padded row stride (words)
constexpr int A_WORDS = 2 * TM * RS;
constexpr int B_WORDS = 2 * TN * RS;
constexpr int STAGE_WORDS = A_WORDS + B_WORDS;
constexpr int SMEM_BYTES = 2 * STAGE_WORDS * 4 + (2 * TM + 2 * TN) * 4;

__device__ __forceinline__ void cp_async16(uint32_t* dst, const uint32_t* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void mma_b1_and(int32_t (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(256, 2) cgemm_b1_mma_kernel(GemmB1Args p) {
  extern __shared__ __align__(16) uint32_t sm[];
  int32_t* popA = reinterpret_cast<int32_t*>(sm + 2 * STAGE_WORDS);  // [2][TM]: |A_r|, |A_i| per beam
  int32_t* popB = popA + 2 * TM;                                     // [2][TN]: |B_r|, |B_i| per sample
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int n0 = blockIdx.x * TN, m0 = blockIdx.y * TM;
  const int nchunks = (p.Kw + KC - 1) / KC;

  for (int b = blockIdx.z; b < p.B; b += gridDim.z) {
    const uint32_t* Ab = p.w + (size_t)2 * b * p.M * p.Kw;
    const uint32_t* Bb = p.x + (size_t)2 * b * p.N * p.Kw;
    auto load_stage = [&](int c, int buf) {
      uint32_t* sA = sm + buf * STAGE_WORDS;
      uint32_t* sB = sA + A_WORDS;
      const int kw0 = c * KC;
#pragma unroll
      for (int i = 0; i < 8; ++i) {  // A: 2 planes x 128 rows x 8 chunks of 16 B
        const int item = tid + i * 256;
        const int pl = item >> 10, row = (item >> 3) & 127, ch = item & 7;
        const int m = m0 + row, kw = kw0 + ch * 4;
        const bool ok = m < p.M && kw < p.Kw;
        cp_async16(sA + (pl * TM + row) * RS + ch * 4, ok ? Ab + ((size_t)pl * p.M + m) * p.Kw + kw : Ab, ok);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // B: 2 planes x 64 rows x 8 chunks
        const int item = tid + i * 256;
        const int pl = item >> 9, row = (item >> 3) & 63, ch = item & 7;
        const int n = n0 + row, kw = kw0 + ch * 4;
        const bool ok = n < p.N && kw < p.Kw;
        cp_async16(sB + (pl * TN + row) * RS + ch * 4, ok ? Bb + ((size_t)pl * p.N + n) * p.Kw + kw : Bb, ok);
      }
      cp_async_commit();
    };

    int32_t acc_re[2][4][4], acc_im[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) { acc_re[i][j][r] = 0; acc_im[i][j][r] = 0; }
    int32_t pop = 0;  // this thread's row (tid < 256: A plane/row) or column (tid < 128: B) popcount
    int32_t popb = 0;

    load_stage(0, 0);
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1;
      if (c + 1 < nchunks) {
        load_stage(c + 1, buf ^ 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const uint32_t* sA = sm + buf * STAGE_WORDS;
      const uint32_t* sB = sA + A_WORDS;
      // popcounts: thread t -> A row-plane t (256 of them); threads < 128 also B row-plane t
      {
        const uint4* ra = reinterpret_cast<const uint4*>(sA + tid * RS);
#pragma unroll
        for (int q = 0; q < KC / 4; ++q) {
          const uint4 v = ra[q];
          pop += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
        }
        if (tid < 2 * TN) {
          const uint4* rb = reinterpret_cast<const uint4*>(sB + tid * RS);
#pragma unroll
          for (int q = 0; q < KC / 4; ++q) {
            const uint4 v = rb[q];
            popb += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
          }
        }
      }
#pragma unroll
      for (int ks = 0; ks < KC / 8; ++ks) {
        if (c * KC + ks * 8 >= p.Kw) break;  // Kw is a multiple of 8: whole 256-bit steps only
        const int w0 = ks * 8 + t4;
        uint32_t ar[2][4], ai[2][4];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r0 = wm + i * 16 + g;
          ar[i][0] = sA[r0 * RS + w0];
          ar[i][1] = sA[(r0 + 8) * RS + w0];
          ar[i][2] = sA[r0 * RS + w0 + 4];
          ar[i][3] = sA[(r0 + 8) * RS + w0 + 4];
          ai[i][0] = sA[(TM + r0) * RS + w0];
          ai[i][1] = sA[(TM + r0 + 8) * RS + w0];
          ai[i][2] = sA[(TM + r0) * RS + w0 + 4];
          ai[i][3] = sA[(TM + r0 + 8) * RS + w0 + 4];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c0 = wn + j * 8 + g;
          const uint32_t br0 = sB[c0 * RS + w0], br1 = sB[c0 * RS + w0 + 4];
          const uint32_t bi0 = sB[(TN + c0) * RS + w0], bi1 = sB[(TN + c0) * RS + w0 + 4];
          if (TCBF_ABLATE(p, 2)) continue;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            mma_b1_and(acc_re[i][j], ar[i], br0, br1);    // P(A_r & B_r)
            mma_b1_and(acc_re[i][j], ai[i], ~bi0, ~bi1);  // P(A_i & ~B_i)
            mma_b1_and(acc_im[i][j], ar[i], bi0, bi1);    // P(A_r & B_i)
            mma_b1_and(acc_im[i][j], ai[i], br0, br1);    // P(A_i & B_r)
          }
        }
      }
      __syncthreads();  // the next iteration's cp.async overwrites the other buffer only after this
    }
    popA[tid] = pop;
    if (tid < 2 * TN) popB[tid] = popb;
    __syncthreads();

    // epilogue: exact complex value (R1b), int32 planar [B][2][M][N]
    const int twoK = 2 * p.K;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rl = wm + i * 16 + g + h * 8;
        const int m = m0 + rl;
        if (m >= p.M) continue;
        const int par = popA[rl], pai = popA[TM + rl];
        int32_t* ore = p.out + ((size_t)(2 * b) * p.M + m) * p.N;
        int32_t* oim = p.out + ((size_t)(2 * b + 1) * p.M + m) * p.N;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int cl = wn + j * 8 + 2 * t4;
          const int n = n0 + cl;
          int vr[2], vi[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int pbr = popB[cl + e], pbi = popB[TN + cl + e];
            vr[e] = 4 * acc_re[i][j][2 * h + e] - 2 * (par + pai + pbr) + 2 * pbi;
            vi[e] = 4 * acc_im[i][j][2 * h + e] - 2 * (par + pai + pbr + pbi) + twoK;
          }
          if (TCBF_ABLATE(p, 1)) continue;
          if ((p.N & 1) == 0 && n + 1 < p.N) {
            *reinterpret_cast<int2*>(ore + n) = make_int2(vr[0], vr[1]);
            *reinterpret_cast<int2*>(oim + n) = make_int2(vi[0], vi[1]);
          } else {
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (n + e < p.N) { ore[n + e] = vr[e]; oim[n + e] = vi[e]; }
          }
        }
      }
    }
    __syncthreads();  // popA/popB and the stage buffers are reused by the next batch entry
  }
}

}  // namespace

cudaError_t launch_gemm_b1_mma(const GemmB1Args& args, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(cgemm_b1_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((args.N + TN - 1) / TN), (unsigned)((args.M + TM - 1) / TM),
            (unsigned)(args.B < 65535 ? args.B : 65535));
  cgemm_b1_mma_kernel<<<grid, 256, SMEM_BYTES, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace tcbf
