// kernels.h -- internal launcher declarations shared by plan.cu and the kernel files.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace tcbf {

struct GemmF16Args {
  int M, N, B;
  int K16;
  int tiles_m, tiles_n, num_tiles, num_kb;
  float* out;  // used by the masked-store epilogue (N % 4 != 0)
};

cudaError_t launch_gemm_f16(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                            const GemmF16Args& args, int block_n, bool tma_store, int num_sms,
                            cudaStream_t stream);

struct GemmB1Args {
  const uint32_t* w;  // [B][2][M][Kw]
  const uint32_t* x;  // [B][2][N][Kw]
  int32_t* out;       // [B][2][M][N]
  int M, N, K, Kw, B;
};
cudaError_t launch_gemm_b1_popc(const GemmB1Args& args, cudaStream_t stream);
cudaError_t launch_gemm_b1_tc(const CUtensorMap& tmC, const GemmB1Args& args, bool tma_store, int num_sms,
                              cudaStream_t stream);

// pack kernels (pack.cu)
cudaError_t launch_pack_f16(const float* src, int layout, int operand, int64_t B, int64_t R, int64_t C,
                            int64_t K16, uint16_t* dst, cudaStream_t stream);
cudaError_t launch_pack_b1(const float* src, int layout, int operand, int64_t B, int64_t R, int64_t C,
                           int64_t Kw, uint32_t* dst, cudaStream_t stream);

}  // namespace tcbf
