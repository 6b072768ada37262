// kernels.h -- internal launcher declarations shared by plan.cu and the kernel files.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace tcbf {

// Ablation switches of the measurement studies in DESIGN.md §4 (skip stores / MMAs / expansion).
// They exist only in TCBF_DEV builds (TCBF_DEBUG env, read once at plan creation); the product
// library compiles them out, so its results never depend on the environment at call time.
#ifdef TCBF_DEV
#define TCBF_ABLATE(args, bit) (((args).debug & (bit)) != 0)
#else
#define TCBF_ABLATE(args, bit) false
#endif

struct GemmF16Args {
  int M, N, B;
  int K16;
  int tiles_m, tiles_n, num_tiles, num_kb;
  float* out;  // used by the masked-store epilogue (N % 4 != 0)
  int debug;   // TCBF_DEV ablation: bit0 skip output stores, bit1 skip MMAs
  int group_m; // tile rows per rasterisation group (tile_coords)
  int splits, kb_per_split;  // K split of the streaming-conversion kernel (fp32 TMA reduce-add)
  unsigned long long* trace;  // TCBF_DEV timeline of the fused kernel (globaltimer stamps), else null
  int multicast;              // interleaved kernel: weight multicast across CTA pairs (0 = off)
};

// fp16 GEMM kernel variants (tile N x K-block x stages x epilogue warps)
enum {
  F16_V_K32_S4_E8 = 0,  // 128x128, BK 32, 4 stages, 8 epilogue warps
  F16_V_K64_S3 = 1,     // 128x128, BK 64, 3 stages, 4 epilogue warps (default 1-CTA tile)
  F16_V_N64 = 2,        // 128x64,  BK 64, 4 stages, 4 epilogue warps (small N)
  F16_V_2CTA_N128 = 3,  // CTA pair, 256x128 tile, BK 64, 4 stages, double-buffered TMEM
  F16_V_2CTA_N256 = 4,  // CTA pair, 256x256 tile, BK 64, 3 stages, single TMEM buffer
  F16_V_COUNT = 5
};
int gemm_f16_block_n(int variant);
cudaError_t launch_gemm_f16_2cta(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                                 const GemmF16Args& args, int block_n, int num_sms, cudaStream_t stream);
int gemm_f16_block_k(int variant);
cudaError_t launch_gemm_f16(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                            const GemmF16Args& args, int variant, int epi, int num_sms,
                            cudaStream_t stream);

int gemm_f16_ileave_block_k();
int gemm_f16_ileave_block_n();
cudaError_t launch_gemm_f16_ileave(const CUtensorMap& tmA, const CUtensorMap& tmX, const CUtensorMap& tmC,
                                   const GemmF16Args& args, int num_sms, cudaStream_t stream);
int gemm_f16_conv_block_k();
int gemm_f16_conv_splits(int tiles, int num_kb, int num_sms);
cudaError_t launch_gemm_f16_conv(const CUtensorMap& tmA, const CUtensorMap& tmX, const CUtensorMap& tmC,
                                 const GemmF16Args& args, int layout, int num_sms, cudaStream_t stream);
bool gemm_f16_smaj_supported(int64_t K16);
// sample-major fused kernel (gemm_f16_smaj.cu): tiles_m = beam tiles, tiles_n = 128-sample tiles
// resident-data interleaved fp16 kernel (gemm_f16_ileave_res.cu): tiles_m = 64-beam tiles,
// tiles_n = 128-sample units, num_kb = K16 / 64 (K16 <= 256)
bool gemm_f16_ileave_res_supported(int64_t K16);
int gemm_f16_ileave_res_beams();
int gemm_f16_ileave_res_samples();
cudaError_t launch_gemm_f16_ileave_res(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmF16Args& args,
                                       int num_sms, cudaStream_t stream);
cudaError_t launch_gemm_f16_smaj(const CUtensorMap& tmW, const GemmF16Args& args, const float* x_src, int layout,
                                 int K, int cluster, int num_sms, cudaStream_t stream);
// data-in-TMEM sample-major fused kernel (gemm_f16_tmem.cu): tiles_m = 64-beam tiles, tiles_n =
// 128-sample units per batch entry, num_kb = K16 / 64 (K16 <= 256)
bool gemm_f16_tmem_supported(int64_t K16);
int gemm_f16_tmem_beams();
int gemm_f16_tmem_raw_rows();
cudaError_t launch_gemm_f16_tmem(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmF16Args& args,
                                 int layout, int wkb, int cluster, int num_sms, cudaStream_t stream);
// the same with 32-beam tiles and half of the next unit staged in TMEM (gemm_f16_tmem2.cu): K16 == 256
bool gemm_f16_tmem2_supported(int64_t K16);
int gemm_f16_tmem2_beams();
cudaError_t launch_gemm_f16_tmem2(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmF16Args& args,
                                  int layout, int wkb, int cluster, int num_sms, cudaStream_t stream);
struct GemmB1Args;
// 1-bit sample-major kernel with the unit's expanded data resident in TMEM (gemm_b1_tmem.cu):
// Kw <= 24 words; 64-beam tiles, 128-sample units, line-store epilogue (any N)
bool gemm_b1_tmem_supported(int64_t Kw);
int gemm_b1_tmem_beams();
cudaError_t launch_gemm_b1_tmem(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmB1Args& a, int num_sms,
                                cudaStream_t stream);

struct GemmB1Args {
  const uint32_t* w;  // [B][2][M][Kw]
  const uint32_t* x;  // [B][2][N][Kw]
  int32_t* out;       // [B][2][M][N]
  int M, N, K, Kw, B;
  int debug;  // TCBF_DEV ablation: bit0 skip stores, bit1 skip MMAs, bit2 skip expansion
  int group_m;  // tile rows per rasterisation group (tile_coords)
  int splits;   // split-K factor (int8 kernel): >1 accumulates exact int32 partials with TMA reduce-add
  int kb_per_split;
  unsigned long long* trace;  // TCBF_DEV timeline (globaltimer stamps) of the swapped kernel, else null
};
cudaError_t launch_gemm_b1_popc(const GemmB1Args& args, cudaStream_t stream);
cudaError_t launch_gemm_b1_mma(const GemmB1Args& args, cudaStream_t stream);  // legacy mma.sync b1 AND
bool gemm_b1_f4_supported(int64_t Kw);
int gemm_b1_f4_block_words();
bool gemm_b1_f4_tma_words(int64_t Kw);
int gemm_b1_f4_store_box_cols(int64_t Kw);
int gemm_b1_f4_swap_beams(int64_t M);  // beams per tile of the swapped small-M kernel (0: not used)
int gemm_b1_f4_swap_box_words();        // packed words per TMA box row of the swapped kernel
cudaError_t launch_gemm_b1_f4_swap(const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmC,
                                   const GemmB1Args& args, int beams, bool tma_store, int num_sms, cudaStream_t stream);
cudaError_t launch_gemm_b1_f4(const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmC,
                              const GemmB1Args& args, bool tma_store, int num_sms, cudaStream_t stream);
cudaError_t launch_gemm_b1_tc(const CUtensorMap& tmC, const GemmB1Args& args, bool tma_store, int num_sms,
                              cudaStream_t stream);

// steering weights (steer.cu)
cudaError_t launch_steering(const double* pos, const double* theta, const double* freq, double c, int64_t B,
                            int64_t M, int64_t K, int layout, float* dst, cudaStream_t stream);

// pack kernels (pack.cu)
cudaError_t launch_pack_f16(const float* src, int layout, int operand, int64_t B, int64_t R, int64_t C,
                            int64_t K16, uint16_t* dst, cudaStream_t stream);
// wpt: 1-bit data pack words per thread (32, 8, 2, 1), 0 = chosen by operand size
cudaError_t launch_pack_b1(const float* src, int layout, int operand, int64_t B, int64_t R, int64_t C,
                           int64_t Kw, int wpt, uint32_t* dst, cudaStream_t stream);

}  // namespace tcbf
