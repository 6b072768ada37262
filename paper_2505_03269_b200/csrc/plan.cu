// plan.cu -- the C ABI (include/tcbf.h): validation, layout arithmetic, TMA descriptor
// encoding and dispatch to the sm_100a kernels.  No exceptions or aborts cross the ABI.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "kernels.h"
#include "plan_internal.h"
#include "tcbf.h"

namespace {

thread_local char g_err[512] = "";
thread_local int g_launches = 0;

tcbf_status fail(tcbf_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

tcbf_status cuda_fail(cudaError_t e, const char* what) {
  return fail(TCBF_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

bool mul_ok(size_t a, size_t b, size_t* out) {
  if (a != 0 && b > SIZE_MAX / a) return false;
  *out = a * b;
  return true;
}

tcbf_status compute_sizes(int64_t M, int64_t N, int64_t K, int64_t B, tcbf_precision p, size_t* wb, size_t* xb,
                          size_t* ob, int64_t* kp) {
  if (M < 1 || N < 1 || K < 1 || B < 1)
    return fail(TCBF_ERR_INVALID_ARG, "M, N, K, batch must be >= 1 (got %lld, %lld, %lld, %lld)", (long long)M,
                (long long)N, (long long)K, (long long)B);
  if (p != TCBF_PREC_F16 && p != TCBF_PREC_B1) return fail(TCBF_ERR_INVALID_ARG, "unknown precision %d", (int)p);
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX || B > INT32_MAX)
    return fail(TCBF_ERR_INVALID_ARG, "dimensions must fit int32");
  if (p == TCBF_PREC_B1 && K >= (int64_t(1) << 30))
    return fail(TCBF_ERR_INVALID_ARG, "1-bit mode requires K < 2^30 so |Re|,|Im| <= 2K fit int32");
  int64_t k = p == TCBF_PREC_F16 ? (K + 63) / 64 * 64 : ((K + 31) / 32 + 7) / 8 * 8;
  size_t elem = p == TCBF_PREC_F16 ? 2 : 4;
  size_t t, w, x, o;
  if (!mul_ok((size_t)B * 2, (size_t)M, &t) || !mul_ok(t, (size_t)k, &t) || !mul_ok(t, elem, &w))
    return fail(TCBF_ERR_INVALID_ARG, "packed weight size overflows size_t");
  // F16 data is consumed MN-major: [B][2][K][Np], Np = round_up(N, 8); B1 data is [B][2][N][Kw]
  const bool dx_ok = p == TCBF_PREC_F16
                         ? (mul_ok((size_t)B * 2, (size_t)K, &t) && mul_ok(t, (size_t)((N + 7) / 8 * 8), &t) &&
                            mul_ok(t, elem, &x))
                         : (mul_ok((size_t)B * 2, (size_t)N, &t) && mul_ok(t, (size_t)k, &t) && mul_ok(t, elem, &x));
  if (!dx_ok) return fail(TCBF_ERR_INVALID_ARG, "packed data size overflows size_t");
  if (!mul_ok((size_t)B * 2, (size_t)M, &t) || !mul_ok(t, (size_t)N, &t) || !mul_ok(t, 4, &o))
    return fail(TCBF_ERR_INVALID_ARG, "output size overflows size_t");
  if (wb) *wb = w;
  if (xb) *xb = x;
  if (ob) *ob = o;
  if (kp) *kp = k;
  return TCBF_OK;
}

tcbf_status check_device(const tcbf_plan* plan) {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev != plan->device)
    return fail(TCBF_ERR_DEVICE_MISMATCH, "current device %d differs from the plan's device %d", dev, plan->device);
  return TCBF_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency).
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

tcbf_status encode_3d(CUtensorMap* map, CUtensorMapDataType dt, size_t elem, const void* base, uint64_t d0,
                      uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1, CUtensorMapSwizzle sw,
                      CUtensorMapL2promotion l2) {
  auto enc = get_encode();
  if (!enc) return fail(TCBF_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * elem, d0 * d1 * elem};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TCBF_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
  return TCBF_OK;
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

}  // namespace

void retain_pool_memory() {
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

void tcbf_internal_set_launches(int n) { g_launches = n; }

tcbf_status tcbf_internal_fail(tcbf_status s, const char* what) { return fail(s, "%s", what); }

tcbf_status tcbf_internal_cuda_fail(cudaError_t e, const char* what) { return cuda_fail(e, what); }

namespace {

// Experiment overrides (DESIGN.md §4 variant studies, tests that force a kernel).  Read ONCE, at
// plan creation; a plan never consults the environment again, so its results and its kernel
// choice are fixed for its lifetime (the immutable plan of SURVEY.md §8b).
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}
bool env_set(const char* name) { return getenv(name) != nullptr; }

// Streaming-conversion kernel units (column tiles x K splits) for an M <= 128 fp16 plan.
int64_t conv_units(const tcbf_plan* p, int* splits) {
  const int64_t tiles = ((p->N + 127) / 128) * p->B;
  const int bk = tcbf::gemm_f16_conv_block_k();
  const int nkb = (int)((p->K + bk - 1) / bk);
  int sp = tiles < INT32_MAX ? tcbf::gemm_f16_conv_splits((int)tiles, nkb, p->num_sms) : 1;
  if (p->conv_splits_override > 0) sp = std::max(1, std::min(p->conv_splits_override, nkb));
  const int kbps = (nkb + sp - 1) / sp;
  sp = (nkb + kbps - 1) / kbps;
  if (splits) *splits = sp;
  return tiles * sp;
}

void choose_kernels(tcbf_plan* p) {
  // fp16 GEMM tile: 128x64 when N <= 64, else 128x128 (BK 64, 3 stages, 4 epilogue warps); CTA
  // pairs (cta_group::2) halve the per-SM shared-memory traffic of the B operand when M spans more
  // than one 128-row tile and K is long enough to be compute-bound (DESIGN.md §4 variant table)
  if (p->N <= 64) p->f16_variant = tcbf::F16_V_N64;
  else if (p->M <= 128 || p->N % 4 != 0) p->f16_variant = tcbf::F16_V_K64_S3;
  else if (p->K >= 2048 && p->N >= 256) p->f16_variant = tcbf::F16_V_2CTA_N256;  // long K: compute-bound
  else if (p->kp > 256) p->f16_variant = tcbf::F16_V_2CTA_N128;                 // mid K (measured +5-8%)
  else p->f16_variant = tcbf::F16_V_K64_S3;                                       // short K: store-bound
  // few tiles (small problems, e.g. square 1024^3: 64 CTAs of 256x128 pairs on 148 SMs): the
  // 128x64 tile fills twice as many SMs (measured 1024^3: 15.2 vs 18.6 us)
  {
    const int64_t pair_ctas = 2 * ((p->M + 255) / 256) * ((p->N + 127) / 128) * p->B;
    const int64_t n64_ctas = ((p->M + 127) / 128) * ((p->N + 63) / 64) * p->B;
    if ((p->f16_variant == tcbf::F16_V_2CTA_N128 || p->f16_variant == tcbf::F16_V_2CTA_N256) &&
        pair_ctas < p->num_sms / 2 && n64_ctas > pair_ctas)
      p->f16_variant = tcbf::F16_V_N64;
  }
  const int v = env_int("TCBF_F16_VARIANT", -1);
  if (v >= 0 && v < tcbf::F16_V_COUNT) p->f16_variant = v;

  // 1-bit: +-1 fp4 (kind::mxf4) tensor cores, exact while 32 Kw <= 2^23; int8 AND form beyond;
  // 2-3 K blocks (256 < K <= 768) with more than 64 beams: the sample-major kernel with the unit's
  // data resident in TMEM and line-store epilogue (radio 1-bit GEMM 1.73-1.91 -> 1.51-1.54 ms; at
  // one K block the beam-major kernel is faster: 372-385 vs 425-440 us for 2.15 GB of output)
  p->b1_kernel = tcbf::gemm_b1_f4_supported(p->kp) ? TCBF_B1K_F4 : TCBF_B1K_I8;
  if (tcbf::gemm_b1_tmem_supported(p->kp) && p->kp > 8 && p->M > 64) p->b1_kernel = TCBF_B1K_TMEM;
  if (const char* e = getenv("TCBF_B1_KERNEL")) {
    if (strcmp(e, "popc") == 0) p->b1_kernel = TCBF_B1K_POPC;
    else if (strcmp(e, "i8") == 0) p->b1_kernel = TCBF_B1K_I8;
    else if (strcmp(e, "bmma") == 0) p->b1_kernel = TCBF_B1K_BMMA;
    else if (strcmp(e, "f4") == 0 && tcbf::gemm_b1_f4_supported(p->kp)) p->b1_kernel = TCBF_B1K_F4;
    else if (strcmp(e, "tmem") == 0 && tcbf::gemm_b1_tmem_supported(p->kp)) p->b1_kernel = TCBF_B1K_TMEM;
  }
  p->b1_swap_beams = (p->b1_kernel == TCBF_B1K_F4 && !env_set("TCBF_NO_SWAP")) ? tcbf::gemm_b1_f4_swap_beams(p->M) : 0;
  // experiment overrides: the swapped kernel (64-beam tiles) for any M; coalesced st.global
  // epilogue instead of TMA stores
  if (env_int("TCBF_B1_SWAP", 0) == 64 && tcbf::gemm_b1_f4_supported(p->kp) &&
      (p->b1_kernel == TCBF_B1K_F4 || p->b1_kernel == TCBF_B1K_TMEM)) {
    p->b1_kernel = TCBF_B1K_F4;
    p->b1_swap_beams = 64;
  }
  p->b1_force_stg = env_int("TCBF_B1_STG", 0) != 0;
  // split-K of the int8 kernel: measured not to shorten the per-SM K chain, so only forced (tests)
  p->b1_splits = 1;
  p->b1_kb_per_split = (int)(p->kp / 4);
  if (p->b1_kernel == TCBF_B1K_I8) {
    const int64_t nkb = p->kp / 4;
    const int64_t sp = std::min<int64_t>(std::max(1, env_int("TCBF_B1_SPLITS", 1)), nkb);
    if (sp > 1) {
      p->b1_kb_per_split = (int)((nkb + sp - 1) / sp);
      p->b1_splits = (int)((nkb + p->b1_kb_per_split - 1) / p->b1_kb_per_split);
    }
  }
  p->pack_wpt = env_int("TCBF_PACK_WPT", 0);

  // tcbf_beamform_raw: data conversion fused into the GEMM where the shape allows it
  const bool no_fused = env_int("TCBF_NO_FUSED", 0) != 0;
  p->f16_multicast = env_int("TCBF_F16_MC", 1) != 0;
  p->conv_splits_override = env_int("TCBF_CONV_SPLITS", 0);
  p->raw_mode = TCBF_RAW_PACK;
  // fused kernel kind: sample-major (coalesced line stores straight from TMEM, any N) by default;
  // the beam-major TMA-store kernel (needs N % 4 == 0) stays selectable for comparison
  // (default: data resident in TMEM, next unit staged in smem; TCBF_F16_FUSED=smaj keeps the data
  // in smem, =beam the beam-major TMA-store kernel)
  // (the TMEM kernel takes the raw data by TMA: 16-byte rows need N % 4 == 0 in either layout;
  // other N take the smem sample-major kernel, chosen here so the plan's kernel name holds)
  p->f16_fused_kind = p->N % 4 == 0 ? TCBF_FUSED_TMEM : TCBF_FUSED_SMAJ;
  // K16 = 256 (the radio shape class): 32-beam tiles, half of the next unit written straight into
  // TMEM, the freed staging spent on a deeper weight ring (gemm_f16_tmem2.cu; TCBF_F16_FUSED=tmem
  // keeps the 64-beam kernel); WKB 4 (one 32 KB stage per tile) measured fastest
  const int tmem32_wkb = env_int("TCBF_TMEM2_WKB", 4) == 2 ? 2 : 4;
  p->tmem32 = tcbf::gemm_f16_tmem2_supported(p->kp) ? tmem32_wkb : 0;
  if (const char* e = getenv("TCBF_F16_FUSED")) {
    if (strcmp(e, "smaj") == 0) p->f16_fused_kind = TCBF_FUSED_SMAJ;
    else if (strcmp(e, "tmem") == 0 && p->N % 4 == 0) {
      p->f16_fused_kind = TCBF_FUSED_TMEM;
      p->tmem32 = 0;
    }
  }
  p->tmem_wkb = env_int("TCBF_TMEM_WKB", 1) == 2 ? 2 : 1;  // K blocks per weight stage
  // weight multicast cluster of the sample-major kernel (TCBF_F16_MC=0 turns multicast off)
  p->smaj_cluster = p->f16_multicast ? 2 : 1;
  p->f16i_resident = tcbf::gemm_f16_ileave_res_supported(p->kp) && !env_set("TCBF_F16I_STREAM");
  // fp16 interleaved data: the data-in-TMEM kernel where it applies (TCBF_F16I=res keeps the
  // kernel that multiplies the interleaved tile as stored, TCBF_F16I_STREAM the streaming one)
  p->f16i_tmem = tcbf::gemm_f16_tmem_supported(p->kp) && !env_set("TCBF_F16I_STREAM");
  if (const char* e = getenv("TCBF_F16I"))
    if (strcmp(e, "res") == 0) p->f16i_tmem = 0;
  if (p->prec == TCBF_PREC_F16 && !no_fused) {
    const bool fusable = p->f16_fused_kind == TCBF_FUSED_TMEM ? tcbf::gemm_f16_tmem_supported(p->kp)
                                                              : tcbf::gemm_f16_smaj_supported(p->kp);
    if (fusable) {
      p->raw_mode = TCBF_RAW_FUSED;
    } else if (p->M <= 128 && p->N % 4 == 0) {
      // every data element enters one tile: stream the fp32 data through the GEMM once; needs
      // enough (column tile x K split) units to occupy the GPU (measured: below a quarter of
      // the SMs, pack + GEMM wins)
      if (conv_units(p, nullptr) >= p->num_sms / 4 || env_set("TCBF_FORCE_STREAM_CONV")) p->raw_mode = TCBF_RAW_STREAM;
    }
  }
  p->debug = 0;
#ifdef TCBF_DEV
  p->debug = env_int("TCBF_DEBUG", 0);
#endif
}

const char* gemm_kernel_name(const tcbf_plan* plan) {
  if (plan->prec == TCBF_PREC_B1) {
    const bool tma = plan->N % 4 == 0;
    switch (plan->b1_kernel) {
      case TCBF_B1K_POPC: return "b1_popc_xor_64x64";
      case TCBF_B1K_BMMA: return "b1_mma_sync_and_128x64";
      case TCBF_B1K_I8: return tma ? "b1_tcgen05_i8_128x128_tma" : "b1_tcgen05_i8_128x128_stg";
      case TCBF_B1K_TMEM: return "b1_tcgen05_mxf4pm1_tmem_128x64";
      default: break;
    }
    if (plan->b1_swap_beams == 32)
      return tma ? "b1_tcgen05_mxf4pm1_swap_128x32_tma" : "b1_tcgen05_mxf4pm1_swap_128x32_stg";
    if (plan->b1_swap_beams == 64)
      return tma ? "b1_tcgen05_mxf4pm1_swap_128x64_tma" : "b1_tcgen05_mxf4pm1_swap_128x64_stg";
    return tma ? "b1_tcgen05_mxf4pm1_atmem_128x128_tma" : "b1_tcgen05_mxf4pm1_atmem_128x128_stg";
  }
  if (plan->N % 4 != 0)
    return plan->f16_variant == tcbf::F16_V_N64 ? "f16_tcgen05_128x64_masked" : "f16_tcgen05_128x128_masked";
  static const char* names[tcbf::F16_V_COUNT] = {
      "f16_tcgen05_128x128_k32s4e8_tma", "f16_tcgen05_128x128_k64s3e4_tma", "f16_tcgen05_128x64_k64s4e4_tma",
      "f16_tcgen05_2cta_256x128_k64s4_tma", "f16_tcgen05_2cta_256x256_k64s3_tma"};
  return names[plan->f16_variant];
}

}  // namespace

namespace {

tcbf_status beamform_f16(const tcbf_plan* plan, const void* w_packed, const void* x_packed, void* out,
                         cudaStream_t st) {
  // Final kernel choice first, so the tensor-map boxes always match the instantiation:
  // TMA bulk store needs N % 4 == 0 (16-B row stride), otherwise the masked-store epilogue
  // (instantiated for the N64 and K64_S3 tiles only).
  int var = plan->f16_variant;
  int epi = 0;
  if (plan->N % 4 != 0) {
    epi = 2;
    if (var != tcbf::F16_V_N64) var = tcbf::F16_V_K64_S3;
  }
  const int bn = tcbf::gemm_f16_block_n(var);
  const int bk = tcbf::gemm_f16_block_k(var);
  const bool use_pair = var == tcbf::F16_V_2CTA_N128 || var == tcbf::F16_V_2CTA_N256;
  CUtensorMap ta, tb, tc;
  // A (weights, K-major [2B][M][K16]): box {BK, 128}, swizzle = BK * 2 bytes
  tcbf_status s = encode_3d(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w_packed, plan->kp, plan->M, 2 * plan->B, bk,
                            128, bk == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (s != TCBF_OK) return s;
  // B (data, MN-major [2B][K][Np]): box {64 columns, BK rows}, 128-byte swizzle; K tail is OOB -> 0
  s = encode_3d(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, x_packed, plan->n_packed, plan->K, 2 * plan->B, 64, bk,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (s != TCBF_OK) return s;
  if (epi == 0) {
    s = encode_3d(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, out, plan->N, plan->M, 2 * plan->B, 32, 32,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE);
    if (s != TCBF_OK) return s;
  } else {
    memset(&tc, 0, sizeof(tc));
  }
  tcbf::GemmF16Args a;
  memset(&a, 0, sizeof(a));
  a.M = (int)plan->M; a.N = (int)plan->N; a.B = (int)plan->B; a.K16 = (int)plan->kp;
  a.tiles_m = (int)((plan->M + (use_pair ? 255 : 127)) / (use_pair ? 256 : 128));
  a.tiles_n = (int)((plan->N + bn - 1) / bn);
  const int64_t nt = (int64_t)a.tiles_m * a.tiles_n * plan->B;
  if (nt > INT32_MAX) return fail(TCBF_ERR_INVALID_ARG, "too many tiles");
  a.num_tiles = (int)nt;
  a.num_kb = (int)(plan->kp / bk);
  a.out = static_cast<float*>(out);
  {  // rasterisation group: keep ~48 MB of weight rows (A_r + A_i, K16 fp16) of a group in L2
    const int64_t rows_per_tile = use_pair ? 256 : 128;
    const int64_t bytes_per_tile_row = rows_per_tile * plan->kp * 4;
    int64_t gm = (48ll << 20) / (bytes_per_tile_row > 0 ? bytes_per_tile_row : 1);
    a.group_m = (int)std::max<int64_t>(1, std::min<int64_t>(gm, a.tiles_m));
  }
  a.debug = plan->debug;
  cudaError_t e = use_pair ? tcbf::launch_gemm_f16_2cta(ta, tb, tc, a, bn, plan->num_sms, st)
                           : tcbf::launch_gemm_f16(ta, tb, tc, a, var, epi, plan->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(e, "beamform kernel launch");
  g_launches = 1;
  return TCBF_OK;
}

tcbf_status beamform_b1(const tcbf_plan* plan, const void* w_packed, const void* x_packed, void* out,
                        cudaStream_t st) {
  tcbf::GemmB1Args a;
  memset(&a, 0, sizeof(a));
  a.w = static_cast<const uint32_t*>(w_packed);
  a.x = static_cast<const uint32_t*>(x_packed);
  a.out = static_cast<int32_t*>(out);
  a.M = (int)plan->M; a.N = (int)plan->N; a.K = (int)plan->K; a.Kw = (int)plan->kp; a.B = (int)plan->B;
  a.debug = plan->debug;
  {  // rasterisation group: 1-bit operands are small; ~16 MB of packed weight rows per group
    const int64_t bytes_per_tile_row = 128 * plan->kp * 8;
    const int64_t tm = (plan->M + 127) / 128;
    a.group_m = (int)std::max<int64_t>(1, std::min<int64_t>((16ll << 20) / bytes_per_tile_row, tm));
  }
  a.splits = plan->b1_splits;
  a.kb_per_split = plan->b1_kb_per_split;
  cudaError_t e;
  if (a.splits > 1) {  // exact int32 partials reduce-added into a zeroed output
    e = cudaMemsetAsync(out, 0, plan->out_bytes, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync (split-K output)");
  }
  const bool tma_store = (plan->N % 4) == 0 && !plan->b1_force_stg;
  tcbf_status s;
  if (plan->b1_kernel == TCBF_B1K_TMEM) {
    // packed words whole rows per box: weights {Kw, 64 beams}, data {Kw, 128 samples}, no swizzle
    CUtensorMap tw, tx;
    s = encode_3d(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, w_packed, plan->kp, plan->M, 2 * plan->B,
                  (uint32_t)plan->kp, (uint32_t)tcbf::gemm_b1_tmem_beams(), CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (s != TCBF_OK) return s;
    s = encode_3d(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, x_packed, plan->kp, plan->N, 2 * plan->B,
                  (uint32_t)plan->kp, 128, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (s != TCBF_OK) return s;
    e = tcbf::launch_gemm_b1_tmem(tw, tx, a, plan->num_sms, st);
  } else if (plan->b1_kernel == TCBF_B1K_BMMA) {
    e = tcbf::launch_gemm_b1_mma(a, st);
  } else if (plan->b1_kernel == TCBF_B1K_POPC) {
    e = tcbf::launch_gemm_b1_popc(a, st);
  } else {
    CUtensorMap tc;
    memset(&tc, 0, sizeof(tc));
    if (plan->b1_swap_beams) {  // few beams: samples on the 128-row MMA dimension, beams on N
      CUtensorMap tw, tx;
      // packed words in boxes of four 256-bit K blocks (128-byte rows, 128-byte swizzle; words past
      // Kw are zero-filled and never expanded)
      const uint32_t bw = (uint32_t)tcbf::gemm_b1_f4_swap_box_words();
      s = encode_3d(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, w_packed, plan->kp, plan->M, 2 * plan->B, bw,
                    (uint32_t)plan->b1_swap_beams, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
      if (s != TCBF_OK) return s;
      s = encode_3d(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, x_packed, plan->kp, plan->N, 2 * plan->B, bw, 128,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
      if (s != TCBF_OK) return s;
      if (tma_store) {  // 32 beams x 32 samples boxes, unswizzled 128-byte rows
        s = encode_3d(&tc, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, out, plan->N, plan->M, 2 * plan->B, 32, 32,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE);
        if (s != TCBF_OK) return s;
      }
#ifdef TCBF_DEV
      const char* trace_file = getenv("TCBF_TRACE");  // dev timeline (tools/trace_swap.py)
      if (trace_file) {
        cudaMalloc(&a.trace, (size_t)plan->num_sms * 1024 * 8);
        cudaMemsetAsync(a.trace, 0, (size_t)plan->num_sms * 1024 * 8, st);
      }
#endif
      e = tcbf::launch_gemm_b1_f4_swap(tw, tx, tc, a, plan->b1_swap_beams, tma_store, plan->num_sms, st);
#ifdef TCBF_DEV
      if (trace_file) {
        std::vector<unsigned long long> h((size_t)plan->num_sms * 1024);
        cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        cudaFree(a.trace);
        if (FILE* f = fopen(trace_file, "wb")) {
          fwrite(h.data(), 8, h.size(), f);
          fclose(f);
        }
      }
#endif
    } else if (plan->b1_kernel == TCBF_B1K_F4) {  // packed words by TMA: box {one 256-bit K block, 128 rows}
      CUtensorMap tw, tx;
      if (tma_store) {
        const bool box16 = tcbf::gemm_b1_f4_store_box_cols(plan->kp) == 16;  // 32 x 16 boxes, 64-byte swizzle
        s = encode_3d(&tc, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, out, plan->N, plan->M, 2 * plan->B, box16 ? 16 : 32, 32,
                      box16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE);
        if (s != TCBF_OK) return s;
      }
      const uint32_t kbw = (uint32_t)tcbf::gemm_b1_f4_block_words();
      s = encode_3d(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, w_packed, plan->kp, plan->M, 2 * plan->B, kbw, 128,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
      if (s != TCBF_OK) return s;
      s = encode_3d(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, x_packed, plan->kp, plan->N, 2 * plan->B, kbw, 128,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
      if (s != TCBF_OK) return s;
      e = tcbf::launch_gemm_b1_f4(tw, tx, tc, a, tma_store, plan->num_sms, st);
    } else {  // int8 AND form: per-warp 32-row x 32-column boxes
      if (tma_store) {
        s = encode_3d(&tc, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, out, plan->N, plan->M, 2 * plan->B, 32, 32,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE);
        if (s != TCBF_OK) return s;
      }
      e = tcbf::launch_gemm_b1_tc(tc, a, tma_store, plan->num_sms, st);
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, "beamform kernel launch");
  g_launches = a.splits > 1 ? 2 : 1;  // memset + kernel when split-K
  return TCBF_OK;
}

}  // namespace

extern "C" {

tcbf_status tcbf_layout_sizes(int64_t M, int64_t N, int64_t K, int64_t batch, tcbf_precision precision,
                              size_t* w_bytes, size_t* x_bytes, size_t* out_bytes, int64_t* k_packed) {
  return compute_sizes(M, N, K, batch, precision, w_bytes, x_bytes, out_bytes, k_packed);
}

tcbf_status tcbf_plan_create(tcbf_plan** plan, int64_t M, int64_t N, int64_t K, int64_t batch,
                             tcbf_precision precision) {
  if (!plan) return fail(TCBF_ERR_INVALID_ARG, "plan out-pointer is NULL");
  *plan = nullptr;
  size_t wb, xb, ob;
  int64_t kp;
  tcbf_status s = compute_sizes(M, N, K, batch, precision, &wb, &xb, &ob, &kp);
  if (s != TCBF_OK) return s;
  int dev = -1, major = 0, minor = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(TCBF_ERR_UNSUPPORTED_DEVICE, "no CUDA device: %s", cudaGetErrorString(e));
  }
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return fail(TCBF_ERR_UNSUPPORTED_DEVICE, "cannot query device %d", dev);
  }
  if (major != 10 || minor != 0)
    return fail(TCBF_ERR_UNSUPPORTED_DEVICE, "device %d is sm_%d%d; this library is built for sm_100a", dev, major,
                minor);
  tcbf_plan* p = new (std::nothrow) tcbf_plan_s;
  if (!p) return fail(TCBF_ERR_ALLOC, "host allocation of the plan failed");
  memset(p, 0, sizeof(*p));
  p->M = M; p->N = N; p->K = K; p->B = batch;
  p->prec = precision;
  p->kp = kp;
  p->device = dev;
  p->num_sms = sms;
  p->w_bytes = wb; p->x_bytes = xb; p->out_bytes = ob;
  p->n_packed = (N + 7) / 8 * 8;
  choose_kernels(p);
  *plan = p;
  return TCBF_OK;
}

tcbf_status tcbf_plan_destroy(tcbf_plan* plan) {
  delete plan;
  return TCBF_OK;
}

tcbf_status tcbf_packed_bytes(const tcbf_plan* plan, tcbf_operand operand, size_t* bytes) {
  if (!plan || !bytes) return fail(TCBF_ERR_INVALID_ARG, "NULL argument");
  if (operand != TCBF_WEIGHTS && operand != TCBF_DATA) return fail(TCBF_ERR_INVALID_ARG, "bad operand");
  *bytes = operand == TCBF_WEIGHTS ? plan->w_bytes : plan->x_bytes;
  return TCBF_OK;
}

tcbf_status tcbf_output_bytes(const tcbf_plan* plan, size_t* bytes) {
  if (!plan || !bytes) return fail(TCBF_ERR_INVALID_ARG, "NULL argument");
  *bytes = plan->out_bytes;
  return TCBF_OK;
}

const char* tcbf_plan_variant(const tcbf_plan* plan) {
  if (!plan) return "none";
  return gemm_kernel_name(plan);
}

const char* tcbf_plan_kernel(const tcbf_plan* plan, tcbf_entry entry) {
  if (!plan) return "none";
  switch (entry) {
    case TCBF_ENTRY_BEAMFORM: return gemm_kernel_name(plan);
    case TCBF_ENTRY_BEAMFORM_RAW:
      if (plan->raw_mode == TCBF_RAW_FUSED)
        return plan->f16_fused_kind == TCBF_FUSED_TMEM ? (plan->tmem32 ? "f16_tcgen05_fused_tmem_128x32"
                                                                        : "f16_tcgen05_fused_tmem_128x64")
                                                       : "f16_tcgen05_fused_smaj_128x128";
      if (plan->raw_mode == TCBF_RAW_STREAM) return "f16_tcgen05_stream_conv_128x128";
      return gemm_kernel_name(plan);  // preceded by the pack kernel
    case TCBF_ENTRY_BEAMFORM_F16I:
      return plan->prec != TCBF_PREC_F16 ? "none"
             : plan->f16i_tmem     ? (plan->tmem32 ? "f16_tcgen05_interleaved_tmem_128x32"
                                                   : "f16_tcgen05_interleaved_tmem_128x64")
             : plan->f16i_resident ? "f16_tcgen05_interleaved_resident_128x64" : "f16_tcgen05_interleaved_smaj_64x128";
  }
  return "none";
}

int tcbf_plan_raw_fused(const tcbf_plan* plan) { return plan && plan->raw_mode != TCBF_RAW_PACK ? 1 : 0; }

tcbf_status tcbf_pack(const tcbf_plan* plan, tcbf_operand operand, const float* src, tcbf_src_layout layout,
                      void* dst, void* stream) {
  g_launches = 0;
  if (!plan || !src || !dst) return fail(TCBF_ERR_INVALID_ARG, "NULL argument");
  if (operand != TCBF_WEIGHTS && operand != TCBF_DATA) return fail(TCBF_ERR_INVALID_ARG, "bad operand");
  if (layout != TCBF_SRC_INTERLEAVED && layout != TCBF_SRC_PLANAR) return fail(TCBF_ERR_INVALID_ARG, "bad layout");
  if (!aligned(src, layout == TCBF_SRC_INTERLEAVED ? 8 : 4) || !aligned(dst, 16))
    return fail(TCBF_ERR_INVALID_ARG, "misaligned src (needs %d B) or dst (needs 16 B)",
                layout == TCBF_SRC_INTERLEAVED ? 8 : 4);
  tcbf_status s = check_device(plan);
  if (s != TCBF_OK) return s;
  const int64_t R = operand == TCBF_WEIGHTS ? plan->M : plan->K;
  const int64_t C = operand == TCBF_WEIGHTS ? plan->K : plan->N;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (plan->prec == TCBF_PREC_F16)
    e = tcbf::launch_pack_f16(src, (int)layout, (int)operand, plan->B, R, C,
                              operand == TCBF_WEIGHTS ? plan->kp : plan->n_packed, static_cast<uint16_t*>(dst), st);
  else
    e = tcbf::launch_pack_b1(src, (int)layout, (int)operand, plan->B, R, C, plan->kp, plan->pack_wpt,
                             static_cast<uint32_t*>(dst), st);
  if (e != cudaSuccess) return cuda_fail(e, "pack kernel launch");
  g_launches = 1;
  return TCBF_OK;
}


tcbf_status tcbf_beamform(const tcbf_plan* plan, const void* w_packed, const void* x_packed, void* out, void* stream) {
  g_launches = 0;
  if (!plan || !w_packed || !x_packed || !out) return fail(TCBF_ERR_INVALID_ARG, "NULL argument");
  if (!aligned(w_packed, 16) || !aligned(x_packed, 16) || !aligned(out, 16))
    return fail(TCBF_ERR_INVALID_ARG, "packed operands and output must be 16-byte aligned");
  tcbf_status s = check_device(plan);
  if (s != TCBF_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return plan->prec == TCBF_PREC_F16 ? beamform_f16(plan, w_packed, x_packed, out, st)
                                     : beamform_b1(plan, w_packed, x_packed, out, st);
}

tcbf_status tcbf_beamform_raw(const tcbf_plan* plan, const void* w_packed, const float* x_src,
                              tcbf_src_layout layout, void* out, void* stream) {
  g_launches = 0;
  if (!plan || !w_packed || !x_src || !out) return fail(TCBF_ERR_INVALID_ARG, "NULL argument");
  if (layout != TCBF_SRC_INTERLEAVED && layout != TCBF_SRC_PLANAR) return fail(TCBF_ERR_INVALID_ARG, "bad layout");
  if (!aligned(w_packed, 16) || !aligned(out, 16) || !aligned(x_src, layout == TCBF_SRC_INTERLEAVED ? 8 : 4))
    return fail(TCBF_ERR_INVALID_ARG, "misaligned pointer");
  tcbf_status s = check_device(plan);
  if (s != TCBF_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // data-in-TMEM kernel (plans with N % 4 == 0): its raw fp32 data comes in by TMA, which needs a
  // 16-byte-aligned source; a source aligned only to 8 (interleaved) or 4 (planar) bytes takes the
  // smem sample-major kernel
  const bool tmem_tma_ok = aligned(x_src, 16);
  if (plan->raw_mode == TCBF_RAW_FUSED && plan->f16_fused_kind == TCBF_FUSED_TMEM && tmem_tma_ok) {
    // weights: the stacked K-major B operand, boxes {64 K, 64 beams} of a plane, 128-byte swizzle
    CUtensorMap tw, tx;
    const int bn = plan->tmem32 ? tcbf::gemm_f16_tmem2_beams() : tcbf::gemm_f16_tmem_beams();
    s = encode_3d(&tw, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w_packed, plan->kp, plan->M, 2 * plan->B, 64,
                  (uint32_t)bn, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (s != TCBF_OK) return s;
    const uint32_t rr = (uint32_t)tcbf::gemm_f16_tmem_raw_rows();
    if (layout == TCBF_SRC_INTERLEAVED)
      s = encode_3d(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x_src, 2 * plan->N, plan->K, plan->B, 256, rr,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    else
      s = encode_3d(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x_src, plan->N, plan->K, 2 * plan->B, 128, rr,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (s != TCBF_OK) return s;
    tcbf::GemmF16Args a;
    memset(&a, 0, sizeof(a));
    a.M = (int)plan->M; a.N = (int)plan->N; a.B = (int)plan->B; a.K16 = (int)plan->kp;
    a.tiles_m = (int)((plan->M + bn - 1) / bn);  // 64- (32-) beam tiles
    a.tiles_n = (int)((plan->N + 127) / 128);    // 128-sample units per batch entry
    a.num_kb = (int)(plan->kp / 64);
    const int64_t nu = (int64_t)a.tiles_n * plan->B;
    if (nu * a.tiles_m > INT32_MAX) return fail(TCBF_ERR_INVALID_ARG, "too many work units");
    a.num_tiles = (int)(nu * a.tiles_m);
    a.out = static_cast<float*>(out);
    a.debug = plan->debug;
#ifdef TCBF_DEV
    const char* trace_file = getenv("TCBF_TRACE");  // dev timeline (tools/trace_smaj.py)
    if (trace_file) {
      cudaMalloc(&a.trace, (size_t)plan->num_sms * 1024 * 8);
      cudaMemsetAsync(a.trace, 0, (size_t)plan->num_sms * 1024 * 8, st);
    }
#endif
    cudaError_t e = plan->tmem32 ? tcbf::launch_gemm_f16_tmem2(tw, tx, a, (int)layout, plan->tmem32, plan->smaj_cluster,
                                                            plan->num_sms, st)
                                 : tcbf::launch_gemm_f16_tmem(tw, tx, a, (int)layout, plan->tmem_wkb, plan->smaj_cluster,
                                                           plan->num_sms, st);
#ifdef TCBF_DEV
    if (trace_file) {
      std::vector<unsigned long long> h((size_t)plan->num_sms * 1024);
      cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      cudaFree(a.trace);
      if (FILE* f = fopen(trace_file, "wb")) {
        fwrite(h.data(), 8, h.size(), f);
        fclose(f);
      }
    }
#endif
    if (e != cudaSuccess) return cuda_fail(e, "fused (data in TMEM) beamform kernel launch");
    g_launches = 1;
    return TCBF_OK;
  }
  if (plan->raw_mode == TCBF_RAW_FUSED &&
      (plan->f16_fused_kind == TCBF_FUSED_SMAJ || plan->f16_fused_kind == TCBF_FUSED_TMEM)) {
    // weights as the stacked K-major B operand: boxes {64 K, 64 beams} of a plane, 128-byte swizzle
    // (a stage is four boxes, split among the CTAs of a multicast cluster)
    CUtensorMap tw;
    s = encode_3d(&tw, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w_packed, plan->kp, plan->M, 2 * plan->B, 64, 64,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (s != TCBF_OK) return s;
    tcbf::GemmF16Args a;
    memset(&a, 0, sizeof(a));
    a.M = (int)plan->M; a.N = (int)plan->N; a.B = (int)plan->B; a.K16 = (int)plan->kp;
    a.tiles_m = (int)((plan->M + 127) / 128);   // beam tiles
    a.tiles_n = (int)((plan->N + 127) / 128);   // 128-sample units per batch entry
    a.num_kb = (int)(plan->kp / 64);
    const int64_t nu = (int64_t)a.tiles_n * plan->B;
    if (nu * a.tiles_m > INT32_MAX) return fail(TCBF_ERR_INVALID_ARG, "too many work units");
    a.num_tiles = (int)(nu * a.tiles_m);
    a.out = static_cast<float*>(out);
    a.debug = plan->debug;
#ifdef TCBF_DEV
    const char* trace_file = getenv("TCBF_TRACE");  // dev timeline (tools/trace_smaj.py)
    if (trace_file) {
      cudaMalloc(&a.trace, (size_t)plan->num_sms * 1024 * 8);
      cudaMemsetAsync(a.trace, 0, (size_t)plan->num_sms * 1024 * 8, st);
    }
#endif
    cudaError_t e = tcbf::launch_gemm_f16_smaj(tw, a, x_src, (int)layout, (int)plan->K, plan->smaj_cluster,
                                               plan->num_sms, st);
#ifdef TCBF_DEV
    if (trace_file) {
      std::vector<unsigned long long> h((size_t)plan->num_sms * 1024);
      cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      cudaFree(a.trace);
      if (FILE* f = fopen(trace_file, "wb")) {
        fwrite(h.data(), 8, h.size(), f);
        fclose(f);
      }
    }
#endif
    if (e != cudaSuccess) return cuda_fail(e, "fused (sample-major) beamform kernel launch");
    g_launches = 1;
    return TCBF_OK;
  }
  if (plan->raw_mode == TCBF_RAW_STREAM && aligned(x_src, 16)) {
    // Small-M plans (one 128-row weight tile): every data element enters one tile, so the
    // streaming kernel converts the fp32 data on the fly (no separate pack pass).
    const int bk = tcbf::gemm_f16_conv_block_k();
    CUtensorMap ta, tx, tc;
    s = encode_3d(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w_packed, plan->kp, plan->M, 2 * plan->B, bk, 128,
                  CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (s != TCBF_OK) return s;
    // raw fp32 data: interleaved [B][K][2N] (box 256 floats = 128 complex x 32 k-rows) or planar
    // [2B][K][N] (box 128 x 32 per plane); out-of-range k / n are zero-filled by the TMA unit
    if (layout == TCBF_SRC_INTERLEAVED)
      s = encode_3d(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x_src, 2 * plan->N, plan->K, plan->B, 256, bk,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    else
      s = encode_3d(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x_src, plan->N, plan->K, 2 * plan->B, 128, bk,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (s != TCBF_OK) return s;
    s = encode_3d(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, out, plan->N, plan->M, 2 * plan->B, 32, 128,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE);
    if (s != TCBF_OK) return s;
    tcbf::GemmF16Args a;
    memset(&a, 0, sizeof(a));
    a.M = (int)plan->M; a.N = (int)plan->N; a.B = (int)plan->B; a.K16 = (int)plan->kp;
    a.tiles_m = 1;
    a.tiles_n = (int)((plan->N + 127) / 128);
    a.group_m = 1;
    const int64_t nt = (int64_t)a.tiles_n * plan->B;
    if (nt * 16 > INT32_MAX) return fail(TCBF_ERR_INVALID_ARG, "too many tiles");
    a.num_tiles = (int)nt;
    a.num_kb = (int)((plan->K + bk - 1) / bk);
    conv_units(plan, &a.splits);
    a.kb_per_split = (a.num_kb + a.splits - 1) / a.splits;
    a.out = static_cast<float*>(out);
    a.debug = plan->debug;
    int launches = 1;
    if (a.splits > 1) {  // partial sums are reduce-added into a zeroed output
      cudaError_t e = cudaMemsetAsync(out, 0, plan->out_bytes, st);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync (split-K output)");
      launches = 2;
    }
    cudaError_t e = tcbf::launch_gemm_f16_conv(ta, tx, tc, a, (int)layout, plan->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(e, "streaming-conversion beamform kernel launch");
    g_launches = launches;
    return TCBF_OK;
  }
  // Pack into stream-ordered scratch, then beamform.  Keep the pool's memory cached between calls
  // (the default release threshold returns it to the driver at every synchronisation, making each
  // call pay a fresh allocation).
  retain_pool_memory();
  void* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, plan->x_bytes, st);
  if (e != cudaSuccess) return fail(TCBF_ERR_ALLOC, "cudaMallocAsync (data scratch): %s", cudaGetErrorString(e));
  s = tcbf_pack(plan, TCBF_DATA, x_src, layout, scratch, stream);
  int launches = s == TCBF_OK ? 1 : 0;
  if (s == TCBF_OK) {
    s = tcbf_beamform(plan, w_packed, scratch, out, stream);
    launches += g_launches;
  }
  cudaFreeAsync(scratch, st);
  g_launches = s == TCBF_OK ? launches : 0;
  return s;
}
tcbf_status tcbf_beamform_f16i(const tcbf_plan* plan, const void* w_packed, const void* x_f16, void* out,
                               void* stream) {
  g_launches = 0;
  if (!plan || !w_packed || !x_f16 || !out) return fail(TCBF_ERR_INVALID_ARG, "NULL argument");
  if (plan->prec != TCBF_PREC_F16) return fail(TCBF_ERR_INVALID_ARG, "tcbf_beamform_f16i needs an F16 plan");
  if (plan->N % 4) return fail(TCBF_ERR_INVALID_ARG, "tcbf_beamform_f16i needs N %% 4 == 0");
  if (!aligned(w_packed, 16) || !aligned(x_f16, 16) || !aligned(out, 16))
    return fail(TCBF_ERR_INVALID_ARG, "operands and output must be 16-byte aligned");
  tcbf_status s = check_device(plan);
  if (s != TCBF_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (plan->f16i_tmem) {
    // data-in-TMEM kernel with the fp16 pairs by TMA ({N, K, B} 32-bit elements, 16-row boxes),
    // de-interleaved into the staged next unit (DESIGN.md §4 NEXT-1)
    CUtensorMap tw, tx;
    const int bn = plan->tmem32 ? tcbf::gemm_f16_tmem2_beams() : tcbf::gemm_f16_tmem_beams();
    s = encode_3d(&tw, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w_packed, plan->kp, plan->M, 2 * plan->B, 64,
                  (uint32_t)bn, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (s != TCBF_OK) return s;
    s = encode_3d(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, x_f16, plan->N, plan->K, plan->B, 128,
                  (uint32_t)tcbf::gemm_f16_tmem_raw_rows(), CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (s != TCBF_OK) return s;
    tcbf::GemmF16Args a;
    memset(&a, 0, sizeof(a));
    a.M = (int)plan->M; a.N = (int)plan->N; a.B = (int)plan->B; a.K16 = (int)plan->kp;
    a.tiles_m = (int)((plan->M + bn - 1) / bn);
    a.tiles_n = (int)((plan->N + 127) / 128);
    a.num_kb = (int)(plan->kp / 64);
    const int64_t nu = (int64_t)a.tiles_n * plan->B;
    if (nu * a.tiles_m > INT32_MAX) return fail(TCBF_ERR_INVALID_ARG, "too many tiles");
    a.num_tiles = (int)(nu * a.tiles_m);
    a.out = static_cast<float*>(out);
    a.debug = plan->debug;
    cudaError_t e = plan->tmem32 ? tcbf::launch_gemm_f16_tmem2(tw, tx, a, 2, plan->tmem32, plan->smaj_cluster,
                                                            plan->num_sms, st)
                                 : tcbf::launch_gemm_f16_tmem(tw, tx, a, 2, plan->tmem_wkb, plan->smaj_cluster,
                                                           plan->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(e, "interleaved-fp16 (data in TMEM) beamform kernel launch");
    g_launches = 1;
    return TCBF_OK;
  }
  if (plan->f16i_resident) {
    // data resident per 128-sample unit, 64-beam tiles: weights box {64 K, 64 beams}; interleaved
    // data as a real [B][K][2N] fp16 matrix, boxes {64 columns, 64 k-rows} (128-byte swizzle)
    CUtensorMap tw, tx;
    const int bb = tcbf::gemm_f16_ileave_res_beams(), bs = tcbf::gemm_f16_ileave_res_samples();
    s = encode_3d(&tw, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w_packed, plan->kp, plan->M, 2 * plan->B, 64, bb,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (s != TCBF_OK) return s;
    s = encode_3d(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, x_f16, 2 * plan->N, plan->K, plan->B, 64, 64,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (s != TCBF_OK) return s;
    tcbf::GemmF16Args a;
    memset(&a, 0, sizeof(a));
    a.multicast = plan->f16_multicast;
    a.M = (int)plan->M; a.N = (int)plan->N; a.B = (int)plan->B; a.K16 = (int)plan->kp;
    a.tiles_m = (int)((plan->M + bb - 1) / bb);
    a.tiles_n = (int)((plan->N + bs - 1) / bs);
    a.num_kb = (int)(plan->kp / 64);
    const int64_t nu = (int64_t)a.tiles_n * plan->B;
    if (nu * a.tiles_m > INT32_MAX) return fail(TCBF_ERR_INVALID_ARG, "too many tiles");
    a.num_tiles = (int)(nu * a.tiles_m);
    a.out = static_cast<float*>(out);
    a.debug = plan->debug;
    cudaError_t e = tcbf::launch_gemm_f16_ileave_res(tw, tx, a, plan->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(e, "interleaved-fp16 (resident) beamform kernel launch");
    g_launches = 1;
    return TCBF_OK;
  }
  const int bk = tcbf::gemm_f16_ileave_block_k(), bnc = tcbf::gemm_f16_ileave_block_n();
  CUtensorMap ta, tx, tc;
  s = encode_3d(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w_packed, plan->kp, plan->M, 2 * plan->B, bk, 128,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (s != TCBF_OK) return s;
  // interleaved data as a real [B][K][2N] fp16 matrix: 64-column x BK-row MN-major boxes
  s = encode_3d(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, x_f16, 2 * plan->N, plan->K, plan->B, 64, bk,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  if (s != TCBF_OK) return s;
  memset(&tc, 0, sizeof(tc));  // output written by coalesced st.global straight from TMEM (no TMA map)
  tcbf::GemmF16Args a;
  memset(&a, 0, sizeof(a));
  a.multicast = plan->f16_multicast;
  a.M = (int)plan->M; a.N = (int)plan->N; a.B = (int)plan->B; a.K16 = (int)plan->kp;
  a.tiles_m = (int)((plan->M + 127) / 128);
  a.tiles_n = (int)((plan->N + bnc - 1) / bnc);
  a.out = static_cast<float*>(out);
  a.debug = plan->debug;
  const int64_t nt = (int64_t)a.tiles_m * a.tiles_n * plan->B;
  if (nt > INT32_MAX) return fail(TCBF_ERR_INVALID_ARG, "too many tiles");
  a.num_tiles = (int)nt;
  a.num_kb = (int)(plan->kp / bk);
  {  // rasterisation group: ~48 MB of weight rows in L2
    const int64_t bytes_per_tile_row = 128 * plan->kp * 4;
    a.group_m = (int)std::max<int64_t>(1, std::min<int64_t>((48ll << 20) / bytes_per_tile_row, a.tiles_m));
  }
  cudaError_t e = tcbf::launch_gemm_f16_ileave(ta, tx, tc, a, plan->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(e, "interleaved-fp16 beamform kernel launch");
  g_launches = 1;
  return TCBF_OK;
}

tcbf_status tcbf_steering_weights(const tcbf_plan* plan, const double* positions, const double* angles,
                                  const double* freqs, double c, tcbf_src_layout layout, float* dst,
                                  void* stream) {
  g_launches = 0;
  if (!plan || !positions || !angles || !freqs || !dst) return fail(TCBF_ERR_INVALID_ARG, "NULL argument");
  if (!(c > 0.0)) return fail(TCBF_ERR_INVALID_ARG, "wave speed must be > 0");
  if (layout != TCBF_SRC_INTERLEAVED && layout != TCBF_SRC_PLANAR) return fail(TCBF_ERR_INVALID_ARG, "bad layout");
  if (!aligned(dst, layout == TCBF_SRC_INTERLEAVED ? 8 : 4) || !aligned(positions, 8) || !aligned(angles, 8) ||
      !aligned(freqs, 8))
    return fail(TCBF_ERR_INVALID_ARG, "misaligned pointer");
  tcbf_status s = check_device(plan);
  if (s != TCBF_OK) return s;
  cudaError_t e = tcbf::launch_steering(positions, angles, freqs, c, plan->B, plan->M, plan->K, (int)layout, dst,
                                        static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "steering kernel launch");
  g_launches = 1;
  return TCBF_OK;
}

int tcbf_last_launch_count(void) { return g_launches; }

const char* tcbf_status_string(tcbf_status status) {
  switch (status) {
    case TCBF_OK: return "TCBF_OK";
    case TCBF_ERR_INVALID_ARG: return "TCBF_ERR_INVALID_ARG";
    case TCBF_ERR_UNSUPPORTED_DEVICE: return "TCBF_ERR_UNSUPPORTED_DEVICE";
    case TCBF_ERR_DEVICE_MISMATCH: return "TCBF_ERR_DEVICE_MISMATCH";
    case TCBF_ERR_ALLOC: return "TCBF_ERR_ALLOC";
    case TCBF_ERR_CUDA: return "TCBF_ERR_CUDA";
  }
  return "TCBF_ERR_UNKNOWN";
}

const char* tcbf_last_error(void) { return g_err; }

}  // extern "C"
