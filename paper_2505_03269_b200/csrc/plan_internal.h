// plan_internal.h -- the plan object behind the opaque tcbf_plan handle (host metadata only).
// Every field is fixed at tcbf_plan_create (kernel choice included, environment overrides read
// there once); the entry points only read it.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "tcbf.h"

enum { TCBF_B1K_POPC = 0, TCBF_B1K_I8 = 1, TCBF_B1K_F4 = 4, TCBF_B1K_BMMA = 5, TCBF_B1K_TMEM = 6 };
enum { TCBF_RAW_PACK = 0, TCBF_RAW_FUSED = 1, TCBF_RAW_STREAM = 2 };
enum { TCBF_FUSED_SMAJ = 0, TCBF_FUSED_TMEM = 2 };

struct tcbf_plan_s {
  int64_t M, N, K, B;
  tcbf_precision prec;
  int64_t kp;   // K16 (fp16 elements) or Kw (uint32 words)
  int device;
  int num_sms;
  int64_t n_packed;  // F16 data row length Np = round_up(N, 8) (MN-major packed data)
  size_t w_bytes, x_bytes, out_bytes;
  // kernel choice (choose_kernels in plan.cu)
  int f16_variant;    // tcbf::F16_V_*
  int f16_multicast;  // fused kernels: weight stages multicast across CTA pairs (TCBF_F16_MC=0: off)
  int f16_fused_kind; // TCBF_FUSED_*: which fused fp32-data kernel tcbf_beamform_raw runs
  int f16i_resident;  // tcbf_beamform_f16i: resident-data kernel (K16 <= 256) instead of the streaming one
  int f16i_tmem;      // tcbf_beamform_f16i: the data-in-TMEM kernel (K16 <= 256), preferred over both
  int smaj_cluster;   // sample-major fused kernel: weight-multicast cluster size (1 or 2)
  int tmem_wkb;       // data-in-TMEM fused kernel: K blocks per weight stage (1 or 2)
  int tmem32;         // data-in-TMEM fused kernel with 32-beam tiles (gemm_f16_tmem2.cu): 0, or its WKB (2/4)
  int raw_mode;       // TCBF_RAW_*: what tcbf_beamform_raw runs
  int conv_splits_override;  // streaming-conversion K split (0 = by shape)
  int b1_kernel;      // TCBF_B1K_*: fp4 +-1 tensor cores (default), int8 AND form, legacy b1 mma.sync, popc
  int b1_swap_beams;  // fp4 swapped small-M kernel: beams per tile (32 / 64), 0 = not used
  int b1_force_stg;   // experiment: st.global epilogue instead of TMA stores
  int b1_splits, b1_kb_per_split;  // int8 split-K (forced only)
  int pack_wpt;       // 1-bit data pack words per thread (0 = by size)
  int debug;          // TCBF_DEV ablation bits (0 in product builds)
};

// shared by the ABI entry points (thread-local state in plan.cu)
__attribute__((visibility("hidden"))) void tcbf_internal_set_launches(int n);
__attribute__((visibility("hidden"))) tcbf_status tcbf_internal_fail(tcbf_status s, const char* what);
__attribute__((visibility("hidden"))) tcbf_status tcbf_internal_cuda_fail(cudaError_t e, const char* what);
// sets the current device's default mempool release threshold to "never" (stream-ordered scratch)
__attribute__((visibility("hidden"))) void retain_pool_memory();
