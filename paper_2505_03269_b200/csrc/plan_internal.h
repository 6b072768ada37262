// plan_internal.h -- the plan object behind the opaque tcbf_plan handle (host metadata only).
#pragma once
#include <cstddef>
#include <cstdint>

#include "tcbf.h"

struct tcbf_plan_s {
  int64_t M, N, K, B;
  tcbf_precision prec;
  int64_t kp;   // K16 (fp16 elements) or Kw (uint32 words)
  int device;
  int num_sms;
  int f16_variant;  // tcbf::F16_V_*
  int64_t n_packed;  // F16 data row length Np = round_up(N, 8) (MN-major packed data)
  int b1_tc;    // 1-bit kernel: 4 = kind::mxf4 (+-1, default), 3 = kind::i8 CTA pair, 2 = kind::f8f6f4 (+-1),
                // 1 = kind::i8 (AND form), 5 = legacy mma.sync b1 AND, 0 = CUDA-core popc
  size_t w_bytes, x_bytes, out_bytes;
};

// launch accounting shared by the ABI entry points (thread-local in plan.cu)
__attribute__((visibility("hidden"))) void tcbf_internal_set_launches(int n);
// sets the current device's default mempool release threshold to "never" (stream-ordered scratch)
__attribute__((visibility("hidden"))) void retain_pool_memory();
