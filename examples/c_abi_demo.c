/*
 * c_abi_demo.c -- the C ABI (include/tcbf.h) used from plain C, no Python: one 16-bit and one
 * 1-bit beamform of a small radio-like problem (M beams x K receivers x N samples x B channels)
 * through tcbf_plan_create / tcbf_pack / tcbf_beamform / tcbf_beamform_raw, checked against a
 * direct double-precision triple loop in this file (the operation of PAPER.md:78-84, Eq. 3).
 *
 * Inputs are small integers (exact in fp16; every fp32 partial sum exact), so the 16-bit result
 * must equal the triple loop exactly; the 1-bit result is checked against the same loop on the
 * signs (value >= 0 -> +1).  Exit code 0 and a final "OK" line on success.
 *
 * Build: gcc -std=c11 -O2 -I include examples/c_abi_demo.c -o c_abi_demo \
 *            -L paper_2505_03269_b200/lib -ltcbf -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,...
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "tcbf.h"

#define CHECK(call)                                                                          \
  do {                                                                                       \
    tcbf_status s_ = (call);                                                                 \
    if (s_ != TCBF_OK) {                                                                     \
      fprintf(stderr, "%s failed: %s (%s)\n", #call, tcbf_status_string(s_), tcbf_last_error()); \
      return 1;                                                                              \
    }                                                                                        \
  } while (0)
#define CUDA(call)                                                                      \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      fprintf(stderr, "%s failed: %s\n", #call, cudaGetErrorString(e_));                \
      return 1;                                                                         \
    }                                                                                   \
  } while (0)

enum { M = 200, N = 300, K = 100, B = 3 };

/* small integers in [-4, 4], a fixed LCG so the run is reproducible */
static float next_val(uint32_t* s) {
  *s = *s * 1664525u + 1013904223u;
  return (float)((int)((*s >> 24) % 9u) - 4);
}

static double sgn(float v) { return v >= 0.f ? 1.0 : -1.0; }

int main(void) {
  const size_t nw = (size_t)B * M * K * 2, nx = (size_t)B * K * N * 2, no = (size_t)B * 2 * M * N;
  float* w = malloc(nw * sizeof(float));  /* interleaved [B][M][K] (re, im) */
  float* x = malloc(nx * sizeof(float));  /* interleaved [B][K][N] (re, im) */
  float* y16 = malloc(no * sizeof(float));
  int32_t* y1 = malloc(no * sizeof(int32_t));
  uint32_t seed = 12345u;
  for (size_t i = 0; i < nw; ++i) w[i] = next_val(&seed);
  for (size_t i = 0; i < nx; ++i) x[i] = next_val(&seed);

  float *dw, *dx;
  CUDA(cudaMalloc((void**)&dw, nw * sizeof(float)));
  CUDA(cudaMalloc((void**)&dx, nx * sizeof(float)));
  CUDA(cudaMemcpy(dw, w, nw * sizeof(float), cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(dx, x, nx * sizeof(float), cudaMemcpyHostToDevice));

  int bad = 0;
  for (int mode = 0; mode < 2; ++mode) {
    const tcbf_precision prec = mode == 0 ? TCBF_PREC_F16 : TCBF_PREC_B1;
    tcbf_plan* plan = NULL;
    CHECK(tcbf_plan_create(&plan, M, N, K, B, prec));
    size_t wb, xb, ob;
    CHECK(tcbf_packed_bytes(plan, TCBF_WEIGHTS, &wb));
    CHECK(tcbf_packed_bytes(plan, TCBF_DATA, &xb));
    CHECK(tcbf_output_bytes(plan, &ob));
    void *wp, *xp, *out;
    CUDA(cudaMalloc(&wp, wb));
    CUDA(cudaMalloc(&xp, xb));
    CUDA(cudaMalloc(&out, ob));
    CHECK(tcbf_pack(plan, TCBF_WEIGHTS, dw, TCBF_SRC_INTERLEAVED, wp, NULL));
    CHECK(tcbf_pack(plan, TCBF_DATA, dx, TCBF_SRC_INTERLEAVED, xp, NULL));
    CHECK(tcbf_beamform(plan, wp, xp, out, NULL));
    CUDA(cudaDeviceSynchronize());
    CUDA(cudaMemcpy(mode == 0 ? (void*)y16 : (void*)y1, out, ob, cudaMemcpyDeviceToHost));
    if (mode == 0) {  /* the fused path from the fp32 source must agree exactly here too */
      CHECK(tcbf_beamform_raw(plan, wp, dx, TCBF_SRC_INTERLEAVED, out, NULL));
      float* yr = malloc(no * sizeof(float));
      CUDA(cudaDeviceSynchronize());
      CUDA(cudaMemcpy(yr, out, ob, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < no; ++i) bad += yr[i] != y16[i];
      printf("f16 raw (%s) vs packed: %d mismatches\n", tcbf_plan_kernel(plan, TCBF_ENTRY_BEAMFORM_RAW), bad);
      free(yr);
    }
    /* direct triple loop: C[b][m][n] = sum_k W[b][m][k] X[b][k][n] */
    int errs = 0;
    for (int b = 0; b < B; ++b)
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          double re = 0.0, im = 0.0;
          for (int k = 0; k < K; ++k) {
            const float* wv = w + (((size_t)b * M + m) * K + k) * 2;
            const float* xv = x + (((size_t)b * K + k) * N + n) * 2;
            const double wr = mode ? sgn(wv[0]) : wv[0], wi = mode ? sgn(wv[1]) : wv[1];
            const double xr = mode ? sgn(xv[0]) : xv[0], xi = mode ? sgn(xv[1]) : xv[1];
            re += wr * xr - wi * xi;
            im += wr * xi + wi * xr;
          }
          const size_t o = (((size_t)b * 2) * M + m) * N + n, oi = o + (size_t)M * N;
          const double gr = mode ? (double)y1[o] : (double)y16[o];
          const double gi = mode ? (double)y1[oi] : (double)y16[oi];
          errs += gr != re || gi != im;
        }
    printf("%s beamform (%s): %d mismatches against the triple loop\n", mode ? "1-bit" : "16-bit",
           tcbf_plan_kernel(plan, TCBF_ENTRY_BEAMFORM), errs);
    bad += errs;
    cudaFree(wp);
    cudaFree(xp);
    cudaFree(out);
    CHECK(tcbf_plan_destroy(plan));
  }
  cudaFree(dw);
  cudaFree(dx);
  free(w);
  free(x);
  free(y16);
  free(y1);
  printf(bad ? "FAILED\n" : "OK\n");
  return bad ? 1 : 0;
}
