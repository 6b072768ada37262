// host_pipeline.cu -- tcbf_beamform_host: the end-to-end call over HOST buffers.
// Batches are streamed through the GPU in chunks on two CUDA streams so that the
// host->device copy of chunk i+1 and the device->host copy of chunk i-1 overlap the
// pack + beamform kernels of chunk i (copy engines and SMs work concurrently).
// Weights are packed once and stay resident (the model matrix is packed
// once, the measurement matrix per ensemble).  Each chunk runs tcbf_beamform_raw.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "plan_internal.h"
#include "tcbf.h"

extern "C" tcbf_status tcbf_beamform_host(const tcbf_plan* plan, const void* w_packed_dev, const float* x_host,
                                          tcbf_src_layout layout, void* out_host) {
  if (!plan || !w_packed_dev || !x_host || !out_host) return TCBF_ERR_INVALID_ARG;
  const int64_t B = plan->B;
  const size_t src_per_b = (size_t)plan->K * plan->N * 2 * sizeof(float);
  const size_t xp_per_b = plan->x_bytes / B;
  const size_t wp_per_b = plan->w_bytes / B;
  const size_t out_per_b = plan->out_bytes / B;
  // chunk: ~192 MiB of device scratch per buffer set, at least one batch entry
  const size_t per_b = src_per_b + out_per_b;  // packed data scratch (if any) is tcbf_beamform_raw's
  int64_t cb = (int64_t)((192ull << 20) / per_b);
  if (cb < 1) cb = 1;
  if (cb > B) cb = B;
  const int64_t nchunks = (B + cb - 1) / cb;

  // Keep the stream-ordered pool's memory between calls (the default release threshold of 0
  // would hand the scratch back to the driver at every synchronize and re-allocate each call).
  retain_pool_memory();
  cudaStream_t st[2] = {nullptr, nullptr};
  void* buf[2] = {nullptr, nullptr};
  tcbf_status status = TCBF_OK;
  int launches = 0;
  for (int i = 0; i < 2; ++i) {
    if (cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking) != cudaSuccess) { status = TCBF_ERR_CUDA; break; }
    if (cudaMallocAsync(&buf[i], per_b * cb, st[i]) != cudaSuccess) { status = TCBF_ERR_ALLOC; break; }
  }
  for (int64_t c = 0; c < nchunks && status == TCBF_OK; ++c) {
    const int s = (int)(c & 1);
    const int64_t b0 = c * cb;
    const int64_t nb = (b0 + cb <= B) ? cb : (B - b0);
    char* d_src = static_cast<char*>(buf[s]);
    char* d_out = d_src + src_per_b * cb;
    tcbf_plan sub = *plan;  // same shape, nb batch entries
    sub.B = nb;
    sub.w_bytes = wp_per_b * nb;
    sub.x_bytes = xp_per_b * nb;
    sub.out_bytes = out_per_b * nb;
    if (cudaMemcpyAsync(d_src, reinterpret_cast<const char*>(x_host) + src_per_b * b0, src_per_b * nb,
                        cudaMemcpyHostToDevice, st[s]) != cudaSuccess) { status = TCBF_ERR_CUDA; break; }
    // pack + beamform (one fused kernel where the plan allows it)
    status = tcbf_beamform_raw(&sub, static_cast<const char*>(w_packed_dev) + wp_per_b * b0,
                               reinterpret_cast<const float*>(d_src), layout, d_out, st[s]);
    if (status != TCBF_OK) break;
    launches += tcbf_last_launch_count();
    if (cudaMemcpyAsync(static_cast<char*>(out_host) + out_per_b * b0, d_out, out_per_b * nb,
                        cudaMemcpyDeviceToHost, st[s]) != cudaSuccess) { status = TCBF_ERR_CUDA; break; }
  }
  for (int i = 0; i < 2; ++i) {
    if (st[i]) {
      if (buf[i]) cudaFreeAsync(buf[i], st[i]);
      if (cudaStreamSynchronize(st[i]) != cudaSuccess && status == TCBF_OK) status = TCBF_ERR_CUDA;
      cudaStreamDestroy(st[i]);
    }
  }
  tcbf_internal_set_launches(launches);
  return status;
}
