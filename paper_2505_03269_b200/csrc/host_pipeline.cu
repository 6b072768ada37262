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

namespace {

constexpr size_t kAlign = 256;  // device scratch sub-buffers start on 256-byte boundaries

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Two copy/compute streams per (thread, device), created on first use and reused by every later
// call on this thread (the call blocks until its work is done, so reuse is safe).
struct ThreadStreams {
  int device = -1;
  cudaStream_t st[2] = {nullptr, nullptr};
  ~ThreadStreams() {
    for (cudaStream_t s : st)
      if (s) cudaStreamDestroy(s);  // best effort at thread exit
  }
};
thread_local ThreadStreams t_streams;

tcbf_status get_streams(int device, cudaStream_t out[2]) {
  if (t_streams.device != device) {
    for (cudaStream_t& s : t_streams.st) {
      if (s) cudaStreamDestroy(s);
      s = nullptr;
    }
    t_streams.device = -1;
    for (cudaStream_t& s : t_streams.st) {
      cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (e != cudaSuccess) return tcbf_internal_cuda_fail(e, "tcbf_beamform_host: cudaStreamCreate");
    }
    t_streams.device = device;
  }
  out[0] = t_streams.st[0];
  out[1] = t_streams.st[1];
  return TCBF_OK;
}

}  // namespace

extern "C" tcbf_status tcbf_beamform_host(const tcbf_plan* plan, const void* w_packed_dev, const float* x_host,
                                          tcbf_src_layout layout, void* out_host) {
  tcbf_internal_set_launches(0);
  if (!plan || !w_packed_dev || !x_host || !out_host)
    return tcbf_internal_fail(TCBF_ERR_INVALID_ARG, "tcbf_beamform_host: NULL argument");
  if (layout != TCBF_SRC_INTERLEAVED && layout != TCBF_SRC_PLANAR)
    return tcbf_internal_fail(TCBF_ERR_INVALID_ARG, "tcbf_beamform_host: bad layout");
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return tcbf_internal_cuda_fail(e, "tcbf_beamform_host: cudaGetDevice");
  if (dev != plan->device)
    return tcbf_internal_fail(TCBF_ERR_DEVICE_MISMATCH, "tcbf_beamform_host: current device differs from the plan's");
  const int64_t B = plan->B;
  const size_t src_per_b = (size_t)plan->K * plan->N * 2 * sizeof(float);
  const size_t wp_per_b = plan->w_bytes / B;
  const size_t out_per_b = plan->out_bytes / B;
  // chunk: ~192 MiB of device scratch per buffer set, at least one batch entry
  int64_t cb = (int64_t)((192ull << 20) / (src_per_b + out_per_b));
  if (cb < 1) cb = 1;
  if (cb > B) cb = B;
  const int64_t nchunks = (B + cb - 1) / cb;
  // [source chunk | output chunk], each 256-byte aligned (the GEMMs need 16-byte aligned outputs,
  // the streaming kernels 16-byte aligned sources; src_per_b * cb alone may be only 8-aligned)
  const size_t src_bytes = round_up(src_per_b * cb, kAlign);
  const size_t set_bytes = src_bytes + round_up(out_per_b * cb, kAlign);

  cudaStream_t st[2];
  tcbf_status status = get_streams(dev, st);
  if (status != TCBF_OK) return status;
  // Keep the stream-ordered pool's memory between calls (the default release threshold of 0
  // would hand the scratch back to the driver at every synchronize and re-allocate each call).
  retain_pool_memory();
  void* buf[2] = {nullptr, nullptr};
  int launches = 0;
  for (int i = 0; i < 2 && status == TCBF_OK; ++i) {
    e = cudaMallocAsync(&buf[i], set_bytes, st[i]);
    if (e != cudaSuccess) {
      buf[i] = nullptr;
      status = tcbf_internal_fail(TCBF_ERR_ALLOC, "tcbf_beamform_host: cudaMallocAsync of the chunk scratch failed");
    }
  }
  for (int64_t c = 0; c < nchunks && status == TCBF_OK; ++c) {
    const int s = (int)(c & 1);
    const int64_t b0 = c * cb;
    const int64_t nb = (b0 + cb <= B) ? cb : (B - b0);
    char* d_src = static_cast<char*>(buf[s]);
    char* d_out = d_src + src_bytes;
    tcbf_plan sub = *plan;  // same shape and kernel choice, nb batch entries
    sub.B = nb;
    sub.w_bytes = wp_per_b * nb;
    sub.x_bytes = plan->x_bytes / B * nb;
    sub.out_bytes = out_per_b * nb;
    e = cudaMemcpyAsync(d_src, reinterpret_cast<const char*>(x_host) + src_per_b * b0, src_per_b * nb,
                        cudaMemcpyHostToDevice, st[s]);
    if (e != cudaSuccess) { status = tcbf_internal_cuda_fail(e, "tcbf_beamform_host: H2D copy"); break; }
    // pack + beamform (one fused kernel where the plan allows it); sets tcbf_last_error on failure
    status = tcbf_beamform_raw(&sub, static_cast<const char*>(w_packed_dev) + wp_per_b * b0,
                               reinterpret_cast<const float*>(d_src), layout, d_out, st[s]);
    if (status != TCBF_OK) break;
    launches += tcbf_last_launch_count();
    e = cudaMemcpyAsync(static_cast<char*>(out_host) + out_per_b * b0, d_out, out_per_b * nb,
                        cudaMemcpyDeviceToHost, st[s]);
    if (e != cudaSuccess) { status = tcbf_internal_cuda_fail(e, "tcbf_beamform_host: D2H copy"); break; }
  }
  for (int i = 0; i < 2; ++i) {
    if (buf[i]) cudaFreeAsync(buf[i], st[i]);
    e = cudaStreamSynchronize(st[i]);
    if (e != cudaSuccess && status == TCBF_OK) status = tcbf_internal_cuda_fail(e, "tcbf_beamform_host: synchronize");
  }
  tcbf_internal_set_launches(status == TCBF_OK ? launches : 0);
  return status;
}
