// steer.cu -- steering-weight generation (Sec. II Eqs. 1-3).
//
// Far-field plane wave: x_k(t) = s(t - tau_k), tau_k = d_k sin(theta) / c (Eq. 2).  For a
// narrowband channel at frequency f the delay is the phase exp(-2 pi i f tau_k), so the weights
// that align the receivers on direction theta_m are (reading R9, raw sum, no 1/K)
//     w[b][m][k] = exp(+2 pi i f_b d_k sin(theta_m) / c).
// The phase in cycles is formed in fp64 and reduced to [-1/2, 1/2] before sincospi, so the fp32
// weights stay accurate for LOFAR-sized baselines (f d / c ~ 1e3-1e5 cycles).
#include <cuda_runtime.h>

#include <cstdint>

namespace tcbf {
namespace {

template <int LAYOUT>
__global__ void steering_kernel(const double* __restrict__ pos, const double* __restrict__ theta,
                                const double* __restrict__ freq, double inv_c, int64_t B, int64_t M, int64_t K,
                                float* __restrict__ dst) {
  const int64_t total = B * M * K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i % K;
    const int64_t bm = i / K;
    const int64_t m = bm % M;
    const int64_t b = bm / M;
    const double cycles = freq[b] * pos[k] * sin(theta[m]) * inv_c;
    const double frac = cycles - rint(cycles);
    double s, c;
    sincospi(2.0 * frac, &s, &c);
    if (LAYOUT == 0) {
      reinterpret_cast<float2*>(dst)[i] = make_float2((float)c, (float)s);
    } else {
      dst[((b * 2 + 0) * M + m) * K + k] = (float)c;
      dst[((b * 2 + 1) * M + m) * K + k] = (float)s;
    }
  }
}

}  // namespace

cudaError_t launch_steering(const double* pos, const double* theta, const double* freq, double c, int64_t B,
                            int64_t M, int64_t K, int layout, float* dst, cudaStream_t stream) {
  const int64_t total = B * M * K;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (layout == 0) steering_kernel<0><<<(unsigned)blocks, 256, 0, stream>>>(pos, theta, freq, 1.0 / c, B, M, K, dst);
  else steering_kernel<1><<<(unsigned)blocks, 256, 0, stream>>>(pos, theta, freq, 1.0 / c, B, M, K, dst);
  return cudaGetLastError();
}

}  // namespace tcbf
