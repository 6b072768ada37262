// Device twin of synth/__init__.py: the counter-based input generator.
// Holds no beamforming arithmetic; integer hashing + exact int->float
// conversion (or table lookup / one fp32 multiply), bit-identical to numpy.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ int adc4(uint32_t bits24) {
  int s = 0;
#pragma unroll
  for (int f = 0; f < 4; ++f) s += (int)((bits24 >> (6 * f)) & 63u) - 32;
  return s;
}

__global__ void gen_kernel(float2* __restrict__ out, int dist, uint64_t base, int64_t total,
                           int64_t offset, const float2* __restrict__ tab) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < total; i += stride) {
    uint64_t h = splitmix64(base ^ (uint64_t)(i + offset));
    uint32_t hi24 = (uint32_t)((h >> 40) & 0xFFFFFFu);
    uint32_t lo24 = (uint32_t)((h >> 16) & 0xFFFFFFu);
    float re, im;
    if (dist == 0) {
      re = __int2float_rn((int)hi24 - 8388608) * 0x1p-23f;
      im = __int2float_rn((int)lo24 - 8388608) * 0x1p-23f;
    } else if (dist == 1 || dist == 4) {
      re = __int2float_rn(adc4(hi24));
      im = __int2float_rn(adc4(lo24));
      if (dist == 4) { re *= 0x1p-7f; im *= 0x1p-7f; }
    } else {
      float2 t = tab[(int)(h >> 52)];
      re = t.x; im = t.y;
      if (dist == 3) {
        float amp = __int2float_rn((int)lo24 + 1) * 0x1p-24f;
        re = __fmul_rn(re, amp);
        im = __fmul_rn(im, amp);
      }
    }
    out[i] = make_float2(re, im);
  }
}

}  // namespace

extern "C" int synth_generate_dev(void* out, int dist, uint64_t base, int64_t B, int64_t R,
                                  int64_t C, int64_t offset, const void* table, void* stream) {
  int64_t total = B * R * C;
  if (total <= 0) return 0;
  int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  gen_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
      (float2*)out, dist, base, total, offset, (const float2*)table);
  return (int)cudaGetLastError();
}
