// Seeded counter-based input generator, device side (libttt_gen.so).
//
// NOT part of the product boundary and holds none of the method's
// arithmetic: it re-implements workload/rng.py's generator so the bench can
// synthesise paper-sized inputs directly in HBM.  tests/test_workload_gen.py
// checks it against the NumPy implementation bit for bit.
#include <cuda_bf16.h>
#include <cstdint>

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

__host__ __device__ inline uint64_t hmix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

uint64_t key_of(uint64_t seed, uint64_t tensor, uint64_t owner, uint64_t layer, int64_t pos) {
  uint64_t k = hmix64(seed ^ 0x243F6A8885A308D3ull);
  k = hmix64(k ^ tensor);
  k = hmix64(k ^ owner);
  k = hmix64(k ^ layer);
  k = hmix64(k ^ (uint64_t)(pos + (1ll << 31)));
  return k;
}

template <bool BF16>
__global__ void gen_kernel(void *out, uint64_t key, size_t n, float amp) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t h = mix64(key + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull);
    const int u = (int)(h >> 40) - (1 << 23);
    float f = __fmul_rn((float)u, 1.1920928955078125e-07f);   // 2^-23
    f = __fmul_rn(f, amp);
    if (BF16)
      static_cast<__nv_bfloat16 *>(out)[i] = __float2bfloat16_rn(f);
    else
      static_cast<float *>(out)[i] = f;
  }
}

}  // namespace

extern "C" int ttt_gen_uniform(void *out, uint64_t seed, uint64_t tensor, uint64_t owner, uint64_t layer,
                               int64_t pos, size_t n, float amp, int bf16, void *stream) {
  const uint64_t key = key_of(seed, tensor, owner, layer, pos);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  size_t blocks = (n + 255) / 256;
  if (blocks > (size_t)sms * 16) blocks = (size_t)sms * 16;
  if (blocks == 0) return 0;
  if (bf16)
    gen_kernel<true><<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(out, key, n, amp);
  else
    gen_kernel<false><<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(out, key, n, amp);
  return (int)cudaGetLastError();
}
