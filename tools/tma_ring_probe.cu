// Probe: can a TMA bulk-copy ring (bytes in flight held in shared memory, not registers / L1)
// stream HBM faster than register LDG batches (~64 KB in flight per SM, capped by both the
// register file and the L1 left beside 164 KB of shared memory)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_ring_probe tools/tma_ring_probe.cu
//   tools/tma_ring_probe <row_bytes> <slots> <consumer_warps> <producers>
// Each CTA streams rows of `row_bytes` (19,456 = one ΔW row at d_ff 9728) into `slots` ring
// slots; consumer warps take slots round-robin, touch every 16-B vector (an FMA chain, like a
// dot product) and release them.  448 MB per launch (one decode READ's bytes).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned s32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_parity(unsigned long long *b, unsigned par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(s32(b)),
               "r"(par)
               : "memory");
}

__global__ void __launch_bounds__(1024, 1) ring(const unsigned char *src, int rows_per_cta, int row_bytes, int slots,
                                                int cw, int prod, float *out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned long long *full = (unsigned long long *)sm, *empty = full + 64;
  unsigned char *buf = sm + 1024;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < slots; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const unsigned char *base = src + (size_t)blockIdx.x * rows_per_cta * row_bytes;
  if (warp == 0) {                                   // producers: lanes 0..prod-1, rows k ≡ lane (mod prod)
    if (lane < prod)
      for (int k = 0; k < rows_per_cta; ++k) {
        const int s = k % slots;
        if (s % prod != lane) continue;                 // a slot always has the same producer lane
        if (k >= slots) wait_parity(empty + s, ((k / slots) - 1) & 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(full + s)), "r"(row_bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         s32(buf + (size_t)s * row_bytes)),
                     "l"(base + (size_t)k * row_bytes), "r"(row_bytes), "r"(s32(full + s))
                     : "memory");
      }
    return;
  }
  if (warp > cw) return;
  float acc = 0.f;
  const int nv = row_bytes / 16;
  // consumer warp w owns slots s ≡ w-1 (mod cw) (cw divides slots): never more than one phase ahead
  for (int k = warp - 1; k < rows_per_cta; k += cw) {
    const int s = k % slots;
    wait_parity(full + s, (k / slots) & 1);
    const float4 *r = (const float4 *)(buf + (size_t)s * row_bytes);
    for (int v = lane; v < nv; v += 32) {
      const float4 a = r[v];
      acc = fmaf(a.x, a.y, acc);
      acc = fmaf(a.z, a.w, acc);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(empty + s)) : "memory");
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main(int argc, char **argv) {
  const int row_bytes = argc > 1 ? atoi(argv[1]) : 19456, slots = argc > 2 ? atoi(argv[2]) : 7,
            prod0 = argc > 4 ? atoi(argv[4]) : 4;
  int prod = prod0;
  int cw = argc > 3 ? atoi(argv[3]) : slots;
  if (slots % cw) cw = slots;                          // a slot's rows stay on one consumer warp
  if (prod > slots) prod = slots;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t per_launch = 448ull << 20;
  const int rows_per_cta = (int)(per_launch / row_bytes / sms);
  const size_t bytes = (size_t)rows_per_cta * row_bytes * sms;
  unsigned char *a, *b;
  float *out;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(a, 1, bytes);
  cudaMemset(b, 1, bytes);
  const size_t smem = 1024 + (size_t)slots * row_bytes;
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int it = 0; it < 20; ++it) {
    cudaEventRecord(e0);
    ring<<<sms, 32 * (cw + 1), smem>>>(it & 1 ? a : b, rows_per_cta, row_bytes, slots, cw, prod, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 3 && ms < best) best = ms;
  }
  printf("row %d slots %d (%zu KB in flight) consumers %d producers %d: %.1f GB/s (%s)\n", row_bytes, slots,
         (size_t)slots * row_bytes / 1024, cw, prod, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
