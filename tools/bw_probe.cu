// HBM read-bandwidth probe: how many bytes in flight per SM does a pure
// streaming read need on this B200?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldnc(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int U>
__global__ void rd(const uint4 *__restrict__ a, size_t n, unsigned *out) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldnc(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n; i += stride) { uint4 v = ldnc(a + i); acc ^= v.x ^ v.w; }
  if (acc == 0x12345678) out[0] = acc;
}

// row-streaming like the READ kernel: each warp reads contiguous 19456-byte rows
template <int U>
__global__ void rows(const uint4 *__restrict__ a, int nrows, int nvec, unsigned *out) {
  unsigned acc = 0;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, W = (gridDim.x * blockDim.x) >> 5;
  for (int r = gw; r < nrows; r += W) {
    const uint4 *row = a + (size_t)r * nvec;
    for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) if (v0 + 32 * u < nvec) v[u] = ldnc(row + v0 + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) if (v0 + 32 * u < nvec) acc ^= v[u].x ^ v[u].w;
    }
  }
  if (acc == 0x12345678) out[0] = acc;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 10;
}

int main1() {
  const size_t bytes = 448ull << 20 << 1;   // 896 MB (> L2); rotate between two halves
  uint4 *buf; unsigned *out;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 4);
  cudaMemset(buf, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t n = bytes / 2 / 16;
  int flip = 0;
  printf("grid-stride read, 448 MB per launch\n");
  for (int th : {256, 512, 1024})
    for (int bpsm : {1, 2, 4})
      for (int U : {4, 8, 16}) {
        if (th * bpsm > 2048) continue;
        float ms = timeit([&] {
          const uint4 *p = buf + (flip ^= 1) * n;
          if (U == 4) rd<4><<<sms * bpsm, th>>>(p, n, out);
          if (U == 8) rd<8><<<sms * bpsm, th>>>(p, n, out);
          if (U == 16) rd<16><<<sms * bpsm, th>>>(p, n, out);
        });
        printf("th %4d  blk/SM %d  U %2d : %.1f GB/s  (inflight/SM %d KB)\n", th, bpsm, U, n * 16 / ms / 1e6,
               th * bpsm * U * 16 / 1024);
      }
  printf("row streaming (19456 B rows), 448 MB per launch\n");
  const int nvec = 1216, nrows = (int)(n / nvec);
  for (int th : {512, 1024})
    for (int U : {4, 8, 16}) {
      float ms = timeit([&] {
        const uint4 *p = buf + (flip ^= 1) * n;
        if (U == 4) rows<4><<<sms, th>>>(p, nrows, nvec, out);
        if (U == 8) rows<8><<<sms, th>>>(p, nrows, nvec, out);
        if (U == 16) rows<16><<<sms, th>>>(p, nrows, nvec, out);
      });
      printf("rows th %4d U %2d : %.1f GB/s\n", th, U, (double)nrows * nvec * 16 / ms / 1e6);
    }
  return 0;
}

// ---------------------------------------------------------------------------
// TMA bulk-copy ring: P producer threads (warp 0) stream S-byte stages into an
// R-stage ring; 15 consumer warps touch one word and release the stage.
__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_wait(unsigned long long *b, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(s32(b)), "r"(par) : "memory");
}
__global__ void __launch_bounds__(512, 1) tma_ring(const unsigned char *src, size_t per_cta, int S, int R, int P, unsigned *out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned long long *full = (unsigned long long *)sm, *empty = full + 128;
  unsigned char *ring = sm + 2048;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < R; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nst = (int)(per_cta / S);
  const unsigned char *base = src + (size_t)blockIdx.x * per_cta;
  if (warp == 0) {
    if (lane < P) {
      for (int k = lane; k < nst; k += P) {
        const int s = k % R;
        if (k >= R) mb_wait(empty + s, ((k / R) - 1) & 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(full + s)), "r"(S) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(s32(ring + (size_t)s * S)), "l"(base + (size_t)k * S), "r"(S), "r"(s32(full + s)) : "memory");
      }
    }
    return;
  }
  unsigned acc = 0;
  for (int k = warp - 1; k < nst; k += 15) {
    const int s = k % R;
    mb_wait(full + s, (k / R) & 1);
    acc ^= ((const unsigned *)(ring + (size_t)s * S))[lane];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(empty + s)) : "memory");
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main2(int S, int P) {
  const size_t bytes = 448ull << 20 << 1;
  unsigned char *buf; unsigned *out;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 4);
  cudaMemset(buf, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int flip = 0;
  printf("TMA bulk ring (448 MB per launch)\n");
  {
    {
      int R = (200 * 1024) / S; if (R > 128) R = 128;
      const size_t per = (448ull << 20) / sms / S * S;
      float ms = timeit([&] {
        tma_ring<<<sms, 512, 2048 + R * S>>>(buf + (flip ^= 1) * (448ull << 20), per, S, R, P, out);
      });
      printf("S %5d R %3d P %d : %.1f GB/s  (%s)\n", S, R, P, per * sms / ms / 1e6,
             cudaGetErrorString(cudaDeviceSynchronize()));
      fflush(stdout);
    }
  }
  return 0;
}
int main(int argc, char **argv) {
  if (argc > 2) return main2(atoi(argv[1]), atoi(argv[2]));
  return main1();
}
