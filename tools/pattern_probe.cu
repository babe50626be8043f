// DRAM access-pattern probe (tools/pattern_probe.cu): 1024-thread persistent CTAs, each warp streams ~16 KB tasks.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint4 ld(const uint4 *p) {
  uint4 r; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)); return r; }
// mode 0: one row (1216 vec) per task, lane-contiguous 4 x 512B per batch
// mode 1: 16 rows x (2 x 64B per row per batch)  [current MMA base pattern], 8 batches per task
// mode 2: 8 rows x (4 x 64B contiguous per row per batch), 8 batches per task
__global__ void __launch_bounds__(1024, 1) k(const uint4 *W, int rows, int nvec, int mode, unsigned *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, tq = lane & 3;
  const int stride = gridDim.x * 32;
  unsigned acc = 0;
  uint4 cur[4], nxt[4];
  if (mode == 0) {
    for (int t = warp * gridDim.x + blockIdx.x; t < rows; t += stride) {
      const uint4 *r = W + (size_t)t * nvec;
      for (int v = lane; v < nvec; v += 128) {
#pragma unroll
        for (int u = 0; u < 4; ++u) cur[u] = v + 32 * u < nvec ? ld(r + v + 32 * u) : make_uint4(0,0,0,0);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc ^= cur[u].x ^ cur[u].w;
      }
    }
  } else if (mode == 1) {
    const int KC = (nvec + 63) / 64, ntask = rows / 16 * KC;
    for (int t = warp * gridDim.x + blockIdx.x; t < ntask; t += stride) {
      const int rb = t / KC, kc = t % KC;
      const uint4 *q = W + (size_t)(rb * 16 + g) * nvec + kc * 64 + tq;
      for (int j = 0; j < 8; ++j) {
        const int v0 = kc * 64 + 8 * j + tq;
        cur[0] = v0 < nvec ? ld(q + 8 * j) : make_uint4(0,0,0,0);
        cur[1] = v0 + 4 < nvec ? ld(q + 8 * j + 4) : make_uint4(0,0,0,0);
        cur[2] = v0 < nvec ? ld(q + 8 * j + 8 * (size_t)nvec) : make_uint4(0,0,0,0);
        cur[3] = v0 + 4 < nvec ? ld(q + 8 * j + 8 * (size_t)nvec + 4) : make_uint4(0,0,0,0);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc ^= cur[u].x ^ cur[u].w;
      }
    }
  } else {
    const int KC = (nvec + 127) / 128, ntask = rows / 8 * KC;
    for (int t = warp * gridDim.x + blockIdx.x; t < ntask; t += stride) {
      const int rb = t / KC, kc = t % KC;
      const uint4 *q = W + (size_t)(rb * 8 + g) * nvec + kc * 128 + tq;
      for (int j = 0; j < 8; ++j) {
        const int v0 = kc * 128 + 16 * j + tq;
#pragma unroll
        for (int u = 0; u < 4; ++u) cur[u] = v0 + 4 * u < nvec ? ld(q + 16 * j + 4 * u) : make_uint4(0,0,0,0);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc ^= cur[u].x ^ cur[u].w;
      }
    }
  }
  (void)nxt;
  if (acc == 0x12345) out[0] = acc;
}
int main() {
  const int nvec = 1216, rows = 2560 * 9;   // 448 MB
  const size_t bytes = (size_t)rows * nvec * 16;
  uint4 *W; unsigned *o; cudaMalloc(&W, 2 * bytes); cudaMalloc(&o, 4); cudaMemset(W, 1, 2 * bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(a);
      k<<<148, 1024>>>(W + (it & 1) * (bytes / 16), rows, nvec, mode, o);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("mode %d: %.1f GB/s (%s)\n", mode, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
}
