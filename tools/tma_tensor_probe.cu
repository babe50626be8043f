// Probe: HBM streaming through TMA *tensor* boxes (128 rows x 64 bf16 = 16 KB, 128-B swizzle)
// into a shared-memory ring, one producer lane + one consumer warp per CTA, 148 persistent CTAs.
// Question for a tcgen05 decode READ: can box streaming match the ~6.8-6.9 TB/s of plain 16-B
// loads (tools/bw_probe.cu), and does the unit order matter?
//   order 0: "wavefront" — unit u = rb * nkb + kb dealt round-robin, so the 148 CTAs read
//            neighbouring 128-B column segments of the same 128 rows at the same time;
//   order 1: each CTA streams whole row blocks (rb = c, c + 148, ...), 148 separate regions.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_tensor_probe tools/tma_tensor_probe.cu -lcuda
//   order g >= 2: groups of g CTAs share each row block (K split g ways), 148/g blocks at a time.
//   tools/tma_tensor_probe <stages> <order>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned s32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_parity(unsigned long long *b, unsigned par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(s32(b)),
               "r"(par)
               : "memory");
}

__global__ void __launch_bounds__(64, 1) ring(const __grid_constant__ CUtensorMap map, int nrb, int nkb, int stages,
                                              int order, unsigned *out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char *sm = (unsigned char *)(((unsigned long long)sm_raw + 1023) & ~1023ull);
  unsigned long long *full = (unsigned long long *)(sm + stages * 16384), *empty = full + 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int units = nrb * nkb;
  // order >= 2: groups of g = order CTAs; group grp sweeps row blocks grp, grp + G, ...; CTA sub of
  // the group takes K blocks [sub * nkb / g, (sub + 1) * nkb / g) of each
  const int g = order >= 2 ? order : 1, G = gridDim.x / g, grp = blockIdx.x / g, sub = blockIdx.x % g;
  const int kb_lo = sub * nkb / g, kb_n = (sub + 1) * nkb / g - kb_lo;
  auto unit = [&](int i, int &rb, int &kb) {   // i-th unit of this CTA
    if (order >= 2) {
      rb = grp + (i / kb_n) * G;
      kb = kb_lo + i % kb_n;
    } else if (order == 0) {
      const int u = blockIdx.x + i * gridDim.x;
      rb = u / nkb;
      kb = u - rb * nkb;
    } else {
      const int per = nkb, r = blockIdx.x + (i / per) * gridDim.x;
      rb = r;
      kb = i % per;
    }
  };
  int n_mine = 0;
  if (order >= 2) n_mine = grp < G ? ((nrb - grp + G - 1) / G) * kb_n : 0;
  else if (order == 0) n_mine = (units - (int)blockIdx.x + gridDim.x - 1) / gridDim.x;
  else n_mine = ((nrb - (int)blockIdx.x + gridDim.x - 1) / gridDim.x) * nkb;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < n_mine; ++i) {
      const int s = i % stages;
      if (i >= stages) wait_parity(empty + s, ((i / stages) - 1) & 1);
      int rb, kb;
      unit(i, rb, kb);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(full + s)), "r"(16384) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              s32(sm + s * 16384)),
          "l"(&map), "r"(kb * 64), "r"(rb * 128), "r"(s32(full + s))
          : "memory");
    }
  } else if (warp == 1) {
    unsigned acc = 0;
    for (int i = 0; i < n_mine; ++i) {
      const int s = i % stages;
      wait_parity(full + s, (i / stages) & 1);
      acc ^= *(const unsigned *)(sm + s * 16384 + lane * 512);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(empty + s)) : "memory");
    }
    if (acc == 0x12345678u) out[0] = acc;
  }
}

int main(int argc, char **argv) {
  const int stages = argc > 1 ? atoi(argv[1]) : 8, order = argc > 2 ? atoi(argv[2]) : 0;
  const int cols = 9728, nkb = cols / 64, nrb = 180;               // 180 x 128 rows = 23040 rows = 448 MB
  const size_t bytes = (size_t)nrb * 128 * cols * 2;
  void *buf;
  unsigned *out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 1, bytes);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)nrb * 128};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 1024 + (size_t)stages * 16384 + 1024;
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) ring<<<sms, 64, smem>>>(map, nrb, nkb, stages, order, out);
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) ring<<<sms, 64, smem>>>(map, nrb, nkb, stages, order, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("tma tensor ring: stages %d (%d KB) order %d: %.1f us per 448 MB launch, %.1f GB/s (%s)\n", stages,
         stages * 16, order, ms / 20 * 1e3, bytes / (ms / 20 / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
