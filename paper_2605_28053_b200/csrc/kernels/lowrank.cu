// NEXT f1 — low-rank delta TTTState (DeltaAdapterState; App. F
// P:1023-1034), READ and WRITE on B200.  Rule (SPEC S:188 / S:215 generalised to
// d_model ≠ d_ff with the shared base, reading xviii):
//     READ   y = W_down · z + Bᵀ (A z)            A [R][d_ff], B [R][d_model] per owner-layer
//     WRITE  m = (1/C) Σ_t z_t;  A' = A + η (A m) mᵀ;  B' = B   (into the shadow slot)
// Payload layout per slot and layer: A (R·d_ff) then B (R·d_model), σ.dtype = bf16.
//
// READ is three launches per layer (the base product is the only dense part):
//   lr_u_kernel      u_b = A_b x_b (one warp per (member, k) dot of length d_ff),
//                    gathers x_b into a contiguous workspace and appends (z, v) to the tail;
//   base GEMM        Y32 = Xg · W_downᵀ on tcgen05 (read_chunk_tc in base-only mode: the
//                    group's rows are the M dimension, W_down is read once per group);
//   lr_finish_kernel y_b = Y32_b + Bᵀ u_b (+ residual), bf16, scattered through μ.
// WRITE is one CTA per member: chunk mean m from the tail, w = A m, A' = A + η w mᵀ,
// B copied; a non-finite candidate raises the group fail flag.
#include <cuda_bf16.h>

#include "../internal.h"

namespace ttt {
namespace {

__device__ __forceinline__ float bf(const __nv_bfloat16 v) { return __bfloat162float(v); }

// one CTA per member b: x_b staged in shared memory once, warps over the rank rows k,
// 4 independent 16-byte loads of A in flight per lane.
constexpr int kUThreads = 1024;                   // 32 warps = 32 rank rows per CTA
__global__ void __launch_bounds__(kUThreads) lr_u_kernel(const LowRankRead p) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint4 *xs = reinterpret_cast<uint4 *>(smem);
  const int b = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int R = p.rank, dff = p.d_ff, dm = p.d_model, nvec = dff / 8;
  const bool first = blockIdx.y == 0;              // rank block 0 also gathers x and appends the tail
  const int o = p.owner_idx[b];
  const uint4 *x4 = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.X) + (size_t)p.x_row[b] * dff);
  uint4 *xg = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.Xg) + (size_t)b * dff);
  uint4 *tz = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.tailZ) + o * p.tz_owner + p.tz_layer +
                                        (size_t)p.tail_pos[b] * dff);
  for (int v = tid; v < nvec; v += kUThreads) {     // stage x; gather for the base GEMM; tail append (a4)
    const uint4 z = x4[v];
    xs[v] = z;
    if (first) {
      xg[v] = z;
      tz[v] = z;
    }
  }
  if (first) {
    const __nv_bfloat16 *vt = static_cast<const __nv_bfloat16 *>(p.Vt) + (size_t)p.v_row[b] * dm;
    __nv_bfloat16 *tv = static_cast<__nv_bfloat16 *>(p.tailV) + o * p.tv_owner + p.tv_layer + (size_t)p.tail_pos[b] * dm;
    for (int i = tid; i < dm; i += kUThreads) tv[i] = vt[i];
  }
  __syncthreads();
  const __nv_bfloat16 *slot = static_cast<const __nv_bfloat16 *>(p.slots) +
                              (2LL * o + p.sel[o]) * p.slot_elems + p.layer_off;
  for (int k = blockIdx.y * (kUThreads / 32) + warp; k < min(R, (blockIdx.y + 1) * (kUThreads / 32));
       k += kUThreads / 32) {
    const uint4 *a4 = reinterpret_cast<const uint4 *>(slot + (size_t)k * dff);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    int v = lane;
    for (; v + 96 < nvec; v += 128) {
      uint4 a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = a4[v + 32 * u];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint4 z = xs[v + 32 * u];
        const __nv_bfloat16 *ah = reinterpret_cast<const __nv_bfloat16 *>(&a[u]);
        const __nv_bfloat16 *zh = reinterpret_cast<const __nv_bfloat16 *>(&z);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[u] = fmaf(bf(ah[e]), bf(zh[e]), acc[u]);
      }
    }
    for (; v < nvec; v += 32) {
      const uint4 a = a4[v], z = xs[v];
      const __nv_bfloat16 *ah = reinterpret_cast<const __nv_bfloat16 *>(&a);
      const __nv_bfloat16 *zh = reinterpret_cast<const __nv_bfloat16 *>(&z);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[0] = fmaf(bf(ah[e]), bf(zh[e]), acc[0]);
    }
    float s = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) p.u[(size_t)b * 64 + k] = s;
  }
}

__global__ void __launch_bounds__(256) lr_finish_kernel(const LowRankRead p) {
  const int b = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= p.n || i >= p.d_model) return;
  const int o = p.owner_idx[b];
  const __nv_bfloat16 *Bm = static_cast<const __nv_bfloat16 *>(p.slots) + (2LL * o + p.sel[o]) * p.slot_elems +
                            p.layer_off + (size_t)p.rank * p.d_ff;
  float y = 0.f;
  for (int ks = 0; ks < p.ksplit; ++ks) y += p.Y32[ks * p.y32_slab + (size_t)b * p.d_model + i];   // fixed order
  for (int k = 0; k < p.rank; ++k) y = fmaf(p.u[(size_t)b * 64 + k], bf(Bm[(size_t)k * p.d_model + i]), y);
  if (p.resid) y += bf(static_cast<const __nv_bfloat16 *>(p.resid)[(size_t)p.y_row[b] * p.d_model + i]);
  static_cast<__nv_bfloat16 *>(p.Y)[(size_t)p.y_row[b] * p.d_model + i] = __float2bfloat16_rn(y);
}

// one CTA per member (grid.x = n), one layer per launch
__global__ void __launch_bounds__(512) lr_write_kernel(const LowRankWrite p) {
  extern __shared__ float sm[];                    // m [d_ff], w [R]
  float *m = sm, *w = sm + p.d_ff;
  const int b = blockIdx.x, o = p.owner_idx[b];
  const int R = p.rank, dff = p.d_ff, dm = p.d_model, C = p.C, nvec = dff / 8;
  const uint4 *Z = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.tailZ) + o * p.tz_owner +
                                                   p.tz_layer);
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {     // chunk mean m: 8 columns per thread, t ascending
    float sacc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int t = 0;
    for (; t + 7 < C; t += 8) {                               // 8 independent 16-byte loads in flight
      uint4 z[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) z[u] = Z[(size_t)(t + u) * nvec + v];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const __nv_bfloat16 *h = reinterpret_cast<const __nv_bfloat16 *>(&z[u]);
#pragma unroll
        for (int e = 0; e < 8; ++e) sacc[e] += bf(h[e]);
      }
    }
    for (; t < C; ++t) {
      const uint4 z = Z[(size_t)t * nvec + v];
      const __nv_bfloat16 *h = reinterpret_cast<const __nv_bfloat16 *>(&z);
#pragma unroll
      for (int e = 0; e < 8; ++e) sacc[e] += bf(h[e]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) m[v * 8 + e] = sacc[e] / (float)C;
  }
  __syncthreads();
  const __nv_bfloat16 *src = static_cast<const __nv_bfloat16 *>(p.slots) + (2LL * o + p.sel[o]) * p.slot_elems +
                             p.layer_off;
  __nv_bfloat16 *dst = static_cast<__nv_bfloat16 *>(p.slots) + (2LL * o + 1 - p.sel[o]) * p.slot_elems + p.layer_off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int k = warp; k < R; k += nw) {                        // w = A m
    const uint4 *a4 = reinterpret_cast<const uint4 *>(src + (size_t)k * dff);
    float s = 0.f;
    for (int v = lane; v < nvec; v += 32) {
      const uint4 a = a4[v];
      const __nv_bfloat16 *h = reinterpret_cast<const __nv_bfloat16 *>(&a);
#pragma unroll
      for (int e = 0; e < 8; ++e) s = fmaf(bf(h[e]), m[v * 8 + e], s);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) w[k] = s;
  }
  __syncthreads();
  bool bad = false;
  const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
  uint4 *d4 = reinterpret_cast<uint4 *>(dst);
  for (int e = threadIdx.x; e < R * nvec; e += blockDim.x) {   // A' = A + η w mᵀ, 8 elements per thread
    const int k = e / nvec, v = e - k * nvec;
    const uint4 a = s4[e];
    const __nv_bfloat16 *h = reinterpret_cast<const __nv_bfloat16 *>(&a);
    uint4 r;
    __nv_bfloat16 *rh = reinterpret_cast<__nv_bfloat16 *>(&r);
    const float ew = p.eta * w[k];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      rh[q] = __float2bfloat16_rn(fmaf(ew, m[v * 8 + q], bf(h[q])));
      bad |= !isfinite(bf(rh[q]));
    }
    d4[e] = r;
  }
  const int nb = R * dm / 8;                                  // B' = B
  for (int e = threadIdx.x; e < nb; e += blockDim.x) d4[R * nvec + e] = s4[R * nvec + e];
  if (bad) atomicOr(p.fail_flag, 1);
}

}  // namespace

cudaError_t launch_lowrank_read(const LowRankRead &p, const ChunkLaunch &base, cudaStream_t s) {
  const size_t smem = (size_t)p.d_ff * 2;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e0 = cudaFuncSetAttribute(lr_u_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e0 != cudaSuccess) return e0;
    configured = smem;
  }
  lr_u_kernel<<<dim3(p.n, (p.rank + 31) / 32), kUThreads, smem, s>>>(p);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = launch_read_chunk(base, s);                  // base-only tcgen05 GEMM into Y32
  if (e != cudaSuccess) return e;
  lr_finish_kernel<<<dim3((p.d_model + 255) / 256, p.n), 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_lowrank_write(const LowRankWrite &p, cudaStream_t s) {
  const size_t smem = ((size_t)p.d_ff + 64) * 4;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(lr_write_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  lr_write_kernel<<<p.n, 512, smem, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace ttt
