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

// one warp per (member b, rank row k)
__global__ void __launch_bounds__(256) lr_u_kernel(const LowRankRead p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int R = p.rank, dff = p.d_ff, dm = p.d_model;
  const int b = warp / R, k = warp - b * R;
  if (b >= p.n) return;
  const int o = p.owner_idx[b];
  const __nv_bfloat16 *x = static_cast<const __nv_bfloat16 *>(p.X) + (size_t)p.x_row[b] * dff;
  const __nv_bfloat16 *slot = static_cast<const __nv_bfloat16 *>(p.slots) +
                              (2LL * o + p.sel[o]) * p.slot_elems + p.layer_off;
  const __nv_bfloat16 *A = slot + (size_t)k * dff;
  const uint4 *a4 = reinterpret_cast<const uint4 *>(A), *x4 = reinterpret_cast<const uint4 *>(x);
  float acc = 0.f;
  for (int v = lane; v < dff / 8; v += 32) {
    const uint4 a = a4[v], z = x4[v];
    const __nv_bfloat16 *ah = reinterpret_cast<const __nv_bfloat16 *>(&a);
    const __nv_bfloat16 *zh = reinterpret_cast<const __nv_bfloat16 *>(&z);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc = fmaf(bf(ah[e]), bf(zh[e]), acc);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) p.u[(size_t)b * 64 + k] = acc;
  if (k == 0) {                                    // gather x_b for the base GEMM; tail append (a4)
    uint4 *xg = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.Xg) + (size_t)b * dff);
    uint4 *tz = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.tailZ) + o * p.tz_owner + p.tz_layer +
                                          (size_t)p.tail_pos[b] * dff);
    for (int v = lane; v < dff / 8; v += 32) {
      const uint4 z = x4[v];
      xg[v] = z;
      tz[v] = z;
    }
    const __nv_bfloat16 *vt = static_cast<const __nv_bfloat16 *>(p.Vt) + (size_t)p.v_row[b] * dm;
    __nv_bfloat16 *tv = static_cast<__nv_bfloat16 *>(p.tailV) + o * p.tv_owner + p.tv_layer + (size_t)p.tail_pos[b] * dm;
    for (int i = lane; i < dm; i += 32) tv[i] = vt[i];
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
  const int R = p.rank, dff = p.d_ff, dm = p.d_model, C = p.C;
  const __nv_bfloat16 *Z = static_cast<const __nv_bfloat16 *>(p.tailZ) + o * p.tz_owner + p.tz_layer;
  for (int j = threadIdx.x; j < dff; j += blockDim.x) {      // chunk mean m (t ascending)
    float s = 0.f;
    for (int t = 0; t < C; ++t) s += bf(Z[(size_t)t * dff + j]);
    m[j] = s / (float)C;
  }
  __syncthreads();
  const __nv_bfloat16 *src = static_cast<const __nv_bfloat16 *>(p.slots) + (2LL * o + p.sel[o]) * p.slot_elems +
                             p.layer_off;
  __nv_bfloat16 *dst = static_cast<__nv_bfloat16 *>(p.slots) + (2LL * o + 1 - p.sel[o]) * p.slot_elems + p.layer_off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int k = warp; k < R; k += nw) {                        // w = A m
    float s = 0.f;
    for (int j = lane; j < dff; j += 32) s = fmaf(bf(src[(size_t)k * dff + j]), m[j], s);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) w[k] = s;
  }
  __syncthreads();
  bool bad = false;
  for (size_t e = threadIdx.x; e < (size_t)R * dff; e += blockDim.x) {   // A' = A + η w mᵀ
    const int k = (int)(e / dff), j = (int)(e - (size_t)k * dff);
    const __nv_bfloat16 a = __float2bfloat16_rn(fmaf(p.eta * w[k], m[j], bf(src[e])));
    bad |= !isfinite(bf(a));
    dst[e] = a;
  }
  for (size_t e = threadIdx.x; e < (size_t)R * dm; e += blockDim.x)     // B' = B
    dst[(size_t)R * dff + e] = src[(size_t)R * dff + e];
  if (bad) atomicOr(p.fail_flag, 1);
}

}  // namespace

cudaError_t launch_lowrank_read(const LowRankRead &p, const ChunkLaunch &base, cudaStream_t s) {
  const int warps = p.n * p.rank;
  lr_u_kernel<<<(warps * 32 + 255) / 256, 256, 0, s>>>(p);
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
