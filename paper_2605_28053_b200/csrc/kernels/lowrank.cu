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
// B copied; a non-finite candidate raises its owner's device fail flag.
#include <cuda_bf16.h>

#include <cstdlib>

#include "../internal.h"

namespace ttt {
namespace {

__device__ __forceinline__ float bf(const __nv_bfloat16 v) { return __bfloat162float(v); }

typedef unsigned long long u64;
__device__ __forceinline__ uint4 ld_stream(const uint4 *q) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(q));
  return r;
}
// acc += a.lo*z.lo + a.hi*z.hi for one packed bf16 pair, fp32 accumulate (FHFMA.BF16)
__device__ __forceinline__ void fma_bf16x2(float &acc, uint32_t a, uint32_t z) {
  asm("{\n\t.reg .b16 al, ah, zl, zh;\n\t"
      "mov.b32 {al, ah}, %1;\n\tmov.b32 {zl, zh}, %2;\n\t"
      "fma.rn.f32.bf16 %0, al, zl, %0;\n\tfma.rn.f32.bf16 %0, ah, zh, %0;\n}"
      : "+f"(acc)
      : "r"(a), "r"(z));
}
__device__ __forceinline__ void dot8(float &acc, const uint4 &a, const uint4 &z) {
  fma_bf16x2(acc, a.x, z.x); fma_bf16x2(acc, a.y, z.y); fma_bf16x2(acc, a.z, z.z); fma_bf16x2(acc, a.w, z.w);
}

// u = A x as warp tasks (member b, rank row k, K segment j of nseg): a persistent grid of
// 1024-thread CTAs on every SM streams A with 4 × 16-byte loads per lane in flight (x from
// L2), each task writes its partial to u[(b·R + k)·nseg + j] and lr_finish sums the nseg
// partials in order (deterministic).  The same launch gathers x into the contiguous
// workspace of the base GEMM (when rows are not already contiguous) and appends the tail.
constexpr int kUThreads = 1024;
__global__ void __launch_bounds__(kUThreads, 1) lr_u_kernel(const LowRankRead p, int gather) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = p.rank, dff = p.d_ff, dm = p.d_model, nvec = dff / 8, S = p.nseg;
  const int gtid = blockIdx.x * kUThreads + tid, gsz = gridDim.x * kUThreads;
  for (int idx = gtid; idx < p.n * nvec; idx += gsz) {       // gather x, append z (a4)
    const int b = idx / nvec, v = idx - b * nvec, o = p.owner_idx[b];
    const uint4 z = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.X) + (size_t)p.x_row[b] * dff)[v];
    if (gather) reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.Xg) + (size_t)b * dff)[v] = z;
    reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.tailZ) + o * p.tz_owner + p.tz_layer +
                              (size_t)p.tail_pos[b] * dff)[v] = z;
  }
  for (int idx = gtid; idx < p.n * dm; idx += gsz) {         // append v
    const int b = idx / dm, i = idx - b * dm, o = p.owner_idx[b];
    (static_cast<__nv_bfloat16 *>(p.tailV) + o * p.tv_owner + p.tv_layer + (size_t)p.tail_pos[b] * dm)[i] =
        (static_cast<const __nv_bfloat16 *>(p.Vt) + (size_t)p.v_row[b] * dm)[i];
  }
  const int n_tasks = p.n * R * S, nw = gridDim.x * (kUThreads / 32);
  for (int t = warp * gridDim.x + blockIdx.x; t < n_tasks; t += nw) {
    const int r = t / S, j = t - r * S, b = r / R, k = r - b * R, o = p.owner_idx[b];
    const uint4 *a4 = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.slots) +
                                                      (2LL * o + p.sel[o]) * p.slot_elems + p.layer_off +
                                                      (size_t)k * dff);
    const uint4 *x4 = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.X) + (size_t)p.x_row[b] * dff);
    const int v0 = nvec * j / S, v1 = nvec * (j + 1) / S;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int v = v0 + lane; v < v1; v += 128) {
      uint4 a[4], z[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool in = v + 32 * u < v1;
        a[u] = in ? ld_stream(a4 + v + 32 * u) : make_uint4(0u, 0u, 0u, 0u);
        z[u] = in ? __ldg(x4 + v + 32 * u) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) dot8(acc[u], a[u], z[u]);
    }
    float s = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) p.u[(size_t)r * S + j] = s;
  }
}

// y_b = Σ_ks Y32[ks]_b + Bᵀ u_b (+ residual): one CTA per (member, 2048 outputs), 8 outputs
// per thread with 16-byte loads; u_b = Σ_j partials (in order) staged in shared memory.
constexpr int kFinThreads = 256;
__global__ void __launch_bounds__(kFinThreads) lr_finish_kernel(const LowRankRead p) {
  __shared__ float us[64];
  const int b = blockIdx.y, o = p.owner_idx[b], R = p.rank, dm = p.d_model, S = p.nseg;
  if (threadIdx.x < R) {
    float u = 0.f;
    for (int j = 0; j < S; ++j) u += p.u[((size_t)b * R + threadIdx.x) * S + j];
    us[threadIdx.x] = u;
  }
  __syncthreads();
  const int i0 = (blockIdx.x * kFinThreads + threadIdx.x) * 8;
  if (i0 >= dm) return;
  const __nv_bfloat16 *Bm = static_cast<const __nv_bfloat16 *>(p.slots) + (2LL * o + p.sel[o]) * p.slot_elems +
                            p.layer_off + (size_t)R * p.d_ff;
  float y[8];
  {
    const float4 *q = reinterpret_cast<const float4 *>(p.Y32 + (size_t)b * dm + i0);
    const float4 lo = q[0], hi = q[1];
    y[0] = lo.x; y[1] = lo.y; y[2] = lo.z; y[3] = lo.w; y[4] = hi.x; y[5] = hi.y; y[6] = hi.z; y[7] = hi.w;
  }
  for (int ks = 1; ks < p.ksplit; ++ks) {                     // fixed slab order
    const float4 *q = reinterpret_cast<const float4 *>(p.Y32 + ks * p.y32_slab + (size_t)b * dm + i0);
    const float4 lo = q[0], hi = q[1];
    y[0] += lo.x; y[1] += lo.y; y[2] += lo.z; y[3] += lo.w; y[4] += hi.x; y[5] += hi.y; y[6] += hi.z; y[7] += hi.w;
  }
  for (int k0 = 0; k0 < R; k0 += 8) {              // 8 B rows' loads in flight
    uint4 bv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      bv[q] = k0 + q < R ? *reinterpret_cast<const uint4 *>(Bm + (size_t)(k0 + q) * dm + i0) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t w[4] = {bv[q].x, bv[q].y, bv[q].z, bv[q].w};
      const float uk = k0 + q < R ? us[k0 + q] : 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        y[2 * e] = fmaf(uk, __uint_as_float(w[e] << 16), y[2 * e]);
        y[2 * e + 1] = fmaf(uk, __uint_as_float(w[e] & 0xffff0000u), y[2 * e + 1]);
      }
    }
  }
  if (p.resid) {
    const uint4 rv = *reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.resid) +
                                                      (size_t)p.y_row[b] * dm + i0);
    const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      y[2 * e] += __uint_as_float(w[e] << 16);
      y[2 * e + 1] += __uint_as_float(w[e] & 0xffff0000u);
    }
  }
  uint32_t out[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    __nv_bfloat162 h = __floats2bfloat162_rn(y[2 * e], y[2 * e + 1]);
    out[e] = *reinterpret_cast<uint32_t *>(&h);
  }
  *reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.Y) + (size_t)p.y_row[b] * dm + i0) =
      make_uint4(out[0], out[1], out[2], out[3]);
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
  if (bad) atomicOr(p.mfail + o, 1);        // per-member flag: the commit resolves members
}

__global__ void __launch_bounds__(256) lr_gather_kernel(const LowRankRead p) {
  const int nvec = p.d_ff / 8;
  for (int idx = blockIdx.x * 256 + threadIdx.x; idx < p.n * nvec; idx += gridDim.x * 256) {
    const int b = idx / nvec, v = idx - b * nvec;
    reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.Xg) + (size_t)b * p.d_ff)[v] =
        reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.X) + (size_t)p.x_row[b] * p.d_ff)[v];
  }
}

}  // namespace

// K segments per A row so the n·R·nseg warp tasks fill whole waves of warps
int lr_segments(int rows, int warps) {
  int best = 1;
  double best_eff = 0;
  for (int S = 1; S <= kMaxLrSeg; ++S) {
    const long long t = (long long)rows * S;
    const double eff = (double)t / ((double)((t + warps - 1) / warps) * warps);
    if (eff > best_eff + 1e-3) {
      best_eff = eff;
      best = S;
    }
  }
  return best;
}

cudaError_t launch_lowrank_read(const LowRankRead &p0, const ChunkLaunch &base0, cudaStream_t s) {
  LowRankRead p = p0;
  ChunkLaunch base = base0;
  const int sms = device_sm_count();
  // TTT_LR_FUSED: 1 (default) base GEMM + u warps + finish in one launch (read_chunk_tc.cu),
  // 2 one-pass tcgen05 GEMM over [W_down; A] + bulk-copy finish (lowrank_tc.cu; measured equal
  // at R = 64 and 8 % slower at R = 16), 0 three launches
  static const int mode = getenv("TTT_LR_FUSED") ? atoi(getenv("TTT_LR_FUSED")) : 1;
  bool identity = true;
  for (int b = 0; b < p.n; ++b) identity &= p.x_row[b] == b;
  if (mode == 2 && lowrank_tc_supported(p.n, p.d_model, p.d_ff, p.rank)) {
    if (!identity) {
      lr_gather_kernel<<<sms * 4, 256, 0, s>>>(p);
      count_launch();
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    return launch_lowrank_tc(p, identity ? p.X : p.Xg, s);
  }
  if (mode != 0 && read_chunk_fused_fits(base.n, p.d_model, base.ksplit)) {
    // one launch: base GEMM on tcgen05 + u = A x warps + tail append + finish (read_chunk_tc.cu)
    if (p.x_row0 >= 0 && p.x_rows_total > 0) {     // contiguous rows of a known buffer: no gather
      base.X = p.X;
      base.x_rowmap = 1;
      base.x_row0 = p.x_row0;
      base.x_rows_total = p.x_rows_total;
    } else if (identity) {
      base.X = p.X;
      base.x_rowmap = 1;
    } else {
      lr_gather_kernel<<<sms * 4, 256, 0, s>>>(p);
      count_launch();
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    base.lr = &p;
    base.lr_ctr = p.ctr;
    base.cooperative = g_live_lowrank_pools.load() > 1;
    return launch_read_chunk(base, s);
  }
  p.nseg = lr_segments(p.n * p.rank, sms * (kUThreads / 32));
  // the base GEMM reads X in place when its rows are 0..n-1 and fill whole 128-row blocks
  int gather = p.n % 128 != 0;
  for (int b = 0; b < p.n; ++b) gather |= p.x_row[b] != b;
  if (!gather) base.X = p.X;
  lr_u_kernel<<<sms, kUThreads, 0, s>>>(p, gather);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = launch_read_chunk(base, s);                  // base-only tcgen05 GEMM into Y32
  if (e != cudaSuccess) return e;
  lr_finish_kernel<<<dim3((p.d_model / 8 + kFinThreads - 1) / kFinThreads, p.n), kFinThreads, 0, s>>>(p);
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
