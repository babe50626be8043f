// a3 + a4 — decode READ: y_b = x_b · (W_down[l] + ΔW_{μ(b)}[l])ᵀ, tail append.
//
// PAPER: ApplyState "apply; keep version" and TailBufferUpdate "append; no
// version bump" (Table 3); READ views are immutable (P:350-352,
// P:403-409).  BASELINE.json north_star: y = x·(W_down + ΔW_owner)ᵀ.
//
// B200 design (DESIGN.md §"READ kernel"): decode READ is a set of GEMVs with
// arithmetic intensity ≈ 2 flop/byte, i.e. HBM-bound by two
// orders of magnitude, so it is a streaming SIMT kernel, not a tensor-core
// GEMM.  One persistent CTA per SM (148 on B200) stages every member's x row
// in shared memory once; warps stream whole 19 KB rows of W_down (read once
// per group) and of each owner's ΔW (read once) with 16-byte
// L1-no-allocate loads, 8 in flight per lane, and FMA in fp32.  A task is
// (matrix m ∈ {base, member 0..n-1}, output row i); each task stores one fp32
// partial, and the last of the n+1 tasks of row i (per-row ticket) sums
// base + delta in a fixed order and writes y (deterministic; no atomics on
// data).  The committed slot is selected through the device active-slot
// table, so a commit enqueued earlier on the stream is visible without a
// host round trip.
#include <cuda_bf16.h>

#include "../internal.h"

namespace ttt {
namespace {

constexpr int kThreads = 512;
constexpr int kUnroll = 8;

__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

template <typename T>
struct Elem;
template <>
struct Elem<__nv_bfloat16> {
  static constexpr int kVec = 8;
  // w (8 bf16) · x (8 bf16) accumulated into acc in element order
  __device__ static __forceinline__ void unpack(const uint4 &v, float (&f)[8]) {
    f[0] = bf_lo(v.x); f[1] = bf_hi(v.x); f[2] = bf_lo(v.y); f[3] = bf_hi(v.y);
    f[4] = bf_lo(v.z); f[5] = bf_hi(v.z); f[6] = bf_lo(v.w); f[7] = bf_hi(v.w);
  }
  __device__ static __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ static __forceinline__ __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};
template <>
struct Elem<float> {
  static constexpr int kVec = 4;
  __device__ static __forceinline__ void unpack(const uint4 &v, float (&f)[4]) {
    f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
  }
  __device__ static __forceinline__ float to_f(float v) { return v; }
  __device__ static __forceinline__ float from_f(float v) { return v; }
};

template <typename T>
__global__ void __launch_bounds__(kThreads, 1) read_decode_kernel(const ReadParams p) {
  using E = Elem<T>;
  constexpr int VN = E::kVec;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint4 *xs = reinterpret_cast<uint4 *>(smem_raw);   // [n][nvec] member x rows

  const int n = p.n, dff = p.d_ff, dm = p.d_model;
  const int nvec = dff / VN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // stage x rows (coalesced, once per CTA)
  for (int idx = tid; idx < n * nvec; idx += kThreads) {
    const int b = idx / nvec, v = idx - b * nvec;
    xs[idx] = reinterpret_cast<const uint4 *>(static_cast<const T *>(p.X) + (size_t)p.x_row[b] * dff)[v];
  }
  __syncthreads();

  // a4 — TailBufferUpdate: CTA b appends member b's (z, v) at its tail index.
  if (blockIdx.x < n) {
    const int b = blockIdx.x, o = p.owner_idx[b];
    uint4 *tz = reinterpret_cast<uint4 *>(static_cast<T *>(p.tailZ) + o * p.tz_owner + p.tz_layer +
                                          (size_t)p.tail_pos[b] * dff);
    for (int v = tid; v < nvec; v += kThreads) tz[v] = xs[b * nvec + v];
    T *tv = static_cast<T *>(p.tailV) + o * p.tv_owner + p.tv_layer + (size_t)p.tail_pos[b] * dm;
    const T *src = static_cast<const T *>(p.Vt) + (size_t)p.v_row[b] * dm;
    for (int i = tid; i < dm; i += kThreads) tv[i] = src[i];
  }

  const long long n_tasks = (long long)(n + 1) * dm;
  const int warps_total = gridDim.x * (kThreads / 32);
  const int gw = blockIdx.x * (kThreads / 32) + warp;
  const int arrivals = n + 1;

  for (long long t = gw; t < n_tasks; t += warps_total) {
    const int m = (int)(t / dm);          // 0 = base W_down, 1+b = member b's ΔW
    const int i = (int)(t - (long long)m * dm);
    const uint4 *row;
    int b = 0;
    if (m == 0) {
      row = reinterpret_cast<const uint4 *>(static_cast<const T *>(p.w_down_l) + (size_t)i * dff);
    } else {
      b = m - 1;
      const int o = p.owner_idx[b];
      const long long slot = 2LL * o + p.sel[o];
      row = reinterpret_cast<const uint4 *>(static_cast<const T *>(p.slots) + slot * p.slot_elems +
                                            p.layer_off + (size_t)i * dff);
    }
    float acc[kMaxReadMembers];
#pragma unroll
    for (int r = 0; r < kMaxReadMembers; ++r) acc[r] = 0.f;

    for (int v0 = lane; v0 < nvec; v0 += 32 * kUnroll) {
      uint4 w[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (v0 + 32 * u < nvec) w[u] = ld_stream(row + v0 + 32 * u);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int v = v0 + 32 * u;
        if (v < nvec) {
          float wf[VN];
          E::unpack(w[u], wf);
          if (m == 0) {
#pragma unroll
            for (int r = 0; r < kMaxReadMembers; ++r) {
              if (r < n) {
                float xf[VN];
                E::unpack(xs[r * nvec + v], xf);
#pragma unroll
                for (int e = 0; e < VN; ++e) acc[r] = fmaf(wf[e], xf[e], acc[r]);
              }
            }
          } else {
            float xf[VN];
            E::unpack(xs[b * nvec + v], xf);
#pragma unroll
            for (int e = 0; e < VN; ++e) acc[0] = fmaf(wf[e], xf[e], acc[0]);
          }
        }
      }
    }
    // warp all-reduce (butterfly: every lane ends with the same sums)
    if (m == 0) {
#pragma unroll
      for (int r = 0; r < kMaxReadMembers; ++r) {
        if (r < n) {
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], off);
        }
      }
      // lane r stores member r's partial (static index select keeps acc in registers)
      float mine = 0.f;
#pragma unroll
      for (int r = 0; r < kMaxReadMembers; ++r) mine = (lane == r) ? acc[r] : mine;
      if (lane < n) p.Pbase[(size_t)lane * dm + i] = mine;
    } else {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], off);
      if (lane == 0) p.Pdelta[(size_t)b * dm + i] = acc[0];
    }
    __syncwarp();
    int old = 0;
    if (lane == 0) {
      __threadfence();
      old = atomicAdd(p.tickets + i, 1);
    }
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old == arrivals - 1) {            // last arrival for row i: combine in fixed order
      __threadfence();
      if (lane < n) {
        float y = __ldcg(p.Pbase + (size_t)lane * dm + i) + __ldcg(p.Pdelta + (size_t)lane * dm + i);
        if (p.resid) y += E::to_f(static_cast<const T *>(p.resid)[(size_t)p.y_row[lane] * dm + i]);
        static_cast<T *>(p.Y)[(size_t)p.y_row[lane] * dm + i] = E::from_f(y);
      }
      if (lane == 0) p.tickets[i] = 0;    // self-reset for the next launch
    }
  }
}

template <typename T>
cudaError_t launch_t(const ReadParams &p, cudaStream_t s) {
  const size_t smem = (size_t)p.n * p.d_ff * sizeof(T);
  static int configured_smem = -1;
  if ((int)smem > configured_smem) {
    cudaError_t e = cudaFuncSetAttribute(read_decode_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 * 1024));
    if (e != cudaSuccess) return e;
    configured_smem = (int)smem;
  }
  const int grid = device_sm_count();
  read_decode_kernel<T><<<grid, kThreads, smem, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_read_decode(int dtype, const ReadParams &p, cudaStream_t s) {
  if (dtype == 1) return launch_t<__nv_bfloat16>(p, s);
  return launch_t<float>(p, s);
}

}  // namespace ttt
