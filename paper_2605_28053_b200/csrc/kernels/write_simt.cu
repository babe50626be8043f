// a5 — WRITE (BoundaryUpdate), SIMT fp32-FFMA version.
//
// PAPER: "the update reads owner r's committed version v and produces one
// dirty candidate state for that owner. The candidate is invisible to later
// READs until committed" (WRITE paragraph; Table 3 BoundaryUpdate
// P:387-390).  Rule: SURVEY.md §8(c) reading i,
//     ΔW̃_{v+1}[i][j] = ΔW_v[i][j] + η · Σ_{t<C} V_c[t][i] · Z_c[t][j].
// The candidate goes to the owner's shadow slot (2·o + 1 − sel[o]); the
// committed slot (2·o + sel[o]) is only read.  A non-finite candidate
// element raises its owner's device fail flag ("finite entries").
//
// This kernel is the true-fp32 path for σ.dtype = fp32 (BJ configs[0]
// tolerance 1e-5 excludes tf32) and the fallback-free reference
// design for bf16 storage when the tcgen05 kernel does not apply.  64×64
// output tile per CTA, 4×4 per thread, K = C streamed through shared memory
// in 32-token slices, fixed summation order t = 0..C−1.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

#include "../internal.h"

namespace ttt {
namespace {

constexpr int TI = 64, TJ = 64, KT = 32, NT = 256;

template <typename T>
__device__ __forceinline__ float ld_f(const T *p);
template <>
__device__ __forceinline__ float ld_f<float>(const float *p) { return *p; }
template <>
__device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16 *p) { return __bfloat162float(*p); }

template <typename T>
__device__ __forceinline__ T st_cvt(float v);
template <>
__device__ __forceinline__ float st_cvt<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 st_cvt<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <typename T>
__global__ void __launch_bounds__(NT) write_simt_kernel(const WriteParams p) {
  __shared__ float Vs[KT][TI];
  __shared__ float Zs[KT][TJ];
  const int b = blockIdx.z;
  const int o = p.owner_idx[b];
  const int i0 = blockIdx.y * TI, j0 = blockIdx.x * TJ;
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int dm = p.d_model, dff = p.d_ff, C = p.C;
  const T *Z = static_cast<const T *>(p.tailZ) + o * p.tz_owner + p.tz_layer;   // [C][d_ff]
  const T *V = static_cast<const T *>(p.tailV) + o * p.tv_owner + p.tv_layer;   // [C][d_model]

  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = 0.f;

  for (int t0 = 0; t0 < C; t0 += KT) {
    for (int idx = tid; idx < KT * TI; idx += NT) {
      const int t = idx / TI, ii = idx % TI;
      Vs[t][ii] = (t0 + t < C && i0 + ii < dm) ? ld_f(V + (size_t)(t0 + t) * dm + i0 + ii) : 0.f;
    }
    for (int idx = tid; idx < KT * TJ; idx += NT) {
      const int t = idx / TJ, jj = idx % TJ;
      Zs[t][jj] = (t0 + t < C && j0 + jj < dff) ? ld_f(Z + (size_t)(t0 + t) * dff + j0 + jj) : 0.f;
    }
    __syncthreads();
    const int kt = min(KT, C - t0);
    for (int t = 0; t < kt; ++t) {
      float a[4], c[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = Vs[t][ty * 4 + q];
        c[q] = Zs[t][tx * 4 + q];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[r][q] = fmaf(a[r], c[q], acc[r][q]);
    }
    __syncthreads();
  }

  const long long src_slot = 2LL * o + p.sel[o];
  const long long dst_slot = 2LL * o + 1 - p.sel[o];
  const T *S = static_cast<const T *>(p.slots) + src_slot * p.slot_elems + p.layer_off;
  T *D = static_cast<T *>(p.slots) + dst_slot * p.slot_elems + p.layer_off;
  bool bad = false;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = i0 + ty * 4 + r;
    if (i >= dm) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + tx * 4 + q;
      if (j >= dff) continue;
      const size_t off = (size_t)i * dff + j;
      const float cand = fmaf(p.eta, acc[r][q], ld_f(S + off));
      const T st = st_cvt<T>(cand);
      bad |= !isfinite(ld_f(&st));
      D[off] = st;
    }
  }
  if (bad) atomicOr(p.mfail + o, 1);        // per-member flag: the commit resolves members
}

// SPEC-compat rule 1 (the CPU program's rank-1 stand-in, S:188 / S:206 / S:215; SURVEY §8(c)
// step 7): m = (1/C) Σ_t z_t over the chunk's tail, ΔW̃ = ΔW_v + η·m mᵀ (square: d_model = d_ff;
// the targets v_t are not used); READ is the unchanged y = (W_down + ΔW)·x with W_down = I.
// One CTA row of the grid per member: every CTA recomputes m (C·d tail reads from L2) into
// shared memory, then writes its share of the d×d candidate.
template <typename T>
__global__ void __launch_bounds__(256) write_rule1_kernel(const WriteParams p) {
  extern __shared__ float m[];
  const int b = blockIdx.y, o = p.owner_idx[b], d = p.d_ff;
  const T *Z = static_cast<const T *>(p.tailZ) + o * p.tz_owner + p.tz_layer;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float s = 0.f;
    for (int t = 0; t < p.C; ++t) s += ld_f(Z + (size_t)t * d + j);
    m[j] = s / (float)p.C;
  }
  __syncthreads();
  const T *S = static_cast<const T *>(p.slots) + (2LL * o + p.sel[o]) * p.slot_elems + p.layer_off;
  T *D = static_cast<T *>(p.slots) + (2LL * o + 1 - p.sel[o]) * p.slot_elems + p.layer_off;
  bool bad = false;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (size_t)d * d;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / d), j = (int)(idx - (size_t)i * d);
    const T st = st_cvt<T>(fmaf(p.eta * m[i], m[j], ld_f(S + idx)));
    bad |= !isfinite(ld_f(&st));
    D[idx] = st;
  }
  if (bad) atomicOr(p.mfail + o, 1);
}

}  // namespace

cudaError_t launch_write_rule1(int dtype, const WriteParams &p, cudaStream_t s) {
  const size_t smem = (size_t)p.d_ff * 4;
  const int per = (int)std::min<size_t>(((size_t)p.d_ff * p.d_ff + 255) / 256, (size_t)device_sm_count());
  dim3 grid(std::max(1, per), p.n);
  if (dtype == 1) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(write_rule1_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    write_rule1_kernel<__nv_bfloat16><<<grid, 256, smem, s>>>(p);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(write_rule1_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    write_rule1_kernel<float><<<grid, 256, smem, s>>>(p);
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_write_simt(int dtype, const WriteParams &p, cudaStream_t s) {
  dim3 grid((p.d_ff + TJ - 1) / TJ, (p.d_model + TI - 1) / TI, p.n);
  if (dtype == 1)
    write_simt_kernel<__nv_bfloat16><<<grid, NT, 0, s>>>(p);
  else
    write_simt_kernel<float><<<grid, NT, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace ttt
