// a3 + a4 — decode READ: y_b = x_b · (W_down[l] + ΔW_{μ(b)}[l])ᵀ, tail append.
//
// PAPER: ApplyState "apply; keep version" and TailBufferUpdate "append; no
// version bump" (Table 3); READ views are immutable (P:350-352,
// P:403-409).  BASELINE.json north_star: y = x·(W_down + ΔW_owner)ᵀ.
//
// B200 design (DESIGN.md §"READ kernel"): decode READ is a set of GEMVs with
// arithmetic intensity ≈ 2 flop/byte — HBM-bound by two orders of
// magnitude — so it is a streaming SIMT kernel, not a tensor-core GEMM.  Its
// speed is set by bytes in flight and by issue slots (tools/bw_probe.cu: a
// pure 16-byte-load stream reaches ~6.8 TB/s with ≥ 64-128 KB in flight per
// SM; a one-thread TMA bulk-copy ring tops out near 4.8 TB/s):
//  * one persistent CTA per SM (148 on B200), 16 warps; every member's x row
//    is staged in shared memory once per CTA;
//  * a task is (matrix m ∈ {W_down, ΔW of member 0..n-1}, output row i); a
//    warp streams the 19 KB row with 16-byte L1-no-allocate loads and keeps
//    the next batch of 8 loads per lane (possibly of its next task) in flight
//    while it consumes the current one;
//  * bf16 products accumulate in fp32 with the mixed-precision FMA
//    `fma.rn.f32.bf16` (SASS FHFMA.BF16 with .H0/.H1 half selects), so a
//    16-byte vector costs 8 FMAs and no unpacking; fp32 uses FFMA2 pairs;
//  * each task stores one fp32 partial; the last of the n+1 tasks of row i
//    (per-row ticket) sums base + delta in a fixed order and writes y, so the
//    result is deterministic and no data goes through atomics.
// The committed slot is selected through the device active-slot table, so a
// commit enqueued earlier on the stream is visible without a host round trip.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "../internal.h"

namespace ttt {
namespace {

// Launch variants (threads per CTA, 16-byte loads per lane per batch): the
// default was chosen by a sweep (TTT_READ_CFG selects another for tuning).

typedef unsigned long long u64;

__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// L2 eviction-priority variants (configs with several READ launches per layer: W_down[l] is kept
// in L2 across the group's launches, the once-read ΔW rows are evicted first)
__device__ __forceinline__ u64 l2_policy(bool last) {
  u64 pol;
  if (last) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ld_stream_hint(const uint4 *p, u64 pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// acc += w.lo*x.lo + w.hi*x.hi for one packed bf16 pair (fp32 accumulate)
__device__ __forceinline__ void fma_bf16x2(float &acc, uint32_t w, uint32_t x) {
  asm("{\n\t.reg .b16 wl, wh, xl, xh;\n\t"
      "mov.b32 {wl, wh}, %1;\n\tmov.b32 {xl, xh}, %2;\n\t"
      "fma.rn.f32.bf16 %0, wl, xl, %0;\n\tfma.rn.f32.bf16 %0, wh, xh, %0;\n}"
      : "+f"(acc)
      : "r"(w), "r"(x));
}
__device__ __forceinline__ u64 pack2(uint32_t lo, uint32_t hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ void ffma2(u64 &acc, u64 a, u64 b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ float hsum2(u64 v) {
  uint32_t lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
  return __uint_as_float(lo) + __uint_as_float(hi);
}

// Per element type: accumulator, 16-byte-vector dot, finish, conversions.
template <typename T> struct Elem;
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kVec = 8;
  typedef float Acc;
  __device__ static __forceinline__ Acc zero() { return 0.f; }
  __device__ static __forceinline__ void dot(Acc &a, const uint4 &w, const uint4 &x) {
    fma_bf16x2(a, w.x, x.x); fma_bf16x2(a, w.y, x.y); fma_bf16x2(a, w.z, x.z); fma_bf16x2(a, w.w, x.w);
  }
  __device__ static __forceinline__ float finish(Acc a) { return a; }
  __device__ static __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ static __forceinline__ __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};
template <> struct Elem<float> {
  static constexpr int kVec = 4;
  typedef u64 Acc;
  __device__ static __forceinline__ Acc zero() { return 0ull; }
  __device__ static __forceinline__ void dot(Acc &a, const uint4 &w, const uint4 &x) {
    ffma2(a, pack2(w.x, w.y), pack2(x.x, x.y));
    ffma2(a, pack2(w.z, w.w), pack2(x.z, x.w));
  }
  __device__ static __forceinline__ float finish(Acc a) { return hsum2(a); }
  __device__ static __forceinline__ float to_f(float v) { return v; }
  __device__ static __forceinline__ float from_f(float v) { return v; }
};

// NEXT f3 — streaming learner (C = 1, every step a WRITE): with FUSE the delta
// tasks also write the candidate row ΔW'[i] = ΔW[i] + η·v_i·x into the owner's
// shadow slot while the pre-update row is in registers (y uses version v,
// reading xvii), so an all-update step streams ΔW once in and once out instead
// of READ + a separate WRITE pass (all-update row P:559).
// The candidate is ΔW + η·(v·x) with v·x exact in fp32 (two 8-bit significands) and ONE fp32
// rounding of the fma — the fp32 value the storage RNE rounds (reading xi); η·v rounded first
// would add a second rounding that shifts ~0.5 % of the bf16 results at η = 0.01.
__device__ __forceinline__ uint32_t upd_bf16x2(uint32_t w, uint32_t x, u64 v2, u64 eta2, uint32_t &expmax) {
  u64 px, r2 = pack2(w << 16, w & 0xffff0000u);
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(px) : "l"(pack2(x << 16, x & 0xffff0000u)), "l"(v2));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r2) : "l"(px), "l"(eta2));
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float((uint32_t)(r2 >> 32))), "f"(__uint_as_float((uint32_t)r2)));
  expmax = __vmaxu2(expmax, r & 0x7f807f80u);
  return r;
}
template <typename T> struct Upd;
template <> struct Upd<__nv_bfloat16> {
  __device__ static __forceinline__ uint4 apply(const uint4 &w, const uint4 &x, float v, float eta, uint32_t &em) {
    const u64 v2 = pack2(__float_as_uint(v), __float_as_uint(v)), e2 = pack2(__float_as_uint(eta), __float_as_uint(eta));
    return make_uint4(upd_bf16x2(w.x, x.x, v2, e2, em), upd_bf16x2(w.y, x.y, v2, e2, em),
                      upd_bf16x2(w.z, x.z, v2, e2, em), upd_bf16x2(w.w, x.w, v2, e2, em));
  }
  __device__ static __forceinline__ bool bad(uint32_t em) {
    return (em & 0x7f80u) == 0x7f80u || (em >> 16) == 0x7f80u;
  }
};
template <> struct Upd<float> {
  __device__ static __forceinline__ uint32_t one(uint32_t w, uint32_t x, float ev, uint32_t &em) {
    const float r = fmaf(ev, __uint_as_float(x), __uint_as_float(w));
    em |= isfinite(r) ? 0u : 1u;
    return __float_as_uint(r);
  }
  __device__ static __forceinline__ uint4 apply(const uint4 &w, const uint4 &x, float v, float eta, uint32_t &em) {
    const float ev = eta * v;
    return make_uint4(one(w.x, x.x, ev, em), one(w.y, x.y, ev, em), one(w.z, x.z, ev, em), one(w.w, x.w, ev, em));
  }
  __device__ static __forceinline__ bool bad(uint32_t em) { return em != 0; }
};

template <typename T, int kThreads, int kU, bool FUSE>
__global__ void __launch_bounds__(kThreads, 1) read_decode_kernel(const ReadParams p) {
  constexpr int kWarps = kThreads / 32;
  using E = Elem<T>;
  using Acc = typename E::Acc;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint4 *xs = reinterpret_cast<uint4 *>(smem_raw);      // [n][nvec] member x rows
  __shared__ const uint4 *s_row0[kMaxReadMembers + 1];  // row-0 base of each matrix
  __shared__ uint4 *s_dst0[kMaxReadMembers];             // FUSE: row-0 base of each shadow slot

  const int n = p.n, dff = p.d_ff, dm = p.d_model;
  const int nvec = dff / E::kVec;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // Programmatic dependent launch (PDL): let the next layer's READ grid be scheduled as our
  // CTAs retire, and overlap our own launch with the previous kernel's tail.  Before
  // griddepcontrol.wait only W_down is touched — no kernel ever writes it — so warps whose
  // first task is a base row issue their first batch early; everything that may depend on
  // earlier kernels in the stream (x, the active-slot table, ΔW, the workspace) waits.
  asm volatile("griddepcontrol.launch_dependents;");
  const int n_tasks = (n + 1) * dm;
  const int stride = gridDim.x * kWarps;
  int t = p.order ? warp * gridDim.x + blockIdx.x : blockIdx.x * kWarps + warp;
  auto load = [&](uint4 (&buf)[kU], const uint4 *row, int v0) {
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (v0 + 32 * u < nvec) buf[u] = ld_stream(row + v0 + 32 * u);
  };
  uint4 cur[kU], nxt[kU];
  int v = lane;
  const uint4 *row = nullptr;
  const bool early = t < dm;                        // first task is a W_down row
  __shared__ __align__(8) unsigned long long s_xbar;
  const bool xtma = p.xtma && (reinterpret_cast<uintptr_t>(p.X) & 15) == 0;   // rows staged by bulk copies
  if (xtma && tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_xbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (early) {
    row = static_cast<const uint4 *>(p.w_down_l) + (size_t)t * nvec;
    load(cur, row, v);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (tid <= n) {
    if (tid == 0) {
      s_row0[0] = static_cast<const uint4 *>(p.w_down_l);
      if (xtma) {                                  // the n x rows: one bulk copy each
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_xbar), bytes = (uint32_t)nvec * 16;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes * n) : "memory");
        for (int b = 0; b < n; ++b)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(xs + (size_t)b * nvec)),
                       "l"(static_cast<const T *>(p.X) + (size_t)p.x_row[b] * dff), "r"(bytes), "r"(bar)
                       : "memory");
      }
    } else {
      const int o = p.owner_idx[tid - 1];
      const long long slot = 2LL * o + p.sel[o];
      s_row0[tid] = reinterpret_cast<const uint4 *>(static_cast<const T *>(p.slots) + slot * p.slot_elems +
                                                    p.layer_off);
      if (FUSE)
        s_dst0[tid - 1] = reinterpret_cast<uint4 *>(static_cast<T *>(const_cast<void *>(p.slots)) +
                                                    (2LL * o + 1 - p.sel[o]) * p.slot_elems + p.layer_off);
    }
  }
  __syncthreads();                                 // row-0 table ready

  auto row_of = [&](int task) {
    const int m = task / dm;
    return s_row0[m] + (size_t)(task - m * dm) * nvec;
  };
  if (!early && t < n_tasks) {
    row = row_of(t);
    load(cur, row, v);
  }

  for (int idx = xtma ? n * nvec : tid; idx < n * nvec; idx += kThreads) {
    const int b = idx / nvec, vv = idx - b * nvec;
    xs[idx] = reinterpret_cast<const uint4 *>(static_cast<const T *>(p.X) + (size_t)p.x_row[b] * dff)[vv];
  }
  // a4 — TailBufferUpdate, spread over every CTA: z rows as 16-byte vectors, v rows as elements.
  {
    const int zq = n * nvec, gtid = blockIdx.x * kThreads + tid, gsz = gridDim.x * kThreads;
    for (int idx = gtid; idx < zq; idx += gsz) {
      const int b = idx / nvec, vv = idx - b * nvec, o = p.owner_idx[b];
      reinterpret_cast<uint4 *>(static_cast<T *>(p.tailZ) + o * p.tz_owner + p.tz_layer +
                                (size_t)p.tail_pos[b] * dff)[vv] =
          reinterpret_cast<const uint4 *>(static_cast<const T *>(p.X) + (size_t)p.x_row[b] * dff)[vv];
    }
    for (int idx = gtid; idx < n * dm; idx += gsz) {
      const int b = idx / dm, i = idx - b * dm, o = p.owner_idx[b];
      (static_cast<T *>(p.tailV) + o * p.tv_owner + p.tv_layer + (size_t)p.tail_pos[b] * dm)[i] =
          (static_cast<const T *>(p.Vt) + (size_t)p.v_row[b] * dm)[i];
    }
  }
  if (xtma)                                        // every thread observes the bulk copies' completion
    asm volatile("{\n\t.reg .pred P;\nXS_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra XS_%=;\n}" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_xbar))
                 : "memory");
  __syncthreads();
  if (t >= n_tasks) return;
  Acc acc[kMaxReadMembers];
#pragma unroll
  for (int r = 0; r < kMaxReadMembers; ++r) acc[r] = E::zero();
  uint32_t expmax = 0;                             // FUSE: non-finite guard of the candidate

  while (true) {
    // next batch: same row, or the first batch of this warp's next task
    int nv = v + 32 * kU, nt = t;
    const uint4 *nrow = row;
    const bool task_end = nv >= nvec;
    if (task_end) {
      nt = t + stride;
      nv = lane;
      if (nt < n_tasks) nrow = row_of(nt);
    }
    const bool more = nt < n_tasks;
    if (more) load(nxt, nrow, nv);

    const int m = t / dm;
    if (m == 0) {                                  // base W_down: every member's x
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (v + 32 * u < nvec) {
#pragma unroll
          for (int r = 0; r < kMaxReadMembers; ++r)
            if (r < n) E::dot(acc[r], cur[u], xs[r * nvec + v + 32 * u]);
        }
      }
    } else {                                       // member b's ΔW: its own x only
      const uint4 *xb = xs + (m - 1) * nvec;
#pragma unroll
      for (int u = 0; u < kU; ++u)                 // kU independent FMA chains
        if (v + 32 * u < nvec) E::dot(acc[u % kMaxReadMembers], cur[u], xb[v + 32 * u]);
      if (FUSE) {
        const int b = m - 1, i = t - m * dm;
        const float ev = E::to_f(static_cast<const T *>(p.Vt)[(size_t)p.v_row[b] * dm + i]);
        uint4 *drow = s_dst0[b] + (size_t)i * nvec;
#pragma unroll
        for (int u = 0; u < kU; ++u)
          // candidate rows are not read again by this step: streaming stores (+2 % measured)
          if (v + 32 * u < nvec) __stcs(drow + v + 32 * u, Upd<T>::apply(cur[u], xb[v + 32 * u], ev, p.eta, expmax));
      }
    }

    if (task_end) {
      const int i = t - m * dm;
      if (m == 0) {
        float mine = 0.f;
#pragma unroll
        for (int r = 0; r < kMaxReadMembers; ++r) {
          if (r < n) {
            float s = E::finish(acc[r]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            mine = (lane == r) ? s : mine;
          }
          acc[r] = E::zero();
        }
        if (lane < n) p.Pbase[(size_t)lane * dm + i] = mine;
      } else {
        float s = E::finish(acc[0]);
#pragma unroll
        for (int r = 1; r < kMaxReadMembers; ++r) s += E::finish(acc[r]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
#pragma unroll
        for (int r = 0; r < kMaxReadMembers; ++r) acc[r] = E::zero();
        if (lane == 0) p.Pdelta[(size_t)(m - 1) * dm + i] = s;
        if (FUSE) {                                // per-member device failure flag (device-side App. H)
          if (Upd<T>::bad(expmax)) atomicOr(p.mfail + p.owner_idx[m - 1], 1);
          expmax = 0;
        }
      }
      __syncwarp();
      int old = 0;
      if (lane == 0) {
        __threadfence();
        old = atomicAdd(p.tickets + i, 1);
      }
      old = __shfl_sync(0xffffffffu, old, 0);
      if (old == n) {                              // last of the n+1 arrivals for row i
        __threadfence();
        if (lane < n) {
          float y = __ldcg(p.Pbase + (size_t)lane * dm + i) + __ldcg(p.Pdelta + (size_t)lane * dm + i);
          if (p.resid) y += E::to_f(static_cast<const T *>(p.resid)[(size_t)p.y_row[lane] * dm + i]);
          static_cast<T *>(p.Y)[(size_t)p.y_row[lane] * dm + i] = E::from_f(y);
        }
        if (lane == 0) p.tickets[i] = 0;           // self-reset for the next launch
      }
    }
    if (!more) break;
#pragma unroll
    for (int u = 0; u < kU; ++u) cur[u] = nxt[u];
    v = nv;
    row = nrow;
    t = nt;
  }
}

// ---------------------------------------------------------------------------
// bf16 READ with the shared base product on tensor cores.  The base term X·W_downᵀ for the
// group's ≤ 8 members is a real (skinny) GEMM — N = 8 members — so it runs as
// mma.sync.m16n8k16 (bf16 in, fp32 accumulate): a base task is 16 rows of W_down × a
// 512-wide K chunk (16 KB, the size of a ΔW row task), the A fragment comes straight from the
// 16-byte streaming loads (K is permuted identically on both operands, so no shuffles) and
// the B fragment is one 16-byte read of the staged x.  That replaces 64 FHFMA + 8 LDS per
// 16 bytes of W_down with ¼ MMA, which the SIMT version spent ~10 % of the launch on.  The
// per-member ΔW rows (GEMVs) stay SIMT.  Row i combines, in a fixed order, the K-chunk
// partials of the base and the member's ΔW partial once all n + KC tasks of row i arrived.
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

constexpr int kMmaThreads = 1024, kMmaChunkVec = 64;   // 512 bf16 of K per base task
constexpr int kXStage = 5;   // x staging loads in flight per thread (sweep: 4 = the compiler's unroll, 5, 6, 8, 10; 5 best)
constexpr int kDU = 4;                                  // ΔW loads per lane per batch (= the preloaded batch)

__host__ __device__ inline int mma_nvp(int nvec) { return (nvec + 127) / 128 * 128; }

template <bool FUSE, bool L2H, bool PRE1 = true>
__global__ void __launch_bounds__(kMmaThreads, 1) read_decode_mma_kernel(const ReadParams p) {
  constexpr int kWarps = kMmaThreads / 32;
  using E = Elem<__nv_bfloat16>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint4 *xs = reinterpret_cast<uint4 *>(smem_raw);      // [8][nvp] member x rows, zero padded
  __shared__ const uint4 *s_row0[kMaxReadMembers + 1];
  __shared__ uint4 *s_dst0[kMaxReadMembers];
  __shared__ int s_next;                                  // per-CTA dynamic task counter (p.dyn)
  __shared__ __align__(8) unsigned long long s_xbar;      // p.xtma: x rows staged by bulk copies

  const int n = p.n, dff = p.d_ff, dm = p.d_model, nvec = dff / 8, nvp = mma_nvp(nvec);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, tq = lane & 3;
  const int KC = p.kc, n_base = (dm + 15) / 16 * KC, n_tasks = n_base + n * dm;
  asm volatile("griddepcontrol.launch_dependents;");
  const int stride = gridDim.x * kWarps;
  int t = p.order ? warp * gridDim.x + blockIdx.x : blockIdx.x * kWarps + warp;
  // Next task of this warp. Static: t + stride. Dynamic (p.dyn, SM-interleaved order): the
  // CTA's task list t ≡ blockIdx.x (mod grid) is handed out by a shared-memory counter, so
  // warps that run ahead take more tasks and the CTA's warps finish together — a static split
  // left a ~15 µs tail where the last warps streamed alone (per-warp bandwidth is latency-bound).
  auto next_task = [&](int tt) -> int {
    if (!p.dyn) return tt + stride;
    int k = 0;
    if (lane == 0) k = atomicAdd(&s_next, 1);
    k = __shfl_sync(0xffffffffu, k, 0);
    return (int)blockIdx.x + (int)gridDim.x * k;
  };
  if (tid == 0) s_next = kWarps;
  const uint4 *W = static_cast<const uint4 *>(p.w_down_l);
  const u64 pol_w = L2H ? l2_policy(true) : 0ull, pol_d = L2H ? l2_policy(false) : 0ull;
  auto ldw = [&](const uint4 *q) { return L2H ? ld_stream_hint(q, pol_w) : ld_stream(q); };
  auto ldd = [&](const uint4 *q) { return L2H ? ld_stream_hint(q, pol_d) : ld_stream(q); };

  // base task tt: rows r0 = 16·(tt / KC) (+g, +g+8) × vectors {8j + tq, 8j + 4 + tq} of K chunk tt % KC
  auto load_base = [&](uint4 (&buf)[4], int tt, int j) {
    const int rb = tt / KC, kc = tt - rb * KC, r = rb * 16 + g, v0 = kc * kMmaChunkVec + 8 * j + tq;
    const uint4 *q = W + (size_t)r * nvec + v0;
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    buf[0] = (r < dm && v0 < nvec) ? ldw(q) : z;
    buf[1] = (r < dm && v0 + 4 < nvec) ? ldw(q + 4) : z;
    buf[2] = (r + 8 < dm && v0 < nvec) ? ldw(q + 8 * (size_t)nvec) : z;
    buf[3] = (r + 8 < dm && v0 + 4 < nvec) ? ldw(q + 8 * (size_t)nvec + 4) : z;
  };
  // ΔW task: 4 × 32 lanes of one row
  auto load_delta = [&](uint4 (&buf)[4], const uint4 *rw, int v0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) buf[u] = v0 + 32 * u < nvec ? ldd(rw + v0 + 32 * u) : make_uint4(0u, 0u, 0u, 0u);
  };

  uint4 cur[4], nxt[4];
  const bool early = t < n_base;                  // base tasks read only W_down before the wait
  if (p.xtma && tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_xbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // r2: a warp whose first task is a ΔW row also requests its first batch before the wait. The
  // active-slot table and the slot bytes are written only by commit / WRITE / control kernels,
  // none of which triggers its dependents early (p.early_delta is cleared when the WRITE's early
  // trigger is switched on), so they completed before this grid was launched.
  const bool pre_delta = p.early_delta && !early && t < n_tasks;
  const uint4 *row = nullptr;
  if (early) load_base(cur, t, 0);
  else if (pre_delta) {
    const int td = t - n_base, m = td / dm, o = p.owner_idx[m];
    row = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.slots) +
                                          (2LL * o + p.sel[o]) * p.slot_elems + p.layer_off) +
          (size_t)(td - m * dm) * nvec;
    load_delta(cur, row, lane);
  }
  auto copy_x = [&]() {                           // the n x rows: one bulk copy each (no registers)
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_xbar), bytes = (uint32_t)dff * 2;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes * n) : "memory");
    for (int b = 0; b < n; ++b)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(xs + (size_t)b * nvp)),
                   "l"(static_cast<const __nv_bfloat16 *>(p.X) + (size_t)p.x_row[b] * dff), "r"(bytes), "r"(bar)
                   : "memory");
  };
  // inside tttstate_serve_step: once an earlier launch of the step has passed its PDL wait (it
  // publishes the step's epoch, below), X — an input of the whole step — is complete and visible,
  // so the bulk copies go out before this launch's wait (read_decode_tc.cu, p.x_epoch)
  bool x_early = false;
  if (p.xtma && p.x_epoch > 0 && tid == 0) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p.xflag) : "memory");
    if (v == p.x_epoch) {
      copy_x();
      x_early = true;
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p.x_epoch > 0 && blockIdx.x == 0 && tid == 0)
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.xflag), "r"(p.x_epoch) : "memory");
  if (tid <= n) {
    if (tid == 0) {
      s_row0[0] = W;
      if (p.xtma && !x_early) copy_x();
    } else {
      const int o = p.owner_idx[tid - 1];
      s_row0[tid] = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.slots) +
                                                    (2LL * o + p.sel[o]) * p.slot_elems + p.layer_off);
      if (FUSE)
        s_dst0[tid - 1] = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(const_cast<void *>(p.slots)) +
                                                    (2LL * o + 1 - p.sel[o]) * p.slot_elems + p.layer_off);
    }
  }
  __syncthreads();
  int v = lane;
  if (!early && t < n_tasks && !pre_delta) {
    const int td = t - n_base, m = td / dm;
    row = s_row0[m + 1] + (size_t)(td - m * dm) * nvec;
    load_delta(cur, row, v);
  }
  // x rows (zero pad / absent members): kXStage loads per thread in flight, then the stores;
  // p.xtma: only the zero padding here, the rows arrive by bulk copy
  if (p.xtma) {
    for (int idx = tid; idx < kMaxReadMembers * nvp; idx += kMmaThreads) {
      const int b = idx / nvp, vv = idx - b * nvp;
      if (b >= n || vv >= nvec) xs[idx] = make_uint4(0u, 0u, 0u, 0u);
    }
  }
  for (int base = p.xtma ? kMaxReadMembers * nvp : tid; base < kMaxReadMembers * nvp; base += kXStage * kMmaThreads) {
    uint4 tmp[kXStage];
#pragma unroll
    for (int e = 0; e < kXStage; ++e) {
      const int idx = base + e * kMmaThreads, b = idx / nvp, vv = idx - b * nvp;
      tmp[e] = (idx < kMaxReadMembers * nvp && b < n && vv < nvec)
                   ? reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.X) + (size_t)p.x_row[b] * dff)[vv]
                   : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int e = 0; e < kXStage; ++e)
      if (base + e * kMmaThreads < kMaxReadMembers * nvp) xs[base + e * kMmaThreads] = tmp[e];
  }
  {                                               // a4 — TailBufferUpdate, spread over every CTA
    const int zq = n * nvec, gtid = blockIdx.x * kMmaThreads + tid, gsz = gridDim.x * kMmaThreads;
    for (int idx = gtid; idx < zq; idx += gsz) {
      const int b = idx / nvec, vv = idx - b * nvec, o = p.owner_idx[b];
      reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.tailZ) + o * p.tz_owner + p.tz_layer +
                                (size_t)p.tail_pos[b] * dff)[vv] =
          reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.X) + (size_t)p.x_row[b] * dff)[vv];
    }
    for (int idx = gtid; idx < n * dm; idx += gsz) {
      const int b = idx / dm, ii = idx - b * dm, o = p.owner_idx[b];
      (static_cast<__nv_bfloat16 *>(p.tailV) + o * p.tv_owner + p.tv_layer + (size_t)p.tail_pos[b] * dm)[ii] =
          (static_cast<const __nv_bfloat16 *>(p.Vt) + (size_t)p.v_row[b] * dm)[ii];
    }
  }
  // base-first warps: the first task's second batch too, while the x rows are still arriving
  // (the registers the LDG/STS x staging used are free with the bulk copies)
  bool pre1 = PRE1 && p.xtma && early;
  if (pre1) load_base(nxt, t, 1);
  if (p.xtma)                                     // every thread observes the bulk copies' completion
    asm volatile("{\n\t.reg .pred P;\nXW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra XW_%=;\n}" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_xbar))
                 : "memory");
  __syncthreads();
  if (t >= n_tasks) return;

  const int target = n + KC;                      // arrivals per output row
  // y_b[i] = Σ_kc base partials + ΔW_b partial, in a fixed order: lane (grp, b) = (lane >> 3,
  // lane & 7) sums slots kc ≡ grp (mod 4) of member b (slot KC = the ΔW partial) with all its
  // loads in flight at once (one L2 round trip for KC ≤ 31), then two xor shuffles add the groups
  auto combine = [&](int i) {
    const int b = lane & 7, grp = lane >> 3;
    float y = 0.f;
    if (b < n) {
      for (int kc0 = grp; kc0 <= KC; kc0 += 32) {
        float part[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int kc = kc0 + 4 * e;
          part[e] = kc < KC ? __ldcg(p.Pbase + ((size_t)kc * kMaxReadMembers + b) * dm + i)
                            : (kc == KC ? __ldcg(p.Pdelta + (size_t)b * dm + i) : 0.f);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) y += part[e];
      }
    }
    y += __shfl_xor_sync(0xffffffffu, y, 8);
    y += __shfl_xor_sync(0xffffffffu, y, 16);
    if (lane < n) {
      if (p.resid) y += E::to_f(static_cast<const __nv_bfloat16 *>(p.resid)[(size_t)p.y_row[lane] * dm + i]);
      static_cast<__nv_bfloat16 *>(p.Y)[(size_t)p.y_row[lane] * dm + i] = E::from_f(y);
    }
    if (lane == 0) p.tickets[i] = 0;              // self-reset for the next launch
  };

  // ---- phase 1: base tasks (16 rows × 512 of K on mma.sync), batches double-buffered
  while (t < n_base) {
    const int rb = t / KC, kc = t - rb * KC, r0 = rb * 16;
    const int nb = min(8, (nvec - kc * kMmaChunkVec + 7) / 8);
    const uint4 *xg = xs + (size_t)g * nvp + kc * kMmaChunkVec + tq;
    float c[4] = {0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < nb; ++j) {
      if (j + 1 < nb && !(pre1 && j == 0)) load_base(nxt, t, j + 1);
      const uint4 b0 = xg[8 * j], b1 = xg[8 * j + 4];
      mma_bf16_16816(c, cur[0].x, cur[2].x, cur[0].y, cur[2].y, b0.x, b0.y);
      mma_bf16_16816(c, cur[0].z, cur[2].z, cur[0].w, cur[2].w, b0.z, b0.w);
      mma_bf16_16816(c, cur[1].x, cur[3].x, cur[1].y, cur[3].y, b1.x, b1.y);
      mma_bf16_16816(c, cur[1].z, cur[3].z, cur[1].w, cur[3].w, b1.z, b1.w);
#pragma unroll
      for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
    }
    pre1 = false;
    const int nt = next_task(t);                  // prefetch the next task's first batch
    if (nt < n_base) load_base(cur, nt, 0);
    else if (nt < n_tasks) {
      const int td = nt - n_base, m = td / dm;
      row = s_row0[m + 1] + (size_t)(td - m * dm) * nvec;
      load_delta(cur, row, lane);
    }
    // c0,c1: row r0+g, members 2tq, 2tq+1; c2,c3: row r0+g+8
    {
      const int r = r0 + g;
      float *P = p.Pbase + ((size_t)kc * kMaxReadMembers + 2 * tq) * dm;
      if (r < dm) {
        P[r] = c[0];
        P[dm + r] = c[1];
      }
      if (r + 8 < dm) {
        P[r + 8] = c[2];
        P[dm + r + 8] = c[3];
      }
    }
    __syncwarp();                                 // the warp's partials, then one release fence
    if (lane == 0) __threadfence();
    __syncwarp();
    int last = 0;
    if (lane < 16 && r0 + lane < dm) last = atomicAdd(p.tickets + r0 + lane, 1) == target - 1;
    unsigned mask = __ballot_sync(0xffffffffu, last);
    if (mask) __threadfence();
    while (mask) {
      const int l = __ffs(mask) - 1;
      mask &= mask - 1;
      combine(r0 + l);
    }
    t = nt;
  }
  if (t >= n_tasks) return;

  // ---- phase 2: ΔW rows (SIMT GEMVs, FHFMA). Plain batches: issue kDU 16-byte loads per
  // lane, then consume them. Measured faster than the register double buffer with
  // cross-task prefetch it replaced (76.7 vs 78.9 µs sustained, 0.90 vs 0.88 burst): with 32
  // warps per SM the other warps already hide a batch's latency, and the simpler loop keeps
  // registers (no spills) and instructions down.
  uint32_t expmax = 0;
  bool have_cur = true;                          // the first ΔW batch is preloaded (before x staging, or by the base phase)
  for (; t < n_tasks; t += stride) {
    const int td = t - n_base, m = td / dm, i = td - m * dm;
    const uint4 *rw = s_row0[m + 1] + (size_t)i * nvec;
    const uint4 *xb = xs + (size_t)m * nvp;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    float ev = 0.f;
    uint4 *drow = nullptr;
    if (FUSE) {
      ev = E::to_f(static_cast<const __nv_bfloat16 *>(p.Vt)[(size_t)p.v_row[m] * dm + i]);
      drow = s_dst0[m] + (size_t)i * nvec;
    }
    for (int v0 = lane; v0 < nvec; v0 += 32 * kDU) {
      uint4 w[kDU];
      if (have_cur) {                            // (kDU == 4: the preloaded batch is this one)
#pragma unroll
        for (int u = 0; u < kDU; ++u) w[u] = cur[u & 3];
        have_cur = false;
      } else {
#pragma unroll
        for (int u = 0; u < kDU; ++u)
          w[u] = v0 + 32 * u < nvec ? ldd(rw + v0 + 32 * u) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < kDU; ++u) E::dot(acc[u & 3], w[u], xb[v0 + 32 * u]);
      if (FUSE) {
#pragma unroll
        for (int u = 0; u < kDU; ++u)
          if (v0 + 32 * u < nvec) __stcs(drow + v0 + 32 * u, Upd<__nv_bfloat16>::apply(w[u], xb[v0 + 32 * u], ev, p.eta, expmax));
      }
    }
    float sum = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (lane == 0) p.Pdelta[(size_t)m * dm + i] = sum;
    if (FUSE) {                                  // per-member device failure flag (device-side App. H)
      if (Upd<__nv_bfloat16>::bad(expmax)) atomicOr(p.mfail + p.owner_idx[m], 1);
      expmax = 0;
    }
    __syncwarp();
    int old = 0;
    if (lane == 0) {
      __threadfence();
      old = atomicAdd(p.tickets + i, 1);
    }
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old == target - 1) {
      __threadfence();
      combine(i);
    }
  }
}

size_t smem_bytes(int n, int d_ff, int esize) { return (size_t)n * d_ff * esize; }

template <typename T, int TH, int U, bool FUSE>
cudaError_t launch_cfg1(const ReadParams &p, cudaStream_t s) {
  const size_t smem = smem_bytes(p.n, p.d_ff, sizeof(T));
  static int configured = -1;
  if ((int)smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(read_decode_kernel<T, TH, U, FUSE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 * 1024));
    if (e != cudaSuccess) return e;
    configured = (int)smem;
  }
  static const bool pdl = !getenv("TTT_PDL") || atoi(getenv("TTT_PDL")) != 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(device_sm_count());
  cfg.blockDim = dim3(TH);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static const int order = getenv("TTT_READ_ORDER") ? atoi(getenv("TTT_READ_ORDER")) : 1;
  static const int xtma = getenv("TTT_READ_XTMA") ? atoi(getenv("TTT_READ_XTMA")) : 1;
  ReadParams q = p;
  q.order = order;
  q.xtma = xtma;
  cudaError_t e = cudaLaunchKernelEx(&cfg, read_decode_kernel<T, TH, U, FUSE>, q);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <typename T, int TH, int U>
cudaError_t launch_cfg(const ReadParams &p, cudaStream_t s) {
  return p.fuse ? launch_cfg1<T, TH, U, true>(p, s) : launch_cfg1<T, TH, U, false>(p, s);
}

int read_cfg() {
  static int cfg = -1;
  if (cfg < 0) {
    const char *e = getenv("TTT_READ_CFG");
    cfg = e ? atoi(e) : 0;
  }
  return cfg;
}

template <typename T>
cudaError_t launch_t(const ReadParams &p, cudaStream_t s) {
  // the fused C = 1 READ + WRITE (f3) streams two row sets per task (read + candidate store):
  // 3 loads per lane per batch measured best for it (87 % vs 85 % of HBM with 4)
  if (read_cfg() == 0 && p.fuse) return launch_cfg<T, 1024, 3>(p, s);
  switch (read_cfg()) {
    case 1: return launch_cfg<T, 1024, 3>(p, s);
    case 2: return launch_cfg<T, 1024, 2>(p, s);
    case 3: return launch_cfg<T, 768, 5>(p, s);
    case 4: return launch_cfg<T, 640, 6>(p, s);
    case 5: return launch_cfg<T, 896, 4>(p, s);
    default: return launch_cfg<T, 1024, 4>(p, s);
  }
}

}  // namespace

bool read_decode_fits(int n, int d_model, int d_ff, int esize) {
  (void)d_model;
  return smem_bytes(n, d_ff, esize) <= 220 * 1024;
}

namespace {
template <bool FUSE, bool L2H>
cudaError_t launch_mma(const ReadParams &p, cudaStream_t s) {
  const size_t smem = (size_t)kMaxReadMembers * mma_nvp(p.d_ff / 8) * 16;
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(read_decode_mma_kernel<FUSE, L2H, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 * 1024));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(read_decode_mma_kernel<FUSE, L2H, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)std::max<size_t>(smem, 48 * 1024));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  static const bool pre1 = !getenv("TTT_READ_PRE1") || atoi(getenv("TTT_READ_PRE1")) != 0;
  static const bool pdl = !getenv("TTT_PDL") || atoi(getenv("TTT_PDL")) != 0;
  static const int order = getenv("TTT_READ_ORDER") ? atoi(getenv("TTT_READ_ORDER")) : 1;
  static const int dyn = getenv("TTT_READ_DYN") ? atoi(getenv("TTT_READ_DYN")) : 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(device_sm_count());
  cfg.blockDim = dim3(kMmaThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static const int xtma = getenv("TTT_READ_XTMA") ? atoi(getenv("TTT_READ_XTMA")) : 1;
  static const int early_delta = getenv("TTT_READ_EARLY_DELTA") ? atoi(getenv("TTT_READ_EARLY_DELTA")) : 1;
  ReadParams q = p;
  q.order = order;
  q.dyn = order == 1 ? dyn : 0;
  q.xtma = xtma;
  q.early_delta = early_delta && !write_tc_triggers_early();
  cudaError_t e = pre1 ? cudaLaunchKernelEx(&cfg, read_decode_mma_kernel<FUSE, L2H, true>, q)
                       : cudaLaunchKernelEx(&cfg, read_decode_mma_kernel<FUSE, L2H, false>, q);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

int read_decode_mma_chunks(int dtype, int d_ff) {
  static const bool on = !getenv("TTT_READ_MMA") || atoi(getenv("TTT_READ_MMA")) != 0;
  if (!on || dtype != 1 || d_ff % 8) return 0;
  if ((size_t)kMaxReadMembers * mma_nvp(d_ff / 8) * 16 > 220 * 1024) return 0;
  return (d_ff / 8 + kMmaChunkVec - 1) / kMmaChunkVec;
}

cudaError_t launch_read_decode(int dtype, const ReadParams &p, cudaStream_t s) {
  static const int l2keep = getenv("TTT_READ_L2KEEP") ? atoi(getenv("TTT_READ_L2KEEP")) : 1;
  static const int persist_mb = getenv("TTT_L2_PERSIST_MB") ? atoi(getenv("TTT_L2_PERSIST_MB")) : 0;
  static bool limit_set = false;
  if (persist_mb > 0 && !limit_set) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)persist_mb << 20);
    limit_set = true;
  }
  // the TMA + tcgen05 READ for every bf16 group (bench.py config 2: 68.8 vs 75.7-76.9 µs).  Groups
  // split over several launches (configs 3 / 5) kept the SIMT kernel while the TMA READ stopped at
  // the PDL wait (0.81 / 0.80 vs 0.84 / 0.83 of the roofline); with its producer streaming past the
  // wait it is faster there too: 0.883 / 0.865 vs 0.853 / 0.841 (TTT_READ_TC_MULTI=0: SIMT for them)
  static const int tc_multi = getenv("TTT_READ_TC_MULTI") ? atoi(getenv("TTT_READ_TC_MULTI")) : 1;
  if (p.kc > 0 && !p.fuse && (!p.l2keep || tc_multi) && p.ptc && read_decode_tc_supported(p.n, p.d_model, p.d_ff)) {
    static const int early_delta = getenv("TTT_READ_EARLY_DELTA") ? atoi(getenv("TTT_READ_EARLY_DELTA")) : 1;
    ReadParams q = p;
    q.early_delta = early_delta && !write_tc_triggers_early();
    const cudaError_t e = launch_read_decode_tc(q, s);   // TMA + tcgen05 (read_decode_tc.cu)
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();                            // no plan for this shape: the SIMT kernel below
  }
  if (p.kc > 0) {
    if (p.l2keep && l2keep) return p.fuse ? launch_mma<true, true>(p, s) : launch_mma<false, true>(p, s);
    return p.fuse ? launch_mma<true, false>(p, s) : launch_mma<false, false>(p, s);
  }
  if (dtype == 1) return launch_t<__nv_bfloat16>(p, s);
  return launch_t<float>(p, s);
}

}  // namespace ttt
