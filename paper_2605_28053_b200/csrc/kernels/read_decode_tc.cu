// a3 + a4 — decode READ on TMA + tcgen05 (bf16, up to 8 members per launch).
//
// PAPER: READ = ApplyState + ReturnOutputs (Table 3, §4.2): for every
// member b of a legal READ group, y_b = x_b·(W_down[l] + ΔW_b[l])ᵀ, the committed slot chosen
// by the device active-slot table, the pool never written; TailBufferUpdate appends (z_t, v_t)
// (P:382-385).  Same operation as read_decode.cu's kernels; this one moves the bytes
// differently.
//
// Why: the operation is a pure HBM stream (448.7 MB per launch at 8 members, AI ≈ 2).  A probe
// of TMA tensor boxes into a shared-memory ring (tools/tma_tensor_probe.cu, r2) streams that
// volume at 6.80–6.83 TB/s with two warps per SM when the boxes are dealt evenly, vs ~6.0 TB/s
// for the 1024-thread register-batch kernel, whose warps run out of rows at different times.
// So: every weight byte arrives as a 128-row × 64-column box (16 KB, 128-byte swizzle) and the
// tensor core does the products — the weight rows are the MMA's A operand (M = 128) and the
// members' x rows its B operand (N = 16: the 8 member rows, rows 8..15 aliased onto them by a
// zero stride), accumulating D[128 rows × 16] in TMEM.  For a ΔW_b box only column b of D is
// wanted (15/16 of that MMA is thrown away — a few % of the tensor pipe, irrelevant next to the
// HBM stream).
//
// Work split: the 1+n matrices (W_down, ΔW_0 … ΔW_{n-1}) × ⌈d_model/128⌉ row blocks are dealt
// round-robin to G groups of g CTAs; CTA `sub` of a group streams K blocks [sub·nkb/g,
// (sub+1)·nkb/g) of each of its group's row blocks, so its slice of the x rows is staged in shared
// memory once.  plan_g picks g to minimise the busiest CTA's boxes, then the smallest x slice
// (most ring stages) and most SMs: at paper dims g = 7, G = 21 (147 CTAs, ≤ 9 row blocks × 22 K blocks).
// Each (row block, K slice) partial goes to a workspace slab; the last of the (1+n)·g arrivals
// for an output row block (per-row-block ticket) sums, in a fixed order, Σ_slices W-partial[b] +
// Σ_slices ΔW_b-partial (+ resid) → bf16 y (deterministic).  Warps: 0 TMA producer (lane 0),
// 1 MMA issuer (lane 0), 2–5 x staging / tail append / epilogue (tcgen05.ld) / combine.  TMEM:
// per row block 4 accumulators of 16 columns (one per K = 16 step of a box, summed in order in
// the epilogue), double-buffered (row block k in k & 1).
//
// Ring stages hold bps = 3 boxes (48 KB) with ONE tcgen05.commit per stage: with a commit per
// 16-KB box the launch took 82.8–97.7 µs (each commit → slot release round trip throttled the
// stream; ncu tensor pipe 3.8 %, so not MMA throughput); 2 / 3 / 4 boxes per stage: 77.6 / 76.6 /
// 78.3 µs in tools/microbench.py.  In bench.py (the 36-layer decode window) it beats the SIMT
// kernel read_decode_mma_kernel: 74.0–74.3 vs 74.7–76.9 µs per launch on power-capped boxes,
// 73.9 µs = 0.929 of HBM at full clock, so it is the default bf16 decode READ for
// groups that fit one launch (≤ 8 members).  Groups split over several launches (configs 3 / 5)
// kept the SIMT kernel (faster there) until the producer streamed past the PDL wait (below); now
// this kernel serves them too (0.883 / 0.865 vs 0.853 / 0.841 of the roofline).  TTT_READ_TC=0
// restores the SIMT kernel everywhere, TTT_READ_TC_MULTI=0 for multi-launch groups; fp32 pools
// and the fused C = 1 READ+WRITE always use it.
//
// Early x (inside tttstate_serve_step): a launch whose step epoch is already published
// stages its x slice before the PDL wait, and the MMA warp never waits (shared memory → TMEM
// only), so the preloaded ring drains while the previous launch finishes: 72.6 µs = 0.945 of HBM
// in bench.py on a power-capped 1,770 MHz box (3,022 vs 2,946 tok/s without it, same box).
//
// Run-ahead: the producer does not stop at the PDL wait once its ring is full — W_down is never
// written and ΔW slots only by kernels that never trigger early (p.early_delta) — so it streams on
// while the MMA warp fills both TMEM buffers; only the epilogue's global writes wait.  72.5 → 68.8
// µs per launch (3,020 → 3,186 tok/s); with the g = 7 plan 68.5 µs = the measured HBM copy peak
// (TTT_READ_TC_RUNAHEAD=0: stop at the wait).
//
// TTT_READ_TC_HYB = h (opt-in, measured not kept): warps 6–9 stream the CTA's last h ΔW row blocks
// through registers next to the TMA ring (more bytes in flight per SM).  h = 1 / 2 / 3: 74.8 / 76.6 /
// 87.4 µs per launch vs 74.2–75.4 default on the same box — the launch is DRAM-rate bound here.
#include <algorithm>
#include <mutex>
#include <cstdio>
#include <cstdlib>

#include "../internal.h"
#include "sm100_ptx.cuh"

namespace ttt {
namespace {

using namespace ptx;

constexpr int kTcThreads = 192;
constexpr int kHybWarps = 4;                       // TTT_READ_TC_HYB: register-streaming ΔW warps (6..9)
constexpr int kHybRows = 4;                        // rows per warp batch (all their loads in flight)
constexpr int kHybLd = 5;                          // 16-B loads per lane per row (K slice ≤ 5·32·8 elements)
constexpr int kTcBK = 64;                          // K elements per box (128 B rows)
constexpr int kTcBoxBytes = 128 * kTcBK * 2;       // 16 KB
constexpr int kTcMaxStages = 12;
#ifndef TTT_TC_COMBINE_BATCH
#define TTT_TC_COMBINE_BATCH 8
#endif
constexpr int kCombineBatch = TTT_TC_COMBINE_BATCH;   // K slices whose partials one combine round trip loads

struct DecTcParams {
  int n, d_model, d_ff, L, layer;
  int g, G, nkb, nrb, n_mat, stages;
  int l2keep;
  const int *sel;
  const void *X, *Vt, *resid;
  void *Y;
  void *tailZ, *tailV;
  long long tz_owner, tv_owner, tz_layer, tv_layer;
  float *Pw;                     // [g][nrb·128][8]   W_down partials per K slice
  float *Pd;                     // [g][nrb·128][8]   ΔW_b partials (column b of record b)
  int *tickets;                  // [nrb] arrivals per output row block (self-resetting)
  int owner_idx[kMaxReadMembers], x_row[kMaxReadMembers], v_row[kMaxReadMembers], y_row[kMaxReadMembers];
  int tail_pos[kMaxReadMembers];
  int trace;                     // TTT_READ_TC_TRACE=1: per-CTA %globaltimer stamps printed at exit
  int pre;                       // W boxes requested before the PDL wait
  int nomma;                     // diagnostic: release ring slots without MMAs (wrong results)
  int bps;                       // boxes per ring stage (one commit per stage)
  int early_delta;               // ΔW boxes may be requested before the PDL wait (slot-table writers never trigger early)
  int hyb;                       // the CTA's last `hyb` ΔW row blocks go to register-streaming warps, not TMA
  const __nv_bfloat16 *slots;    // slot array (the tmD tensor: [n_slot_layers][d_model][d_ff])
  int *xflag;                    // serve_step epoch word (ReadParams::xflag)
  int x_epoch;                   // > 0: inside tttstate_serve_step
  int runahead;                  // producer streams past the ring fill before the PDL wait (early_delta only)
};

template <int ID, int COUNT>
__device__ __forceinline__ void named_bar() {
  asm volatile("barrier.sync %0, %1;" ::"n"(ID), "n"(COUNT) : "memory");
}
// 32 lanes × 8 consecutive 32-bit TMEM columns
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kTcThreads + 32 * kHybWarps, 1)
    read_decode_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmD,
                          const DecTcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages, g = p.g, grp = blockIdx.x / g, sub = blockIdx.x - grp * g;
  const int kb_lo = sub * p.nkb / g, kb_hi = (sub + 1) * p.nkb / g, nkq = kb_hi - kb_lo;
  unsigned char *xs = smem + (size_t)S * p.bps * kTcBoxBytes;  // [nkq][8 rows][128 B] swizzled x slice
  u64 *bars = reinterpret_cast<u64 *>(xs + (size_t)nkq * 1024);
  u64 *full = bars, *empty = bars + kTcMaxStages, *t_full = bars + 2 * kTcMaxStages, *t_empty = t_full + 2;
  u64 *x_ready = t_empty + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(x_ready + 1);
  __shared__ int s_last, s_last_h, s_xe;
  __shared__ unsigned long long ts[7];
  auto stamp = [&](int i) {
    if (p.trace) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[i] = t;
    }
  };
  if (threadIdx.x == 0) stamp(0);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_rb = p.n_mat * p.nrb;                              // row blocks over all matrices
  const int my_rbs = grp < p.G ? (n_rb - grp + p.G - 1) / p.G : 0;
  auto rb_of = [&](int k, int &m, int &rbi) {                    // k-th row block of this group
    const int r = grp + k * p.G;
    m = r / p.nrb;
    rbi = r - m * p.nrb;
  };
  // hybrid split: the last h row blocks (ΔW only) are streamed by warps 6.. through registers
  int h = 0;
  while (h < p.hyb && h + 1 < my_rbs && (grp + (my_rbs - 1 - h) * p.G) / p.nrb > 0) ++h;
  const int kt = my_rbs - h;                                     // row blocks through TMA + tcgen05

  // combine output row block rbi (fixed order), by the 128 threads t of the last-arriving group
  auto combine = [&](const int rbi, const int t) {
    const int rows_pad = p.nrb * 128, dm = p.d_model, n = p.n;
    __threadfence();
    const int i = rbi * 128 + t;
    if (i < dm) {
      // y_b = Σ_slices W-partial[b] + Σ_slices ΔW_b-partial, slices ascending; the loads of
      // kCombineBatch slices are issued together (one L2 round trip at the g = 8 plan)
      float w[8], d[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) w[e] = d[e] = 0.f;
      for (int s0 = 0; s0 < g; s0 += kCombineBatch) {
        float4 lw[kCombineBatch][2], ld[kCombineBatch][2];
#pragma unroll
        for (int u = 0; u < kCombineBatch; ++u) {
          const bool ok = s0 + u < g;
          const float4 *pw = reinterpret_cast<const float4 *>(p.Pw + ((size_t)(s0 + u) * rows_pad + i) * 8);
          const float4 *pd = reinterpret_cast<const float4 *>(p.Pd + ((size_t)(s0 + u) * rows_pad + i) * 8);
          const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
          lw[u][0] = ok ? __ldcg(pw) : z;
          lw[u][1] = ok ? __ldcg(pw + 1) : z;
          ld[u][0] = ok ? __ldcg(pd) : z;
          ld[u][1] = ok ? __ldcg(pd + 1) : z;
        }
#pragma unroll
        for (int u = 0; u < kCombineBatch; ++u) {
          if (s0 + u >= g) break;
          w[0] += lw[u][0].x; w[1] += lw[u][0].y; w[2] += lw[u][0].z; w[3] += lw[u][0].w;
          w[4] += lw[u][1].x; w[5] += lw[u][1].y; w[6] += lw[u][1].z; w[7] += lw[u][1].w;
          d[0] += ld[u][0].x; d[1] += ld[u][0].y; d[2] += ld[u][0].z; d[3] += ld[u][0].w;
          d[4] += ld[u][1].x; d[5] += ld[u][1].y; d[6] += ld[u][1].z; d[7] += ld[u][1].w;
        }
      }
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        if (b >= n) break;
        float y = w[b] + d[b];
        if (p.resid)
          y += __bfloat162float(static_cast<const __nv_bfloat16 *>(p.resid)[(size_t)p.y_row[b] * dm + i]);
        static_cast<__nv_bfloat16 *>(p.Y)[(size_t)p.y_row[b] * dm + i] = __float2bfloat16_rn(y);
      }
    }
    if (t == 0) p.tickets[rbi] = 0;                         // self-reset for the next launch
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(t_full + i, 1);
      mbar_init(t_empty + i, 4);
    }
    mbar_init(x_ready, 128);                          // every warp-2..5 thread
    mbar_init_fence();
  }
  if (warp == 1) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  asm volatile("griddepcontrol.launch_dependents;");

  if (warp == 0) {
    if (lane == 0 && my_rbs > 0) {                          // ---------------- TMA producer
      tma_prefetch(&tmW);
      tma_prefetch(&tmD);
      const u64 pol_w = p.l2keep ? policy_evict_last() : 0ull;
      int it = 0;
      // W_down is never written by any kernel: this group's W boxes may be requested before the
      // PDL wait (ΔW boxes need the slot table, written by commits)
      bool waited = false;
      for (int k = 0; k < kt; ++k) {
        int m, rbi;
        rb_of(k, m, rbi);
        int coord2 = p.layer;
        if (m > 0) {
          if (!waited && !p.early_delta) {                  // (see read_decode.cu: p.early_delta)
            asm volatile("griddepcontrol.wait;" ::: "memory");
            waited = true;
          }
          const int o = p.owner_idx[m - 1];
          coord2 = (2 * o + p.sel[o]) * p.L + p.layer;
        }
        for (int kb = kb_lo; kb < kb_hi; kb += p.bps, ++it) {   // a stage = bps boxes (consecutive K blocks)
          const int s = it % S, nb = min(p.bps, kb_hi - kb);
          if (it >= p.pre || it >= S) {
            // (pre-wait prefetch budget used: wait now — unless nothing this producer loads can be
            // written by an earlier grid: W_down never, ΔW slots only by kernels that never
            // trigger early (p.early_delta); TTT_READ_TC_RUNAHEAD=0 keeps the wait)
            if (!waited && !(p.runahead && p.early_delta)) {
              asm volatile("griddepcontrol.wait;" ::: "memory");
              waited = true;
            }
            if (it >= S) mbar_wait(empty + s, ((it / S) - 1) & 1);
          }
          mbar_expect_tx(full + s, (uint32_t)nb * kTcBoxBytes);
          for (int i = 0; i < nb; ++i) {
            unsigned char *dst = smem + ((size_t)s * p.bps + i) * kTcBoxBytes;
            if (m == 0) {
              if (p.l2keep) tma_load_3d_hint(dst, &tmW, full + s, (kb + i) * kTcBK, rbi * 128, 0, pol_w);
              else tma_load_3d(dst, &tmW, full + s, (kb + i) * kTcBK, rbi * 128, 0);
            } else {
              tma_load_3d(dst, &tmD, full + s, (kb + i) * kTcBK, rbi * 128, coord2);
            }
          }
        }
      }
      if (!waited && !(p.runahead && p.early_delta)) asm volatile("griddepcontrol.wait;" ::: "memory");
    }
  } else if (warp == 1) {                                   // ---------------- MMA issuer
    // (reads only this CTA's shared memory and writes TMEM: no PDL wait; x_ready gates it)
    if (my_rbs > 0) {
      mbar_wait(x_ready, 0);
      if (lane == 0) stamp(1);
      tc_fence_after();
      // N = 16: B rows 8..15 alias rows 0..7 (SBO = 0), i.e. D columns 8..15 repeat 0..7 (unused)
      const uint32_t idesc = idesc_bf16(128, 16, 0, 0);
      const uint32_t xb0 = smem_u32(xs);
      int it = 0;
      for (int k = 0; k < kt; ++k) {
        const uint32_t acc = tmem + (uint32_t)((k & 1) * 64);   // 4 accumulators of 16 columns (one per K=16 step)
        if (k >= 2) {
          mbar_wait(t_empty + (k & 1), ((k >> 1) - 1) & 1);
          tc_fence_after();
        }
        for (int kb = kb_lo; kb < kb_hi; kb += p.bps, ++it) {
          const int s = it % S, nb = min(p.bps, kb_hi - kb);
          const bool last = kb + nb >= kb_hi;
          mbar_wait(full + s, (it / S) & 1);
          tc_fence_after();
          if (lane == 0 && p.nomma) {                       // diagnostic (TTT_READ_TC_NOMMA): stream only
            mbar_arrive(empty + s);
            if (last) mbar_arrive(t_full + (k & 1));
          } else if (lane == 0) {
            for (int i = 0; i < nb; ++i) {
              const uint32_t a0 = smem_u32(smem + ((size_t)s * p.bps + i) * kTcBoxBytes);
              const uint32_t b0 = xb0 + (uint32_t)(kb + i - kb_lo) * 1024;
#pragma unroll
              for (int kk = 0; kk < kTcBK / 16; ++kk)
                mma_bf16(acc + kk * 16, smem_desc_sw128(a0 + kk * 32, 16, 1024), smem_desc_sw128(b0 + kk * 32, 16, 0),
                         idesc, (kb > kb_lo || i > 0) ? 1u : 0u);
            }
            mma_commit(empty + s);
            if (last) mma_commit(t_full + (k & 1));
          }
          __syncwarp();
        }
      }
    }
  } else if (warp < 6) {                                    // ---------------- warps 2-5
    const int q = warp & 3, et = threadIdx.x - 64;
    // Inside tttstate_serve_step X is an input of the whole step (written before the call, never
    // during it).  Once an earlier launch of this step has passed its PDL wait — it publishes the
    // step's epoch in *xflag below — everything that wrote X has completed and is visible, so this
    // launch stages its x slice before its own wait, while the previous launch drains, instead of
    // after it with the ring already full.  Otherwise (the step's first launch, read_apply) the x
    // loads follow the wait.
    bool xe = false;
    if (p.x_epoch > 0) {
      if (et == 0) {
        int v;
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p.xflag) : "memory");
        s_xe = v == p.x_epoch;
      }
      named_bar<1, 128>();
      xe = s_xe;
    }
    if (!xe) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 64) stamp(5);
    const int n = p.n, dff = p.d_ff, dm = p.d_model;
    if (my_rbs > 0) {
      // x slice → shared memory, K-major 128-byte-swizzled 8-row atoms: 16-B chunk c of row r in
      // atom kbl at kbl·1024 + r·128 + ((c ^ r)·16); rows n..7 zero.  Plain 16-B loads, all of a
      // thread's chunks in flight at once (one round trip; TMA one-row boxes took ~9 µs here: a
      // fixed cost per tiny box), then fence.proxy.async so the MMA (async proxy) sees them.
      constexpr int kXPer = 24;
      const int chunks = nkq * 64;
      for (int i0 = et; i0 < chunks; i0 += 128 * kXPer) {
        uint4 v[kXPer];
#pragma unroll
        for (int u = 0; u < kXPer; ++u) {
          const int i = i0 + u * 128, kbl = i >> 6, r = (i >> 3) & 7, c = i & 7;
          const int kel = (kb_lo + kbl) * kTcBK + c * 8;
          v[u] = make_uint4(0u, 0u, 0u, 0u);
          if (i < chunks && r < n && kel < dff)
            v[u] = *reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.X) + (size_t)p.x_row[r] * dff +
                                                    kel);
        }
#pragma unroll
        for (int u = 0; u < kXPer; ++u) {
          const int i = i0 + u * 128, kbl = i >> 6, r = (i >> 3) & 7, c = i & 7;
          if (i < chunks) *reinterpret_cast<uint4 *>(xs + (size_t)kbl * 1024 + r * 128 + ((c ^ r) << 4)) = v[u];
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes → MMA (async proxy)
      mbar_arrive(x_ready);
    }
    if (xe) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p.x_epoch > 0 && blockIdx.x == 0 && et == 0)        // this launch is past its wait: publish
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.xflag), "r"(p.x_epoch) : "memory");
    {                                                       // a4 — TailBufferUpdate, spread over every CTA
      const int zq = n * (dff / 8), gtid = blockIdx.x * 128 + et, gsz = gridDim.x * 128;
      for (int idx = gtid; idx < zq; idx += gsz) {
        const int b = idx / (dff / 8), vv = idx - b * (dff / 8), o = p.owner_idx[b];
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
    const int rows_pad = p.nrb * 128;
    for (int k = 0; k < kt; ++k) {
      int m, rbi;
      rb_of(k, m, rbi);
      mbar_wait(t_full + (k & 1), (k >> 1) & 1);
      if (et == 0 && k == 0) stamp(2);
      tc_fence_after();
      uint32_t r[8];
      {   // the 4 independent accumulator chains (a dependent chain of N = 16 MMAs was latency-bound),
          // summed in a fixed order
        const uint32_t t0 = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((k & 1) * 64);
        uint32_t r1[8], r2[8], r3[8];
        tmem_ld8(t0, r);
        tmem_ld8(t0 + 16, r1);
        tmem_ld8(t0 + 32, r2);
        tmem_ld8(t0 + 48, r3);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          r[e] = __float_as_uint(((__uint_as_float(r[e]) + __uint_as_float(r1[e])) + __uint_as_float(r2[e])) +
                                 __uint_as_float(r3[e]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(t_empty + (k & 1));
      const int row = rbi * 128 + q * 32 + lane;           // < rows_pad; rows ≥ d_model are zero boxes
      if (m == 0) {                                         // W_down partial: all 8 member columns
        float4 *d4 = reinterpret_cast<float4 *>(p.Pw + ((size_t)sub * rows_pad + row) * 8);
        __stcg(d4, make_float4(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]), __uint_as_float(r[3])));
        __stcg(d4 + 1, make_float4(__uint_as_float(r[4]), __uint_as_float(r[5]), __uint_as_float(r[6]), __uint_as_float(r[7])));
      } else {                                              // ΔW_b partial: column b only, same record layout
        const int b = m - 1;
        float v = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (e == b) v = __uint_as_float(r[e]);
        __stcg(p.Pd + ((size_t)sub * rows_pad + row) * 8 + b, v);
      }
      named_bar<1, 128>();                                  // the row block's partials are stored
      if (et == 0) {
        __threadfence();
        s_last = atomicAdd(p.tickets + rbi, 1) == p.n_mat * g - 1;
      }
      named_bar<1, 128>();
      if (s_last) combine(rbi, et);                         // output row block rbi (fixed order)
    }
  } else if (h > 0) {                                       // ---------------- warps 6..: hybrid ΔW rows
    // The CTA's last h ΔW row blocks, K slice [kb_lo, kb_hi), streamed through registers (16-B
    // loads, kHybRows rows × kHybLd loads per lane in flight) next to the TMA ring, so the SM has the
    // ring's and the registers' bytes in flight at once; products against the swizzled x slice in
    // shared memory, a fixed-order warp reduction, then the same partial record, ticket and
    // combine as the tcgen05 epilogue.
    const int hw = warp - 6, ht = threadIdx.x - kTcThreads;
    const int rows_pad = p.nrb * 128, dff = p.d_ff, kel0 = kb_lo * kTcBK, klen = min(nkq * kTcBK, dff - kel0);
    const int nch = klen >> 3;                                // 16-B chunks in the K slice
    if (!p.early_delta) asm volatile("griddepcontrol.wait;" ::: "memory");
    bool xwait = true;
    for (int j = 0; j < h; ++j) {
      int m, rbi;
      rb_of(kt + j, m, rbi);
      const int b = m - 1, o = p.owner_idx[b];
      const __nv_bfloat16 *base = p.slots + ((size_t)((2 * o + p.sel[o]) * p.L + p.layer) * p.d_model) * dff + kel0;
      for (int r0 = hw * kHybRows; r0 < 128; r0 += kHybWarps * kHybRows) {
        uint4 v[kHybRows][kHybLd];
#pragma unroll
        for (int rr = 0; rr < kHybRows; ++rr) {
          const int row = rbi * 128 + r0 + rr;
#pragma unroll
          for (int u = 0; u < kHybLd; ++u) {
            const int c = lane + 32 * u;
            v[rr][u] = make_uint4(0u, 0u, 0u, 0u);
            if (row < p.d_model && c < nch) v[rr][u] = __ldcs(reinterpret_cast<const uint4 *>(base + (size_t)row * dff) + c);
          }
        }
        if (xwait) {
          asm volatile("griddepcontrol.wait;" ::: "memory");
          mbar_wait(x_ready, 0);
          xwait = false;
        }
        float acc[kHybRows];
#pragma unroll
        for (int rr = 0; rr < kHybRows; ++rr) acc[rr] = 0.f;
#pragma unroll
        for (int u = 0; u < kHybLd; ++u) {
          const int c = lane + 32 * u;
          if (c < nch) {
            const uint4 xv = *reinterpret_cast<const uint4 *>(xs + (size_t)(c >> 3) * 1024 + b * 128 + (((c & 7) ^ b) << 4));
            const __nv_bfloat162 *x2 = reinterpret_cast<const __nv_bfloat162 *>(&xv);
#pragma unroll
            for (int rr = 0; rr < kHybRows; ++rr) {
              const __nv_bfloat162 *w2 = reinterpret_cast<const __nv_bfloat162 *>(&v[rr][u]);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 wf = __bfloat1622float2(w2[e]), xf = __bfloat1622float2(x2[e]);
                acc[rr] = fmaf(wf.x, xf.x, acc[rr]);
                acc[rr] = fmaf(wf.y, xf.y, acc[rr]);
              }
            }
          }
        }
#pragma unroll
        for (int rr = 0; rr < kHybRows; ++rr) {
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) acc[rr] += __shfl_xor_sync(0xffffffffu, acc[rr], off);
          const int row = rbi * 128 + r0 + rr;
          if (lane == 0) __stcg(p.Pd + ((size_t)sub * rows_pad + row) * 8 + b, acc[rr]);
        }
      }
      named_bar<2, 32 * kHybWarps>();                       // the row block's partials are stored
      if (ht == 0) {
        __threadfence();
        s_last_h = atomicAdd(p.tickets + rbi, 1) == p.n_mat * g - 1;
      }
      named_bar<2, 32 * kHybWarps>();
      if (s_last_h) combine(rbi, ht);
    }
    if (xwait) asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (threadIdx.x == 64) stamp(3);
  tc_fence_before();
  __syncwarp();
  __syncthreads();
  if (warp == 1) tmem_dealloc<128>(tmem);
  if (p.trace && threadIdx.x == 0) {
    stamp(4);
    printf("DTC %d %llu %llu %llu %llu %llu %d %llu\n", (int)blockIdx.x, ts[0], ts[1], ts[2], ts[3], ts[4], p.layer,
           ts[5]);
  }
}

// g (CTAs per row block): first the K blocks of the busiest CTA, ⌈rbs / G⌉ · ⌈nkb / g⌉, are
// minimised; then, among the g within 5 % of that minimum whose ring is as deep as any (a box's
// slot is held until its MMAs complete, so bytes in flight = ring − slots in MMA), the one that
// streams on the most SMs (G · g).  Since the producer streams past the PDL wait, consecutive
// launches overlap and a CTA that finishes early starts the next launch's boxes, so the SMs in use
// count more than the last CTA of one launch: at paper dims g = 7 (147 SMs, busiest CTA 198
// boxes) measured 3,194–3,198 tok/s vs 3,152 for g = 8 (144 SMs, 190 boxes), g = 5 / 6 3,174–3,190;
// g = 10 / 12 (row blocks of 16 / 13 boxes: the per-row-block epilogue no longer hides) 2,824–2,942.
int plan_g(int n_rb, int nkb, int sms, int *G_out, int *stages_out) {
  static const int st_env = getenv("TTT_READ_TC_STAGES") ? atoi(getenv("TTT_READ_TC_STAGES")) : kTcMaxStages;
  const int gmax = std::min({sms, nkb, kTcMaxG});                  // (kTcMaxG: the partials workspace)
  auto stages_of = [&](int g) {
    const int nkq = (nkb + g - 1) / g;
    return std::min(st_env, (int)((227 * 1024 - 4096 - (size_t)nkq * 1024) / kTcBoxBytes));
  };
  auto cost_of = [&](int g) { const int G = sms / g; return ((n_rb + G - 1) / G) * ((nkb + g - 1) / g); };
  int best_cost = 1 << 30, best_st = 0;
  for (int g = 1; g <= gmax; ++g)
    if (stages_of(g) >= 4) best_cost = std::min(best_cost, cost_of(g));
  if (best_cost == 1 << 30) return 0;
  for (int g = 1; g <= gmax; ++g)
    if (stages_of(g) >= 4 && cost_of(g) * 100 <= best_cost * 105) best_st = std::max(best_st, stages_of(g));
  int best = 0, best_used = 0, best_c = 1 << 30;
  for (int g = 1; g <= gmax; ++g) {
    if (stages_of(g) != best_st || cost_of(g) * 100 > best_cost * 105) continue;
    const int G = sms / g, used = std::min(G, n_rb) * g, c = cost_of(g);
    if (used > best_used || (used == best_used && c < best_c)) {
      best = g;
      best_used = used;
      best_c = c;
    }
  }
  *G_out = sms / best;
  *stages_out = best_st;
  return best;
}

}  // namespace

bool read_decode_tc_supported(int n, int d_model, int d_ff) {
  static const int on = getenv("TTT_READ_TC") ? atoi(getenv("TTT_READ_TC")) : 1;   // TTT_READ_TC=0: the SIMT kernel
  return on && n >= 1 && n <= kMaxReadMembers && d_model >= 128 && d_ff % 8 == 0 && d_ff >= kTcBK &&
         ptx::encode_fn() != nullptr;
}

cudaError_t launch_read_decode_tc(const ReadParams &rp, cudaStream_t s) {
  DecTcParams p{};
  p.n = rp.n; p.d_model = rp.d_model; p.d_ff = rp.d_ff; p.L = rp.L; p.layer = rp.layer;
  p.nkb = (rp.d_ff + kTcBK - 1) / kTcBK;
  p.nrb = (rp.d_model + 127) / 128;
  p.n_mat = 1 + rp.n;
  const int sms = device_sm_count();
  static const int bps = getenv("TTT_READ_TC_BPS") ? std::max(1, std::min(4, atoi(getenv("TTT_READ_TC_BPS")))) : 3;
  p.bps = bps;
  // host fast path (r2: this launch cost 19.3 µs of host time vs 13.9 for the SIMT kernel): the
  // plan and both tensor maps are memoised per (layer's W_down, slot array, shape, group size)
  struct Memo {
    const void *w, *slots;
    long long nsl;
    int n, dm, dff, g, G, stages;
    CUtensorMap mW, mD;
  };
  static Memo memo[64];
  static std::mutex memo_mu;
  const size_t h = ((size_t)rp.layer * 8 + (size_t)rp.n) & 63;   // (layers' W_down are 64 · 4 KB multiples apart)
  Memo hit{};
  bool have = false;
  {
    std::lock_guard<std::mutex> lock(memo_mu);
    const Memo &m = memo[h];
    if (m.w == rp.w_down_l && m.slots == rp.slots && m.nsl == rp.n_slot_layers && m.n == rp.n && m.dm == rp.d_model &&
        m.dff == rp.d_ff && m.g > 0) {
      hit = m;
      have = true;
    }
  }
  if (have) {
    p.g = hit.g;
    p.G = hit.G;
    p.stages = hit.stages;
  } else {
    p.g = plan_g(p.n_mat * p.nrb, p.nkb, sms, &p.G, &p.stages);
    p.stages = std::max(2, p.stages / bps);
  }
  static const int g_env = getenv("TTT_READ_TC_G") ? atoi(getenv("TTT_READ_TC_G")) : 0;
  if (g_env > 0 && g_env <= std::min(sms, kTcMaxG)) {   // tuning override
    p.g = g_env;
    p.G = sms / g_env;
    const int nkq_e = (p.nkb + p.g - 1) / p.g;
    p.stages = std::max(2, std::min(kTcMaxStages, (int)((227 * 1024 - 4096 - (size_t)nkq_e * 1024) / kTcBoxBytes)) / bps);
  }
  // no plan for this shape: cudaErrorNotSupported, and launch_read_decode runs the SIMT kernel
  if (p.g == 0 || (size_t)p.g * p.nrb * 128 * 8 * 2 * sizeof(float) > rp.ptc_bytes) return cudaErrorNotSupported;
  p.l2keep = rp.l2keep;
  p.early_delta = rp.early_delta;
  static const int trace = getenv("TTT_READ_TC_TRACE") ? atoi(getenv("TTT_READ_TC_TRACE")) : 0;
  p.trace = trace;
  static const int pre = getenv("TTT_READ_TC_PRE") ? atoi(getenv("TTT_READ_TC_PRE")) : 1 << 20;
  p.pre = pre;
  static const int nomma = getenv("TTT_READ_TC_NOMMA") ? atoi(getenv("TTT_READ_TC_NOMMA")) : 0;
  p.nomma = nomma;
  static const int hyb = getenv("TTT_READ_TC_HYB") ? atoi(getenv("TTT_READ_TC_HYB")) : 0;
  p.hyb = ((p.nkb + p.g - 1) / p.g) * kTcBK <= kHybLd * 32 * 8 ? hyb : 0;   // (K slice within the warps' loads)
  p.slots = static_cast<const __nv_bfloat16 *>(rp.slots);
  p.xflag = rp.xflag;
  static const int runahead = getenv("TTT_READ_TC_RUNAHEAD") ? atoi(getenv("TTT_READ_TC_RUNAHEAD")) : 1;
  p.runahead = runahead;
  p.x_epoch = rp.xflag ? rp.x_epoch : 0;
  p.sel = rp.sel;
  p.X = rp.X; p.Vt = rp.Vt; p.resid = rp.resid; p.Y = rp.Y;
  p.tailZ = rp.tailZ; p.tailV = rp.tailV;
  p.tz_owner = rp.tz_owner; p.tv_owner = rp.tv_owner; p.tz_layer = rp.tz_layer; p.tv_layer = rp.tv_layer;
  p.Pw = rp.ptc;
  p.Pd = rp.ptc + (size_t)p.g * p.nrb * 128 * 8;
  p.tickets = rp.tickets;
  for (int b = 0; b < rp.n; ++b) {
    p.owner_idx[b] = rp.owner_idx[b];
    p.x_row[b] = rp.x_row[b];
    p.v_row[b] = rp.v_row[b];
    p.y_row[b] = rp.y_row[b];
    p.tail_pos[b] = rp.tail_pos[b];
  }
  CUtensorMap mW, mD;
  if (have) {
    mW = hit.mW;
    mD = hit.mD;
  } else {
    if (!cached_map(&mW, rp.w_down_l, rp.d_ff, rp.d_model, 1, kTcBK, 128) ||
        !cached_map(&mD, rp.slots, rp.d_ff, rp.d_model, (uint64_t)rp.n_slot_layers, kTcBK, 128))
      return cudaErrorInvalidValue;
    if (g_env == 0) {
      std::lock_guard<std::mutex> lock(memo_mu);
      memo[h] = Memo{rp.w_down_l, rp.slots, rp.n_slot_layers, rp.n, rp.d_model, rp.d_ff, p.g, p.G, p.stages, mW, mD};
    }
  }
  const int nkq = (p.nkb + p.g - 1) / p.g;
  const size_t smem = 1024 + (size_t)p.stages * p.bps * kTcBoxBytes + (size_t)nkq * 1024 + (2 * kTcMaxStages + 6) * 8 + 16;
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(read_decode_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  static const bool pdl = !getenv("TTT_PDL") || atoi(getenv("TTT_PDL")) != 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(kTcThreads + (p.hyb > 0 ? 32 * kHybWarps : 0));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, read_decode_tc_kernel, mW, mD, p);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace ttt
