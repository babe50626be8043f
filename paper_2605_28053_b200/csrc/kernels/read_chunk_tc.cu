// NEXT f2 — chunk-granular READ (prefill / long-context state build) on tcgen05.
//
// PAPER: a request's READ steps inside one TTT chunk all observe the same
// committed version v (READ "keeps version", Table 3; the version
// changes only at commit), so the C tokens of a chunk can be applied
// as one matrix product before the boundary WRITE (chunk boundaries "every
// C_ttt generated tokens"; prefill builds the state the decode
// trace starts from, 32K/64K contexts P:601-602):
//     Y_b[t, :] = z_t · (W_down[l] + ΔW_b[l])ᵀ,   t = 0 .. C-1, all at version v,
// and the chunk's (z_t, v_t) are appended to the owner's tail.  This is the one
// regime where READ is a dense contraction (AI ≈ 4·C·E / (2.25·E·2) ≈ 227
// flop/B at C=128 with 8 owners sharing W_down), so it runs on
// tensor cores: TN GEMM M = C (tokens), N = d_model, K = d_ff, A = X_b (K-major),
// B = W_down[l] and B' = ΔW_b[l] (both K-major rows of the weight), two MMAs
// per K=16 step into ONE fp32 TMEM accumulator — W + ΔW is never rounded.
//  * 1 persistent CTA per SM, tiles (member, N-block); N-blocks have two widths
//    (w_hi, w_hi−16 ≤ 160) chosen so the tiles fill the 148 SMs (d_model 2560 × 8
//    members: 18 blocks per member = 16 × 144 + 2 × 128 → 144 CTAs instead of 128);
//  * warp 0 TMA producer (4-stage ring of X / W / ΔW 64-wide K blocks, 128 B
//    swizzle), warp 1 TMEM alloc + single-thread MMA issue, warps 2-5
//    epilogue (tcgen05.ld → bf16 → Y); during the mainloop the epilogue warps
//    of each of a member's N-tiles append 1/nt of the chunk to the tail.
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "../internal.h"
#include "sm100_ptx.cuh"

namespace ttt {
namespace {

using namespace ptx;

constexpr int BM = 128, BK = 64, kStages = 4;
#ifndef TTT_LR_STAGES
#define TTT_LR_STAGES 4
#endif
// fused low-rank READ ring depth (r2: 3 stages — a smaller shared-memory carveout, more L1 for
// the u-warps' register streams — measured R = 16 31.3 vs 30.1 µs, R = 64 54.5 vs 54.4 µs)
constexpr int kStagesLR = TTT_LR_STAGES;
constexpr int kThreads = 192;
#ifndef TTT_LR_UW
#define TTT_LR_UW 16
#endif
constexpr int kUW = TTT_LR_UW;                    // fused low-rank mode: u = A x warps per CTA
constexpr int kThreadsLR = kThreads + 32 * kUW;
#ifndef TTT_LR_UB
#define TTT_LR_UB 12
#endif
constexpr int kUB = TTT_LR_UB;                    // fused low-rank: 16-byte loads of A per lane per batch

// fused low-rank READ (NEXT f1) extras: the u = A x stream, the tail append and the finish
// y = Σ_ks Y32 + Bᵀu (+ resid) run inside the base-GEMM launch (one launch per layer)
struct LrFused {
  const void *slots;
  long long slot_elems, layer_off;
  int R;
  const void *Xsrc, *resid;
  void *Yout;
  float *u;                      // [n][R]
  float *bu;                     // [n][d_model] Bᵀu per member (fp32)
  int *ctr;                      // [0] members whose Bᵀu is done, [1] CTAs exited, [2..] slab tickets per (row block, N block)
  const int *x_row, *v_row, *y_row, *tail_pos;   // device member table (MemberTable rows 1-4)
};

struct ChunkParams {
  int n, d_model, d_ff, C, L, layer;
  const int *sel;
  const void *X, *Vt;
  void *Y;
  void *tailZ, *tailV;
  long long tz_owner, tv_owner, tz_layer, tv_layer;
  int delta, append, valid_rows, ksplit;
  int nt, w_hi, h;               // N blocks per member; blocks j < h are w_hi wide, the rest w_hi - 16
  float *Y32;
  long long y32_slab;
  int x_rowmap;                  // X map is [rows][d_ff]: row block b starts at row x_row0 + 128·b
  int x_row0;
  int cooperative;               // LR: launch cooperatively (co-residency guaranteed)
  int trace;                     // LR: TTT_LR_PRINT=1 prints per-CTA %globaltimer phase stamps (profiling)
  int early_dep;                 // PDL: trigger the dependent launch at entry (TTT_CHUNK_EARLY_DEP)
  const int *owner_idx;          // device member table row 0
  LrFused lr;
  int *xflag;                    // LR inside tttstate_serve_step: epoch word (ReadParams::xflag)
  int x_epoch;                   //   > 0: X rows may be read before the PDL wait once published
};

__device__ __forceinline__ uint4 ld_stream(const uint4 *q) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(q));
  return r;
}
__device__ __forceinline__ void fma_bf16x2(float &acc, uint32_t a, uint32_t z) {
  asm("{\n\t.reg .b16 al, ah, zl, zh;\n\t"
      "mov.b32 {al, ah}, %1;\n\tmov.b32 {zl, zh}, %2;\n\t"
      "fma.rn.f32.bf16 %0, al, zl, %0;\n\tfma.rn.f32.bf16 %0, ah, zh, %0;\n}"
      : "+f"(acc)
      : "r"(a), "r"(z));
}
// named barrier among a subset of warps (non-.aligned form: callers may arrive diverged,
// e.g. after the single spinning thread of the finish gate)
template <int ID, int COUNT>
__device__ __forceinline__ void named_bar() {
  asm volatile("barrier.sync %0, %1;" ::"n"(ID), "n"(COUNT) : "memory");
}
__device__ __forceinline__ int ld_volatile(const int *q) {
  int v;
  asm volatile("ld.volatile.global.b32 %0, [%1];" : "=r"(v) : "l"(q));
  return v;
}

// f1 finish, run by the 4 epilogue warps + the kUW u warps of the CTA after named barrier 2:
// y = Σ_ks Y32[ks] + Bᵀu (+ resid) for this tile's columns and its 1/KS share of the rows,
// 8 outputs per item with the R loads of u and B issued 8 at a time.
template <int BN>
__device__ __forceinline__ void lr_finish(const ChunkParams &p, int b, int j, int ks, int n0, int width, int ft) {
  named_bar<2, 128 + 32 * kUW>();
  const LrFused &lr = p.lr;
  const int KS = p.ksplit;
  const int rows = min(BM, p.valid_rows - b * BM), r_lo = rows * ks / KS, r_hi = rows * (ks + 1) / KS;
  const int cpr = width / 8, items = (r_hi - r_lo) * cpr, dm = p.d_model;
  for (int itm = ft; itm < items; itm += 128 + 32 * kUW) {
    const int rr = b * BM + r_lo + itm / cpr, c = n0 + 8 * (itm % cpr);
    float y[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) y[e] = 0.f;
    for (int q0 = 0; q0 < KS; q0 += 4) {           // fixed slab order, 4 slabs' loads in flight
      float4 lo[4], hi[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q0 + q < KS) {
          const float4 *s4 = reinterpret_cast<const float4 *>(p.Y32 + (q0 + q) * p.y32_slab + (size_t)rr * dm + c);
          lo[q] = __ldcg(s4);
          hi[q] = __ldcg(s4 + 1);
        } else {
          lo[q] = hi[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        y[0] += lo[q].x; y[1] += lo[q].y; y[2] += lo[q].z; y[3] += lo[q].w;
        y[4] += hi[q].x; y[5] += hi[q].y; y[6] += hi[q].z; y[7] += hi[q].w;
      }
    }
    {                                              // + Bᵀu (computed by the member's u warps)
      const float4 *b4 = reinterpret_cast<const float4 *>(lr.bu + (size_t)rr * dm + c);
      const float4 lo = __ldcg(b4), hi = __ldcg(b4 + 1);
      y[0] += lo.x; y[1] += lo.y; y[2] += lo.z; y[3] += lo.w; y[4] += hi.x; y[5] += hi.y; y[6] += hi.z; y[7] += hi.w;
    }
    if (lr.resid) {
      const uint4 rv = *reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(lr.resid) +
                                                        (size_t)lr.y_row[rr] * dm + c);
      const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        y[2 * h] += __uint_as_float(w[h] << 16);
        y[2 * h + 1] += __uint_as_float(w[h] & 0xffff0000u);
      }
    }
    uint32_t out[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      __nv_bfloat162 h2 = __floats2bfloat162_rn(y[2 * h], y[2 * h + 1]);
      out[h] = *reinterpret_cast<uint32_t *>(&h2);
    }
    *reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(lr.Yout) + (size_t)lr.y_row[rr] * dm + c) =
        make_uint4(out[0], out[1], out[2], out[3]);
  }
}

template <int BN, bool LR>   // BN: largest N-block (smem stage size); actual widths are runtime
__global__ void __launch_bounds__(LR ? kThreadsLR : kThreads, 1)
    read_chunk_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                         const __grid_constant__ CUtensorMap tmD, const ChunkParams p) {
  constexpr int kTmemCols = BN <= 128 ? 128 : 256;
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;   // stage slots sized for BN rows
  const uint32_t b_box = (uint32_t)p.w_hi * BK * 2;                   // bytes one B box actually lands
  constexpr uint32_t STAGE = A_BYTES + (LR ? 1 : 2) * B_BYTES;      // low-rank base mode has no ΔW box
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kStages = LR ? kStagesLR : ::ttt::kStages;          // ring depth of this mode
  u64 *bars = reinterpret_cast<u64 *>(smem + kStages * STAGE);
  u64 *full = bars, *empty = bars + kStages, *t_full = bars + 2 * kStages, *t_empty = t_full + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(t_empty + 1);
  uint4 *xs_lr = reinterpret_cast<uint4 *>(smem + kStages * STAGE + 512);   // LR: one member's x row
  float *us_lr = reinterpret_cast<float *>(smem + kStages * STAGE + 256);   // LR: u_m = A_m x_m (≤ 64)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = p.nt, nk_all = p.d_ff / BK, KS = p.ksplit;
  __shared__ unsigned long long ts[8];              // LR profiling stamps (p.trace)
  auto stamp = [&](int i) {
    if (LR && p.trace) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[i] = t;
    }
  };
  if (threadIdx.x == 0) stamp(0);
  auto n0_of = [&](int j) { return j < p.h ? j * p.w_hi : p.h * p.w_hi + (j - p.h) * (p.w_hi - 16); };
  auto width_of = [&](int j) { return j < p.h ? p.w_hi : p.w_hi - 16; };
  const int n_tiles = p.n * nt * KS;
  // tile u -> (member / row block b, N block j, K range ks)
  auto decode = [&](int u, int &b, int &j, int &kb0, int &kb1) {
    const int ks = u % KS, bj = u / KS;
    b = bj / nt;
    j = bj - b * nt;
    kb0 = nk_all * ks / KS;
    kb1 = nk_all * (ks + 1) / KS;
  };

  // LR inside tttstate_serve_step (read_decode_tc.cu, x_epoch): once an earlier launch of the step
  // has passed its PDL wait and published the step's epoch, X is complete and visible, and the
  // slot table, member table and low-rank state are written only by kernels that never trigger
  // their dependents early — so the producer (X, W_down boxes), the MMA warp (shared memory →
  // TMEM) and the u warps' x staging and u = A x (shared memory) run before this launch's wait;
  // every global write (tail, slabs, Bᵀu, counters) stays behind it.
  __shared__ int s_xe;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(t_full, 1);
    mbar_init(t_empty, 4);
    mbar_init_fence();
    int v = 0;
    if (LR && p.x_epoch > 0) asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p.xflag) : "memory");
    s_xe = LR && p.x_epoch > 0 && v == p.x_epoch;
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const bool xe = s_xe != 0;
  // PDL: the prologue above (barriers, TMEM, tensor-map prefetch) overlaps the previous
  // kernel's tail; everything below may depend on it (X, slots, sel, workspace, counters).
  if (p.early_dep) asm volatile("griddepcontrol.launch_dependents;");
  // low-rank launch: W_down is never written by any kernel, so the first tile's first W boxes
  // are requested before the wait and stream while the previous kernel drains (X, the slot
  // table and the rest after it): -1 % per layer at R = 16 / 64; the chunk READ measured
  // 1.5-2 % slower with it, so it keeps the plain order
  int npre = 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmW);
    tma_prefetch(&tmD);
  }
  if (LR && warp == 0 && lane == 0 && (int)blockIdx.x < n_tiles) {
    int b, j, kb0, kb1;
    decode(blockIdx.x, b, j, kb0, kb1);
    npre = min(kStages, kb1 - kb0);
    for (int i = 0; i < npre; ++i) {
      mbar_expect_tx(full + i, A_BYTES + (p.delta ? 2 : 1) * b_box);
      tma_load_3d(smem + i * STAGE + A_BYTES, &tmW, full + i, (kb0 + i) * BK, n0_of(j), p.layer);
    }
  }
  if (!xe) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) stamp(1);

  if (warp == 0) {
    if (lane == 0) {                                        // ---------------- TMA producer
      int it = 0;
      for (int u = blockIdx.x; u < n_tiles; u += gridDim.x) {
        int b, j, kb0, kb1;
        decode(u, b, j, kb0, kb1);
        const int o = p.delta ? p.owner_idx[b] : 0;
        const int slot_l = p.delta ? (2 * o + p.sel[o]) * p.L + p.layer : 0;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % kStages;
          if (it >= kStages) mbar_wait(empty + s, ((it / kStages) - 1) & 1);
          unsigned char *st = smem + s * STAGE;
          const bool pre = it < npre;                       // W box (and the expect) already issued
          if (!pre) mbar_expect_tx(full + s, A_BYTES + (p.delta ? 2 : 1) * b_box);
          if (p.x_rowmap) tma_load_3d(st, &tmX, full + s, kb * BK, p.x_row0 + b * BM, 0);
          else tma_load_3d(st, &tmX, full + s, kb * BK, 0, b);
          if (!pre) tma_load_3d(st + A_BYTES, &tmW, full + s, kb * BK, n0_of(j), p.layer);
          if (p.delta) tma_load_3d(st + A_BYTES + B_BYTES, &tmD, full + s, kb * BK, n0_of(j), slot_l);
        }
      }
    }
  } else if (warp == 1) {                                   // ---------------- MMA issuer
    int it = 0, k = 0;
    for (int u = blockIdx.x; u < n_tiles; u += gridDim.x, ++k) {
      int b, j, kb0, kb1;
      decode(u, b, j, kb0, kb1);
      const uint32_t idesc = idesc_bf16(BM, width_of(j), 0, 0);
      if (k > 0) mbar_wait(t_empty, (k - 1) & 1);
      tc_fence_after();
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % kStages;
        mbar_wait(full + s, (it / kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a0 = smem_u32(smem + s * STAGE);
          const uint32_t w0 = a0 + A_BYTES, d0 = w0 + B_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {        // K=16 step = 32 bytes inside the 128 B swizzle row
            const u64 ad = smem_desc_sw128(a0 + kk * 32, 16, 1024);
            mma_bf16(tmem, ad, smem_desc_sw128(w0 + kk * 32, 16, 1024), idesc, ((kb - kb0) | kk) ? 1u : 0u);
            if (p.delta) mma_bf16(tmem, ad, smem_desc_sw128(d0 + kk * 32, 16, 1024), idesc, 1u);
          }
          mma_commit(empty + s);
          if (kb == kb1 - 1) mma_commit(t_full);
        }
        __syncwarp();
      }
    }
    if (lane == 0) stamp(2);                                // last MMA issued
  } else if (warp < 6) {                                    // ---------------- epilogue warps 2-5
    const int q = warp & 3, row = q * 32 + lane;            // token index t in the chunk
    const int et = threadIdx.x - 64;
    if (xe) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (LR && p.x_epoch > 0 && blockIdx.x == 0 && et == 0)  // past this launch's wait: publish
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.xflag), "r"(p.x_epoch) : "memory");
    int k = 0;
    for (int u = blockIdx.x; u < n_tiles; u += gridDim.x, ++k) {
      int b, j, kb0, kb1;
      decode(u, b, j, kb0, kb1);
      const int ks = u % KS;
      if (p.append) {                                        // a4: tile j appends slice j of the chunk to the tail
        const int o = p.owner_idx[b];
        auto copy_slice = [&](const uint4 *src, uint4 *dst, size_t total) {
          const size_t lo = total * j / nt, hi = total * (j + 1) / nt;
          size_t v = lo + et;
          for (; v + 3 * 128 < hi; v += 4 * 128) {           // 4 independent 16-B loads in flight per thread
            const uint4 a0 = src[v], a1 = src[v + 128], a2 = src[v + 256], a3 = src[v + 384];
            dst[v] = a0; dst[v + 128] = a1; dst[v + 256] = a2; dst[v + 384] = a3;
          }
          for (; v < hi; v += 128) dst[v] = src[v];
        };
        copy_slice(reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.X) + (size_t)b * p.C * p.d_ff),
                   reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.tailZ) + o * p.tz_owner + p.tz_layer),
                   (size_t)p.C * p.d_ff / 8);
        copy_slice(reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.Vt) + (size_t)b * p.C * p.d_model),
                   reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.tailV) + o * p.tv_owner + p.tv_layer),
                   (size_t)p.C * p.d_model / 8);
      }
      mbar_wait(t_full, k & 1);
      tc_fence_after();
      const int n0 = n0_of(j), width = width_of(j);
      __nv_bfloat16 *yrow = static_cast<__nv_bfloat16 *>(p.Y) + ((size_t)b * p.C + row) * p.d_model + n0;
      float *yrow32 = p.Y32 ? p.Y32 + ks * p.y32_slab + ((size_t)b * p.C + row) * p.d_model + n0 : nullptr;
      const bool valid = row < p.C && (!p.Y32 || b * p.C + row < p.valid_rows);
      // f1 split-K slab (fp32): each lane's tcgen05.ld row is transposed through shared memory
      // (the TMA ring is idle once the single tile's MMAs retired) so a warp store writes 8 rows ×
      // 64 contiguous bytes instead of 32 rows × 16 bytes (trace r2: this epilogue took 3.5 µs, now
      // 2.1; R = 16 31.6 -> 29.4 µs per layer, R = 64 56.3 -> 54.2; 32-column steps measured 30.8 µs)
      float *stg = LR ? reinterpret_cast<float *>(smem) + q * (32 * 17) : nullptr;
#pragma unroll 1
      for (int c = 0; c < width / 16; ++c) {      // 16 accumulator columns at a time
        uint32_t r[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 16), r);
        if (LR && yrow32) {
#pragma unroll
          for (int e = 0; e < 16; ++e) stg[lane * 17 + e] = __uint_as_float(r[e]);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rr = i * 8 + (lane >> 2), c4 = (lane & 3) * 4, grow = b * p.C + q * 32 + rr;
            if (q * 32 + rr < p.C && grow < p.valid_rows) {
              const float *sp = stg + rr * 17 + c4;
              *reinterpret_cast<float4 *>(p.Y32 + ks * p.y32_slab + (size_t)grow * p.d_model + n0 + c * 16 + c4) =
                  make_float4(sp[0], sp[1], sp[2], sp[3]);
            }
          }
          __syncwarp();
        } else if (valid && yrow32) {
          float4 *d4 = reinterpret_cast<float4 *>(yrow32 + c * 16);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            d4[v] = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]), __uint_as_float(r[4 * v + 2]),
                                __uint_as_float(r[4 * v + 3]));
        } else if (valid) {
          uint32_t o8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
            o8[e] = *reinterpret_cast<uint32_t *>(&h2);
          }
          uint4 *dst = reinterpret_cast<uint4 *>(yrow + c * 16);
          dst[0] = make_uint4(o8[0], o8[1], o8[2], o8[3]);
          dst[1] = make_uint4(o8[4], o8[5], o8[6], o8[7]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(t_empty);
      if (LR) {                                    // f1: arm the finish of this tile
        named_bar<1, 128>();                       // this CTA's slab is written
        if (et == 0) stamp(3);
        if (et == 0) {
          int *tick = p.lr.ctr + 2 + b * nt + j;
          __threadfence();
          atomicAdd(tick, 1);
          while (ld_volatile(tick) < KS) __nanosleep(64);            // every K slab of the tile
          while (ld_volatile(p.lr.ctr) < p.valid_rows) __nanosleep(64);   // every member's Bᵀu
          __threadfence();
          stamp(6);
        }
        lr_finish<BN>(p, b, j, ks, n0, width, et);   // with the u warps (named barrier 2)
      }
    }
  } else if (LR) {                                          // ---------------- u = A x warps (f1)
    // CTA c owns members c, c + grid, ...: x_m staged in shared memory once, the kUW warps
    // stream the R rows of A_m (8 × 16-byte loads per lane in flight), then append (z, v).
    const LrFused &lr = p.lr;
    const int uw = warp - 6, ut = uw * 32 + lane, R = lr.R, dff = p.d_ff, dm = p.d_model, nvec = dff / 8;
    for (int m = blockIdx.x; m < p.valid_rows; m += gridDim.x) {
      const int o = p.owner_idx[m];
      const uint4 *x4 = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(lr.Xsrc) +
                                                        (size_t)lr.x_row[m] * dff);
      uint4 *tz = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.tailZ) + o * p.tz_owner + p.tz_layer +
                                            (size_t)lr.tail_pos[m] * dff);
      named_bar<3, 32 * kUW>();   // previous member's rows done
      auto append_v = [&]() {                        // a4: append v_m
        const uint4 *vs = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.Vt) +
                                                          (size_t)lr.v_row[m] * dm);
        uint4 *tv = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.tailV) + o * p.tv_owner + p.tv_layer +
                                              (size_t)lr.tail_pos[m] * dm);
        for (int v = ut; v < dm / 8; v += 32 * kUW) tv[v] = vs[v];
      };
      for (int v = ut; v < nvec; v += 32 * kUW) {    // stage x_m; a4: append z_m (after the wait if xe)
        const uint4 z = x4[v];
        xs_lr[v] = z;
        if (!xe) tz[v] = z;
      }
      if (!xe) append_v();
      named_bar<3, 32 * kUW>();   // x_m staged
      const __nv_bfloat16 *A = static_cast<const __nv_bfloat16 *>(lr.slots) + (2LL * o + p.sel[o]) * lr.slot_elems +
                               lr.layer_off;
      for (int k = uw; k < R; k += kUW) {
        const uint4 *a4 = reinterpret_cast<const uint4 *>(A + (size_t)k * dff);
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int v = lane; v < nvec; v += 32 * kUB) {
          uint4 a[kUB];
#pragma unroll
          for (int q = 0; q < kUB; ++q) a[q] = v + 32 * q < nvec ? ld_stream(a4 + v + 32 * q) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
          for (int q = 0; q < kUB; ++q) {
            if (v + 32 * q < nvec) {
              const uint4 z = xs_lr[v + 32 * q];
              float &ac = acc[q & 3];
              fma_bf16x2(ac, a[q].x, z.x); fma_bf16x2(ac, a[q].y, z.y);
              fma_bf16x2(ac, a[q].z, z.z); fma_bf16x2(ac, a[q].w, z.w);
            }
          }
        }
        float sum = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
        if (lane == 0) us_lr[k] = sum;
      }
      named_bar<3, 32 * kUW>();   // u_m complete (shared memory)
      if (ut == 0) stamp(4);
      if (xe) asm volatile("griddepcontrol.wait;" ::: "memory");   // global writes from here on: behind the wait
      // Bᵀu_m: 8 outputs per thread, the R rows of B_m streamed 8 loads at a time
      const uint4 *B4 = reinterpret_cast<const uint4 *>(A + (size_t)R * dff);
      for (int i8 = ut; i8 < dm / 8; i8 += 32 * kUW) {
        float y[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) y[e] = 0.f;
        for (int k0 = 0; k0 < R; k0 += 8) {
          uint4 bv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            bv[q] = k0 + q < R ? ld_stream(B4 + (size_t)(k0 + q) * (dm / 8) + i8) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float uk = k0 + q < R ? us_lr[k0 + q] : 0.f;
            const uint32_t w[4] = {bv[q].x, bv[q].y, bv[q].z, bv[q].w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              y[2 * h] = fmaf(uk, __uint_as_float(w[h] << 16), y[2 * h]);
              y[2 * h + 1] = fmaf(uk, __uint_as_float(w[h] & 0xffff0000u), y[2 * h + 1]);
            }
          }
        }
        float4 *o4 = reinterpret_cast<float4 *>(lr.bu + (size_t)m * dm + 8 * i8);
        o4[0] = make_float4(y[0], y[1], y[2], y[3]);
        o4[1] = make_float4(y[4], y[5], y[6], y[7]);
      }
      named_bar<3, 32 * kUW>();   // Bᵀu_m written
      if (ut == 0) stamp(5);
      if (ut == 0) {
        __threadfence();
        atomicAdd(lr.ctr, 1);
      }
      if (xe) {                                      // a4 appends, off the u -> Bᵀu -> gate chain
        for (int v = ut; v < nvec; v += 32 * kUW) tz[v] = xs_lr[v];
        append_v();
      }
    }
    int b, j, kb0, kb1;                            // this CTA's (single) tile
    decode(blockIdx.x, b, j, kb0, kb1);
    lr_finish<BN>(p, b, j, blockIdx.x % KS, n0_of(j), width_of(j), 128 + uw * 32 + lane);
  }
  tc_fence_before();
  __syncwarp();                                    // warp 0: the producer lane rejoins its warp
  __syncthreads();
  if (warp == 1) tmem_dealloc<kTmemCols>(tmem);
  if (LR && p.trace && threadIdx.x == 0) {
    stamp(7);
    printf("LRT %d %llu %llu %llu %llu %llu %llu %llu %llu %d\n", (int)blockIdx.x, ts[0], ts[1], ts[2], ts[3], ts[4],
           ts[5], ts[6], ts[7], p.layer);
  }
  if (LR && threadIdx.x == 0) {                    // the last CTA out re-arms the counters
    __threadfence();
    if (atomicAdd(p.lr.ctr + 1, 1) == (int)gridDim.x - 1) {
      p.lr.ctr[0] = 0;
      for (int g = 0; g < p.n * nt; ++g) p.lr.ctr[2 + g] = 0;
      __threadfence();
      p.lr.ctr[1] = 0;
    }
  }
}

template <int BN, bool LR>
size_t smem_bytes(int d_ff) {   // LR: stages without the ΔW box, plus one x row
  return 1024 + (size_t)(LR ? kStagesLR : kStages) * (BM * BK * 2 + (LR ? 1 : 2) * BN * BK * 2) + 256 +
         (LR ? 256 + (size_t)d_ff * 2 : 0);
}

template <int BN, bool LR>
cudaError_t launch_bn(const CUtensorMap &mX, const CUtensorMap &mW, const CUtensorMap &mD, const ChunkParams &p,
                      cudaStream_t s) {
  const size_t smem = smem_bytes<BN, LR>(p.d_ff);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(read_chunk_tc_kernel<BN, LR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  const int tiles = p.n * p.nt * p.ksplit;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min(device_sm_count(), tiles));
  cfg.blockDim = dim3(LR ? kThreadsLR : kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  // the fused low-rank launch spin-waits across CTAs: a cooperative launch makes the driver
  // guarantee that every CTA is co-resident (also against other streams' kernels)
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (LR && p.cooperative) ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, read_chunk_tc_kernel<BN, LR>, mX, mW, mD, p);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

// N-block plan: T blocks per member of widths w_hi (h of them) and w_hi - 16, w_hi ≤ 160,
// minimising waves × per-tile smem traffic (A 128 rows + two B blocks of w_hi rows).
struct NPlan {
  int T = 0, w_hi = 0, h = 0;
};
NPlan plan_n(int d_model, int tiles_per_block_unit, int sms) {
  NPlan best;
  double best_cost = 1e30;
  for (int T = (d_model + 159) / 160; T <= d_model / 16; ++T) {
    const int w_hi = ((d_model + T - 1) / T + 15) / 16 * 16;
    if (w_hi > 160 || w_hi < 16) continue;
    const int w_lo = w_hi - 16;
    int h = (d_model - T * w_lo) / 16;            // blocks of width w_hi
    if (T * w_lo + 16 * h != d_model || h < 0 || h > T) continue;
    if (w_lo == 0 && h < T) continue;
    const long long tiles = (long long)T * tiles_per_block_unit;
    const long long waves = (tiles + sms - 1) / sms;
    const double cost = (double)waves * (128 + 2 * w_hi);
    // equal cost: prefer more blocks while they still fit one wave (more SMs streaming)
    const bool more = cost < best_cost + 1e-9 && T > best.T && tiles <= sms;
    if (cost < best_cost - 1e-9 || more) {
      best_cost = std::min(best_cost, cost);
      best = {T, w_hi, h};
    }
  }
  return best;
}

}  // namespace

// Tensor-map encode cache (host): decode-time launches reuse the same handful of maps per
// layer, so encoding is done once per (base, dims, box).
bool cached_map(CUtensorMap *m, const void *base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
                int swizzle_bytes) {
  struct Entry {
    const void *base;
    uint64_t d0, d1, d2;
    uint32_t b0, b1;
    int sw;
    CUtensorMap map;
  };
  static Entry cache[128];
  static int n_used = 0, next = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < n_used; ++i) {
    const Entry &e = cache[i];
    if (e.base == base && e.d0 == d0 && e.d1 == d1 && e.d2 == d2 && e.b0 == b0 && e.b1 == b1 && e.sw == swizzle_bytes) {
      *m = e.map;
      return true;
    }
  }
  if (!ptx::make_map_bf16_3d(m, base, d0, d1, d2, b0, b1, swizzle_bytes)) return false;
  Entry &e = cache[next];
  e = Entry{base, d0, d1, d2, b0, b1, swizzle_bytes, *m};
  next = (next + 1) % 128;
  n_used = n_used < 128 ? n_used + 1 : 128;
  return true;
}

// fused low-rank READ needs every tile of the launch resident at once (one CTA per SM)
bool read_chunk_fused_fits(int row_blocks, int d_model, int ksplit) {
  const int sms = device_sm_count();
  const NPlan np = plan_n(d_model, row_blocks * std::max(1, ksplit), sms);
  return np.T > 0 && row_blocks * np.T * std::max(1, ksplit) <= sms;
}

bool read_chunk_supported(int d_model, int d_ff, int C) {
  return C >= 1 && C <= BM && d_ff % BK == 0 && d_model % 16 == 0 && d_model >= 128 &&
         ptx::encode_fn() != nullptr;
}

cudaError_t launch_read_chunk(const ChunkLaunch &cl, cudaStream_t s) {
  ChunkParams p{};
  p.n = cl.n;
  p.d_model = cl.d_model;
  p.d_ff = cl.d_ff;
  p.C = cl.C;
  p.L = cl.L;
  p.layer = cl.layer;
  p.sel = cl.sel;
  p.X = cl.X;
  p.Vt = cl.Vt;
  p.Y = cl.Y;
  p.tailZ = cl.tailZ;
  p.tailV = cl.tailV;
  p.tz_owner = cl.tz_owner;
  p.tv_owner = cl.tv_owner;
  p.tz_layer = cl.tz_layer;
  p.tv_layer = cl.tv_layer;
  p.delta = cl.delta;
  p.append = cl.append;
  p.valid_rows = cl.valid_rows;
  p.Y32 = cl.Y32;
  p.ksplit = cl.ksplit < 1 ? 1 : cl.ksplit;
  p.y32_slab = cl.y32_slab;
  p.x_rowmap = cl.x_rowmap;
  p.x_row0 = cl.x_row0;
  p.cooperative = cl.cooperative;
  static const int lr_print = getenv("TTT_LR_PRINT") ? atoi(getenv("TTT_LR_PRINT")) : 0;
  p.trace = lr_print;
  static const int early_dep = getenv("TTT_CHUNK_EARLY_DEP") ? atoi(getenv("TTT_CHUNK_EARLY_DEP")) : 1;
  p.early_dep = early_dep;
  if (!cl.d_members) return cudaErrorInvalidValue;
  p.owner_idx = cl.d_members;
  const int sms = device_sm_count();
  const NPlan np = plan_n(cl.d_model, cl.n * std::max(1, cl.ksplit), sms);
  if (np.T == 0) return cudaErrorInvalidValue;
  p.nt = np.T;
  p.w_hi = np.w_hi;
  p.h = np.h;
  const bool fused = cl.lr != nullptr;
  if (!fused && cl.delta && !cl.x_rowmap && !cl.Y32) {
    // few members: the wide split-K kernel moves fewer L2 -> SM bytes per CTA (read_chunk_wide.cu)
    // (both costs: per-CTA L2 -> SM bytes / bytes in flight, see plan_read_chunk_wide).  Opt-in
    // (TTT_CHUNK_WIDE=1 forces it, =-1 lets the model choose): measured r2 at 8 members it is
    // slower than this kernel at every K block (16 / 32 / 64: 163 / 125 / 162 vs 101.5 µs), see
    // DESIGN §5 f2, so the default keeps the narrow tiles.
    static const int wide_env = getenv("TTT_CHUNK_WIDE") ? atoi(getenv("TTT_CHUNK_WIDE")) : 0;
    static const int wide_bk = getenv("TTT_WIDE_BK") ? atoi(getenv("TTT_WIDE_BK")) : 32;
    WidePlan wp;
    if (wide_env != 0 && cl.wide_slab && plan_read_chunk_wide(cl.n, cl.d_model, cl.d_ff, sms, wide_bk, &wp)) {
      const long long waves = ((long long)cl.n * np.T + sms - 1) / sms;
      const double stage = BM * BK * 2 + 2.0 * 160 * BK * 2;
      const double narrow = (double)waves * cl.d_ff * 2 * (BM + 2 * np.w_hi) / ((kStages - 1) * stage);
      if (wide_env == 1 || wp.cost < 0.95 * narrow) return launch_read_chunk_wide(cl, wp, s);
    }
  }
  if (fused) {
    // every tile must be resident at once: the finish waits on the other K slabs of its tile
    if (cl.n * np.T * p.ksplit > sms || cl.lr_ctr == nullptr) return cudaErrorInvalidValue;
    const LowRankRead &q = *cl.lr;
    p.lr.slots = q.slots;
    p.lr.slot_elems = q.slot_elems;
    p.lr.layer_off = q.layer_off;
    p.lr.R = q.rank;
    p.lr.Xsrc = q.X;
    p.lr.resid = q.resid;
    p.lr.Yout = q.Y;
    p.lr.u = q.u;
    p.lr.bu = q.Y32 + (size_t)kMaxKSplit * q.y32_slab;
    p.lr.ctr = cl.lr_ctr;
    p.lr.x_row = cl.d_members + kMaxGroup;
    p.lr.v_row = cl.d_members + 2 * kMaxGroup;
    p.lr.y_row = cl.d_members + 3 * kMaxGroup;
    p.lr.tail_pos = cl.d_members + 4 * kMaxGroup;
    p.Vt = q.Vt;
    p.tailZ = q.tailZ;
    p.tailV = q.tailV;
    p.tz_owner = q.tz_owner;
    p.tv_owner = q.tv_owner;
    p.tz_layer = q.tz_layer;
    p.tv_layer = q.tv_layer;
    static const bool lr_early_x = !getenv("TTT_LR_EARLY_X") || atoi(getenv("TTT_LR_EARLY_X")) != 0;
    p.xflag = q.xflag;
    p.x_epoch = lr_early_x && cl.x_rowmap && q.xflag ? q.x_epoch : 0;   // (a gathered Xg is written in the step)
  }
  CUtensorMap mX, mW, mD;
  const bool xmap_ok = cl.x_rowmap ? cached_map(&mX, cl.X, cl.d_ff,
                                                (uint64_t)(cl.x_rows_total > 0 ? cl.x_rows_total : cl.valid_rows), 1,
                                                BK, BM)
                                   : cached_map(&mX, cl.X, cl.d_ff, cl.C, cl.n, BK, BM);
  if (!xmap_ok || !cached_map(&mW, cl.w_down, cl.d_ff, cl.d_model, cl.L, BK, np.w_hi) ||
      !cached_map(&mD, cl.delta ? cl.slots : cl.w_down, cl.d_ff, cl.d_model,
                  cl.delta ? (uint64_t)cl.max_slots * cl.L : (uint64_t)cl.L, BK, np.w_hi))
    return cudaErrorInvalidValue;
  if (fused) {
    p.n = (cl.lr->n + BM - 1) / BM;                // tiles index row blocks; members via p.lr
    p.valid_rows = cl.lr->n;
    return launch_bn<160, true>(mX, mW, mD, p, s);
  }
  return launch_bn<160, false>(mX, mW, mD, p, s);
}

}  // namespace ttt
