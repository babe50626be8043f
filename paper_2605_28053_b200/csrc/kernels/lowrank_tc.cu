// NEXT f1 — low-rank delta READ in ONE pass over HBM (DeltaAdapterState, P:348,
// P:477-479; App. F; rule S:188 generalised, reading xviii):
//     y_m = W_down · z_m + B_mᵀ (A_m z_m)        A_m [R][d_ff], B_m [R][d_model]
//
// Both contractions over d_ff are one tcgen05 GEMM.  The group's members are the
// M rows (X = [z_0 … z_{n-1}], 128-row blocks) and the N dimension is W_down's
// d_model rows followed by every member's R rows of A (BN = 256-row tiles; an A
// tile holds 256/R members' A, loaded as 256/R TMA boxes from the owners' slots):
//     P = X · [W_down ; A_0 ; A_1 ; …]ᵀ      (fp32, TMEM)
// Column block (d_model + m·R … + R) of row m is u_m = A_m z_m; the rest of an A
// tile's rows are other members' products and are dropped (the tensor pipe has the
// headroom: 11.5 GFLOP per 104 MB at R = 16, AI 110 < the 253 flop/B ridge, so the
// launch stays HBM-bound).  K (d_ff) is split in KS slabs so the (row block,
// N tile, slab) tiles fill the SMs; every slab writes fp32 partials (Y32 for W
// tiles, U for A tiles).  A second, PDL-chained launch (the kernel boundary is the
// grid-wide gate) finishes 1/grid of the outputs per CTA:
//     u_m = Σ_ks U[ks][m]   (fixed order),   y_m = Σ_ks Y32[ks][m] + B_mᵀ u_m (+ resid) → bf16.
// W_down, A and B are read once per layer (B by the finish), X once per N tile (L2).
// The tail append (a4) runs in warps 6-11 while the first tile streams.
//
// Warp roles: 0 TMA producer (4-stage ring of X 128×64 + W/A 256×64 bf16 boxes,
// 128-B swizzle), 1 TMEM alloc + single-thread tcgen05.mma issue (M=128, N=256,
// K=16; two 256-column accumulators), 2-5 epilogue (tcgen05.ld → fp32 partials),
// 6-11 tail append.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "../internal.h"
#include "sm100_ptx.cuh"

namespace ttt {

namespace {

using namespace ptx;

#ifndef TTT_LR_BN
#define TTT_LR_BN 256
#endif
constexpr int BM = 128, BN = TTT_LR_BN, BK = 64, kStages = 4;
constexpr int kThreads = 384;
constexpr uint32_t X_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE = X_BYTES + B_BYTES;

struct TcParams {
  int n, d_model, d_ff, R, KS, nW, mpt, T, layer, L, rows;   // rows: padded row count of the Y32/U slabs
  int nA0, units0;                                           // row block 0: A tiles, W + A tiles
  int nA1;                                                   // row block 1 (n > 128)
  const int *sel;
  const void *slots;
  long long slot_elems, layer_off;
  const void *X, *Vt, *resid;
  void *Y;
  float *Y32, *U;
  long long y32_slab;
  void *tailZ, *tailV;
  long long tz_owner, tv_owner, tz_layer, tv_layer;
  int owner_idx[kMaxGroup], x_row[kMaxGroup], v_row[kMaxGroup], y_row[kMaxGroup], tail_pos[kMaxGroup];
  int trace;                                                 // TTT_LR_TRACE=1: %globaltimer per CTA phase
};

__device__ unsigned long long g_lr_trace[8 * 1024 * 4];   // [launch % 8][cta][main entry, main done, finish entry, exit]
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}


struct Tile {
  int b, isA, j, ks, kb0, kb1;
};
// tile u -> (row block b, W tile j or A tile j, K slab ks); units of block 0 first
__device__ __forceinline__ Tile decode(const TcParams &p, int u) {
  Tile t;
  t.ks = u % p.KS;
  int unit = u / p.KS;
  t.b = unit < p.units0 ? 0 : 1;
  if (t.b) unit -= p.units0;
  t.isA = unit >= p.nW;
  t.j = t.isA ? unit - p.nW : unit;
  const int nk = p.d_ff / BK;
  t.kb0 = nk * t.ks / p.KS;
  t.kb1 = nk * (t.ks + 1) / p.KS;
  return t;
}
__device__ __forceinline__ int members_in_block(const TcParams &p, int b) { return min(BM, p.n - b * BM); }

__global__ void __launch_bounds__(kThreads, 1)
    read_lowrank_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                           const __grid_constant__ CUtensorMap tmA, const TcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  u64 *bars = reinterpret_cast<u64 *>(smem + kStages * STAGE);
  u64 *full = bars, *empty = bars + kStages, *t_full = bars + 2 * kStages, *t_empty = t_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(t_empty + 2);
  int *slot_s = reinterpret_cast<int *>(smem + kStages * STAGE + 128);        // A tile: members' slot·L + layer

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(t_full + a, 1);
      mbar_init(t_empty + a, 4);
    }
    mbar_init_fence();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmW);
    tma_prefetch(&tmA);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: the prologue overlaps the previous kernel (the last layer's finish).  W_down is never
  // written by any kernel, so the first W tile's first stages are requested before the wait;
  // X, A (slot selector), tails and the partial buffers only after it.
  asm volatile("griddepcontrol.launch_dependents;");
  int npre = 0;
  if (warp == 0 && lane == 0) {
    const Tile t0 = decode(p, blockIdx.x);
    if (!t0.isA) {
      npre = min(kStages, t0.kb1 - t0.kb0);
      for (int i = 0; i < npre; ++i) {
        mbar_expect_tx(full + i, X_BYTES + B_BYTES);
        tma_load_3d(smem + i * STAGE + X_BYTES, &tmW, full + i, (t0.kb0 + i) * BK, t0.j * BN, p.layer);
      }
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p.trace && threadIdx.x == 0) g_lr_trace[(p.trace - 1) * 4096 + blockIdx.x * 4] = gtimer();

  if (warp == 0) {
    if (lane == 0) {                                        // ---------------- TMA producer
      int it = 0;
      for (int u = blockIdx.x; u < p.T; u += gridDim.x) {
        const Tile t = decode(p, u);
        int nm = 0;
        if (t.isA) {
          const int nb = members_in_block(p, t.b);
          nm = min(p.mpt, nb - t.j * p.mpt);
          for (int i = 0; i < nm; ++i) {
            const int o = p.owner_idx[t.b * BM + t.j * p.mpt + i];
            slot_s[i] = (2 * o + p.sel[o]) * p.L + p.layer;
          }
        }
        const uint32_t bytes = X_BYTES + (t.isA ? (uint32_t)nm * p.R * BK * 2 : B_BYTES);
        for (int kb = t.kb0; kb < t.kb1; ++kb, ++it) {
          const int s = it % kStages;
          if (it >= kStages) mbar_wait(empty + s, ((it / kStages) - 1) & 1);
          unsigned char *st = smem + s * STAGE;
          if (it < npre) {                                  // W box already in flight
            tma_load_3d(st, &tmX, full + s, kb * BK, t.b * BM, 0);
            continue;
          }
          mbar_expect_tx(full + s, bytes);
          tma_load_3d(st, &tmX, full + s, kb * BK, t.b * BM, 0);
          if (!t.isA) {
            tma_load_3d(st + X_BYTES, &tmW, full + s, kb * BK, t.j * BN, p.layer);
          } else {
            for (int i = 0; i < nm; ++i)
              tma_load_3d(st + X_BYTES + i * p.R * BK * 2, &tmA, full + s, kb * BK, 0, slot_s[i]);
          }
        }
      }
    }
  } else if (warp == 1) {                                   // ---------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16(BM, BN, 0, 0);
    int it = 0, k = 0;
    for (int u = blockIdx.x; u < p.T; u += gridDim.x, ++k) {
      const Tile t = decode(p, u);
      const int acc = k & 1;
      if (k >= 2) mbar_wait(t_empty + acc, ((k >> 1) - 1) & 1);
      tc_fence_after();
      for (int kb = t.kb0; kb < t.kb1; ++kb, ++it) {
        const int s = it % kStages;
        mbar_wait(full + s, (it / kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a0 = smem_u32(smem + s * STAGE), b0 = a0 + X_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma_bf16(tmem + acc * BN, smem_desc_sw128(a0 + kk * 32, 16, 1024), smem_desc_sw128(b0 + kk * 32, 16, 1024),
                     idesc, ((kb - t.kb0) | kk) ? 1u : 0u);
          mma_commit(empty + s);
          if (kb == t.kb1 - 1) mma_commit(t_full + acc);
        }
        __syncwarp();
      }
    }
  } else if (warp < 6) {                                    // ---------------- epilogue warps 2-5
    const int q = warp & 3, row = q * 32 + lane;            // TMEM lane = member row in the block
    int k = 0;
    for (int u = blockIdx.x; u < p.T; u += gridDim.x, ++k) {
      const Tile t = decode(p, u);
      const int acc = k & 1;
      mbar_wait(t_full + acc, (k >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + acc * BN + ((uint32_t)(q * 32) << 16);
      const int m = t.b * BM + row;
      const bool valid = row < members_in_block(p, t.b);
      if (!t.isA) {                                          // W tile: fp32 partial of W_down·z
        const int n0 = t.j * BN, ncols = min(BN, p.d_model - n0);
        float *dst = p.Y32 + (size_t)t.ks * p.y32_slab + (size_t)m * p.d_model + n0;
#pragma unroll 1
        for (int c = 0; c < ncols; c += 32) {
          uint32_t r[32];
          tmem_ld32(taddr + (uint32_t)c, r);
          if (valid) {
#pragma unroll
            for (int v = 0; v < 8; ++v)
              if (c + 4 * v < ncols)
                reinterpret_cast<float4 *>(dst + c)[v] =
                    make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
          }
        }
      } else {                                               // A tile: u partial of the member's own R columns
        const int mg0 = t.j * p.mpt, nm = min(p.mpt, members_in_block(p, t.b) - mg0);
        const int i = row - mg0, lo = i * p.R;
        const bool mine = valid && i >= 0 && i < nm;
        // warp-uniform: only warps whose 32 rows meet [mg0, mg0 + nm) read TMEM
        if (mg0 < q * 32 + 32 && mg0 + nm > q * 32) {
          float *dst = p.U + ((size_t)t.ks * p.rows + m) * p.R;
#pragma unroll 1
          for (int c = 0; c < nm * p.R; c += 32) {
            uint32_t r[32];
            tmem_ld32(taddr + (uint32_t)c, r);
            if (mine && c < lo + p.R && c + 32 > lo) {
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (c + e >= lo && c + e < lo + p.R) dst[c + e - lo] = __uint_as_float(r[e]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(t_empty + acc);
    }
  } else {                                                  // ---------------- warps 6-11: a4 tail append
    const int nz = p.d_ff / 8, nv = p.d_model / 8, per = nz + nv;
    const long long total = (long long)p.n * per;
    const long long lo = total * blockIdx.x / gridDim.x, hi = total * (blockIdx.x + 1) / gridDim.x;
    for (long long v = lo + (threadIdx.x - 192); v < hi; v += kThreads - 192) {
      const int m = (int)(v / per), e = (int)(v - (long long)m * per), o = p.owner_idx[m];
      if (e < nz) {
        const uint4 z = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.X) +
                                                        (size_t)p.x_row[m] * p.d_ff)[e];
        reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.tailZ) + o * p.tz_owner + p.tz_layer +
                                  (size_t)p.tail_pos[m] * p.d_ff)[e] = z;
      } else {
        const uint4 w = reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.Vt) +
                                                        (size_t)p.v_row[m] * p.d_model)[e - nz];
        reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.tailV) + o * p.tv_owner + p.tv_layer +
                                  (size_t)p.tail_pos[m] * p.d_model)[e - nz] = w;
      }
    }
  }
  tc_fence_before();
  __syncwarp();                                             // warp 0: the producer lane rejoins its warp
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);

  if (p.trace && threadIdx.x == 0) g_lr_trace[(p.trace - 1) * 4096 + blockIdx.x * 4 + 1] = gtimer();
}

// y_m = Σ_ks Y32[ks][m] + B_mᵀ (Σ_ks U[ks][m]) (+ resid) → bf16.  CTA = (member m, column part
// h of S): one thread issues bulk copies (cp.async.bulk, mbarrier complete_tx) of the member's
// KS partial rows and of B_m's rows (kFinRows per chunk, double-buffered) into shared memory, so
// the bytes stream at the copy engine's rate instead of through per-thread load round trips;
// the 256 threads then reduce from shared memory in a fixed order (slabs ascending, r ascending).
// PDL-chained after read_lowrank_tc_kernel: the kernel boundary is the grid-wide gate.
constexpr int kFinThreads = 256, kFinMaxG = 2;   // ≤ kFinMaxG 8-column groups per thread
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, u64 *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__global__ void __launch_bounds__(kFinThreads, 1) lr_finish_tc_kernel(const TcParams p, int S, int cols, int cr) {
  extern __shared__ __align__(128) unsigned char fsm[];
  u64 *bar = reinterpret_cast<u64 *>(fsm);                          // [0] partials, [1..2] B buffers
  float *u = reinterpret_cast<float *>(fsm + 64);                   // u_m (≤ 64)
  float *P = reinterpret_cast<float *>(fsm + 64 + 256);             // [KS][cols] fp32
  __nv_bfloat16 *Bb = reinterpret_cast<__nv_bfloat16 *>(P + (size_t)p.KS * cols);   // [1 or 2][cr][cols]
  const int tid = threadIdx.x, R = p.R, KS = p.KS, dm = p.d_model;
  const int m = blockIdx.x / S, c0 = (blockIdx.x % S) * cols, nc = min(cols, dm - c0);
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(bar + i, 1);
    mbar_init_fence();
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p.trace && tid == 0 && blockIdx.x < 1024) g_lr_trace[(p.trace - 1) * 4096 + blockIdx.x * 4 + 2] = gtimer();
  const int o = p.owner_idx[m];
  const __nv_bfloat16 *Bm = static_cast<const __nv_bfloat16 *>(p.slots) + (2LL * o + p.sel[o]) * p.slot_elems +
                            p.layer_off + (size_t)R * p.d_ff;
  const int nch = (R + cr - 1) / cr;
  auto issue_chunk = [&](int ch) {
    const int rows = min(cr, R - ch * cr), buf = ch & 1;
    mbar_expect_tx(bar + 1 + buf, (uint32_t)(rows * nc * 2));
    for (int r = 0; r < rows; ++r)
      bulk_g2s(Bb + ((size_t)buf * cr + r) * cols, Bm + (size_t)(ch * cr + r) * dm + c0, nc * 2, bar + 1 + buf);
  };
  if (tid == 0) {
    mbar_expect_tx(bar, (uint32_t)(KS * nc * 4));
    for (int ks = 0; ks < KS; ++ks)
      bulk_g2s(P + (size_t)ks * cols, p.Y32 + ks * p.y32_slab + (size_t)m * dm + c0, nc * 4, bar);
    for (int ch = 0; ch < min(2, nch); ++ch) issue_chunk(ch);
  }
  if (tid < R) {                                                     // u_m = Σ_ks U[ks][m] (slabs ascending)
    float v[kMaxKSplit];
#pragma unroll
    for (int ks = 0; ks < kMaxKSplit; ++ks) v[ks] = ks < KS ? __ldcg(p.U + ((size_t)ks * p.rows + m) * R + tid) : 0.f;
    float sum = 0.f;
#pragma unroll
    for (int ks = 0; ks < kMaxKSplit; ++ks) sum += v[ks];
    u[tid] = sum;
  }
  __syncthreads();
  const int ng = nc / 8;
  float y[kFinMaxG][8];
  mbar_wait(bar, 0);
#pragma unroll
  for (int gi = 0; gi < kFinMaxG; ++gi) {
    const int g = tid + gi * kFinThreads;
#pragma unroll
    for (int e = 0; e < 8; ++e) y[gi][e] = 0.f;
    if (g < ng)
      for (int ks = 0; ks < KS; ++ks) {
        const float4 a = reinterpret_cast<const float4 *>(P + (size_t)ks * cols + 8 * g)[0];
        const float4 b = reinterpret_cast<const float4 *>(P + (size_t)ks * cols + 8 * g)[1];
        y[gi][0] += a.x; y[gi][1] += a.y; y[gi][2] += a.z; y[gi][3] += a.w;
        y[gi][4] += b.x; y[gi][5] += b.y; y[gi][6] += b.z; y[gi][7] += b.w;
      }
  }
  for (int ch = 0; ch < nch; ++ch) {                                 // + Bᵀu, B rows ascending
    const int rows = min(cr, R - ch * cr), buf = ch & 1;
    mbar_wait(bar + 1 + buf, (ch >> 1) & 1);
#pragma unroll
    for (int gi = 0; gi < kFinMaxG; ++gi) {
      const int g = tid + gi * kFinThreads;
      if (g < ng)
        for (int r = 0; r < rows; ++r) {
          const float uk = u[ch * cr + r];
          const uint4 bv = *reinterpret_cast<const uint4 *>(Bb + ((size_t)buf * cr + r) * cols + 8 * g);
          const uint32_t w[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
          for (int hh = 0; hh < 4; ++hh) {
            y[gi][2 * hh] = fmaf(uk, __uint_as_float(w[hh] << 16), y[gi][2 * hh]);
            y[gi][2 * hh + 1] = fmaf(uk, __uint_as_float(w[hh] & 0xffff0000u), y[gi][2 * hh + 1]);
          }
        }
    }
    __syncthreads();                                                 // buffer consumed
    if (tid == 0 && ch + 2 < nch) issue_chunk(ch + 2);
  }
#pragma unroll
  for (int gi = 0; gi < kFinMaxG; ++gi) {
    const int g = tid + gi * kFinThreads;
    if (g >= ng) continue;
    const int c = c0 + 8 * g;
    if (p.resid) {
      const uint4 rv = *reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.resid) +
                                                        (size_t)p.y_row[m] * dm + c);
      const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
      for (int hh = 0; hh < 4; ++hh) {
        y[gi][2 * hh] += __uint_as_float(w[hh] << 16);
        y[gi][2 * hh + 1] += __uint_as_float(w[hh] & 0xffff0000u);
      }
    }
    uint32_t out[4];
#pragma unroll
    for (int hh = 0; hh < 4; ++hh) {
      __nv_bfloat162 h2 = __floats2bfloat162_rn(y[gi][2 * hh], y[gi][2 * hh + 1]);
      out[hh] = *reinterpret_cast<uint32_t *>(&h2);
    }
    *reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.Y) + (size_t)p.y_row[m] * dm + c) =
        make_uint4(out[0], out[1], out[2], out[3]);
  }
  if (p.trace) {
    __syncthreads();
    if (tid == 0 && blockIdx.x < 1024) g_lr_trace[(p.trace - 1) * 4096 + blockIdx.x * 4 + 3] = gtimer();
  }
}


size_t smem_bytes() { return 1024 + (size_t)kStages * STAGE + 256; }

// 3-D bf16 map with an explicit outer stride: A rows of (slot, layer) = [R][d_ff] at slot·L + layer
bool make_map_a(CUtensorMap *m, const void *base, uint64_t d_ff, uint64_t R, uint64_t n_outer, uint64_t outer_bytes) {
  struct Entry {
    const void *base;
    uint64_t d_ff, R, n_outer, outer_bytes;
    CUtensorMap map;
  };
  static Entry cache[16];
  static int n_used = 0, next = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < n_used; ++i) {
    const Entry &e = cache[i];
    if (e.base == base && e.d_ff == d_ff && e.R == R && e.n_outer == n_outer && e.outer_bytes == outer_bytes) {
      *m = e.map;
      return true;
    }
  }
  auto fn = ptx::encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d_ff, R, n_outer};
  cuuint64_t strides[2] = {d_ff * 2, outer_bytes};
  cuuint32_t box[3] = {BK, (cuuint32_t)R, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  cache[next] = Entry{base, d_ff, R, n_outer, outer_bytes, *m};
  next = (next + 1) % 16;
  n_used = n_used < 16 ? n_used + 1 : 16;
  return true;
}

size_t fin_smem(int cols, int KS, int cr, int R) {
  return 64 + 256 + (size_t)KS * cols * 4 + (cr < R ? 2 : 1) * (size_t)cr * cols * 2;
}
// finish split: S column parts per member (cols a multiple of 16, S·cols ≥ d_model > (S-1)·cols),
// the fewest parts whose n·S CTAs cover the SMs; B_m's rows all in flight (cr = R) when that fits
// ~110 KB (2 CTAs per SM, so the grid is one wave: a second wave delays the PDL launch of the
// next layer by ~8 µs, measured), else double-buffered chunks of cr rows (a multiple of 4)
struct FinPlan {
  int S = 1, cols = 0, cr = 4;
};
FinPlan fin_plan(int n, int d_model, int KS, int R, int sms) {
  FinPlan f;
  f.S = std::max(1, std::min({8, (sms + n - 1) / n, d_model / 16}));
  f.cols = ((d_model + f.S - 1) / f.S + 15) / 16 * 16;
  f.S = (d_model + f.cols - 1) / f.cols;
  constexpr size_t kBudget = 110 * 1024;
  if (fin_smem(f.cols, KS, R, R) <= kBudget) {
    f.cr = R;
  } else {
    f.cr = 4;
    while (f.cr + 4 < R && fin_smem(f.cols, KS, f.cr + 4, R) <= kBudget) f.cr += 4;
  }
  return f;
}

struct Plan {
  int KS = 0, nW = 0, mpt = 0, nA0 = 0, nA1 = 0, units = 0, T = 0, grid = 0;
};
Plan make_plan(int n, int d_model, int d_ff, int R, int sms) {
  Plan pl;
  pl.nW = (d_model + BN - 1) / BN;
  pl.mpt = BN / R;
  const int n0 = std::min(n, BM), n1 = n - n0;
  pl.nA0 = (n0 + pl.mpt - 1) / pl.mpt;
  pl.nA1 = n1 > 0 ? (n1 + pl.mpt - 1) / pl.mpt : 0;
  pl.units = pl.nW + pl.nA0 + (n1 > 0 ? pl.nW + pl.nA1 : 0);
  // K slabs: minimise waves / KS (time per launch ∝ waves × K per slab), fewest slabs on ties;
  // at least 4 K blocks of 64 per slab
  const int nk = d_ff / BK;
  double best = 1e30;
  for (int ks = 1; ks <= std::min(kMaxKSplit, std::max(1, nk / 4)); ++ks) {
    const long long tiles = (long long)pl.units * ks;
    const double cost = (double)((tiles + sms - 1) / sms) / ks;
    if (cost < best - 1e-9) {
      best = cost;
      pl.KS = ks;
    }
  }
  pl.T = pl.units * pl.KS;
  pl.grid = std::min(pl.T, sms);
  return pl;
}

}  // namespace

bool lowrank_tc_supported(int n, int d_model, int d_ff, int rank) {
  if (n < 1 || n > 2 * BM || rank < 8 || rank > 64 || rank % 8 || BN % rank || d_ff % BK || d_model % 16 ||
      ptx::encode_fn() == nullptr)
    return false;
  const int sms = device_sm_count();
  const Plan pl = make_plan(n, d_model, d_ff, rank, sms);
  const FinPlan fp = fin_plan(n, d_model, pl.KS, rank, sms);
  return fp.cols / 8 <= kFinMaxG * kFinThreads && fin_smem(fp.cols, pl.KS, fp.cr, rank) <= 200 * 1024;
}

cudaError_t launch_lowrank_tc(const LowRankRead &q, const void *X, cudaStream_t s) {
  const int sms = device_sm_count();
  const Plan pl = make_plan(q.n, q.d_model, q.d_ff, q.rank, sms);
  TcParams p{};
  p.n = q.n; p.d_model = q.d_model; p.d_ff = q.d_ff; p.R = q.rank; p.KS = pl.KS; p.nW = pl.nW; p.mpt = pl.mpt;
  p.T = pl.T; p.layer = q.layer; p.L = q.L;
  p.rows = (q.n + BM - 1) / BM * BM;
  p.nA0 = pl.nA0; p.nA1 = pl.nA1; p.units0 = pl.nW + pl.nA0;
  p.sel = q.sel; p.slots = q.slots; p.slot_elems = q.slot_elems; p.layer_off = q.layer_off;
  p.X = q.X; p.Vt = q.Vt; p.resid = q.resid; p.Y = q.Y;
  p.Y32 = q.Y32; p.U = q.u; p.y32_slab = q.y32_slab;
  p.tailZ = q.tailZ; p.tailV = q.tailV;
  p.tz_owner = q.tz_owner; p.tv_owner = q.tv_owner; p.tz_layer = q.tz_layer; p.tv_layer = q.tv_layer;
  for (int b = 0; b < q.n; ++b) {
    p.owner_idx[b] = q.owner_idx[b];
    p.x_row[b] = q.x_row[b];
    p.v_row[b] = q.v_row[b];
    p.y_row[b] = q.y_row[b];
    p.tail_pos[b] = q.tail_pos[b];
  }
  CUtensorMap mX, mW, mA;
  const long long E = (long long)q.rank * (q.d_ff + q.d_model);   // payload elements per (slot, layer)
  if (!cached_map(&mX, X, q.d_ff, (uint64_t)q.n, 1, BK, BM) ||
      !cached_map(&mW, q.w_down, q.d_ff, q.d_model, q.L, BK, BN) ||
      !make_map_a(&mA, q.slots, q.d_ff, q.rank, (uint64_t)q.max_slots * q.L, (uint64_t)E * 2))
    return cudaErrorInvalidValue;
  const size_t smem = smem_bytes();
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(read_lowrank_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  static const int trace = getenv("TTT_LR_TRACE") ? atoi(getenv("TTT_LR_TRACE")) : 0;
  static int n_traced = 0;
  p.trace = trace ? 1 + (n_traced++ % 8) : 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, read_lowrank_tc_kernel, mX, mW, mA, p);
  count_launch();
  if (e != cudaSuccess) return e;
  const FinPlan fp = fin_plan(q.n, q.d_model, pl.KS, q.rank, sms);
  const size_t fsmem = fin_smem(fp.cols, pl.KS, fp.cr, q.rank);
  static size_t fconfigured = 0;
  if (fsmem > fconfigured) {
    e = cudaFuncSetAttribute(lr_finish_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
    if (e != cudaSuccess) return e;
    fconfigured = fsmem;
  }
  cfg.gridDim = dim3(q.n * fp.S);
  cfg.blockDim = dim3(kFinThreads);
  cfg.dynamicSmemBytes = fsmem;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, lr_finish_tc_kernel, p, fp.S, fp.cols, fp.cr);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace ttt

// debug hook (not part of the ABI header): copy the last traced launch's per-CTA timestamps
extern "C" int ttt_debug_lr_trace(unsigned long long *host, int n) {
  return (int)cudaMemcpyFromSymbol(host, ttt::g_lr_trace, sizeof(unsigned long long) * (size_t)n);
}
