// NEXT f2 — chunk-granular READ (prefill), wide-tile split-K variant for small groups.
//
// Same operation as read_chunk_tc.cu (PAPER: READ keeps the version, Table 3 P:378-381;
// one chunk of C tokens per member at version v, boundaries every C_ttt tokens P:160-161):
//     Y_b[t, :] = z_t · (W_down[l] + ΔW_b[l])ᵀ,   t = 0 .. C-1,
// with the chunk's (z_t, v_t) appended to the owner's tail.
//
// Why a second kernel.  With few members (config 2b: 8 owners, 2560 × 9728) the narrow-tile
// kernel gives every CTA one (member, 144-column) tile over the whole K: each CTA streams its
// member's X (2.5 MB), its W_down rows and its ΔW rows from L2, 1.17 GB of L2 -> SM traffic per
// layer, which the chip delivers in ~100 µs (r2 ncu: L2 -> SM is the bound, tensor pipe 53 %;
// ablation without ΔW: ingress -35 %, time -23 %; multicast cut LTS reads but not SM ingress).
// Here a CTA owns a wider tile (up to 512 accumulator columns of TMEM) and 1/KS of K, and may
// hold MPC = 2 members that share each W_down box:
//   * ingress per CTA = (K/KS)·2·(MPC·128 + (1+MPC)·w) bytes (8 members: 6.4–7.0 MB per CTA
//     instead of 8.1 MB, e.g. MPC = 2, w ≈ 213, KS = 3 or MPC = 1, w = 288, KS = 2);
//   * split-K partials are combined in a fixed order (deterministic): CTA ks owns 1/KS of the
//     tile's 16-column chunks, writes the other chunks' fp32 partials to a workspace slab, and
//     after the tile's ticket shows all KS slabs, bulk-copies the other CTAs' partials of its own
//     chunks into shared memory and adds them to its TMEM accumulator in ks order;
//   * ring: K blocks of 32 (64-byte swizzle) so 3 stages of ~60 KB fit.
// Every CTA of the grid is resident at once (grid ≤ SM count, one CTA per SM, cooperative
// launch), which the ticket wait needs.
//
// Measured r2 (parity-green, NOT the default — TTT_CHUNK_WIDE=1 selects it): at 8 members
// 125–163 µs per layer vs 101.5 µs for the narrow kernel (K blocks of 16 / 32 / 64 elements);
// ncu: fewer L2 -> SM bytes but fewer bytes in flight per SM, and 32-byte rows saturate the
// SM -> L2 request path (DESIGN §5 f2, profiles/r2/read_chunk_wide_ncu.txt).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "../internal.h"
#include "sm100_ptx.cuh"

namespace ttt {
namespace {

using namespace ptx;

constexpr int WBM = 128;                           // rows (tokens) per tile
constexpr int kWThreads = 192;                     // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kWMaxStages = 12;
constexpr int kChunkFloats = WBM * 16;             // one 16-column fp32 partial chunk: 8 KB
constexpr int kSmemAvail = 232448 - 2048;          // dynamic shared memory for the ring (+ barriers, alignment)

struct WideParams {
  int n, d_model, d_ff, C, L, layer;
  int mpc, T, KS, w_hi, h;       // N blocks: j < h are w_hi wide, the rest w_hi - 32
  int stages;
  uint32_t stage_bytes;
  const int *sel, *owner_idx;
  const void *X, *Vt;
  void *Y, *tailZ, *tailV;
  long long tz_owner, tv_owner, tz_layer, tv_layer;
  int append;
  float *slab;                   // [tiles][mpc·w_hi/16][128][16] fp32 partials
  int *tickets;                  // [n/mpc · T] self-resetting arrival counters
};

__device__ __forceinline__ int ld_acquire(const int *q) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(q) : "memory");
  return v;
}
template <int ID, int COUNT>
__device__ __forceinline__ void named_bar() {
  asm volatile("barrier.sync %0, %1;" ::"n"(ID), "n"(COUNT) : "memory");
}

// WBK: K elements per ring stage (16 / 32 / 64 → 32- / 64- / 128-byte swizzled rows)
template <int WBK>
__global__ void __launch_bounds__(kWThreads, 1)
    read_chunk_wide_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmWh,
                           const __grid_constant__ CUtensorMap tmWl, const __grid_constant__ CUtensorMap tmDh,
                           const __grid_constant__ CUtensorMap tmDl, const WideParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  u64 *bars = reinterpret_cast<u64 *>(smem + S * p.stage_bytes);
  u64 *full = bars, *empty = bars + kWMaxStages, *t_full = bars + 2 * kWMaxStages, *f_bar = t_full + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(f_bar + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mpc = p.mpc, KS = p.KS;
  // tile (one per CTA): u = ((group · T) + j) · KS + ks
  const int u = blockIdx.x, ks = u % KS, gj = u / KS, g = gj / p.T, j = gj - g * p.T;
  const int n0 = j < p.h ? j * p.w_hi : p.h * p.w_hi + (j - p.h) * (p.w_hi - 32);
  const int width = j < p.h ? p.w_hi : p.w_hi - 32, half = width / 2;
  const int nk = p.d_ff / WBK, kb0 = nk * ks / KS, kb1 = nk * (ks + 1) / KS;
  constexpr int RB = WBK * 2;                              // bytes per swizzled row
  constexpr uint32_t WA_BYTES = WBM * RB;                  // one member's X box
  const uint32_t WB_BYTES = (uint32_t)p.w_hi * RB;         // stage slot of one weight block

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(t_full, 1);
    mbar_init(f_bar, 1);
    mbar_init_fence();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(j < p.h ? &tmWh : &tmWl);
    tma_prefetch(j < p.h ? &tmDh : &tmDl);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {                                        // ---------------- TMA producer
      const CUtensorMap *mW = j < p.h ? &tmWh : &tmWl, *mD = j < p.h ? &tmDh : &tmDl;
      int slot_l[2] = {0, 0};
#pragma unroll
      for (int m = 0; m < 2; ++m)
        if (m < mpc) {
          const int o = p.owner_idx[g * mpc + m];
          slot_l[m] = (2 * o + p.sel[o]) * p.L + p.layer;
        }
      const uint32_t tx = mpc * WA_BYTES + (1 + mpc) * (uint32_t)width * RB;
      int it = 0;
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % S;
        if (it >= S) mbar_wait(empty + s, ((it / S) - 1) & 1);
        unsigned char *st = smem + s * p.stage_bytes;
        mbar_expect_tx(full + s, tx);
        unsigned char *wst = st + mpc * WA_BYTES;
        tma_load_3d(wst, mW, full + s, kb * WBK, n0, p.layer);
        tma_load_3d(wst + half * RB, mW, full + s, kb * WBK, n0 + half, p.layer);
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          if (m >= mpc) break;
          tma_load_3d(st + m * WA_BYTES, &tmX, full + s, kb * WBK, 0, g * mpc + m);
          unsigned char *dst = wst + (1 + m) * WB_BYTES;
          tma_load_3d(dst, mD, full + s, kb * WBK, n0, slot_l[m]);
          tma_load_3d(dst + half * RB, mD, full + s, kb * WBK, n0 + half, slot_l[m]);
        }
      }
    }
  } else if (warp == 1) {                                   // ---------------- MMA issuer
    const uint32_t idesc = idesc_bf16(WBM, half, 0, 0);
    int it = 0;
    for (int kb = kb0; kb < kb1; ++kb, ++it) {
      const int s = it % S;
      mbar_wait(full + s, (it / S) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(smem + s * p.stage_bytes), w0 = a0 + mpc * WA_BYTES;
#pragma unroll
        for (int kk = 0; kk < WBK / 16; ++kk) {             // K = 16 step = 32 B inside the swizzled row
          for (int m = 0; m < mpc; ++m) {
            const u64 ad = smem_desc_swz<RB>(a0 + m * WA_BYTES + kk * 32);
            const uint32_t d0 = w0 + (1 + m) * WB_BYTES;
#pragma unroll
            for (int q = 0; q < 2; ++q) {                   // the two N halves of the tile
              const uint32_t acc = tmem + (uint32_t)(m * p.w_hi + q * half);
              const uint32_t boff = (uint32_t)(q * half * RB) + kk * 32;
              mma_bf16(acc, ad, smem_desc_swz<RB>(w0 + boff), idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
              mma_bf16(acc, ad, smem_desc_swz<RB>(d0 + boff), idesc, 1u);
            }
          }
        }
        mma_commit(empty + s);
        if (kb == kb1 - 1) mma_commit(t_full);
      }
      __syncwarp();
    }
  } else {                                                  // ---------------- epilogue warps 2-5
    const int q = warp & 3, row = q * 32 + lane, et = threadIdx.x - 64;
    if (p.append) {                                         // a4: this tile appends slice (j, ks) of its members' chunks
      const int part = j * KS + ks, parts = p.T * KS;
      auto copy_slice = [&](const uint4 *src, uint4 *dst, size_t total) {
        const size_t lo = total * part / parts, hi = total * (part + 1) / parts;
        size_t v = lo + et;
        for (; v + 3 * 128 < hi; v += 4 * 128) {
          const uint4 a0 = src[v], a1 = src[v + 128], a2 = src[v + 256], a3 = src[v + 384];
          dst[v] = a0; dst[v + 128] = a1; dst[v + 256] = a2; dst[v + 384] = a3;
        }
        for (; v < hi; v += 128) dst[v] = src[v];
      };
      for (int m = 0; m < mpc; ++m) {
        const int b = g * mpc + m, o = p.owner_idx[b];
        copy_slice(reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.X) + (size_t)b * p.C * p.d_ff),
                   reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.tailZ) + o * p.tz_owner + p.tz_layer),
                   (size_t)p.C * p.d_ff / 8);
        copy_slice(reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(p.Vt) + (size_t)b * p.C * p.d_model),
                   reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.tailV) + o * p.tv_owner + p.tv_layer),
                   (size_t)p.C * p.d_model / 8);
      }
    }
    mbar_wait(t_full, 0);
    tc_fence_after();
    // 16-column chunks of the tile, member-major; CTA k finishes chunks [c_lo(k), c_lo(k+1))
    const int cpm = width / 16, NC = mpc * cpm;
    auto c_lo = [&](int k) { return (k * NC + KS - 1) / KS; };
    const int my0 = c_lo(ks), my1 = c_lo(ks + 1);
    const int cmax = mpc * p.w_hi / 16;                     // slab chunks per CTA
    auto taddr = [&](int c) {
      const int m = c / cpm, cc = c - m * cpm;
      return tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(m * p.w_hi + cc * 16);
    };
    if (KS > 1) {
      float *own = p.slab + (size_t)u * cmax * kChunkFloats;
      for (int c = 0; c < NC; ++c) {                        // partials of the chunks other CTAs finish
        if (c >= my0 && c < my1) continue;
        uint32_t r[16];
        tmem_ld16(taddr(c), r);
        float4 *d4 = reinterpret_cast<float4 *>(own + (size_t)c * kChunkFloats + row * 16);
#pragma unroll
        for (int v = 0; v < 4; ++v)
          __stcg(d4 + v, make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                     __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3])));
      }
      named_bar<1, 128>();
      if (et == 0) {
        int *tick = p.tickets + gj;
        __threadfence();
        atomicAdd(tick, 1);
        while (ld_acquire(tick) < KS) __nanosleep(32);
        __threadfence();
      }
      named_bar<1, 128>();
    }
    // finish own chunks in batches that fit the (now idle) ring: the other KS-1 partials of a
    // chunk land in shared memory by bulk copies, then y = Σ_ks part[ks] (ks ascending) -> bf16
    const int per = KS > 1 ? (int)((S * p.stage_bytes) / ((uint32_t)(KS - 1) * kChunkFloats * 4)) : NC;
    float *stg = reinterpret_cast<float *>(smem);
    int phase = 0;
    for (int c0 = my0; c0 < my1; c0 += per) {
      const int c1 = min(my1, c0 + per);
      if (KS > 1) {
        if (et == 0) {
          // the previous batch was read through the generic proxy; the bulk copies write via the async proxy
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(f_bar, (uint32_t)((c1 - c0) * (KS - 1)) * kChunkFloats * 4);
          for (int c = c0; c < c1; ++c)
            for (int k = 0, i = 0; k < KS; ++k) {
              if (k == ks) continue;
              const float *src = p.slab + ((size_t)(gj * KS + k) * cmax + c) * kChunkFloats;
              bulk_g2s(stg + ((size_t)(c - c0) * (KS - 1) + i) * kChunkFloats, src, kChunkFloats * 4, f_bar);
              ++i;
            }
        }
        mbar_wait(f_bar, phase);
        phase ^= 1;
      }
      for (int c = c0; c < c1; ++c) {
        uint32_t r[16];
        tmem_ld16(taddr(c), r);
        float y[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) y[e] = 0.f;
        for (int k = 0, i = 0; k < KS; ++k) {
          if (k == ks) {
#pragma unroll
            for (int e = 0; e < 16; ++e) y[e] += __uint_as_float(r[e]);
            continue;
          }
          // row-major 64-B rows: read the 4 float4 rotated by (row >> 1) & 3 (no bank conflicts)
          const float4 *s4 = reinterpret_cast<const float4 *>(stg + ((size_t)(c - c0) * (KS - 1) + i) * kChunkFloats +
                                                              row * 16);
          const int rot = (row >> 1) & 3;
          const float4 f0 = s4[rot], f1 = s4[(rot + 1) & 3], f2 = s4[(rot + 2) & 3], f3 = s4[(rot + 3) & 3];
#pragma unroll
          for (int v = 0; v < 4; ++v) {                     // float4 v was loaded as f_{(v - rot) & 3}
            const int k = (v - rot) & 3;
            const float4 f = k == 0 ? f0 : k == 1 ? f1 : k == 2 ? f2 : f3;
            y[4 * v] += f.x; y[4 * v + 1] += f.y; y[4 * v + 2] += f.z; y[4 * v + 3] += f.w;
          }
          ++i;
        }
        if (row < p.C) {
          const int m = c / cpm, cc = c - m * cpm;
          uint32_t o8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(y[2 * e], y[2 * e + 1]);
            o8[e] = *reinterpret_cast<uint32_t *>(&h2);
          }
          uint4 *dst = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.Y) +
                                                 ((size_t)(g * mpc + m) * p.C + row) * p.d_model + n0 + cc * 16);
          dst[0] = make_uint4(o8[0], o8[1], o8[2], o8[3]);
          dst[1] = make_uint4(o8[4], o8[5], o8[6], o8[7]);
        }
      }
      named_bar<1, 128>();                                  // staging buffer free for the next batch
    }
    if (KS > 1 && et == 0) {                                // the tile's last finisher re-arms its ticket
      if (atomicAdd(p.tickets + gj, 1) == 2 * KS - 1) p.tickets[gj] = 0;
    }
  }
  tc_fence_before();
  __syncwarp();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace

// Plan (MPC, T, KS, widths) for n members with K blocks of bk: minimise the modelled time of
// one wave (every tile resident at once) = per-CTA L2 -> SM bytes / bytes in flight (the ring
// minus the stage being consumed: r2 ncu of both chunk kernels, ~2-2.5 µs effective TMA round
// trips, rate = in-flight / latency), widths multiples of 32 (two N halves of 16-multiples),
// MPC·w_hi ≤ 512 TMEM columns, ≥ 3 ring stages.  False when no single-wave plan exists.
bool plan_read_chunk_wide(int n, int d_model, int d_ff, int sms, int bk, WidePlan *out) {
  WidePlan best{};
  double best_cost = 1e30;
  if (bk != 16 && bk != 32 && bk != 64) return false;
  if (d_ff % bk) return false;
  const int nk = d_ff / bk;
  for (int mpc = 1; mpc <= 2; ++mpc) {
    if (n % mpc) continue;
    const int groups = n / mpc;
    for (int T = 1; T <= d_model / 32; ++T) {
      const int w_lo = d_model / T / 32 * 32;
      if (w_lo < 32) break;
      int w_hi = w_lo + 32, h = (d_model - T * w_lo) / 32;
      if (T * w_lo + 32 * h != d_model || h > T) continue;
      if (h == 0) w_hi = w_lo;                                // all blocks w_lo wide: plan as w_hi = w_lo, h = T
      const int hh = h == 0 ? T : h;
      if (mpc * w_hi > 512 || w_hi / 2 > 256) continue;
      const int stage = ((mpc * WBM + (1 + mpc) * w_hi) * bk * 2 + 1023) / 1024 * 1024;
      const int stages = std::min(kWMaxStages, kSmemAvail / stage);
      if (stages < 3) continue;
      for (int KS = 1; KS <= 8; ++KS) {
        const long long tiles = (long long)groups * T * KS;
        if (tiles > sms) break;
        if (nk / KS < 2 * stages) break;
        const double kbytes = (double)((nk + KS - 1) / KS) * bk * 2 * (mpc * WBM + (1 + mpc) * w_hi);
        const double fin = KS > 1 ? 2.0 * (KS - 1) / KS * mpc * w_hi * WBM * 4 : 0.0;
        const double cost = (kbytes + fin) / ((double)(stages - 1) * stage);
        if (cost < best_cost) {
          best_cost = cost;
          best = WidePlan{mpc, T, KS, w_hi, hh, stages, stage, cost, (int)tiles, bk};
        }
      }
    }
  }
  if (best.T == 0) return false;
  *out = best;
  return true;
}

template <int BK>
cudaError_t launch_wide_bk(const CUtensorMap *maps, const WideParams &p, const WidePlan &pl, cudaStream_t s) {
  const size_t smem = 1024 + (size_t)pl.stages * pl.stage_bytes + (2 * kWMaxStages + 2) * 8 + 16;
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(read_chunk_wide_kernel<BK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.tiles);
  cfg.blockDim = dim3(kWThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  // split-K tiles spin on their ticket: co-residency of the whole grid is required
  static const int coop = getenv("TTT_WIDE_COOP") ? atoi(getenv("TTT_WIDE_COOP")) : 1;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pl.KS > 1 && coop) ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, read_chunk_wide_kernel<BK>, maps[0], maps[1], maps[2], maps[3], maps[4], p);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_read_chunk_wide(const ChunkLaunch &cl, const WidePlan &pl, cudaStream_t s) {
  WideParams p{};
  p.n = cl.n; p.d_model = cl.d_model; p.d_ff = cl.d_ff; p.C = cl.C; p.L = cl.L; p.layer = cl.layer;
  p.mpc = pl.mpc; p.T = pl.T; p.KS = pl.KS; p.w_hi = pl.w_hi; p.h = pl.h;
  p.stages = pl.stages; p.stage_bytes = (uint32_t)pl.stage_bytes;
  p.sel = cl.sel; p.owner_idx = cl.d_members;
  p.X = cl.X; p.Vt = cl.Vt; p.Y = cl.Y; p.tailZ = cl.tailZ; p.tailV = cl.tailV;
  p.tz_owner = cl.tz_owner; p.tv_owner = cl.tv_owner; p.tz_layer = cl.tz_layer; p.tv_layer = cl.tv_layer;
  p.append = cl.append;
  p.slab = cl.wide_slab;
  p.tickets = cl.wide_tickets;
  if (!p.owner_idx || (pl.KS > 1 && (!p.slab || !p.tickets))) return cudaErrorInvalidValue;
  if ((size_t)pl.tiles * pl.mpc * pl.w_hi / 16 * kChunkFloats * 4 > cl.wide_slab_bytes) return cudaErrorInvalidValue;
  CUtensorMap maps[5];
  const int w_lo = pl.h == pl.T ? pl.w_hi : pl.w_hi - 32, bk = pl.bk, sw = 2 * bk;
  const uint64_t dslots = (uint64_t)cl.max_slots * cl.L;
  if (!cached_map(&maps[0], cl.X, cl.d_ff, cl.C, cl.n, bk, WBM, sw) ||
      !cached_map(&maps[1], cl.w_down, cl.d_ff, cl.d_model, cl.L, bk, pl.w_hi / 2, sw) ||
      !cached_map(&maps[2], cl.w_down, cl.d_ff, cl.d_model, cl.L, bk, w_lo / 2, sw) ||
      !cached_map(&maps[3], cl.slots, cl.d_ff, cl.d_model, dslots, bk, pl.w_hi / 2, sw) ||
      !cached_map(&maps[4], cl.slots, cl.d_ff, cl.d_model, dslots, bk, w_lo / 2, sw))
    return cudaErrorInvalidValue;
  switch (bk) {
    case 16: return launch_wide_bk<16>(maps, p, pl, s);
    case 32: return launch_wide_bk<32>(maps, p, pl, s);
    case 64: return launch_wide_bk<64>(maps, p, pl, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ttt
