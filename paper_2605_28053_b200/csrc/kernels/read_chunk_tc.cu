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
#include "../internal.h"
#include "sm100_ptx.cuh"

namespace ttt {
namespace {

using namespace ptx;

constexpr int BM = 128, BK = 64, kStages = 4;
constexpr int kThreads = 192;

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
  int owner_idx[kMaxGroup];
};

template <int BN>   // BN: largest N-block (smem stage size); actual widths are runtime
__global__ void __launch_bounds__(kThreads, 1)
    read_chunk_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                         const __grid_constant__ CUtensorMap tmD, const ChunkParams p) {
  constexpr int kTmemCols = BN <= 128 ? 128 : 256;
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;   // stage slots sized for BN rows
  const uint32_t b_box = (uint32_t)p.w_hi * BK * 2;                   // bytes one B box actually lands
  constexpr uint32_t STAGE = A_BYTES + 2 * B_BYTES;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  u64 *bars = reinterpret_cast<u64 *>(smem + kStages * STAGE);
  u64 *full = bars, *empty = bars + kStages, *t_full = bars + 2 * kStages, *t_empty = t_full + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(t_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = p.nt, nk_all = p.d_ff / BK, KS = p.ksplit;
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

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(t_full, 1);
    mbar_init(t_empty, 4);
    mbar_init_fence();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {                                        // ---------------- TMA producer
      tma_prefetch(&tmX);
      tma_prefetch(&tmW);
      tma_prefetch(&tmD);
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
          mbar_expect_tx(full + s, A_BYTES + (p.delta ? 2 : 1) * b_box);
          tma_load_3d(st, &tmX, full + s, kb * BK, 0, b);
          tma_load_3d(st + A_BYTES, &tmW, full + s, kb * BK, n0_of(j), p.layer);
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
  } else {                                                  // ---------------- epilogue warps 2-5
    const int q = warp & 3, row = q * 32 + lane;            // token index t in the chunk
    const int et = threadIdx.x - 64;
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
#pragma unroll 1
      for (int c = 0; c < width / 16; ++c) {      // 16 accumulator columns at a time
        uint32_t r[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 16), r);
        if (valid && yrow32) {
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
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kTmemCols>(tmem);
}

template <int BN>
size_t smem_bytes() {
  return 1024 + (size_t)kStages * (BM * BK * 2 + 2 * BN * BK * 2) + 256;
}

template <int BN>
cudaError_t launch_bn(const CUtensorMap &mX, const CUtensorMap &mW, const CUtensorMap &mD, const ChunkParams &p,
                      cudaStream_t s) {
  const size_t smem = smem_bytes<BN>();
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(read_chunk_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int tiles = p.n * p.nt * p.ksplit;
  read_chunk_tc_kernel<BN><<<std::min(device_sm_count(), tiles), kThreads, smem, s>>>(mX, mW, mD, p);
  count_launch();
  return cudaGetLastError();
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
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = {T, w_hi, h};
    }
  }
  return best;
}

}  // namespace

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
  for (int b = 0; b < cl.n; ++b) p.owner_idx[b] = cl.owner_idx[b];
  const int sms = device_sm_count();
  const NPlan np = plan_n(cl.d_model, cl.n * std::max(1, cl.ksplit), sms);
  if (np.T == 0) return cudaErrorInvalidValue;
  p.nt = np.T;
  p.w_hi = np.w_hi;
  p.h = np.h;
  CUtensorMap mX, mW, mD;
  if (!ptx::make_map_bf16_3d(&mX, cl.X, cl.d_ff, cl.C, cl.n, BK, BM) ||
      !ptx::make_map_bf16_3d(&mW, cl.w_down, cl.d_ff, cl.d_model, cl.L, BK, np.w_hi) ||
      !ptx::make_map_bf16_3d(&mD, cl.delta ? cl.slots : cl.w_down, cl.d_ff, cl.d_model,
                             cl.delta ? (uint64_t)cl.max_slots * cl.L : (uint64_t)cl.L, BK, np.w_hi))
    return cudaErrorInvalidValue;
  return launch_bn<160>(mX, mW, mD, p, s);
}

}  // namespace ttt
