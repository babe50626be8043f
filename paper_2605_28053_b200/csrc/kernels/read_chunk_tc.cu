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
//  * 1 persistent CTA per SM, tiles (member, N-block of BN = 160 or 128);
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
  float *Y32;
  long long y32_slab;
  int owner_idx[kMaxGroup];
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    read_chunk_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                         const __grid_constant__ CUtensorMap tmD, const ChunkParams p) {
  constexpr int kTmemCols = BN <= 128 ? 128 : 256;
  constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;
  constexpr uint32_t STAGE = A_BYTES + 2 * B_BYTES;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  u64 *bars = reinterpret_cast<u64 *>(smem + kStages * STAGE);
  u64 *full = bars, *empty = bars + kStages, *t_full = bars + 2 * kStages, *t_empty = t_full + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(t_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = p.d_model / BN, nk_all = p.d_ff / BK, KS = p.ksplit;
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
          mbar_expect_tx(full + s, p.delta ? STAGE : A_BYTES + B_BYTES);
          tma_load_3d(st, &tmX, full + s, kb * BK, 0, b);
          tma_load_3d(st + A_BYTES, &tmW, full + s, kb * BK, j * BN, p.layer);
          if (p.delta) tma_load_3d(st + A_BYTES + B_BYTES, &tmD, full + s, kb * BK, j * BN, slot_l);
        }
      }
    }
  } else if (warp == 1) {                                   // ---------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16(BM, BN, 0, 0);
    int it = 0, k = 0;
    for (int u = blockIdx.x; u < n_tiles; u += gridDim.x, ++k) {
      int b, j, kb0, kb1;
      decode(u, b, j, kb0, kb1);
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
      __nv_bfloat16 *yrow = static_cast<__nv_bfloat16 *>(p.Y) + ((size_t)b * p.C + row) * p.d_model + j * BN;
      float *yrow32 = p.Y32 ? p.Y32 + ks * p.y32_slab + ((size_t)b * p.C + row) * p.d_model + j * BN : nullptr;
      const bool valid = row < p.C && (!p.Y32 || b * p.C + row < p.valid_rows);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32), r);
        if (valid && yrow32) {
          float4 *d4 = reinterpret_cast<float4 *>(yrow32 + c * 32);
#pragma unroll
          for (int v = 0; v < 8; ++v)
            d4[v] = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]), __uint_as_float(r[4 * v + 2]),
                                __uint_as_float(r[4 * v + 3]));
        } else if (valid) {
          uint32_t o16[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
            o16[e] = *reinterpret_cast<uint32_t *>(&h);
          }
          uint4 *dst = reinterpret_cast<uint4 *>(yrow + c * 32);
#pragma unroll
          for (int v = 0; v < 4; ++v) dst[v] = make_uint4(o16[4 * v], o16[4 * v + 1], o16[4 * v + 2], o16[4 * v + 3]);
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
  const int tiles = p.n * (p.d_model / BN) * p.ksplit;
  read_chunk_tc_kernel<BN><<<std::min(device_sm_count(), tiles), kThreads, smem, s>>>(mX, mW, mD, p);
  count_launch();
  return cudaGetLastError();
}

// wave efficiency of BN on this device (tiles / (waves * SMs))
double wave_eff(int tiles, int sms) {
  const int waves = (tiles + sms - 1) / sms;
  return (double)tiles / ((double)waves * sms);
}

}  // namespace

bool read_chunk_supported(int d_model, int d_ff, int C) {
  return C >= 1 && C <= BM && d_ff % BK == 0 && (d_model % 160 == 0 || d_model % 128 == 0) &&
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
  const bool can160 = cl.d_model % 160 == 0, can128 = cl.d_model % 128 == 0;
  const bool use160 =
      can160 && (!can128 || wave_eff(cl.n * (cl.d_model / 160) * std::max(1, cl.ksplit), sms) >=
                                 wave_eff(cl.n * (cl.d_model / 128) * std::max(1, cl.ksplit), sms));
  const int BN = use160 ? 160 : 128;
  CUtensorMap mX, mW, mD;
  if (!ptx::make_map_bf16_3d(&mX, cl.X, cl.d_ff, cl.C, cl.n, BK, BM) ||
      !ptx::make_map_bf16_3d(&mW, cl.w_down, cl.d_ff, cl.d_model, cl.L, BK, BN) ||
      !ptx::make_map_bf16_3d(&mD, cl.delta ? cl.slots : cl.w_down, cl.d_ff, cl.d_model,
                             cl.delta ? (uint64_t)cl.max_slots * cl.L : (uint64_t)cl.L, BK, BN))
    return cudaErrorInvalidValue;
  return use160 ? launch_bn<160>(mX, mW, mD, p, s) : launch_bn<128>(mX, mW, mD, p, s);
}

}  // namespace ttt
