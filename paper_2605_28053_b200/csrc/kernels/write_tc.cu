// a5 — WRITE (BoundaryUpdate) on 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// PAPER: the update "reads owner r's committed version v and produces one
// dirty candidate state for that owner ... invisible to later READs until
// committed" (WRITE paragraph P:410-417; Table 3 BoundaryUpdate P:387-390).
// Rule (SURVEY.md §8(c) reading i):
//     ΔW̃_{v+1}[i][j] = ΔW_v[i][j] + η · Σ_{t<C} V_c[t][i] · Z_c[t][j]
// i.e. a GEMM with M = d_model (i), N = d_ff (j), K = C, whose operands are
// the owner's tail rings exactly as READ appended them: V_c [C][d_model] and
// Z_c [C][d_ff] are both MN-major (MN contiguous), which UMMA reads natively
// (instruction-descriptor a_major = b_major = MN) — no transpose pass.
//
// B200 design (DESIGN.md §"WRITE kernel"): AI ≈ C/2 = 64 flop/B at C = 128,
// below the ridge (≈ 213-253), so the kernel is HBM-bound on ΔW bytes (read
// v, write v+1); tensor cores are needed because SIMT FFMA would be ~5×
// slower than the HBM bound at C = 128.
//  * persistent, 1 CTA per SM; the (member, j-block, i-block) 128×128 tiles
//    of one layer are split into 148 contiguous ranges; j-major order keeps
//    the Z_c tile (B operand) resident while V_c tiles (A) stream;
//  * warp 0: TMA producer (A ring ×2, B, committed-ΔW tile ring ×2);
//    warp 1: TMEM allocator + single-thread tcgen05.mma issuer
//    (M=128, N=128, K=16 per instruction, fp32 accumulate), commits to
//    mbarriers; warps 2-5: epilogue — tcgen05.ld 32 columns per thread, fp32
//    ΔW_v + η·acc, RNE to bf16 in place in the swizzled staging tile, TMA
//    store to the shadow slot; two TMEM accumulators overlap MMA(t+1) with
//    epilogue(t);
//  * the committed slot 2o+sel[o] is read and the shadow slot 2o+1−sel[o]
//    written (device active-slot table); a non-finite candidate raises its
//    owner's device fail flag and the commit kernel refuses
//    that member (control.cu: device-side App. H resolution).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "../internal.h"

namespace ttt {
namespace {

constexpr int BM = 128, BN = 128;
constexpr int kEpiThreads = 256;                 // 8 epilogue warps: 2 per TMEM lane quarter
constexpr int kThreads = 64 + kEpiThreads;      // producer warp, MMA warp, 8 epilogue warps
constexpr int kTmemCols = 2 * BN;                 // two fp32 accumulators of 128 columns
constexpr int kBox = BM * 128;                    // one 128-row x 64-column bf16 box (16 KB)
#ifndef TTT_WRITE_SB
#define TTT_WRITE_SB 7
#endif
#ifndef TTT_WRITE_ST
#define TTT_WRITE_ST 3
#endif
constexpr int kSB = TTT_WRITE_SB;                 // committed-ΔW box ring depth (3.5 tiles ahead)
constexpr int kST = TTT_WRITE_ST;                 // TMA stores in flight (read side); kSB - kST boxes of load lookahead

typedef unsigned long long u64;

struct TcParams {
  int n, d_model, d_ff, C, L, layer;
  const int *sel;
  float eta;
  int *mfail;
  int owner_idx[kMaxGroup];
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(u64 *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(u64 *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64 *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, u64 *bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, const void *src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
// UMMA shared-memory descriptor (sm_100): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version 1 [46,48), base offset 0, layout SWIZZLE_128B = 2 [61,64).
__device__ __forceinline__ u64 smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  u64 d = 0;
  d |= (u64)((addr >> 4) & 0x3FFF);
  d |= (u64)((lbo >> 4) & 0x3FFF) << 16;
  d |= (u64)((sbo >> 4) & 0x3FFF) << 32;
  d |= (u64)1 << 46;
  d |= (u64)2 << 61;
  return d;
}
// kind::f16 instruction descriptor: D fp32, A/B bf16, A and B MN-major, M=128, N=128.
__host__ __device__ constexpr uint32_t instr_desc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, u64 adesc, u64 bdesc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(u64 *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ u64 pack_u2(uint32_t lo, uint32_t hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ u64 pack_f2(float lo, float hi) { return pack_u2(__float_as_uint(lo), __float_as_uint(hi)); }
// v = a*b + v on fp32 pairs (FFMA2)
__device__ __forceinline__ void ffma2(u64 &v, u64 a, u64 b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(v) : "l"(a), "l"(b));
}
// fp32 pair -> packed bf16x2 (low half = first element), round to nearest even
__device__ __forceinline__ uint32_t cvt_bf16x2(u64 v) {
  uint32_t lo, hi, r;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float(hi)), "f"(__uint_as_float(lo)));
  return r;
}

struct Tile {
  int b, jb, ib;
};

__global__ void __launch_bounds__(kThreads, 1)
    write_tc_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmZ,
                    const __grid_constant__ CUtensorMap tmW, const TcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned carve-up: A ring [2][C x 128], B [C x 128], S (ΔW tile) ring [2][128 x 128]
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int C = p.C;
  const uint32_t a_bytes = (uint32_t)C * BM * 2, b_bytes = (uint32_t)C * BN * 2;
  unsigned char *sA = smem;                       // 2 stages
  unsigned char *sB = sA + 2 * a_bytes;
  unsigned char *sS = sB + b_bytes;               // kSB boxes of 16 KB
  u64 *bars = reinterpret_cast<u64 *>(sS + kSB * kBox);
  u64 *a_full = bars, *a_empty = bars + 2, *b_full = bars + 4, *b_empty = bars + 5;
  u64 *t_full = bars + 6, *t_empty = bars + 8, *s_full = bars + 10, *s_empty = bars + 10 + kSB;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 10 + 2 * kSB);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mb = p.d_model / BM, nb = p.d_ff / BN;
  const int per_member = mb * nb;
  const int n_tiles = p.n * per_member;
  const int t0 = (int)((long long)n_tiles * blockIdx.x / gridDim.x);
  const int t1 = (int)((long long)n_tiles * (blockIdx.x + 1) / gridDim.x);
  auto tile_of = [&](int t) {
    Tile r;
    r.b = t / per_member;
    const int rem = t - r.b * per_member;
    r.jb = rem / mb;
    r.ib = rem - r.jb * mb;
    return r;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(a_full + s, 1);
      mbar_init(a_empty + s, 1);
      mbar_init(t_full + s, 1);
      mbar_init(t_empty + s, kEpiThreads / 32);
    }
    for (int s = 0; s < kSB; ++s) {
      mbar_init(s_full + s, 1);
      mbar_init(s_empty + s, 1);
    }
    mbar_init(b_full, 1);
    mbar_init(b_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  // PDL: only the prologue above overlaps the previous kernel (the layer's READ or WRITE);
  // the tails, slots and the active-slot table are read after the wait.
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch(&tmV);
      tma_prefetch(&tmZ);
      tma_prefetch(&tmW);
      int k = 0, kb = 0, strip = -1, nstrip = 0;
      for (int t = t0; t < t1; ++t, ++k) {
        const Tile tl = tile_of(t);
        const int o = p.owner_idx[tl.b];
        const int tail_idx = o * p.L + p.layer;
        const int sid = tl.b * nb + tl.jb;
        if (sid != strip) {                       // new (member, j-block): reload the resident Z_c tile
          if (nstrip > 0) mbar_wait(b_empty, (nstrip - 1) & 1);
          mbar_expect_tx(b_full, b_bytes);
          for (int h = 0; h < BN / 64; ++h)
            tma_load_3d(sB + h * (C * 128), &tmZ, b_full, tl.jb * BN + 64 * h, 0, tail_idx);
          strip = sid;
          ++nstrip;
        }
        const int s = k & 1;
        if (k >= 2) mbar_wait(a_empty + s, ((k >> 1) - 1) & 1);
        mbar_expect_tx(a_full + s, a_bytes);
        for (int h = 0; h < BM / 64; ++h)
          tma_load_3d(sA + s * a_bytes + h * (C * 128), &tmV, a_full + s, tl.ib * BM + 64 * h, 0, tail_idx);
        const int src_slot = 2 * o + p.sel[o];
        for (int h = 0; h < BN / 64; ++h, ++kb) {
          const int sb = kb % kSB;
          if (kb >= kSB) mbar_wait(s_empty + sb, ((kb / kSB) - 1) & 1);
          mbar_expect_tx(s_full + sb, kBox);
          tma_load_3d(sS + sb * kBox, &tmW, s_full + sb, tl.jb * BN + 64 * h, tl.ib * BM, src_slot * p.L + p.layer);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = instr_desc();
    int k = 0, strip = -1, nstrip = 0;
    for (int t = t0; t < t1; ++t, ++k) {
      const Tile tl = tile_of(t);
      const int sid = tl.b * nb + tl.jb;
      if (sid != strip) {
        mbar_wait(b_full, nstrip & 1);
        strip = sid;
        ++nstrip;
      }
      const int s = k & 1, acc = k & 1;
      mbar_wait(a_full + s, (k >> 1) & 1);
      if (k >= 2) mbar_wait(t_empty + acc, ((k >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t a0 = smem_u32(sA + s * a_bytes), b0 = smem_u32(sB);
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * BN);
        for (int kk = 0; kk < C / 16; ++kk) {
          // K step of 16 rows = two 8-row swizzle atoms = 2048 bytes; LBO = one 64-wide MN box
          const u64 ad = smem_desc(a0 + kk * 2048, (uint32_t)C * 128, 1024);
          const u64 bd = smem_desc(b0 + kk * 2048, (uint32_t)C * 128, 1024);
          mma_bf16(tmem_d, ad, bd, idesc, kk > 0 ? 1u : 0u);
        }
        mma_commit(a_empty + s);                  // A stage free once these MMAs retire
        mma_commit(t_full + acc);                 // accumulator ready for the epilogue
        const bool last_of_strip = (t + 1 >= t1) || (tile_of(t + 1).b * nb + tile_of(t + 1).jb != sid);
        if (last_of_strip) mma_commit(b_empty);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2-9)
    const int q = warp & 3;                       // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;             // which 32-column half of each 64-column box
    const int row = q * 32 + lane;                // output row within the tile
    const int et = threadIdx.x - 64;
    uint32_t expmax = 0;                          // max exponent field seen (non-finite guard)
    const u64 eta2 = pack_f2(p.eta, p.eta);
    int k = 0, kb = 0;
    for (int t = t0; t < t1; ++t, ++k) {
      const Tile tl = tile_of(t);
      const int acc = k & 1;
      mbar_wait(t_full + acc, (k >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int o = p.owner_idx[tl.b];
      const int dst_slot = 2 * o + 1 - p.sel[o];
      for (int h = 0; h < BN / 64; ++h, ++kb) {
        const int sb = kb % kSB;
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + h * 64 + half * 32), r);
        if (h == BN / 64 - 1) {                   // this warp has drained its part of the accumulator
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(t_empty + acc);
        }
        mbar_wait(s_full + sb, (kb / kSB) & 1);
        unsigned char *rowp = sS + sb * kBox + row * 128;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int ch = (half * 4 + u) ^ (row & 7);  // 128-byte swizzle: 16-byte chunk ^ (row % 8)
          uint4 *ptr = reinterpret_cast<uint4 *>(rowp + ch * 16);
          uint4 w = *ptr;
          uint32_t *wv = reinterpret_cast<uint32_t *>(&w);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            // (ΔW_v lo, hi) + η·(acc lo, hi) in fp32x2, one RNE pack to bf16x2
            u64 a2 = pack_u2(r[u * 8 + 2 * e], r[u * 8 + 2 * e + 1]);
            u64 v2 = pack_u2(wv[e] << 16, wv[e] & 0xffff0000u);
            ffma2(v2, eta2, a2);
            const uint32_t ob = cvt_bf16x2(v2);
            expmax = __vmaxu2(expmax, ob & 0x7f807f80u);
            wv[e] = ob;
          }
          *ptr = w;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // smem writes -> TMA store
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
        if (et == 0) {
          tma_store_3d(&tmW, sS + sb * kBox, tl.jb * BN + 64 * h, tl.ib * BM, dst_slot * p.L + p.layer);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kST) : "memory");   // box kb-kST read out
          if (kb >= kST) mbar_arrive(s_empty + (kb - kST) % kSB);
        }
      }
      // per-member non-finite guard: flag this tile's owner (the commit resolves members)
      if ((expmax & 0x7f80u) == 0x7f80u || (expmax >> 16) == 0x7f80u) atomicOr(p.mfail + o, 1);
      expmax = 0;
    }
    if (et == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols));
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_map(CUtensorMap *m, void *base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * 2, d0 * d1 * 2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

size_t smem_bytes(int C) { return 1024 + 2 * (size_t)C * BM * 2 + (size_t)C * BN * 2 + (size_t)kSB * kBox + 512; }

}  // namespace

bool write_tc_supported(int d_model, int d_ff, int C) {
  return d_model % BM == 0 && d_ff % BN == 0 && C % 16 == 0 && C >= 16 && C <= 128 && smem_bytes(C) <= 227 * 1024 &&
         encode_fn() != nullptr;
}

cudaError_t launch_write_tc(const WriteParams &wp, cudaStream_t s) {
  // Tensor maps over the whole arena regions: tails V [owners*L][C][d_model],
  // Z [owners*L][C][d_ff]; pool slots [n_slots*L][d_model][d_ff].
  const int L = (int)(wp.tz_owner / ((long long)wp.C * wp.d_ff));
  const long long n_slots_L = wp.max_slots * (long long)L;
  CUtensorMap mV, mZ, mW;
  if (!make_map(&mV, const_cast<void *>(wp.tailV), wp.d_model, wp.C, (uint64_t)wp.max_owners * L, 64, wp.C) ||
      !make_map(&mZ, const_cast<void *>(wp.tailZ), wp.d_ff, wp.C, (uint64_t)wp.max_owners * L, 64, wp.C) ||
      !make_map(&mW, wp.slots, wp.d_ff, wp.d_model, (uint64_t)n_slots_L, 64, BM))
    return cudaErrorInvalidValue;
  TcParams p{};
  p.n = wp.n;
  p.d_model = wp.d_model;
  p.d_ff = wp.d_ff;
  p.C = wp.C;
  p.L = L;
  p.layer = (int)(wp.layer_off / ((long long)wp.d_model * wp.d_ff));
  p.sel = wp.sel;
  p.eta = wp.eta;
  p.mfail = wp.mfail;
  for (int b = 0; b < wp.n; ++b) p.owner_idx[b] = wp.owner_idx[b];
  const size_t smem = smem_bytes(wp.C);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(write_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  const int tiles = wp.n * (wp.d_model / BM) * (wp.d_ff / BN);
  const int grid = std::min(device_sm_count(), tiles);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, write_tc_kernel, mV, mZ, mW, p);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace ttt
