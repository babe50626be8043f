// C-ABI implementation: TTTState pool (double-slot arena + host mirror),
// READ/WRITE/commit enqueue with validation-before-side-effects, control
// operations (snapshot / rollback / fork), sync and test hooks.
//
// Contract sources: ownership rule P:233-246; Eq. 2-3; StateView
// P:346-352; primitives Table 3; Alg. 1 P:442-466;
// SPEC state_core S:56-146 and executor S:355-409 for error conventions.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_set>

#include "pool.h"

#include <nvtx3/nvToolsExt.h>

// NVTX ranges around the hot-path entry points (SURVEY §5 tracing): no-ops unless a tool
// (Nsight Systems / ncu --nvtx) is attached; `ncu --nvtx --nvtx-include "read_apply/"` filters
namespace {
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace ttt {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};
static std::atomic<int> g_write_impl{0};
static std::atomic<int> g_test_hook{0};   // tttstate_set_test_hook (stress negative control)
// Live device low-rank pools in this process: the fused low-rank READ spin-waits across its
// CTAs, so with two such pools (two streams) its launches become cooperative (co-residency
// guaranteed by the driver); a lone pool keeps the cheaper PDL launch.
std::atomic<int> g_live_lowrank_pools{0};

void count_launch(int n) { g_launches += n; }

int device_sm_count() {
  static int cached_dev = -1, cached = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    cached_dev = dev;
  }
  return cached;
}

void set_last_error(const std::string &msg) { g_last_error = msg; }

static ttt_status fail(ttt_status s, const std::string &msg) {
  g_last_error = std::string(tttstate_status_name(s)) + ": " + msg;
  return s;
}

static ttt_status cuda_fail(cudaError_t e, const char *what) {
  return fail(TTT_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(expr)                                   \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr);  \
  } while (0)

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t payload_elems(const ttt_shape &s) {
  return s.backend == TTT_LOW_RANK ? (size_t)s.rank * (s.d_ff + s.d_model) : (size_t)s.d_model * s.d_ff;
}

Layout compute_layout(const ttt_shape &s, int max_owners, int n_ckpt) {
  const size_t es = s.dtype == TTT_BF16 ? 2 : 4;
  const size_t E = payload_elems(s);
  const size_t slot = (size_t)s.n_layers * E * es;
  Layout L;
  size_t off = 0;
  L.slots = off;   off = align_up(off + slot * (2 * (size_t)max_owners + n_ckpt), 1024);
  L.tailZ = off;   off = align_up(off + (size_t)max_owners * s.n_layers * s.chunk * s.d_ff * es, 1024);
  L.tailV = off;   off = align_up(off + (size_t)max_owners * s.n_layers * s.chunk * s.d_model * es, 1024);
  L.sel = off;     off = align_up(off + (size_t)max_owners * 4, 256);
  L.ver = off;     off = align_up(off + (size_t)max_owners * 8, 256);
  L.flags = off;   off = align_up(off + 64, 256);                  // fail_count, refusal-log counter
  L.mfail = off;   off = align_up(off + (size_t)max_owners * 4, 256);  // per-owner device-failure flags
  L.rlog = off;    off = align_up(off + (size_t)kRefusalLog * sizeof(RefusalRec), 256);
  L.members = off; off = align_up(off + sizeof(MemberTable), 256);
  // READ partials: base K-chunk slabs [kc][8][d_model] (kc ≤ ⌈d_ff/512⌉) + ΔW [8][d_model]
  L.P = off;       off = align_up(off + ((size_t)(s.d_ff + 511) / 512 + 1) * kMaxReadMembers * s.d_model * 4, 256);
  L.tickets = off; off = align_up(off + (size_t)s.d_model * 4, 1024);
  if (s.backend == TTT_FAST_WEIGHT && s.dtype == TTT_BF16) {                     // decode READ on tcgen05
    L.ptc_bytes = (size_t)2 * kTcMaxG * ((s.d_model + 127) / 128 * 128) * 8 * 4;
    L.ptc = off; off = align_up(off + L.ptc_bytes, 1024);
  }
  L.xflag = off; off = align_up(off + 4, 1024);
  if (s.backend == TTT_FAST_WEIGHT && s.dtype == TTT_BF16 && s.chunk <= 128) {   // wide chunk READ (f2)
    L.wtick = off; off = align_up(off + (size_t)kWideMaxTiles * 4, 1024);
    L.wslab = off; off = align_up(off + kWideSlabBytes, 1024);
  }
  if (s.backend == TTT_LOW_RANK) {
    const size_t rows = align_up((size_t)max_owners, 128);
    L.Xg = off;  off = align_up(off + rows * s.d_ff * es, 1024);
    L.Y32 = off; off = align_up(off + (size_t)(kMaxKSplit + 1) * rows * s.d_model * 4, 1024);   // + Bᵀu slab
    L.U = off;   off = align_up(off + (size_t)max_owners * 64 * kMaxLrSeg * 4, 1024);
    L.Ctr = off; off = align_up(off + (8 + rows / 128 * ((size_t)s.d_model / 16 + 1)) * 4, 1024);
  }
  L.total = off;
  return L;
}

static ttt_status check_shape(const ttt_shape *s) {
  if (!s) return fail(TTT_E_INVALID_ARG, "null shape");
  if (s->backend != TTT_FAST_WEIGHT && s->backend != TTT_LOW_RANK)
    return fail(TTT_E_SHAPE, "backend must be fast-weight (τ=0) or low-rank (τ=1)");
  if (s->backend == TTT_LOW_RANK &&
      (s->rank < 1 || s->rank > 64 || s->dtype != TTT_BF16 || !read_chunk_supported(s->d_model, s->d_ff, 128)))
    return fail(TTT_E_SHAPE, "low-rank: rank in [1,64], bf16, d_ff % 64 == 0, d_model % 16 == 0 (>= 128)");
  if (s->dtype != TTT_BF16 && s->dtype != TTT_FP32) return fail(TTT_E_SHAPE, "dtype");
  if (s->d_model <= 0 || s->d_ff <= 0 || s->chunk <= 0 || s->n_layers <= 0)
    return fail(TTT_E_SHAPE, "non-positive dimension");
  const int vec = s->dtype == TTT_BF16 ? 8 : 4;
  if (s->d_ff % vec) return fail(TTT_E_SHAPE, "d_ff must be a multiple of 8 (bf16) / 4 (fp32)");
  if (s->d_model % 4) return fail(TTT_E_SHAPE, "d_model must be a multiple of 4");
  if (s->rule != 0 && !(s->rule == 1 && s->backend == TTT_FAST_WEIGHT && s->d_model == s->d_ff))
    return fail(TTT_E_SHAPE, "rule 1 (SPEC mean rule) needs the fast-weight backend and d_model == d_ff");
  return TTT_OK;
}

}  // namespace ttt

using namespace ttt;

// ---------------------------------------------------------------- helpers
namespace {

ttt_status find_owner(ttt_pool *p, uint64_t owner, OwnerRec **out) {
  auto it = p->owners.find(owner);
  if (it == p->owners.end()) return fail(TTT_E_UNKNOWN_OWNER, "owner " + std::to_string(owner));
  *out = &it->second;
  return TTT_OK;
}

// Key homogeneity (Eq. 3) against this pool, known owners, injective μ.
ttt_status check_group(ttt_pool *p, const ttt_group *g, std::vector<OwnerRec *> &recs) {
  if (!p || !g || !g->owner_map) return fail(TTT_E_INVALID_ARG, "null pool/group");
  if (g->n < 1 || g->n > kMaxGroup) return fail(TTT_E_CAPACITY, "group size must be in [1, 256]");
  if (g->backend != p->sh.backend || g->shape_id != p->shape_id || g->placement != p->placement)
    return fail(TTT_E_MIXED_KEY, "group key (τ,σ,π) does not match the pool");
  if (g->effect != TTT_READ && g->effect != TTT_WRITE) return fail(TTT_E_INVALID_ARG, "effect");
  recs.resize(g->n);
  const uint64_t epoch = ++p->stamp_epoch;         // μ injective: each record visited once per call
  for (int b = 0; b < g->n; ++b) {
    ttt_status st = find_owner(p, g->owner_map[b], &recs[b]);
    if (st != TTT_OK) return st;
    if (recs[b]->stamp == epoch)
      return fail(TTT_E_OWNER_COLLISION, "owner " + std::to_string(g->owner_map[b]) + " twice in μ");
    recs[b]->stamp = epoch;
  }
  return TTT_OK;
}

void clear_applied(OwnerRec &r) {
  std::fill(r.applied.begin(), r.applied.end(), 0);
  r.n_applied = 0;
  r.chunk_mode = false;
  r.fused_layers = 0;
}

// A pinned checkpoint in the shadow slot must move to the checkpoint pool
// before a WRITE overwrites the shadow (K5 checkpoint write).
bool pinned_in_shadow(const OwnerRec &r) { return r.has_ckpt && r.ckpt_pool < 0 && r.ckpt_sel == 1 - r.sel; }

void release_device(ttt_pool *p) {
  for (cudaEvent_t e : p->ev_ring)
    if (e) cudaEventDestroy(e);
  p->ev_ring.clear();
  if (p->hstate) cudaFreeHost(p->hstate);
  p->hstate = p->hstate_dev = nullptr;
}

// Lazy confirmation of an owner's latest write_commit (the host mirror advanced optimistically):
// wait for that commit's event — normally long complete — and take the device's outcome from the
// mapped host record.  A member the device refused (non-finite candidate, control.cu) returns to
// the version and slot it kept.  Called by every entry point that relies on the host's
// (version, sel) of this owner: snapshot, rollback, fork, free, version, and WRITE paths that may
// evict a pinned checkpoint.
ttt_status confirm(ttt_pool *p, OwnerRec &r) {
  if (!r.pending_seq) return TTT_OK;
  CUDA_TRY(cudaEventSynchronize(p->ev_ring[r.pending_seq % p->ev_ring.size()]));
  const volatile HostOwnerState *h = p->hstate + r.idx;
  if (h->seq != r.pending_seq)
    return fail(TTT_E_CUDA, "commit outcome record missing for seq " + std::to_string(r.pending_seq));
  r.version = h->version;
  r.sel = h->sel;
  r.pending_seq = 0;
  return TTT_OK;
}

// Upload a chunk / low-rank READ group's member table unless the device copy already holds it
// (every layer of a decode step reuses the same rows and tail positions: one upload per step).
cudaError_t upload_members(ttt_pool *p, const MemberTable &t, int n, cudaStream_t s) {
  bool same = p->m_n == n;
  for (int k = 0; k < 5 && same; ++k) same = std::memcmp(t.a[k], p->m_last.a[k], (size_t)n * sizeof(int)) == 0;
  if (same) return cudaSuccess;
  cudaError_t e = launch_member_upload(t, n, p->d_members(), s);
  if (e != cudaSuccess) return e;
  for (int k = 0; k < 5; ++k) std::memcpy(p->m_last.a[k], t.a[k], (size_t)n * sizeof(int));
  p->m_n = n;
  return cudaSuccess;
}

cudaError_t evict_pinned(ttt_pool *p, OwnerRec &r, cudaStream_t s) {
  const int c = p->free_ckpt.back();
  p->free_ckpt.pop_back();
  cudaError_t e = launch_copy(p->slot_ptr(2LL * p->max_owners + c), p->slot_ptr(2LL * r.idx + r.ckpt_sel),
                              p->slot_bytes(), s);
  r.ckpt_pool = c;
  return e;
}

}  // namespace

extern "C" {

const char *tttstate_last_error(void) { return g_last_error.c_str(); }

const char *tttstate_status_name(ttt_status s) {
  switch (s) {
    case TTT_OK: return "TTT_OK";
    case TTT_E_UNKNOWN_OWNER: return "TTT_E_UNKNOWN_OWNER";
    case TTT_E_DUPLICATE_OWNER: return "TTT_E_DUPLICATE_OWNER";
    case TTT_E_VERSION_MISMATCH: return "TTT_E_VERSION_MISMATCH";
    case TTT_E_OWNER_COLLISION: return "TTT_E_OWNER_COLLISION";
    case TTT_E_MIXED_KEY: return "TTT_E_MIXED_KEY";
    case TTT_E_DOUBLE_WRITE: return "TTT_E_DOUBLE_WRITE";
    case TTT_E_TAIL_NOT_FULL: return "TTT_E_TAIL_NOT_FULL";
    case TTT_E_NO_CHECKPOINT: return "TTT_E_NO_CHECKPOINT";
    case TTT_E_WRITE_FAILED: return "TTT_E_WRITE_FAILED";
    case TTT_E_POOL_FULL: return "TTT_E_POOL_FULL";
    case TTT_E_SHAPE: return "TTT_E_SHAPE";
    case TTT_E_TAIL_FULL: return "TTT_E_TAIL_FULL";
    case TTT_E_WRONG_EFFECT: return "TTT_E_WRONG_EFFECT";
    case TTT_E_NOT_APPLIED: return "TTT_E_NOT_APPLIED";
    case TTT_E_ALREADY_APPLIED: return "TTT_E_ALREADY_APPLIED";
    case TTT_E_CAPACITY: return "TTT_E_CAPACITY";
    case TTT_E_INVALID_ARG: return "TTT_E_INVALID_ARG";
    case TTT_E_CUDA: return "TTT_E_CUDA";
    case TTT_E_NO_DEVICE: return "TTT_E_NO_DEVICE";
  }
  return "TTT_E_?";
}

int64_t tttstate_launch_count(void) { return g_launches.load(); }

int32_t tttstate_set_write_impl(int32_t impl) { return g_write_impl.exchange(impl); }
int32_t tttstate_set_test_hook(int32_t flags) { return g_test_hook.exchange(flags); }

// ---------------------------------------------------------------- pool
ttt_status tttstate_pool_bytes(const ttt_shape *shape, int32_t max_owners, int32_t n_ckpt, size_t *bytes_out) {
  ttt_status st = check_shape(shape);
  if (st != TTT_OK) return st;
  if (max_owners < 1 || n_ckpt < 0 || !bytes_out) return fail(TTT_E_INVALID_ARG, "max_owners/n_ckpt/out");
  *bytes_out = compute_layout(*shape, max_owners, n_ckpt).total;
  return TTT_OK;
}

ttt_status tttstate_pool_create(const ttt_shape *shape, int32_t shape_id, int32_t placement, int32_t max_owners,
                                int32_t n_ckpt, void *dev_arena, size_t arena_bytes, const void *w_down,
                                ttt_pool **out) {
  ttt_status st = check_shape(shape);
  if (st != TTT_OK) return st;
  if (!out || max_owners < 1 || n_ckpt < 0) return fail(TTT_E_INVALID_ARG, "out/max_owners/n_ckpt");
  Layout lay = compute_layout(*shape, max_owners, n_ckpt);
  if (dev_arena) {
    if (arena_bytes < lay.total) return fail(TTT_E_INVALID_ARG, "arena too small");
    if (reinterpret_cast<uintptr_t>(dev_arena) % 1024) return fail(TTT_E_INVALID_ARG, "arena not 1024-aligned");
    if (!w_down) return fail(TTT_E_INVALID_ARG, "w_down is required for rule 0");
  }
  auto *p = new ttt_pool();
  p->sh = *shape;
  p->shape_id = shape_id;
  p->placement = placement;
  p->max_owners = max_owners;
  p->n_ckpt = n_ckpt;
  p->host_only = dev_arena == nullptr;
  p->arena = static_cast<unsigned char *>(dev_arena);
  p->arena_bytes = arena_bytes;
  p->w_down = w_down;
  p->esize = shape->dtype == TTT_BF16 ? 2 : 4;
  p->E = (long long)payload_elems(*shape);
  p->Ew = (long long)shape->d_model * shape->d_ff;
  p->slot_elems = p->E * shape->n_layers;
  p->tz_owner = (long long)shape->n_layers * shape->chunk * shape->d_ff;
  p->tv_owner = (long long)shape->n_layers * shape->chunk * shape->d_model;
  p->lay = lay;
  for (int i = max_owners - 1; i >= 0; --i) p->free_idx.push_back(i);
  for (int c = n_ckpt - 1; c >= 0; --c) p->free_ckpt.push_back(c);
  if (!p->host_only) {
    cudaError_t e = cudaMemset(p->arena + lay.sel, 0, lay.total - lay.sel);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    // commit outcomes: pinned device-mapped host memory (24 B per owner; not device memory)
    if (e == cudaSuccess)
      e = cudaHostAlloc(reinterpret_cast<void **>(&p->hstate), (size_t)max_owners * sizeof(HostOwnerState),
                        cudaHostAllocMapped);
    if (e == cudaSuccess) {
      std::memset(p->hstate, 0, (size_t)max_owners * sizeof(HostOwnerState));
      e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&p->hstate_dev), p->hstate, 0);
    }
    p->ev_ring.assign(kEventRing, nullptr);
    for (int k = 0; k < kEventRing && e == cudaSuccess; ++k)
      e = cudaEventCreateWithFlags(&p->ev_ring[k], cudaEventDisableTiming);
    if (e != cudaSuccess) {
      release_device(p);
      delete p;
      return cuda_fail(e, "pool tables init");
    }
  }
  if (!p->host_only && shape->backend == TTT_LOW_RANK) g_live_lowrank_pools.fetch_add(1);
  *out = p;
  return TTT_OK;
}

ttt_status tttstate_pool_destroy(ttt_pool *pool) {
  if (pool && !pool->host_only && pool->sh.backend == TTT_LOW_RANK) g_live_lowrank_pools.fetch_sub(1);
  if (pool) release_device(pool);
  delete pool;
  return TTT_OK;
}

ttt_status tttstate_alloc(ttt_pool *p, uint64_t owner, const void *init, uint64_t v0, uint64_t *v_out,
                          void *stream) {
  if (!p) return fail(TTT_E_INVALID_ARG, "null pool");
  if (p->owners.count(owner)) return fail(TTT_E_DUPLICATE_OWNER, "owner " + std::to_string(owner));
  if (p->free_idx.empty()) return fail(TTT_E_POOL_FULL, "no free owner slot");
  if (init && p->host_only) return fail(TTT_E_NO_DEVICE, "init bytes need a device pool");
  const int idx = p->free_idx.back();
  if (!p->host_only) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (init)
      CUDA_TRY(cudaMemcpyAsync(p->slot_ptr(2LL * idx), init, p->slot_bytes(), cudaMemcpyDeviceToDevice, s));
    else
      CUDA_TRY(cudaMemsetAsync(p->slot_ptr(2LL * idx), 0, p->slot_bytes(), s));
    CUDA_TRY(launch_set_state(p->d_sel(), p->d_ver(), p->d_mfail(), idx, 0, v0, s));
  }
  p->free_idx.pop_back();
  OwnerRec r;
  r.idx = idx;
  r.version = v0;
  r.applied.assign(p->sh.n_layers, 0);
  p->owners.emplace(owner, std::move(r));
  if (v_out) *v_out = v0;
  return TTT_OK;
}

ttt_status tttstate_free(ttt_pool *p, uint64_t owner) {
  if (!p) return fail(TTT_E_INVALID_ARG, "null pool");
  OwnerRec *r;
  ttt_status st = find_owner(p, owner, &r);
  if (st != TTT_OK) return st;
  if (r->ckpt_pool >= 0) p->free_ckpt.push_back(r->ckpt_pool);
  p->free_idx.push_back(r->idx);
  p->owners.erase(owner);
  return TTT_OK;
}

ttt_status tttstate_tail_load(ttt_pool *p, uint64_t owner, int32_t n, const void *Z, const void *V,
                              void *stream) {
  if (!p) return fail(TTT_E_INVALID_ARG, "null pool");
  OwnerRec *r;
  ttt_status st = find_owner(p, owner, &r);
  if (st != TTT_OK) return st;
  if (n < 0 || n > p->sh.chunk - 1) return fail(TTT_E_INVALID_ARG, "n must be in [0, C-1]");
  if (r->tail_len != 0 || r->n_applied != 0) return fail(TTT_E_TAIL_FULL, "tail not empty");
  if (n == 0) return TTT_OK;
  if (p->host_only) return fail(TTT_E_NO_DEVICE, "host-only pool");
  if (!Z || !V) return fail(TTT_E_INVALID_ARG, "null Z/V");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const ttt_shape &sh = p->sh;
  for (int l = 0; l < sh.n_layers; ++l) {
    unsigned char *tz = p->arena + p->lay.tailZ + ((size_t)r->idx * p->tz_owner + (size_t)l * sh.chunk * sh.d_ff) * p->esize;
    unsigned char *tv = p->arena + p->lay.tailV + ((size_t)r->idx * p->tv_owner + (size_t)l * sh.chunk * sh.d_model) * p->esize;
    CUDA_TRY(cudaMemcpyAsync(tz, static_cast<const unsigned char *>(Z) + (size_t)l * n * sh.d_ff * p->esize,
                             (size_t)n * sh.d_ff * p->esize, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(tv, static_cast<const unsigned char *>(V) + (size_t)l * n * sh.d_model * p->esize,
                             (size_t)n * sh.d_model * p->esize, cudaMemcpyDeviceToDevice, s));
  }
  r->tail_len = n;
  return TTT_OK;
}

ttt_status tttstate_version(ttt_pool *p, uint64_t owner, uint64_t *v_out) {
  if (!p || !v_out) return fail(TTT_E_INVALID_ARG, "null arg");
  OwnerRec *r;
  ttt_status st = find_owner(p, owner, &r);
  if (st != TTT_OK) return st;
  if ((st = confirm(p, *r)) != TTT_OK) return st;
  *v_out = r->version;
  return TTT_OK;
}

ttt_status tttstate_tail_len(ttt_pool *p, uint64_t owner, int32_t *len_out) {
  if (!p || !len_out) return fail(TTT_E_INVALID_ARG, "null arg");
  OwnerRec *r;
  ttt_status st = find_owner(p, owner, &r);
  if (st != TTT_OK) return st;
  *len_out = r->tail_len;
  return TTT_OK;
}

ttt_status tttstate_next_event(ttt_pool *p, uint64_t owner, int64_t clock, ttt_event *out) {
  if (!p || !out) return fail(TTT_E_INVALID_ARG, "null arg");
  OwnerRec *r;
  ttt_status st = find_owner(p, owner, &r);
  if (st != TTT_OK) return st;
  out->owner = owner;
  out->effect = r->tail_len == p->sh.chunk - 1 ? TTT_WRITE : TTT_READ;   // reading ii
  out->backend = p->sh.backend;
  out->shape_id = p->shape_id;
  out->placement = p->placement;
  out->expected_version = r->version;
  out->ready_step = clock;
  return TTT_OK;
}

ttt_status tttstate_next_events(ttt_pool *p, const uint64_t *owners, int32_t n, int64_t clock, ttt_event *out) {
  if (!p || (n > 0 && (!owners || !out)) || n < 0) return fail(TTT_E_INVALID_ARG, "null arg / negative n");
  for (int i = 0; i < n; ++i) {                    // validate every owner before writing any event
    OwnerRec *r;
    ttt_status st = find_owner(p, owners[i], &r);
    if (st != TTT_OK) return st;
  }
  for (int i = 0; i < n; ++i) tttstate_next_event(p, owners[i], clock, out + i);
  return TTT_OK;
}

ttt_status validate_group(ttt_pool *p, const ttt_group *g, const uint64_t *expected_versions) {
  std::vector<OwnerRec *> recs;
  ttt_status st = check_group(p, g, recs);
  if (st != TTT_OK) return st;
  if (expected_versions)
    for (int b = 0; b < g->n; ++b)
      if (recs[b]->version != expected_versions[b])
        return fail(TTT_E_VERSION_MISMATCH, "owner " + std::to_string(g->owner_map[b]));
  return TTT_OK;
}

}  // extern "C"

namespace {

// read_apply after check_group (serve_step resolves the group once for all layers)
ttt_status read_apply_recs(ttt_pool *p, const ttt_group *g, std::vector<OwnerRec *> &recs, int32_t layer,
                           const void *X, const int32_t *x_rows, const void *Vt, const int32_t *v_rows, void *Y,
                           const int32_t *y_rows, const void *resid, cudaStream_t s, long long x_rows_total = 0) {
  ttt_status st;
  const ttt_shape &sh = p->sh;
  if (layer < 0 || layer >= sh.n_layers) return fail(TTT_E_SHAPE, "layer out of range");
  for (int b = 0; b < g->n; ++b) {
    OwnerRec &r = *recs[b];
    const bool boundary = r.tail_len == sh.chunk - 1;
    if (r.tail_len >= sh.chunk) return fail(TTT_E_TAIL_FULL, "owner " + std::to_string(g->owner_map[b]));
    if ((g->effect == TTT_WRITE) != boundary)
      return fail(TTT_E_WRONG_EFFECT, "owner " + std::to_string(g->owner_map[b]) +
                                          (boundary ? " is at a chunk boundary (WRITE step)" : " is not at a boundary"));
    if (r.applied[layer]) return fail(TTT_E_ALREADY_APPLIED, "owner " + std::to_string(g->owner_map[b]));
    if (r.chunk_mode) return fail(TTT_E_WRONG_EFFECT, "owner " + std::to_string(g->owner_map[b]) + " is mid-chunk");
  }
  // f3: with C = 1 every step is a WRITE whose evidence is this token only, so the
  // candidate is written here, in the same pass over ΔW (write_commit then only commits).
  const bool fuse = g->effect == TTT_WRITE && sh.chunk == 1 && sh.backend == TTT_FAST_WEIGHT && sh.rule == 0 &&
                    g_write_impl.load() != 1;
  int need_evict = 0;
  if (fuse)
    for (int b = 0; b < g->n; ++b)
      if (recs[b]->n_applied == 0 && recs[b]->has_ckpt) {   // pinned_in_shadow needs the confirmed slot
        if ((st = confirm(p, *recs[b])) != TTT_OK) return st;
        need_evict += pinned_in_shadow(*recs[b]);
      }
  if (need_evict > (int)p->free_ckpt.size()) return fail(TTT_E_POOL_FULL, "no free checkpoint slot for a pinned snapshot");
  if (p->host_only) return fail(TTT_E_NO_DEVICE, "host-only pool");
  if (!X || !Vt || !Y) return fail(TTT_E_INVALID_ARG, "null X/Vt/Y");
  if (fuse)
    for (int b = 0; b < g->n; ++b)
      if (recs[b]->n_applied == 0 && pinned_in_shadow(*recs[b])) CUDA_TRY(evict_pinned(p, *recs[b], s));
  if (sh.backend == TTT_LOW_RANK) {                 // NEXT f1: u = A x, base GEMM, y = base + Bᵀu
    LowRankRead lp{};
    lp.n = g->n; lp.d_model = sh.d_model; lp.d_ff = sh.d_ff; lp.rank = sh.rank;
    lp.X = X; lp.Vt = Vt; lp.resid = resid; lp.Y = Y;
    lp.Xg = p->arena + p->lay.Xg;
    lp.Y32 = reinterpret_cast<float *>(p->arena + p->lay.Y32);
    lp.u = reinterpret_cast<float *>(p->arena + p->lay.U);
    lp.slots = p->arena + p->lay.slots;
    lp.slot_elems = p->slot_elems;
    lp.layer_off = (long long)layer * p->E;
    lp.sel = p->d_sel();
    lp.tailZ = p->arena + p->lay.tailZ;
    lp.tailV = p->arena + p->lay.tailV;
    lp.tz_owner = p->tz_owner; lp.tv_owner = p->tv_owner;
    lp.tz_layer = (long long)layer * sh.chunk * sh.d_ff;
    lp.tv_layer = (long long)layer * sh.chunk * sh.d_model;
    for (int b = 0; b < g->n; ++b) {
      lp.owner_idx[b] = recs[b]->idx;
      lp.x_row[b] = x_rows ? x_rows[b] : b;
      lp.v_row[b] = v_rows ? v_rows[b] : b;
      lp.y_row[b] = y_rows ? y_rows[b] : b;
      lp.tail_pos[b] = recs[b]->tail_len;
    }
    if (x_rows_total > 0) {                         // serve_step knows the X buffer: contiguous rows need no gather
      bool contiguous = true;
      for (int b = 0; b < g->n; ++b) contiguous &= lp.x_row[b] == lp.x_row[0] + b;
      if (contiguous && lp.x_row[0] >= 0 && lp.x_row[0] + g->n <= x_rows_total) {
        lp.x_row0 = lp.x_row[0];
        lp.x_rows_total = x_rows_total;
      }
    }
    {
      MemberTable mt;
      for (int b = 0; b < g->n; ++b) {
        mt.a[0][b] = lp.owner_idx[b];
        mt.a[1][b] = lp.x_row[b];
        mt.a[2][b] = lp.v_row[b];
        mt.a[3][b] = lp.y_row[b];
        mt.a[4][b] = lp.tail_pos[b];
      }
      CUDA_TRY(upload_members(p, mt, g->n, s));
    }
    ChunkLaunch cl{};
    cl.d_members = p->d_members();
    cl.n = (g->n + 127) / 128; cl.d_model = sh.d_model; cl.d_ff = sh.d_ff; cl.C = 128; cl.L = sh.n_layers;
    cl.layer = layer; cl.max_slots = 1; cl.sel = p->d_sel();
    cl.X = lp.Xg; cl.w_down = p->w_down; cl.slots = p->w_down;
    cl.delta = 0; cl.append = 0; cl.Y32 = lp.Y32; cl.valid_rows = g->n;
    // split K so the base GEMM (one or two 128-row blocks) covers the SMs; slabs summed in order.
    // ~2/3 of the SM count in (row block, 160-wide) units: plan_n then narrows the N blocks to
    // fill the SMs, and each tile keeps a longer K range (measured: 6 slabs beat 9 by 4 % at
    // 128 members, d 2560 / 9728)
    const int ntile = cl.n * ((sh.d_model + 159) / 160);
    cl.ksplit = std::max(1, std::min({kMaxKSplit, 2 * device_sm_count() / (3 * ntile), sh.d_ff / 64}));
    if (const char *e = getenv("TTT_LR_KS")) cl.ksplit = std::max(1, std::min({kMaxKSplit, atoi(e), sh.d_ff / 64}));
    cl.y32_slab = (long long)align_up((size_t)p->max_owners, 128) * sh.d_model;
    lp.ksplit = cl.ksplit;
    lp.y32_slab = cl.y32_slab;
    lp.ctr = reinterpret_cast<int *>(p->arena + p->lay.Ctr);
    lp.w_down = p->w_down;
    lp.L = sh.n_layers;
    lp.layer = layer;
    lp.max_slots = 2 * p->max_owners + p->n_ckpt;
    lp.xflag = reinterpret_cast<int *>(p->arena + p->lay.xflag);
    lp.x_epoch = p->step_epoch;
    cudaError_t e = launch_lowrank_read(lp, cl, s);
    if (e != cudaSuccess) return cuda_fail(e, "low-rank READ");
    for (int b = 0; b < g->n; ++b) {
      recs[b]->applied[layer] = 1;
      recs[b]->n_applied += 1;
    }
    return TTT_OK;
  }
  int per = std::min(kMaxReadMembers, g->n);
  while (per > 1 && !read_decode_fits(per, sh.d_model, sh.d_ff, (int)p->esize)) --per;
  if (!read_decode_fits(per, sh.d_model, sh.d_ff, (int)p->esize))
    return fail(TTT_E_SHAPE, "d_ff row slices exceed shared memory");
  for (int b0 = 0; b0 < g->n; b0 += per) {
    ReadParams rp{};
    rp.X = X; rp.Vt = Vt; rp.resid = resid; rp.Y = Y;
    rp.w_down_l = static_cast<const unsigned char *>(p->w_down) + (size_t)layer * p->Ew * p->esize;
    rp.slots = p->arena + p->lay.slots;
    rp.slot_elems = p->slot_elems;
    rp.layer_off = (long long)layer * p->E;
    rp.sel = p->d_sel();
    rp.tailZ = p->arena + p->lay.tailZ;
    rp.tailV = p->arena + p->lay.tailV;
    rp.tz_owner = p->tz_owner; rp.tv_owner = p->tv_owner;
    rp.tz_layer = (long long)layer * sh.chunk * sh.d_ff;
    rp.tv_layer = (long long)layer * sh.chunk * sh.d_model;
    // tensor-core base for plain READs; the f3 fused READ+WRITE keeps the all-SIMT kernel
    // (its candidate stores need the registers: 82 % vs 79 % of HBM measured)
    rp.kc = fuse ? 0 : read_decode_mma_chunks(sh.dtype, sh.d_ff);
    rp.Pbase = reinterpret_cast<float *>(p->arena + p->lay.P);
    rp.Pdelta = rp.Pbase + (size_t)std::max(1, rp.kc) * kMaxReadMembers * sh.d_model;
    rp.tickets = reinterpret_cast<int *>(p->arena + p->lay.tickets);
    rp.n = std::min(per, g->n - b0);
    rp.l2keep = g->n > per;                        // several launches read this layer's W_down
    rp.d_model = sh.d_model; rp.d_ff = sh.d_ff;
    rp.fuse = fuse ? 1 : 0;
    rp.eta = p->eta;
    rp.mfail = p->d_mfail();
    for (int k = 0; k < rp.n; ++k) {
      const int b = b0 + k;
      rp.owner_idx[k] = recs[b]->idx;
      rp.x_row[k] = x_rows ? x_rows[b] : b;
      rp.v_row[k] = v_rows ? v_rows[b] : b;
      rp.y_row[k] = y_rows ? y_rows[b] : b;
      rp.tail_pos[k] = recs[b]->tail_len;
    }
    rp.L = sh.n_layers;
    rp.layer = layer;
    rp.n_slot_layers = (long long)(2 * p->max_owners + p->n_ckpt) * sh.n_layers;
    rp.ptc = p->lay.ptc_bytes ? reinterpret_cast<float *>(p->arena + p->lay.ptc) : nullptr;
    rp.ptc_bytes = p->lay.ptc_bytes;
    rp.xflag = reinterpret_cast<int *>(p->arena + p->lay.xflag);
    rp.x_epoch = p->step_epoch;
    cudaError_t e = launch_read_decode(sh.dtype, rp, s);
    if (e != cudaSuccess) return cuda_fail(e, "read_decode launch");
  }
  for (int b = 0; b < g->n; ++b) {
    recs[b]->applied[layer] = 1;
    recs[b]->n_applied += 1;
    if (fuse) recs[b]->fused_layers += 1;
  }
  return TTT_OK;
}

}  // namespace

extern "C" {

ttt_status read_apply(ttt_pool *p, const ttt_group *g, int32_t layer, const void *X, const int32_t *x_rows,
                      const void *Vt, const int32_t *v_rows, void *Y, const int32_t *y_rows,
                      const void *resid, void *stream) {
  NvtxRange nvtx_("read_apply");
  std::vector<OwnerRec *> recs;
  ttt_status st = check_group(p, g, recs);
  if (st != TTT_OK) return st;
  return read_apply_recs(p, g, recs, layer, X, x_rows, Vt, v_rows, Y, y_rows, resid, static_cast<cudaStream_t>(stream));
}

ttt_status tttstate_set_eta(ttt_pool *p, float eta) {
  if (!p) return fail(TTT_E_INVALID_ARG, "null pool");
  p->eta = eta;
  return TTT_OK;
}

ttt_status tttstate_step_done(ttt_pool *p, const ttt_group *g) {
  std::vector<OwnerRec *> recs;
  ttt_status st = check_group(p, g, recs);
  if (st != TTT_OK) return st;
  if (g->effect != TTT_READ) return fail(TTT_E_WRONG_EFFECT, "step_done is for READ groups (write_commit ends a WRITE step)");
  for (int b = 0; b < g->n; ++b) {
    // a READ step ends below the boundary: an owner at C-1 (or one whose chunk was applied by
    // read_apply_chunk) must end its step with write_commit
    if (recs[b]->chunk_mode || recs[b]->tail_len >= p->sh.chunk - 1)
      return fail(TTT_E_WRONG_EFFECT, "owner " + std::to_string(g->owner_map[b]) + " is at a chunk boundary (WRITE step)");
    if (recs[b]->n_applied != p->sh.n_layers)
      return fail(TTT_E_NOT_APPLIED, "owner " + std::to_string(g->owner_map[b]));
  }
  for (int b = 0; b < g->n; ++b) {
    recs[b]->tail_len += 1;
    clear_applied(*recs[b]);
  }
  return TTT_OK;
}

ttt_status read_apply_chunk(ttt_pool *p, const ttt_group *g, int32_t layer, const void *X, const void *Vt,
                            void *Y, void *stream) {
  NvtxRange nvtx_("read_apply_chunk");
  std::vector<OwnerRec *> recs;
  ttt_status st = check_group(p, g, recs);
  if (st != TTT_OK) return st;
  const ttt_shape &sh = p->sh;
  if (g->effect != TTT_WRITE) return fail(TTT_E_WRONG_EFFECT, "a whole chunk ends in its boundary WRITE");
  if (layer < 0 || layer >= sh.n_layers) return fail(TTT_E_SHAPE, "layer out of range");
  if (sh.backend != TTT_FAST_WEIGHT || sh.dtype != TTT_BF16 || !read_chunk_supported(sh.d_model, sh.d_ff, sh.chunk))
    return fail(TTT_E_SHAPE, "chunk READ needs bf16, d_ff % 64 == 0, d_model % 16 == 0 (>= 128), C <= 128");
  for (int b = 0; b < g->n; ++b) {
    OwnerRec &r = *recs[b];
    if (r.tail_len != 0 || (r.n_applied > 0 && !r.chunk_mode))
      return fail(TTT_E_TAIL_FULL, "owner " + std::to_string(g->owner_map[b]) + " is not at a chunk start");
    if (r.applied[layer]) return fail(TTT_E_ALREADY_APPLIED, "owner " + std::to_string(g->owner_map[b]));
  }
  if (p->host_only) return fail(TTT_E_NO_DEVICE, "host-only pool");
  if (!X || !Vt || !Y) return fail(TTT_E_INVALID_ARG, "null X/Vt/Y");
  ChunkLaunch cl{};
  cl.n = g->n; cl.d_model = sh.d_model; cl.d_ff = sh.d_ff; cl.C = sh.chunk; cl.L = sh.n_layers; cl.layer = layer;
  cl.max_slots = 2 * p->max_owners + p->n_ckpt;
  cl.sel = p->d_sel();
  cl.X = X; cl.Vt = Vt; cl.Y = Y;
  cl.w_down = p->w_down;
  cl.slots = p->arena + p->lay.slots;
  cl.tailZ = p->arena + p->lay.tailZ;
  cl.tailV = p->arena + p->lay.tailV;
  cl.tz_owner = p->tz_owner; cl.tv_owner = p->tv_owner;
  cl.tz_layer = (long long)layer * sh.chunk * sh.d_ff;
  cl.tv_layer = (long long)layer * sh.chunk * sh.d_model;
  for (int b = 0; b < g->n; ++b) cl.owner_idx[b] = recs[b]->idx;
  {
    MemberTable mt;
    std::memset(&mt, 0, sizeof(mt));
    for (int b = 0; b < g->n; ++b) mt.a[0][b] = recs[b]->idx;
    CUDA_TRY(upload_members(p, mt, g->n, static_cast<cudaStream_t>(stream)));
  }
  cl.d_members = p->d_members();
  if (p->lay.wslab) {
    cl.wide_slab = reinterpret_cast<float *>(p->arena + p->lay.wslab);
    cl.wide_slab_bytes = kWideSlabBytes;
    cl.wide_tickets = reinterpret_cast<int *>(p->arena + p->lay.wtick);
  }
  cudaError_t e = launch_read_chunk(cl, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "read_chunk launch");
  for (int b = 0; b < g->n; ++b) {
    OwnerRec &r = *recs[b];
    r.applied[layer] = 1;
    r.n_applied += 1;
    r.chunk_mode = true;
    if (r.n_applied == sh.n_layers) r.tail_len = sh.chunk - 1;   // C entries in the tail; boundary token applied
  }
  return TTT_OK;
}

// ---------------------------------------------------------------- WRITE + commit
}  // extern "C"

namespace {

ttt_status write_commit_recs(ttt_pool *p, const ttt_group *g, std::vector<OwnerRec *> &recs, float eta,
                             const uint32_t *fail_mask, uint64_t *new_versions, cudaStream_t s) {
  ttt_status st;
  const ttt_shape &sh = p->sh;
  if (g->effect != TTT_WRITE) return fail(TTT_E_WRONG_EFFECT, "write_commit needs a WRITE group");
  int need_evict = 0, n_fused = 0;
  for (int b = 0; b < g->n; ++b) {
    OwnerRec &r = *recs[b];
    if (r.tail_len != sh.chunk - 1) return fail(TTT_E_TAIL_NOT_FULL, "owner " + std::to_string(g->owner_map[b]));
    if (r.n_applied != sh.n_layers) return fail(TTT_E_NOT_APPLIED, "owner " + std::to_string(g->owner_map[b]));
    n_fused += r.fused_layers == sh.n_layers;
  }
  for (int b = 0; b < g->n; ++b)
    if (recs[b]->has_ckpt) {                        // pinned_in_shadow needs the confirmed slot
      if ((st = confirm(p, *recs[b])) != TTT_OK) return st;
      need_evict += pinned_in_shadow(*recs[b]);
    }
  const bool fused = n_fused == g->n;               // every candidate already written by read_apply (f3)
  if (n_fused != 0 && !fused) return fail(TTT_E_INVALID_ARG, "group mixes fused and unfused members");
  if (fused && eta != p->eta) return fail(TTT_E_INVALID_ARG, "eta differs from the pool's fused-path eta");
  if (!fused && need_evict > (int)p->free_ckpt.size())
    return fail(TTT_E_POOL_FULL, "no free checkpoint slot for a pinned snapshot");
  const int impl = g_write_impl.load();
  const bool use_tc = sh.rule == 0 && sh.dtype == TTT_BF16 && impl != 1 &&
                      write_tc_supported(sh.d_model, sh.d_ff, sh.chunk, sh.n_layers);
  if (!fused && impl == 2 && !use_tc) return fail(TTT_E_SHAPE, "tcgen05 WRITE kernel does not support this shape");
  bool forced = false;
  if (fail_mask)
    for (int b = 0; b < g->n; ++b) forced |= (fail_mask[b / 32] >> (b % 32)) & 1u;
  if (p->host_only) return fail(TTT_E_NO_DEVICE, "host-only pool");
  CommitParams cp{};
  cp.sel = p->d_sel();
  cp.version = p->d_ver();
  cp.mfail = p->d_mfail();
  cp.fail_count = p->d_fail_count();
  cp.rlog_count = p->d_rlog_count();
  cp.rlog = p->d_rlog();
  cp.hstate = p->hstate_dev;
  cp.seq = forced ? 0 : p->commit_seq + 1;
  cp.forced_fail = forced ? 1 : 0;
  cp.n = g->n;
  for (int b = 0; b < g->n; ++b) {
    cp.owner_idx[b] = recs[b]->idx;
    cp.owner_id[b] = g->owner_map[b];
  }
  const bool partial = forced && (g_test_hook.load() & TTT_HOOK_NO_GROUP_ATOMICITY);
  cp.partial = partial ? 1 : 0;
  if (partial)
    for (int b = 0; b < g->n; ++b) cp.fail_bits[b / 32] = fail_mask[b / 32];
  bool committed = false;                           // commit fused into the WRITE kernel
  if (!fused && sh.backend == TTT_LOW_RANK) {
    for (int b = 0; b < g->n; ++b)
      if (pinned_in_shadow(*recs[b])) CUDA_TRY(evict_pinned(p, *recs[b], s));
    LowRankWrite lw{};
    lw.n = g->n; lw.d_model = sh.d_model; lw.d_ff = sh.d_ff; lw.rank = sh.rank; lw.C = sh.chunk;
    lw.slots = p->arena + p->lay.slots;
    lw.slot_elems = p->slot_elems;
    lw.sel = p->d_sel();
    lw.tailZ = p->arena + p->lay.tailZ;
    lw.tz_owner = p->tz_owner;
    lw.eta = eta;
    lw.mfail = p->d_mfail();
    for (int b = 0; b < g->n; ++b) lw.owner_idx[b] = recs[b]->idx;
    for (int l = 0; l < sh.n_layers; ++l) {
      lw.layer_off = (long long)l * p->E;
      lw.tz_layer = (long long)l * sh.chunk * sh.d_ff;
      cudaError_t e = launch_lowrank_write(lw, s);
      if (e != cudaSuccess) return cuda_fail(e, "low-rank write launch");
    }
  } else if (!fused) {
    for (int b = 0; b < g->n; ++b)                  // preserve pinned checkpoints sitting in the shadow slot
      if (pinned_in_shadow(*recs[b])) CUDA_TRY(evict_pinned(p, *recs[b], s));
    WriteParams wp{};
    wp.slots = p->arena + p->lay.slots;
    wp.slot_elems = p->slot_elems;
    wp.sel = p->d_sel();
    wp.tailZ = p->arena + p->lay.tailZ;
    wp.tailV = p->arena + p->lay.tailV;
    wp.tz_owner = p->tz_owner; wp.tv_owner = p->tv_owner;
    wp.eta = eta;
    wp.mfail = p->d_mfail();
    wp.n = g->n; wp.d_model = sh.d_model; wp.d_ff = sh.d_ff; wp.C = sh.chunk;
    wp.max_owners = p->max_owners; wp.max_slots = 2 * p->max_owners + p->n_ckpt;
    for (int b = 0; b < g->n; ++b) wp.owner_idx[b] = recs[b]->idx;
    if (use_tc) {                                   // every layer in one launch, commit fused
      static const bool fuse_commit = !getenv("TTT_WRITE_FUSE_COMMIT") || atoi(getenv("TTT_WRITE_FUSE_COMMIT")) != 0;
      cudaError_t e = launch_write_tc(wp, fuse_commit ? &cp : nullptr, p->d_wctr(), s);
      if (e != cudaSuccess) return cuda_fail(e, "write launch");
      committed = fuse_commit;
    } else {
      for (int l = 0; l < sh.n_layers; ++l) {
        wp.layer_off = (long long)l * p->E;
        wp.tz_layer = (long long)l * sh.chunk * sh.d_ff;
        wp.tv_layer = (long long)l * sh.chunk * sh.d_model;
        cudaError_t e = sh.rule == 1 ? launch_write_rule1(sh.dtype, wp, s) : launch_write_simt(sh.dtype, wp, s);
        if (e != cudaSuccess) return cuda_fail(e, "write launch");
      }
    }
  }
  if (!committed) CUDA_TRY(launch_commit(cp, s));
  if (partial)                                    // the broken contract the negative control needs
    for (int b = 0; b < g->n; ++b) {
      if ((fail_mask[b / 32] >> (b % 32)) & 1u) continue;
      OwnerRec &r = *recs[b];
      r.sel ^= 1;
      r.version += 1;
      r.tail_len = 0;
      clear_applied(r);
    }
  if (forced) return fail(TTT_E_WRITE_FAILED, "injected failure: group not committed");
  // optimistic host mirror: every member at v+1 unless the device refuses it (confirm())
  const uint64_t seq = ++p->commit_seq;
  CUDA_TRY(cudaEventRecord(p->ev_ring[seq % p->ev_ring.size()], s));
  for (int b = 0; b < g->n; ++b) {
    OwnerRec &r = *recs[b];
    r.sel ^= 1;
    r.version += 1;
    r.tail_len = 0;
    r.pending_seq = seq;
    clear_applied(r);
    if (new_versions) new_versions[b] = r.version;
  }
  return TTT_OK;
}

}  // namespace

extern "C" {

ttt_status write_commit(ttt_pool *p, const ttt_group *g, float eta, const uint32_t *fail_mask,
                        uint64_t *new_versions, void *stream) {
  NvtxRange nvtx_("write_commit");
  std::vector<OwnerRec *> recs;
  ttt_status st = check_group(p, g, recs);
  if (st != TTT_OK) return st;
  return write_commit_recs(p, g, recs, eta, fail_mask, new_versions, static_cast<cudaStream_t>(stream));
}

ttt_status tttstate_last_commit_seq(ttt_pool *p, uint64_t *seq_out) {
  if (!p || !seq_out) return fail(TTT_E_INVALID_ARG, "null arg");
  *seq_out = p->commit_seq;
  return TTT_OK;
}

// ---------------------------------------------------------------- control
ttt_status tttstate_snapshot(ttt_pool *p, uint64_t owner, void *stream) {
  NvtxRange nvtx_("tttstate_snapshot");
  (void)stream;
  if (!p) return fail(TTT_E_INVALID_ARG, "null pool");
  OwnerRec *r;
  ttt_status st = find_owner(p, owner, &r);
  if (st != TTT_OK) return st;
  if ((st = confirm(p, *r)) != TTT_OK) return st;   // pin the committed (confirmed) slot only
  if (r->ckpt_pool >= 0) p->free_ckpt.push_back(r->ckpt_pool);
  r->has_ckpt = true;
  r->ckpt_v = r->version;
  r->ckpt_sel = r->sel;      // pin the committed slot: O(1), no bytes move
  r->ckpt_pool = -1;
  return TTT_OK;
}

ttt_status rollback(ttt_pool *p, uint64_t owner, uint64_t *v_out, void *stream) {
  NvtxRange nvtx_("rollback");
  if (!p) return fail(TTT_E_INVALID_ARG, "null pool");
  OwnerRec *r;
  ttt_status st = find_owner(p, owner, &r);
  if (st != TTT_OK) return st;
  if (!r->has_ckpt) return fail(TTT_E_NO_CHECKPOINT, "owner " + std::to_string(owner));
  if (p->host_only) return fail(TTT_E_NO_DEVICE, "host-only pool");
  // No confirmation needed (and no host wait right after a speculative WRITE): the restored
  // (slot, version) come from the checkpoint, and a copy back from the checkpoint pool may land
  // in either slot of the pair; the pending commit's outcome is superseded by the rollback
  // (its refusal record, if any, is still logged for tttstate_refusals).
  r->pending_seq = 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int new_sel;
  if (r->ckpt_pool < 0) {
    new_sel = r->ckpt_sel;                       // re-point to the pinned slot
  } else {
    new_sel = 1 - r->sel;                        // copy the checkpoint back into the shadow slot
    CUDA_TRY(launch_copy(p->slot_ptr(2LL * r->idx + new_sel), p->slot_ptr(2LL * p->max_owners + r->ckpt_pool),
                         p->slot_bytes(), s));
  }
  CUDA_TRY(launch_set_state(p->d_sel(), p->d_ver(), p->d_mfail(), r->idx, new_sel, r->ckpt_v, s));
  r->sel = new_sel;
  r->version = r->ckpt_v;
  r->tail_len = 0;
  clear_applied(*r);
  if (v_out) *v_out = r->version;
  return TTT_OK;
}

ttt_status tttstate_fork(ttt_pool *p, uint64_t src, uint64_t dst, void *stream) {
  NvtxRange nvtx_("tttstate_fork");
  if (!p) return fail(TTT_E_INVALID_ARG, "null pool");
  OwnerRec *rs;
  ttt_status st = find_owner(p, src, &rs);
  if (st != TTT_OK) return st;
  if (p->owners.count(dst)) return fail(TTT_E_DUPLICATE_OWNER, "owner " + std::to_string(dst));
  if (p->free_idx.empty()) return fail(TTT_E_POOL_FULL, "no free owner slot");
  if (p->host_only) return fail(TTT_E_NO_DEVICE, "host-only pool");
  if ((st = confirm(p, *rs)) != TTT_OK) return st;   // copy the committed (confirmed) slot
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int idx = p->free_idx.back();
  CUDA_TRY(launch_copy(p->slot_ptr(2LL * idx), p->slot_ptr(2LL * rs->idx + rs->sel), p->slot_bytes(), s));
  CUDA_TRY(launch_set_state(p->d_sel(), p->d_ver(), p->d_mfail(), idx, 0, rs->version, s));
  p->free_idx.pop_back();
  OwnerRec r;
  r.idx = idx;
  r.version = rs->version;
  r.applied.assign(p->sh.n_layers, 0);
  p->owners.emplace(dst, std::move(r));
  return TTT_OK;
}

ttt_status tttstate_sync(ttt_pool *p, void *stream, int32_t *n_failed_out) {
  NvtxRange nvtx_("tttstate_sync");
  if (!p) return fail(TTT_E_INVALID_ARG, "null pool");
  if (n_failed_out) *n_failed_out = 0;
  if (p->host_only) return TTT_OK;
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  for (auto &kv : p->owners) {                       // every pending commit is complete now
    ttt_status st = confirm(p, kv.second);
    if (st != TTT_OK) return st;
  }
  int count = 0;
  CUDA_TRY(cudaMemcpy(&count, p->d_fail_count(), sizeof(int), cudaMemcpyDeviceToHost));
  if (count == p->fail_seen) return TTT_OK;
  const int nf = count - p->fail_seen;
  p->fail_seen = count;
  if (n_failed_out) *n_failed_out = nf;
  return fail(TTT_E_WRITE_FAILED, std::to_string(nf) + " group(s) had members refused on the device");
}

ttt_status tttstate_refusals(ttt_pool *p, uint64_t *owners, uint64_t *versions, uint64_t *seqs, int32_t cap,
                             int32_t *n_out, void *stream) {
  if (!p || !n_out || cap < 0 || (cap > 0 && (!owners || !versions || !seqs))) return fail(TTT_E_INVALID_ARG, "null arg");
  *n_out = 0;
  if (p->host_only) return TTT_OK;
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  int count = 0;
  CUDA_TRY(cudaMemcpy(&count, p->d_rlog_count(), sizeof(int), cudaMemcpyDeviceToHost));
  const int avail = count - p->rlog_read;
  if (avail > kRefusalLog) return fail(TTT_E_CAPACITY, "refusal log overflowed (drain more often)");
  const int n = std::min(avail, cap);
  std::vector<RefusalRec> recs(n);
  for (int k = 0; k < n; ++k)
    CUDA_TRY(cudaMemcpy(&recs[k], p->d_rlog() + (p->rlog_read + k) % kRefusalLog, sizeof(RefusalRec),
                        cudaMemcpyDeviceToHost));
  for (int k = 0; k < n; ++k) {
    owners[k] = recs[k].owner;
    versions[k] = recs[k].version;
    seqs[k] = recs[k].seq;
  }
  p->rlog_read += n;
  *n_out = n;
  return TTT_OK;
}

// ---------------------------------------------------------------- one serving-loop iteration
ttt_status tttstate_serve_step(ttt_pool *p, ttt_planner *pl, const uint64_t *owners, int32_t n, int64_t clock,
                               const ttt_step_io *io, float eta, const uint64_t *fail_owners, int32_t n_fail,
                               ttt_step_out *out, void *stream) {
  NvtxRange nvtx_("tttstate_serve_step");
  if (!p || !pl || !io || !out || n < 0 || (n > 0 && !owners) || n_fail < 0 || (n_fail > 0 && !fail_owners))
    return fail(TTT_E_INVALID_ARG, "null arg / negative count");
  if (!out->groups || !out->owner_buf || out->group_cap < 0 || out->owner_cap < 0)
    return fail(TTT_E_INVALID_ARG, "null output buffers");
  out->n_groups = out->n_rejected = out->n_read = out->n_write = out->n_injected = 0;
  if (p->host_only) return fail(TTT_E_NO_DEVICE, "host-only pool");
  if (!io->X || !io->Vt || !io->Y) return fail(TTT_E_INVALID_ARG, "null X/Vt/Y");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // owner -> token row; validate every owner before any side effect
  std::unordered_map<uint64_t, int32_t> row;
  row.reserve(2 * (size_t)n + 1);
  for (int i = 0; i < n; ++i) {
    OwnerRec *r;
    ttt_status st = find_owner(p, owners[i], &r);
    if (st != TTT_OK) return st;
    if (!row.emplace(owners[i], io->rows ? io->rows[i] : i).second)
      return fail(TTT_E_OWNER_COLLISION, "owner " + std::to_string(owners[i]) + " listed twice");
  }
  // a1 NextStep: an event for every listed owner without one pending in the planner
  std::unordered_set<uint64_t> pend;
  planner_pending_owners(pl, pend);
  std::vector<ttt_event> ev;
  ev.reserve(n);
  for (int i = 0; i < n; ++i)
    if (!pend.count(owners[i])) {
      ev.emplace_back();
      tttstate_next_event(p, owners[i], clock, &ev.back());
    }
  // a2 LegalGroups (no side effect on error)
  int32_t n_groups = 0, n_rej = 0;
  ttt_status st = plan_batch(pl, ev.data(), (int32_t)ev.size(), clock, out->groups, out->group_cap, out->owner_buf,
                             out->owner_cap, &n_groups, out->rejected, out->rej_cap, &n_rej);
  if (st != TTT_OK) return st;
  out->n_groups = n_groups;
  out->n_rejected = n_rej;
  std::unordered_set<uint64_t> failing(fail_owners, fail_owners + n_fail);
  const size_t es = p->esize;
  std::vector<OwnerRec *> recs, one;
  std::vector<int32_t> rows;
  size_t off = 0;
  // X / Vt are inputs of the whole step: READ launches after the step's first may stage x early
  struct EpochScope {
    ttt_pool *p;
    ~EpochScope() { p->step_epoch = 0; }
  } epoch_scope{p};
  static const bool early_x = !getenv("TTT_READ_EARLY_X") || atoi(getenv("TTT_READ_EARLY_X")) != 0;
  if (early_x) {
    p->epoch_ctr = p->epoch_ctr >= (1 << 30) ? 1 : p->epoch_ctr + 1;
    p->step_epoch = p->epoch_ctr;
  }
  for (int k = 0; k < n_groups; ++k) {
    const ttt_group &g = out->groups[k];
    if ((st = check_group(p, &g, recs)) != TTT_OK) return st;
    if (out->injected) out->injected[k] = 0;
    rows.resize(g.n);
    for (int b = 0; b < g.n; ++b) {
      auto it = row.find(g.owner_map[b]);
      if (it == row.end()) return fail(TTT_E_UNKNOWN_OWNER, "planner issued an owner outside this step");
      rows[b] = it->second;
      if (out->v_before) out->v_before[off + b] = recs[b]->version;
      if (out->member_seq) out->member_seq[off + b] = 0;
    }
    for (int l = 0; l < p->sh.n_layers; ++l) {    // a3 + a4: one dependent READ launch per layer
      const unsigned char *X = static_cast<const unsigned char *>(io->X) + (size_t)l * io->x_layer_stride * es;
      const unsigned char *V = static_cast<const unsigned char *>(io->Vt) + (size_t)l * io->v_layer_stride * es;
      unsigned char *Y = static_cast<unsigned char *>(io->Y) + (size_t)l * io->y_layer_stride * es;
      const unsigned char *R = io->resid ? static_cast<const unsigned char *>(io->resid) + (size_t)l * io->r_layer_stride * es
                                         : nullptr;
      if ((st = read_apply_recs(p, &g, recs, l, X, rows.data(), V, rows.data(), Y, rows.data(), R, s, io->rows_total)) !=
          TTT_OK)
        return st;
    }
    if (g.effect == TTT_READ) {                    // UpdateKVAndTailMetadata
      for (int b = 0; b < g.n; ++b) {
        recs[b]->tail_len += 1;
        clear_applied(*recs[b]);
      }
      out->n_read += g.n;
    } else {                                       // a5 + a6 (+ App. H fallback on an injected failure)
      std::vector<uint32_t> mask((g.n + 31) / 32, 0u);
      bool any = false;
      for (int b = 0; b < g.n; ++b)
        if (failing.count(g.owner_map[b])) {
          mask[b / 32] |= 1u << (b % 32);
          any = true;
        }
      const bool prof = io->ev_write_begin && io->ev_write_end && out->n_write == 0;
      if (prof) CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(io->ev_write_begin), s));
      st = write_commit_recs(p, &g, recs, eta, any ? mask.data() : nullptr, nullptr, s);
      if (prof && st == TTT_OK) CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(io->ev_write_end), s));
      if (st == TTT_OK) {
        for (int b = 0; b < g.n; ++b)
          if (out->member_seq) out->member_seq[off + b] = p->commit_seq;
      } else if (st == TTT_E_WRITE_FAILED && any) {
        if (out->injected) out->injected[k] = 1;
        out->n_injected += 1;
        for (int b = 0; b < g.n; ++b) {            // serial singletons in μ order
          ttt_group g1 = g;
          g1.n = 1;
          g1.owner_map = g.owner_map + b;
          one.assign(1, recs[b]);
          if ((st = write_commit_recs(p, &g1, one, eta, nullptr, nullptr, s)) != TTT_OK) return st;
          if (out->member_seq) out->member_seq[off + b] = p->commit_seq;
        }
      } else {
        return st;
      }
      out->n_write += g.n;
    }
    off += g.n;
  }
  return TTT_OK;
}

// ---------------------------------------------------------------- test hooks
ttt_status tttstate_read_slot_raw(ttt_pool *p, uint64_t owner, int32_t which, int32_t layer, void *host_dst,
                                  void *stream) {
  if (!p || !host_dst) return fail(TTT_E_INVALID_ARG, "null arg");
  OwnerRec *r;
  ttt_status st = find_owner(p, owner, &r);
  if (st != TTT_OK) return st;
  if (p->host_only) return fail(TTT_E_NO_DEVICE, "host-only pool");
  if (layer < 0 || layer >= p->sh.n_layers) return fail(TTT_E_SHAPE, "layer");
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  long long slot;
  if (which == 0 || which == 1) {
    slot = 2LL * r->idx + which;
  } else if (which == 2) {
    if (r->ckpt_pool < 0) return fail(TTT_E_NO_CHECKPOINT, "checkpoint is not in the checkpoint pool");
    slot = 2LL * p->max_owners + r->ckpt_pool;
  } else {                                       // -1: committed slot per the device table
    int dsel = 0;
    CUDA_TRY(cudaMemcpy(&dsel, p->d_sel() + r->idx, 4, cudaMemcpyDeviceToHost));
    slot = 2LL * r->idx + dsel;
  }
  CUDA_TRY(cudaMemcpy(host_dst, p->slot_ptr(slot) + (size_t)layer * p->E * p->esize, (size_t)p->E * p->esize,
                      cudaMemcpyDeviceToHost));
  return TTT_OK;
}

ttt_status tttstate_read_payload(ttt_pool *p, uint64_t owner, int32_t layer, void *host_dst, void *stream) {
  return tttstate_read_slot_raw(p, owner, -1, layer, host_dst, stream);
}

ttt_status tttstate_read_tail(ttt_pool *p, uint64_t owner, int32_t layer, void *host_Z, void *host_V,
                              void *stream) {
  if (!p || !host_Z || !host_V) return fail(TTT_E_INVALID_ARG, "null arg");
  OwnerRec *r;
  ttt_status st = find_owner(p, owner, &r);
  if (st != TTT_OK) return st;
  if (p->host_only) return fail(TTT_E_NO_DEVICE, "host-only pool");
  if (layer < 0 || layer >= p->sh.n_layers) return fail(TTT_E_SHAPE, "layer");
  const ttt_shape &sh = p->sh;
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  CUDA_TRY(cudaMemcpy(host_Z, p->arena + p->lay.tailZ + ((size_t)r->idx * p->tz_owner + (size_t)layer * sh.chunk * sh.d_ff) * p->esize,
                      (size_t)sh.chunk * sh.d_ff * p->esize, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(host_V, p->arena + p->lay.tailV + ((size_t)r->idx * p->tv_owner + (size_t)layer * sh.chunk * sh.d_model) * p->esize,
                      (size_t)sh.chunk * sh.d_model * p->esize, cudaMemcpyDeviceToHost));
  return TTT_OK;
}

ttt_status tttstate_device_version(ttt_pool *p, uint64_t owner, uint64_t *v_out, void *stream) {
  if (!p || !v_out) return fail(TTT_E_INVALID_ARG, "null arg");
  OwnerRec *r;
  ttt_status st = find_owner(p, owner, &r);
  if (st != TTT_OK) return st;
  if (p->host_only) return fail(TTT_E_NO_DEVICE, "host-only pool");
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  unsigned long long v = 0;
  CUDA_TRY(cudaMemcpy(&v, p->d_ver() + r->idx, 8, cudaMemcpyDeviceToHost));
  *v_out = v;
  return TTT_OK;
}

}  // extern "C"
