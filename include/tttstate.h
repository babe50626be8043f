/*
 * tttstate.h — C ABI of the B200-native RW-TTT hot path (arxiv 2605.28053).
 *
 * The path: batched execution of request-owned, versioned TTT state during
 * decode (BASELINE.json north_star; SURVEY.md §8(a) rows a1–a7):
 *   a1  tttstate_next_event   NextStep / event e=(r,τ,σ,ρ,v)         Eq. 2, Alg. 1
 *   a2  plan_batch            LegalGroups (κ buckets, B, w, μ)       Eq. 3-4, §4.3
 *   a3  read_apply            ApplyState y = x·(W_down + ΔW_μ(b))ᵀ   Table 3, READ P:403-409
 *   a4  (fused in read_apply) TailBufferUpdate                      Table 3
 *   a5  write_commit          BoundaryUpdate into the shadow slot    Table 3, WRITE P:410-417
 *   a6  (fused in write_commit) group-atomic Commit v -> v+1         P:391-394, CONTROL P:418-423
 *   a7  tttstate_snapshot / rollback / tttstate_fork, failed write
 * The WRITE rule is SURVEY.md §8(c) reading i: ΔW_{v+1} = ΔW_v + η·V_cᵀZ_c
 * (the paper delegates the rule to the backend).
 *
 * Conventions (every entry point):
 *  - Returns ttt_status; no exception crosses the ABI.  tttstate_last_error()
 *    gives a human-readable message for the calling thread's last failure.
 *  - Validation happens before any side effect: a call that returns an error
 *    leaves every owner's (version, committed bytes, tail) unchanged
 *    (SPEC S:359).  The one exception is TTT_E_WRITE_FAILED, which by
 *    definition has run the update and *not* committed it.
 *  - Device pointers are stream-ordered on the `stream` argument (a
 *    cudaStream_t passed as void*, NULL = legacy default stream).  No call
 *    blocks the host except tttstate_sync, tttstate_refusals and the test hooks
 *    (read_payload / read_slot_raw / read_tail / device_version), and — only
 *    while an earlier write_commit of the same owner is still unconfirmed —
 *    the calls that confirm it (see "Commit confirmation" below).  All compute
 *    calls on one pool must be issued on one stream (or otherwise serialised):
 *    a pool owns one device workspace.
 *  - Ownership: the caller owns the device arena, W_down, X, targets, Y and
 *    streams; the library never allocates device memory.  The pool owns the
 *    slot assignment, tails, version tables and checkpoints inside the arena,
 *    plus a small pinned device-mapped HOST block (24 B per owner) into which
 *    the commit kernel writes each member's post-commit (version, slot).
 *  - Commit confirmation.  write_commit never waits for its kernels: the host
 *    mirror moves every member to v+1 at once (no host sync on the decode
 *    path).  The device may still refuse a member whose candidate is not
 *    finite (App. H fallback resolved on the device, reading xx):
 *    that member keeps v and its committed bytes, and its chunk's evidence is
 *    dropped.  An owner's latest commit is "confirmed" (the mirror corrected
 *    from the device's record, waiting on that commit's event, normally long
 *    complete) by every call that relies on its committed version or slot:
 *    tttstate_version, tttstate_snapshot, tttstate_fork (source),
 *    write_commit / fused read_apply of an owner holding a checkpoint, and
 *    tttstate_sync (all owners).  READ launches use the device slot table, so
 *    they always see the device's committed state.
 *  - Layouts are row-major.  Element type of every operand (ΔW, W_down, X,
 *    targets, Y, residual) is the pool's σ.dtype: TTT_BF16 (uint16 bf16
 *    bits) or TTT_FP32.  Accumulation is fp32 in every kernel.
 *  - A pool created with dev_arena == NULL is host-only: the state machine,
 *    planner and validation work (tests on a CPU box), every call that must
 *    touch the device returns TTT_E_NO_DEVICE.  There is no CPU fallback.
 */
#ifndef TTTSTATE_H
#define TTTSTATE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TTT_OK = 0,
  TTT_E_UNKNOWN_OWNER = 1,     /* owner not registered in this pool */
  TTT_E_DUPLICATE_OWNER = 2,   /* alloc/fork target already registered */
  TTT_E_VERSION_MISMATCH = 3,  /* expected v != committed V(r) (Eq. 3) */
  TTT_E_OWNER_COLLISION = 4,   /* μ not injective */
  TTT_E_MIXED_KEY = 5,         /* group members differ in ρ/τ/σ/π (Eq. 3) */
  TTT_E_DOUBLE_WRITE = 6,      /* a second WRITE for an owner with one pending */
  TTT_E_TAIL_NOT_FULL = 7,     /* write_commit before the chunk's C entries exist */
  TTT_E_NO_CHECKPOINT = 8,     /* rollback without snapshot */
  TTT_E_WRITE_FAILED = 9,      /* group ran, NOT committed; versions and bytes intact */
  TTT_E_POOL_FULL = 10,        /* no free owner / checkpoint slot */
  TTT_E_SHAPE = 11,            /* unsupported or inconsistent shape */
  TTT_E_TAIL_FULL = 12,        /* append past C (the boundary should have fired) */
  TTT_E_WRONG_EFFECT = 13,     /* e.g. write_commit on a READ group */
  TTT_E_NOT_APPLIED = 14,      /* step_done/write_commit before every layer was applied */
  TTT_E_ALREADY_APPLIED = 15,  /* read_apply twice for one (owner, layer, token) */
  TTT_E_CAPACITY = 16,         /* output buffer too small */
  TTT_E_INVALID_ARG = -1,
  TTT_E_CUDA = -2,
  TTT_E_NO_DEVICE = -3
} ttt_status;

enum { TTT_READ = 0, TTT_WRITE = 1 };                              /* ρ */
enum { TTT_FP32 = 0, TTT_BF16 = 1 };                               /* σ.dtype */
enum { TTT_FAST_WEIGHT = 0, TTT_LOW_RANK = 1, TTT_STREAMING = 2 }; /* τ */
enum { TTT_MODE_SERIAL = 0, TTT_MODE_PHASE = 1, TTT_MODE_FULL = 2 };

/* τ + σ of one pool.  rule 0: ΔW += η·V_cᵀZ_c (reading i).
 * rule 1 (SPEC-compat, S:188 / S:215; fast-weight backend, d_model == d_ff):
 * ΔW += η·m mᵀ with m the mean of the chunk's z; READ is unchanged, so the
 * caller passes W_down = I to get SPEC's y = x + ΔW·x.
 * backend: TTT_FAST_WEIGHT (rank 0) or TTT_LOW_RANK (NEXT f1: payload A
 * [rank][d_ff] then B [rank][d_model] per layer, bf16, 1 <= rank <= 64).  */
typedef struct {
  int32_t backend, dtype, d_model, d_ff, chunk, rank, n_layers, rule;
} ttt_shape;

/* Eq. 2: e_i = (r_i, τ_i, σ_i, ρ_i, v_i), plus placement π and ready step. 40 bytes. */
typedef struct {
  uint64_t owner;
  int32_t effect, backend, shape_id, placement;
  uint64_t expected_version;
  int64_t ready_step;
} ttt_event;

/* A legal group G with its injective owner map μ: slot b -> owner_map[b]. */
typedef struct {
  int32_t effect, backend, shape_id, placement;
  int32_t n, _reserved;
  const uint64_t *owner_map;
  int64_t issue_step;
} ttt_group;

typedef struct ttt_pool ttt_pool;
typedef struct ttt_planner ttt_planner;

const char *tttstate_last_error(void);
const char *tttstate_status_name(ttt_status s);

/* ------------------------------------------------------------------ pool */
/* Bytes of device arena a pool needs: double-slot ΔW [2·max_owners + n_ckpt]
 * [L][d_model][d_ff], tails [max_owners][L][C][d_ff + d_model], device
 * tables and kernel workspace (DESIGN.md §"HBM layout").                    */
ttt_status tttstate_pool_bytes(const ttt_shape *shape, int32_t max_owners, int32_t n_ckpt,
                               size_t *bytes_out);

/* Create a pool inside `dev_arena` (device memory the caller owns, ≥ the
 * bytes above, 1024-byte aligned) for shape `shape`, interned as σ id
 * `shape_id`, placement π = `placement` (the device rank).  `w_down` is the
 * shared base [L][d_model][d_ff] on the device; it is borrowed, not copied.
 * dev_arena == NULL makes a host-only pool (see header comment).            */
ttt_status tttstate_pool_create(const ttt_shape *shape, int32_t shape_id, int32_t placement,
                                int32_t max_owners, int32_t n_ckpt, void *dev_arena,
                                size_t arena_bytes, const void *w_down, ttt_pool **out);
ttt_status tttstate_pool_destroy(ttt_pool *pool);

/* Register `owner` at version v0 (v0 = 0 for a fresh state).
 * init == NULL: ΔW = 0; else device [L][d_model][d_ff] copied in.  Empty tail. */
ttt_status tttstate_alloc(ttt_pool *pool, uint64_t owner, const void *init, uint64_t v0,
                          uint64_t *v_out, void *stream);
ttt_status tttstate_free(ttt_pool *pool, uint64_t owner);

/* Seed an empty tail with n ≤ C−1 entries (bursty starts, reading xv):
 * Z device [L][n][d_ff], V device [L][n][d_model].                          */
ttt_status tttstate_tail_load(ttt_pool *pool, uint64_t owner, int32_t n, const void *Z,
                              const void *V, void *stream);

ttt_status tttstate_version(ttt_pool *pool, uint64_t owner, uint64_t *v_out);
ttt_status tttstate_tail_len(ttt_pool *pool, uint64_t owner, int32_t *len_out);

/* a1 — NextStep: fills e=(r, τ, σ, ρ, v=V(r), π, ready_step=clock);
 * ρ = WRITE iff this step's token completes the chunk (reading ii).         */
ttt_status tttstate_next_event(ttt_pool *pool, uint64_t owner, int64_t clock, ttt_event *out);
/* a1 for n owners at once (one host call per serving step): out[i] as above for owners[i].
 * Host-only. Validation first: an unknown owner fails the whole call and writes nothing. */
ttt_status tttstate_next_events(ttt_pool *pool, const uint64_t *owners, int32_t n, int64_t clock, ttt_event *out);

/* ---------------------------------------------------------------- planner */
ttt_status ttt_planner_create(int32_t mode, int32_t B, int32_t w, ttt_planner **out);
ttt_status ttt_planner_destroy(ttt_planner *pl);
/* V(r) for events with shape_id == pool's σ id are looked up in `pool`.     */
ttt_status ttt_planner_attach(ttt_planner *pl, ttt_pool *pool);
ttt_status ttt_planner_pending(ttt_planner *pl, int32_t *n_out);

/* a2 — LegalGroups: add `events` (ready at `clock`) to the κ=(ρ,τ,σ,π)
 * buckets, reject version-mismatched or duplicate-owner events into
 * `rejected` (never issued), and emit every group that is due:
 * the B oldest (ready_step, owner) of a bucket, or the whole bucket once its
 * oldest member has waited w steps (reading ix).  Groups are written to
 * `out` (their owner_map points into `owner_buf`), in κ order.             */
ttt_status plan_batch(ttt_planner *pl, const ttt_event *events, int32_t n, int64_t clock,
                      ttt_group *out, int32_t cap, uint64_t *owner_buf, int32_t owner_cap,
                      int32_t *n_out, ttt_event *rejected, int32_t rej_cap, int32_t *n_rej);

/* Eq. 3 + owner-map clause for an externally formed group: homogeneous key
 * (checked against the pool's τ/σ/π), injective μ, v_b == V(μ(b)).          */
ttt_status validate_group(ttt_pool *pool, const ttt_group *g, const uint64_t *expected_versions);

/* ------------------------------------------------------------ operators */
/* a3 + a4 — READ for layer `layer` of every member b of group g (READ or
 * WRITE group; the WRITE step's own token is applied with version v):
 *   Y[y_rows[b], :] = X[x_rows[b], :] · (W_down[layer] + ΔW_{μ(b)}[layer])ᵀ (+ resid[y_rows[b], :])
 * X: [*, d_ff], Vt: [*, d_model] update targets, Y/resid: [*, d_model], all
 * device, σ.dtype.  *_rows == NULL means row b.  The committed slot is read
 * through the device active-slot table, never written.  (z=X row, v=Vt row)
 * is appended to the owner's layer-`layer` tail at the token's tail index.
 * Errors: TTT_E_ALREADY_APPLIED, TTT_E_TAIL_FULL, TTT_E_OWNER_COLLISION,
 * TTT_E_UNKNOWN_OWNER, TTT_E_SHAPE (layer out of range).                     */
ttt_status read_apply(ttt_pool *pool, const ttt_group *g, int32_t layer, const void *X,
                      const int32_t *x_rows, const void *Vt, const int32_t *v_rows, void *Y,
                      const int32_t *y_rows, const void *resid, void *stream);

/* NEXT f2 — chunk-granular READ (prefill): for every member b of WRITE group g,
 * whose tail is empty, apply all C tokens of its next chunk at the committed
 * version v in one tensor-core GEMM per layer and append them to the tail:
 *   Y[b, t, :] = X[b, t, :] · (W_down[layer] + ΔW_{μ(b)}[layer])ᵀ,  t < C
 * X [n][C][d_ff], Vt [n][C][d_model], Y [n][C][d_model], device, bf16 only.
 * After every layer was applied the chunk's boundary token counts as applied:
 * call write_commit(g) to commit v+1 (same group).  Paper: READs of a chunk
 * keep version v (Table 3); chunk boundaries every C_ttt tokens
 * (P:160-161).  Errors: TTT_E_SHAPE (not bf16 / d_ff % 64 / d_model % 128 or
 * 160 / C > 128), TTT_E_TAIL_FULL (not at a chunk start), TTT_E_ALREADY_APPLIED. */
ttt_status read_apply_chunk(ttt_pool *pool, const ttt_group *g, int32_t layer, const void *X, const void *Vt,
                            void *Y, void *stream);

/* NEXT f3 — streaming learner (C = 1): η used when read_apply of a WRITE group
 * writes the candidate ΔW + η·v·xᵀ in the same pass (default 0.01f); the
 * following write_commit must pass the same η and then only commits.        */
ttt_status tttstate_set_eta(ttt_pool *pool, float eta);

/* UpdateKVAndTailMetadata for a READ group once every layer was applied:
 * tail length += 1 per member (Alg. 1 line 13).                             */
ttt_status tttstate_step_done(ttt_pool *pool, const ttt_group *g);

/* a5 + a6 — WRITE for every member of WRITE group g, then group-atomic commit:
 * for every layer, ΔW̃ = ΔW_v + η·Σ_{t<C} v_t z_tᵀ is written into each
 * member's shadow slot (fp32 accumulate, one rounding to σ.dtype); then one
 * commit kernel publishes active ^= 1, V += 1 for all members iff no member
 * failed (fail_mask bit b set = injected failure of member b; a non-finite
 * candidate element = device-detected failure).  On return tails are
 * cleared and new_versions[b] (host, may be NULL) = v+1 — provisional until
 * confirmed (header "Commit confirmation").  An injected failure returns
 * TTT_E_WRITE_FAILED with versions, committed bytes and tails intact (the
 * caller retries as singletons, App. H fallback).  A
 * device-detected failure fails the group on the device, which resolves the
 * singleton retries at once: members with finite candidates commit (their
 * retry would write the same bytes), the others keep v (refusal records:
 * tttstate_refusals; counted by tttstate_sync).  fail_mask: host array of
 * ceil(n/32) words or NULL.                                                 */
ttt_status write_commit(ttt_pool *pool, const ttt_group *g, float eta, const uint32_t *fail_mask,
                        uint64_t *new_versions, void *stream);

/* a7 — c_r^v <- s_r^v: pins the committed slot (O(1)); latest wins. */
ttt_status tttstate_snapshot(ttt_pool *pool, uint64_t owner, void *stream);
/* a7 — restore the checkpointed slot and version, clear the tail
 * (reading vii), keep the checkpoint.  v_out may be NULL.      */
ttt_status rollback(ttt_pool *pool, uint64_t owner, uint64_t *v_out, void *stream);
/* a7 — new lineage dst from src's committed state, same v, empty tail (reading viii). */
ttt_status tttstate_fork(ttt_pool *pool, uint64_t src, uint64_t dst, void *stream);

/* Synchronise `stream` and confirm every pending commit.  Returns
 * TTT_E_WRITE_FAILED (and n_failed_out > 0) if groups had members refused on
 * the device since the last sync; those members are at the version they
 * kept, with empty tails.                                                    */
ttt_status tttstate_sync(ttt_pool *pool, void *stream, int32_t *n_failed_out);
/* Drain the device refusal records (synchronises `stream`): for each member the
 * device refused, its owner id, the version it kept and the commit sequence
 * number of the write_commit that ran it (tttstate_last_commit_seq).  Returns
 * at most cap records per call, oldest first; TTT_E_CAPACITY if more than
 * 4096 records accumulated between drains.                                   */
ttt_status tttstate_refusals(ttt_pool *pool, uint64_t *owners, uint64_t *versions, uint64_t *seqs,
                             int32_t cap, int32_t *n_out, void *stream);
/* Sequence number of the pool's latest successful write_commit (0 before any). */
ttt_status tttstate_last_commit_seq(ttt_pool *pool, uint64_t *seq_out);

/* ------------------------------------------------------- one serving step */
/* Inputs/outputs of one decode step: the token of owners[i] sits at row rows[i]
 * of every layer's X [*, d_ff], Vt [*, d_model], Y / resid [*, d_model]; layer
 * l's matrices start x/v/y/r_layer_stride ELEMENTS after layer l−1's.  Device
 * memory, σ.dtype.  rows == NULL: row i.  resid may be NULL.  X and Vt are
 * inputs of the whole step: fully written (on `stream`, or before it) when the
 * call is made, not aliasing Y / resid, and not written while the step's
 * launches run — the step's later READ launches stage their x rows before their
 * PDL wait once its first launch has passed it (TTT_READ_EARLY_X=0: never).  */
typedef struct {
  const void *X;
  int64_t x_layer_stride;
  const void *Vt;
  int64_t v_layer_stride;
  void *Y;
  int64_t y_layer_stride;
  const void *resid;
  int64_t r_layer_stride;
  const int32_t *rows;
  void *ev_write_begin, *ev_write_end;   /* profiling (may be NULL): cudaEvent_t recorded right before the
                                          * step's first WRITE group's WRITE launches and after its commit */
  int64_t rows_total;                    /* rows of each layer's X / Vt / Y (0: unknown).  Lets a low-rank
                                          * group with contiguous rows skip the gather of its X rows */
} ttt_step_io;

/* Host buffers the step fills (caller-owned).  groups/owner_buf as plan_batch;
 * v_before[j] (may be NULL) = the version issued member j's token used;
 * member_seq[j] (may be NULL) = the commit sequence number that published (or
 * tried to publish) member j's WRITE, 0 for READ members; injected[k] (may be
 * NULL) = 1 if WRITE group k hit an injected failure and ran the singleton
 * fallback.  Members are numbered in owner_buf order.                          */
typedef struct {
  ttt_group *groups;
  int32_t group_cap;
  int32_t owner_cap;
  uint64_t *owner_buf;
  uint64_t *v_before;
  uint64_t *member_seq;
  int32_t *injected;
  int32_t rej_cap;
  int32_t _pad;
  ttt_event *rejected;
  int32_t n_groups, n_rejected, n_read, n_write, n_injected, _pad2;
} ttt_step_out;

/* One iteration of Alg. 1 for the owners listed, in one call (no
 * per-layer host round trips, no host sync — SURVEY App. B "Launch and
 * overhead"):  a1 NextStep for every listed owner without an event pending in
 * the planner (w > 0 holds events across steps) -> a2 plan_batch at `clock`
 * (rejected events are returned, never issued; re-extract them next step) ->
 * for every group, L dependent read_apply launches (a3 + a4) -> READ groups:
 * step done; WRITE groups: write_commit (a5 + a6, η = eta).  Owners in
 * fail_owners get an injected WRITE failure on this step's first attempt; such
 * a group is retried as serial singletons in μ order (App. H).
 * Validation (owners known and distinct, buffers, planner capacity) happens
 * before any side effect; a CUDA error after launches began returns TTT_E_CUDA. */
ttt_status tttstate_serve_step(ttt_pool *pool, ttt_planner *pl, const uint64_t *owners, int32_t n, int64_t clock,
                               const ttt_step_io *io, float eta, const uint64_t *fail_owners, int32_t n_fail,
                               ttt_step_out *out, void *stream);

/* Test hooks (blocking): committed ΔW[layer] of owner -> host [d_model][d_ff];
 * tail entries -> host Z [C][d_ff], V [C][d_model]; device version table.    */
ttt_status tttstate_read_payload(ttt_pool *pool, uint64_t owner, int32_t layer, void *host_dst,
                                 void *stream);
ttt_status tttstate_read_slot_raw(ttt_pool *pool, uint64_t owner, int32_t which, int32_t layer,
                                  void *host_dst, void *stream);
ttt_status tttstate_read_tail(ttt_pool *pool, uint64_t owner, int32_t layer, void *host_Z,
                              void *host_V, void *stream);
ttt_status tttstate_device_version(ttt_pool *pool, uint64_t owner, uint64_t *v_out, void *stream);

/* Kernel counters (for bench.py's gpu_launches claim): kernels launched by
 * this library since load.                                                  */
int64_t tttstate_launch_count(void);
/* Select the WRITE kernel: 0 = auto (tcgen05 for bf16 when available),
 * 1 = SIMT fp32-FFMA kernel, 2 = tcgen05 kernel.  Returns previous value.   */
int32_t tttstate_set_write_impl(int32_t impl);
/* Test hook for the stress suite's negative control ("disable
 * rollback (test hook) -> MidGroupWriteFail scenario fails").  flags =
 * TTT_HOOK_NO_GROUP_ATOMICITY breaks the group-atomic commit of write_commit
 * (P:418-423): when an injected fail bit is set, the members whose bit
 * is clear are published anyway (a non-atomic selective commit) and the call
 * still returns TTT_E_WRITE_FAILED.  Process-wide; 0 restores the contract.
 * Never set outside tests.  Returns the previous flags.                     */
#define TTT_HOOK_NO_GROUP_ATOMICITY 1
int32_t tttstate_set_test_hook(int32_t flags);

#ifdef __cplusplus
}
#endif
#endif /* TTTSTATE_H */
