// Internal declarations shared by the host library (pool/planner/api) and
// the sm_100a kernels.  Not part of the public ABI (that is include/tttstate.h).
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace ttt {

constexpr int kMaxLrSeg = 16;          // low-rank READ: max K segments per A row
constexpr int kMaxReadMembers = 8;     // members per READ launch (X rows staged in smem)
constexpr int kMaxGroup = 256;         // members per group (planner B cap)
constexpr int kMaxKSplit = 16;         // low-rank base GEMM split-K slabs

// a3 + a4: decode READ over one layer for ≤ kMaxReadMembers members.
struct ReadParams {
  const void *X, *Vt, *resid;
  void *Y;
  const void *w_down_l;          // [d_model][d_ff] of this layer
  const void *slots;             // pool slot array base
  long long slot_elems;          // elements per slot (L * d_model * d_ff)
  long long layer_off;           // layer * d_model * d_ff
  const int *sel;                // device active-slot selector per owner index
  void *tailZ, *tailV;           // tail ring bases
  long long tz_owner, tv_owner;  // elements per owner (L*C*d_ff, L*C*d_model)
  long long tz_layer, tv_layer;  // layer offset in elements (layer*C*d_ff, layer*C*d_model)
  float *Pbase, *Pdelta;         // [kMaxReadMembers][d_model] partial sums
  int *tickets;                  // [d_model] arrival counters (self-resetting)
  int n, d_model, d_ff;
  int owner_idx[kMaxReadMembers];
  int x_row[kMaxReadMembers], v_row[kMaxReadMembers], y_row[kMaxReadMembers];
  int tail_pos[kMaxReadMembers];
  int fuse;                      // f3: also write ΔW + η·v·xᵀ to the shadow slot (C = 1)
  float eta;
  int *mfail;                    // [max_owners] per-owner device-failure flags (non-finite candidate)
  int order;                     // task order: 0 CTA-major, 1 SM-interleaved (balanced bytes per SM)
  int dyn;                       // per-CTA dynamic task hand-out (SM-interleaved order only)
  int kc;                        // > 0: tensor-core base (bf16), Pbase holds kc K-chunk slabs [kc][8][d_model]
  int l2keep;                    // not the group's last launch of this layer: keep W_down in L2 (evict_last)
  int xtma;                      // tensor-core-base kernel: stage the x rows with bulk copies (TMA)
  int early_delta;               // tensor-core-base kernel: first ΔW batch requested before the PDL wait
  // TMA + tcgen05 READ (read_decode_tc.cu): tensor-map extents and its partial-sum workspace
  int L, layer;
  long long n_slot_layers;       // pool slots × L (third extent of the slot tensor map)
  float *ptc;                    // [2][g][⌈d_model/128⌉·128][8] fp32 partials
  size_t ptc_bytes;
  // inside tttstate_serve_step (x_epoch > 0): X is an input of the whole step, so a launch may stage
  // its x rows before the PDL wait once an earlier launch of the same step has passed its wait and
  // published x_epoch in *xflag (device word; see read_decode_tc.cu)
  int *xflag;
  int x_epoch;
};

// a5: chunk update of one layer for every member (shadow slot <- ΔW_v + η VᵀZ).
struct WriteParams {
  void *slots;
  long long slot_elems, layer_off;
  const int *sel;
  const void *tailZ, *tailV;
  long long tz_owner, tv_owner, tz_layer, tv_layer;
  float eta;
  int *mfail;                    // [max_owners] per-owner device-failure flags (non-finite candidate)
  int n, d_model, d_ff, C;
  int max_owners, max_slots;     // tensor-map extents (tails, pool slots)
  int owner_idx[kMaxGroup];
};

// Post-commit state of one owner, written by the commit kernel into pinned device-mapped
// host memory (read by the host only after the commit's event completed).
struct HostOwnerState {
  unsigned long long version, seq;
  int sel, pad;
};
// One device-refused member (non-finite candidate), appended by the commit kernel.
struct RefusalRec {
  unsigned long long owner, version, seq;   // owner id, version it stays at, commit sequence number
  unsigned long long pad;
};
constexpr int kRefusalLog = 4096;          // records kept in the device ring (drained by tttstate_refusals)

// a6: group commit with the App. H fallback resolved on the device.
struct CommitParams {
  int *sel;
  unsigned long long *version;
  int *mfail;          // [max_owners] per-owner device-failure flags set by the WRITE kernels (cleared here)
  int *fail_count;     // cumulative groups with a device-refused member (read by tttstate_sync)
  int *rlog_count;     // refusal-log append counter
  RefusalRec *rlog;    // [kRefusalLog] ring
  HostOwnerState *hstate;   // mapped host [max_owners]: post-commit (version, sel, seq)
  unsigned long long seq;   // this commit's sequence number
  int forced_fail;     // injected failure (host-known): nothing publishes
  int n;
  int owner_idx[kMaxGroup];
  unsigned long long owner_id[kMaxGroup];
  int partial;         // test hook (TTT_HOOK_NO_GROUP_ATOMICITY): publish members with no fail bit
  unsigned fail_bits[kMaxGroup / 32];
};

// NEXT f2: chunk-granular READ of C tokens per member at one version (tcgen05).
struct ChunkLaunch {
  int n, d_model, d_ff, C, L, layer, max_slots;
  const int *sel;
  const void *X, *Vt, *w_down, *slots;
  void *Y, *tailZ, *tailV;
  long long tz_owner, tv_owner, tz_layer, tv_layer;
  int delta = 1;                 // 0: base product only (low-rank READ's X·W_downᵀ)
  int append = 1;                // append the chunk to the tail
  float *Y32 = nullptr;          // non-null: fp32 output rows b*C + t (< valid_rows) instead of bf16 Y
  int valid_rows = 0;
  int ksplit = 1;                // base mode: K split in `ksplit` ranges, slab ks at Y32 + ks*y32_slab
  long long y32_slab = 0;
  int owner_idx[kMaxGroup];
  const struct LowRankRead *lr = nullptr;   // non-null: fused low-rank READ (u = A x, finish) in this launch
  int *lr_ctr = nullptr;                    // fused mode counters [u_done, exit, tickets...], zero at rest
  int x_rowmap = 0;                         // X is [rows][d_ff] (2-D map, rows past n zero-filled)
  int x_row0 = 0;                           // x_rowmap: the group's first row in X (TMA row coordinate offset)
  long long x_rows_total = 0;               // x_rowmap: rows of the X buffer (0: the group's rows only)
  int cooperative = 0;                      // fused mode: cooperative launch (several low-rank pools live)
  const int *d_members = nullptr;           // device member table [5][kMaxGroup]: owner_idx, x_row, v_row,
                                            // y_row, tail_pos (kernel params stay small: see MemberTable)
  float *wide_slab = nullptr;               // wide split-K chunk READ: fp32 partial slabs (pool workspace)
  size_t wide_slab_bytes = 0;
  int *wide_tickets = nullptr;              //   and its per-tile arrival counters (zero at rest)
};

// Wide-tile split-K chunk READ plan (read_chunk_wide.cu): MPC members per CTA sharing each
// W_down box, T N-blocks (j < h: w_hi wide, else w_hi - 32), K split KS ways, one wave.
struct WidePlan {
  int mpc = 0, T = 0, KS = 0, w_hi = 0, h = 0, stages = 0, stage_bytes = 0;
  double cost = 0;               // modelled time: L2 -> SM bytes per CTA / bytes in flight
  int tiles = 0;
  int bk = 16;                   // K elements per ring stage (16 / 32 / 64)
};
constexpr int kWideMaxTiles = 160;          // workspace sizing: tiles per launch (≤ SM count)
constexpr size_t kWideSlabBytes = (size_t)kWideMaxTiles * 512 * 128 * 4;   // 512 TMEM columns x 128 rows fp32
bool plan_read_chunk_wide(int n, int d_model, int d_ff, int sms, int bk, WidePlan *out);
cudaError_t launch_read_chunk_wide(const ChunkLaunch &cl, const WidePlan &pl, cudaStream_t s);

// Per-member arrays of a chunk / low-rank READ group, kept in the pool's device workspace
// instead of the kernel parameters (parameter block ~7 KB -> ~0.6 KB; host per low-rank launch
// 18.0 -> 16.5 µs, r2): the table changes at most once per decode step (every layer of a step
// sees the same rows and tail positions), so it is uploaded by one small kernel when it changes.
struct MemberTable {
  int a[5][kMaxGroup];           // owner_idx, x_row, v_row, y_row, tail_pos
};
cudaError_t launch_member_upload(const MemberTable &t, int n, int *dst, cudaStream_t s);

// NEXT f1: low-rank delta READ / WRITE (DeltaAdapterState).
struct LowRankRead {
  int n, d_model, d_ff, rank;
  int x_row0 = -1;               // >= 0: the members' X rows are x_row0 .. x_row0 + n - 1 of a buffer
  long long x_rows_total = 0;    //   with x_rows_total rows (no gather: the GEMM's TMA map offsets them)
  const void *X, *Vt, *resid;
  void *Y, *Xg;
  float *Y32, *u;                // [ksplit][rows][d_model] base product slabs, [n·R][nseg] A·x partials
  int ksplit;
  int nseg;                      // A rows split into nseg K segments (one warp task each)
  int *ctr;                      // fused-mode counters (see ChunkLaunch::lr_ctr)
  long long y32_slab;
  const void *slots;
  long long slot_elems, layer_off;
  const int *sel;
  void *tailZ, *tailV;
  long long tz_owner, tv_owner, tz_layer, tv_layer;
  int owner_idx[kMaxGroup], x_row[kMaxGroup], v_row[kMaxGroup], y_row[kMaxGroup], tail_pos[kMaxGroup];
  const void *w_down = nullptr;  // [L][d_model][d_ff] (tensor maps of the one-pass kernel)
  int L = 0, layer = 0, max_slots = 0;
  int *xflag = nullptr;          // serve_step epoch word / epoch (ReadParams::xflag, x_epoch)
  int x_epoch = 0;
};
struct LowRankWrite {
  int n, d_model, d_ff, rank, C;
  void *slots;
  long long slot_elems, layer_off;
  const int *sel;
  const void *tailZ;
  long long tz_owner, tz_layer;
  float eta;
  int *mfail;                    // [max_owners] per-owner device-failure flags (non-finite candidate)
  int owner_idx[kMaxGroup];
};
bool read_chunk_fused_fits(int row_blocks, int d_model, int ksplit);
extern std::atomic<int> g_live_lowrank_pools;
cudaError_t launch_lowrank_read(const LowRankRead &p, const ChunkLaunch &base, cudaStream_t s);
cudaError_t launch_lowrank_write(const LowRankWrite &p, cudaStream_t s);
bool lowrank_tc_supported(int n, int d_model, int d_ff, int rank);
cudaError_t launch_lowrank_tc(const LowRankRead &p, const void *X, cudaStream_t s);   // one-pass READ

int device_sm_count();
bool read_chunk_supported(int d_model, int d_ff, int C);
cudaError_t launch_read_chunk(const ChunkLaunch &cl, cudaStream_t s);
cudaError_t launch_read_decode(int dtype, const ReadParams &p, cudaStream_t s);
bool read_decode_fits(int n, int d_model, int d_ff, int esize);
bool read_decode_tc_supported(int n, int d_model, int d_ff);
cudaError_t launch_read_decode_tc(const ReadParams &p, cudaStream_t s);
constexpr int kTcMaxG = 40;            // READ-tc workspace sizing: CTAs per row block
int read_decode_mma_chunks(int dtype, int d_ff);   // > 0: the bf16 tensor-core-base READ applies (its K chunks)
cudaError_t launch_write_simt(int dtype, const WriteParams &p, cudaStream_t s);
cudaError_t launch_write_rule1(int dtype, const WriteParams &p, cudaStream_t s);   // SPEC-compat rule 1 (square)
// bf16, tcgen05: every layer in one launch; cp != nullptr fuses the group commit (last CTA, `arrive`)
cudaError_t launch_write_tc(const WriteParams &p, const CommitParams *cp, int *arrive, cudaStream_t s);
bool write_tc_supported(int d_model, int d_ff, int C, int n_layers);
bool write_tc_triggers_early();   // TTT_WRITE_EARLY_DEP: the WRITE (+ fused commit) triggers dependents at entry
cudaError_t launch_commit(const CommitParams &p, cudaStream_t s);
cudaError_t launch_copy(void *dst, const void *src, size_t bytes, cudaStream_t s);
cudaError_t launch_set_state(int *sel, unsigned long long *version, int *mfail, int idx, int sel_v,
                             unsigned long long ver, cudaStream_t s);

void count_launch(int n = 1);

}  // namespace ttt
