// Host-side records of the TTTState pool (double-slot HBM arena + host mirror).
#pragma once
#include <cstdint>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/tttstate.h"
#include "internal.h"

namespace ttt {

// One owner's host mirror (authoritative for planning; the device tables
// sel[]/version[] are authoritative for kernels; tttstate_sync reconciles).
struct OwnerRec {
  uint64_t stamp = 0;         // group-validation visit mark (μ injectivity check without allocation)
  int idx = -1;               // owner index: slots 2*idx (+0/+1)
  int sel = 0;                // active slot of the pair
  uint64_t version = 0;       // V(r)
  int tail_len = 0;           // completed tokens in the current chunk
  std::vector<uint8_t> applied;   // per layer: current token appended
  int n_applied = 0;
  bool chunk_mode = false;    // current chunk applied by read_apply_chunk (f2)
  int fused_layers = 0;       // f3: layers whose candidate read_apply already wrote (C = 1)
  bool has_ckpt = false;      // c_r^v
  uint64_t ckpt_v = 0;
  int ckpt_sel = 0;           // pinned pair slot (when ckpt_pool < 0)
  int ckpt_pool = -1;         // checkpoint-pool slot index (>= 0 when evicted)
  uint64_t pending_seq = 0;   // latest write_commit of this owner not yet confirmed (0: confirmed)
};

struct Layout {
  size_t slots = 0, tailZ = 0, tailV = 0, sel = 0, ver = 0, flags = 0, mfail = 0, rlog = 0, P = 0, tickets = 0;
  size_t members = 0;                              // MemberTable (chunk / low-rank READ groups)
  size_t wslab = 0, wtick = 0;                     // wide split-K chunk READ workspace (bf16 fast-weight)
  size_t ptc = 0, ptc_bytes = 0;                   // TMA + tcgen05 decode READ partials (bf16 fast-weight)
  size_t xflag = 0;                                // serve_step epoch published after a READ's PDL wait
  size_t Xg = 0, Y32 = 0, U = 0, Ctr = 0, total = 0;   // low-rank READ workspace
};

Layout compute_layout(const ttt_shape &s, int max_owners, int n_ckpt);
void planner_pending_owners(const ttt_planner *pl, std::unordered_set<uint64_t> &out);
void set_last_error(const std::string &msg);
constexpr int kEventRing = 64;   // commit events kept (a newer record of a slot is a later point on the stream)

}  // namespace ttt

struct ttt_pool {
  ttt_shape sh{};
  uint64_t stamp_epoch = 0;
  int shape_id = 0, placement = 0, max_owners = 0, n_ckpt = 0;
  bool host_only = true;
  unsigned char *arena = nullptr;
  size_t arena_bytes = 0;
  const void *w_down = nullptr;
  size_t esize = 4;
  long long E = 0, Ew = 0, slot_elems = 0, tz_owner = 0, tv_owner = 0;   // E: payload / layer, Ew: W_down / layer
  ttt::Layout lay;
  std::unordered_map<uint64_t, ttt::OwnerRec> owners;
  std::vector<int> free_idx, free_ckpt;
  int fail_seen = 0;          // device fail_count already reported by tttstate_sync
  int rlog_read = 0;          // refusal-log records already drained (tttstate_refusals)
  float eta = 0.01f;          // η used by the fused C = 1 path (tttstate_set_eta)
  // lazy commit confirmation: write_commit advances the host mirror optimistically and records
  // an event; the commit kernel writes each member's post-commit (version, sel, seq) into
  // pinned device-mapped host memory, read back only when a call needs the confirmed state
  uint64_t commit_seq = 0;
  int step_epoch = 0;          // > 0 while tttstate_serve_step issues its launches (ReadParams::x_epoch)
  int epoch_ctr = 0;
  std::vector<cudaEvent_t> ev_ring;                 // event recorded after commit seq k: ev_ring[k % size]
  ttt::HostOwnerState *hstate = nullptr;            // [max_owners], cudaHostAllocMapped (host view)
  ttt::HostOwnerState *hstate_dev = nullptr;        // the same memory as the kernels address it
  ttt::MemberTable m_last{};                        // member table last uploaded to lay.members
  int m_n = -1;

  // device pointers (valid when !host_only)
  unsigned char *slot_ptr(long long slot) const {
    return arena + lay.slots + (size_t)slot * (size_t)slot_elems * esize;
  }
  size_t slot_bytes() const { return (size_t)slot_elems * esize; }
  int *d_sel() const { return reinterpret_cast<int *>(arena + lay.sel); }
  unsigned long long *d_ver() const { return reinterpret_cast<unsigned long long *>(arena + lay.ver); }
  int *d_fail_count() const { return reinterpret_cast<int *>(arena + lay.flags); }
  int *d_rlog_count() const { return reinterpret_cast<int *>(arena + lay.flags + 16); }
  int *d_mfail() const { return reinterpret_cast<int *>(arena + lay.mfail); }
  int *d_members() const { return reinterpret_cast<int *>(arena + lay.members); }
  int *d_wctr() const { return reinterpret_cast<int *>(arena + lay.flags + 32); }   // fused-commit arrivals
  ttt::RefusalRec *d_rlog() const { return reinterpret_cast<ttt::RefusalRec *>(arena + lay.rlog); }
};
