// Host-side records of the TTTState pool (double-slot HBM arena + host mirror).
#pragma once
#include <cstdint>
#include <string>
#include <unordered_map>
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
};

struct Layout {
  size_t slots = 0, tailZ = 0, tailV = 0, sel = 0, ver = 0, flags = 0, P = 0, tickets = 0;
  size_t Xg = 0, Y32 = 0, U = 0, Ctr = 0, total = 0;   // low-rank READ workspace
};

Layout compute_layout(const ttt_shape &s, int max_owners, int n_ckpt);

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
  int fail_seen = 0;
  float eta = 0.01f;          // η used by the fused C = 1 path (tttstate_set_eta)

  // device pointers (valid when !host_only)
  unsigned char *slot_ptr(long long slot) const {
    return arena + lay.slots + (size_t)slot * (size_t)slot_elems * esize;
  }
  size_t slot_bytes() const { return (size_t)slot_elems * esize; }
  int *d_sel() const { return reinterpret_cast<int *>(arena + lay.sel); }
  unsigned long long *d_ver() const { return reinterpret_cast<unsigned long long *>(arena + lay.ver); }
  int *d_fail_flag() const { return reinterpret_cast<int *>(arena + lay.flags); }
  int *d_fail_count() const { return reinterpret_cast<int *>(arena + lay.flags + 16); }
};
