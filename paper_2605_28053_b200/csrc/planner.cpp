// a2 — TTT-aware batch planner (host, C++).
//
// PAPER §4.3: "For each ready transition e_i, the planner
// computes κ_i = (ρ_i, τ_i, σ_i, π_i) ... The owner-local version v_i is
// checked against the committed version V(r_i) ... Requests with different
// keys are never co-issued ... For each key, the planner emits a group at
// target batch size B or waits at most w decode steps for compatible
// arrivals. When the wait budget expires, it issues the current legal prefix
// after owner-version and owner-map checks."  Legality: Eq. 3;
// bounded waiting: Eq. 4.  Readings: over-full
// buckets take the B oldest by (ready_step, owner id), the wait timer runs
// from the oldest member (ix); mismatched versions are rejected to the
// caller for revalidation, never issued (x).  Modes: serial / phase grouping
// / full (Table 4).
#include <algorithm>
#include <map>
#include <string>
#include <tuple>
#include <unordered_set>
#include <vector>

#include "pool.h"

#include <nvtx3/nvToolsExt.h>

struct ttt_planner {
  int mode = TTT_MODE_FULL, B = 8, w = 0;
  std::vector<ttt_pool *> pools;
  using Key = std::tuple<int32_t, int32_t, int32_t, int32_t>;   // (ρ, τ, σ, π)
  std::map<Key, std::vector<ttt_event>> buckets;
};

namespace {

ttt_status perr(ttt_status s, const char *m) {
  ttt::set_last_error(std::string(tttstate_status_name(s)) + ": " + m);   // tttstate_last_error()
  return s;
}

// V(r) for an event: the attached pool of its (σ, π).  false if unknown.
bool lookup_version(const ttt_planner *pl, const ttt_event &e, uint64_t *v) {
  for (ttt_pool *p : pl->pools) {
    if (p->shape_id != e.shape_id || p->placement != e.placement || p->sh.backend != e.backend) continue;
    auto it = p->owners.find(e.owner);
    if (it == p->owners.end()) return false;
    *v = it->second.version;
    return true;
  }
  return false;
}

bool older(const ttt_event &a, const ttt_event &b) {
  return a.ready_step != b.ready_step ? a.ready_step < b.ready_step : a.owner < b.owner;
}

}  // namespace

namespace ttt {

void planner_pending_owners(const ttt_planner *pl, std::unordered_set<uint64_t> &out) {
  for (auto &kv : pl->buckets)
    for (auto &e : kv.second) out.insert(e.owner);
}

}  // namespace ttt

extern "C" {

ttt_status ttt_planner_create(int32_t mode, int32_t B, int32_t w, ttt_planner **out) {
  if (!out || B < 1 || B > ttt::kMaxGroup || w < 0 || mode < TTT_MODE_SERIAL || mode > TTT_MODE_FULL)
    return perr(TTT_E_INVALID_ARG, "mode/B/w");
  auto *pl = new ttt_planner();
  pl->mode = mode;
  pl->B = B;
  pl->w = w;
  *out = pl;
  return TTT_OK;
}

ttt_status ttt_planner_destroy(ttt_planner *pl) {
  delete pl;
  return TTT_OK;
}

ttt_status ttt_planner_attach(ttt_planner *pl, ttt_pool *pool) {
  if (!pl || !pool) return perr(TTT_E_INVALID_ARG, "null");
  pl->pools.push_back(pool);
  return TTT_OK;
}

ttt_status ttt_planner_pending(ttt_planner *pl, int32_t *n_out) {
  if (!pl || !n_out) return perr(TTT_E_INVALID_ARG, "null");
  int n = 0;
  for (auto &kv : pl->buckets) n += (int)kv.second.size();
  *n_out = n;
  return TTT_OK;
}

ttt_status plan_batch(ttt_planner *pl, const ttt_event *events, int32_t n, int64_t clock, ttt_group *out,
                      int32_t cap, uint64_t *owner_buf, int32_t owner_cap, int32_t *n_out, ttt_event *rejected,
                      int32_t rej_cap, int32_t *n_rej) {
  nvtxRangePushA("plan_batch");
  struct Pop {
    ~Pop() { nvtxRangePop(); }
  } pop_;
  if (!pl || (n > 0 && !events) || !n_out || !n_rej || n < 0) return perr(TTT_E_INVALID_ARG, "null arg");
  auto buckets = pl->buckets;                        // work on a copy: no side effect on error
  std::vector<ttt_event> rej;
  std::unordered_set<uint64_t> pending;
  for (auto &kv : buckets)
    for (auto &e : kv.second) pending.insert(e.owner);
  // steps 1, 2, 5: key, version check, one pending transition per owner (μ injective)
  for (int k = 0; k < n; ++k) {
    const ttt_event &e = events[k];
    uint64_t v;
    if (!lookup_version(pl, e, &v) || v != e.expected_version || pending.count(e.owner)) {
      rej.push_back(e);
      continue;
    }
    buckets[ttt_planner::Key(e.effect, e.backend, e.shape_id, e.placement)].push_back(e);
    pending.insert(e.owner);
  }
  // pending transitions whose owner moved (rollback) are stale: revalidate
  for (auto &kv : buckets) {
    std::vector<ttt_event> keep;
    for (auto &e : kv.second) {
      uint64_t v;
      if (lookup_version(pl, e, &v) && v == e.expected_version)
        keep.push_back(e);
      else
        rej.push_back(e);
    }
    kv.second.swap(keep);
  }
  // steps 3, 4: per key (in key order), full groups of B, then the expired prefix
  struct G {
    ttt_planner::Key key;
    std::vector<uint64_t> owners;
  };
  std::vector<G> groups;
  for (auto &kv : buckets) {
    auto &b = kv.second;
    std::stable_sort(b.begin(), b.end(), older);
    const int eff = std::get<0>(kv.first);
    const int capB = (pl->mode == TTT_MODE_SERIAL || (pl->mode == TTT_MODE_PHASE && eff == TTT_WRITE)) ? 1 : pl->B;
    size_t i = 0;
    while (b.size() - i >= (size_t)capB) {
      G g{kv.first, {}};
      for (int k = 0; k < capB; ++k) g.owners.push_back(b[i + k].owner);
      groups.push_back(std::move(g));
      i += capB;
    }
    if (i < b.size() && clock - b[i].ready_step >= pl->w) {
      G g{kv.first, {}};
      for (; i < b.size(); ++i) g.owners.push_back(b[i].owner);
      groups.push_back(std::move(g));
    }
    b.erase(b.begin(), b.begin() + i);
  }
  size_t n_owners = 0;
  for (auto &g : groups) n_owners += g.owners.size();
  if ((int)groups.size() > cap || (int)n_owners > owner_cap || (int)rej.size() > rej_cap ||
      (!groups.empty() && (!out || !owner_buf)) || (!rej.empty() && !rejected))
    return perr(TTT_E_CAPACITY, "output buffers too small");
  size_t off = 0;
  for (size_t k = 0; k < groups.size(); ++k) {
    ttt_group &o = out[k];
    o.effect = std::get<0>(groups[k].key);
    o.backend = std::get<1>(groups[k].key);
    o.shape_id = std::get<2>(groups[k].key);
    o.placement = std::get<3>(groups[k].key);
    o.n = (int32_t)groups[k].owners.size();
    o._reserved = 0;
    std::copy(groups[k].owners.begin(), groups[k].owners.end(), owner_buf + off);
    o.owner_map = owner_buf + off;
    o.issue_step = clock;
    off += groups[k].owners.size();
  }
  for (size_t k = 0; k < rej.size(); ++k) rejected[k] = rej[k];
  for (auto it = buckets.begin(); it != buckets.end();)
    it = it->second.empty() ? buckets.erase(it) : std::next(it);
  pl->buckets.swap(buckets);
  *n_out = (int32_t)groups.size();
  *n_rej = (int32_t)rej.size();
  return TTT_OK;
}

}  // extern "C"
