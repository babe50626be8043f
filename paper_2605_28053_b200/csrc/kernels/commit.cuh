// a6 — the group commit as a device function: run by commit_kernel (one CTA) and by the
// last CTA of the tcgen05 WRITE kernel (fused commit, arrival counter).  Semantics in
// control.cu's header comment (group-atomic + App. H fallback resolved on the device).
#pragma once
#include "../internal.h"

namespace ttt {

// Every thread of the calling CTA must call this (it ends in a CTA-wide __syncthreads_or).
__device__ __forceinline__ void commit_members(const CommitParams &p) {
  int bad_any = 0;
  for (int b = threadIdx.x; b < p.n; b += blockDim.x) {
    const int o = p.owner_idx[b];
    const int bad = *reinterpret_cast<volatile int *>(p.mfail + o);
    if (p.forced_fail) {                         // injected: the host runs the singleton retries
      // (the flag stays: a fused C = 1 candidate is not recomputed by its retry; rollback /
      // alloc / fork clear it through set_state_kernel)
      if (p.partial && !((p.fail_bits[b / 32] >> (b % 32)) & 1u)) {   // test hook (negative control)
        p.sel[o] ^= 1;
        p.version[o] += 1ull;
      }
      continue;
    }
    p.mfail[o] = 0;                              // resolved here; the next WRITE raises it again if it must
    if (!bad) {
      p.sel[o] ^= 1;
      p.version[o] += 1ull;
    } else {
      const int k = atomicAdd(p.rlog_count, 1);
      RefusalRec r;
      r.owner = p.owner_id[b];
      r.version = p.version[o];
      r.seq = p.seq;
      r.pad = 0;
      p.rlog[k % kRefusalLog] = r;
    }
    bad_any |= bad;
    HostOwnerState h;
    h.version = p.version[o];
    h.seq = p.seq;
    h.sel = p.sel[o];
    h.pad = 0;
    p.hstate[o] = h;                             // posted writes into mapped host memory
  }
  if (__syncthreads_or(bad_any) && threadIdx.x == 0) atomicAdd(p.fail_count, 1);
  __threadfence_system();
}

}  // namespace ttt
