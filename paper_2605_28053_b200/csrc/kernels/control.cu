// a6 / a7 — commit, checkpoint copy and state set kernels.
//
// Commit: "Commit publishes a dirty state
// as owner r's next version only after the WRITE group succeeds ... The
// version counter changes here, not inside the backend update".  Group-atomic
// (SURVEY.md §8(c) reading vi) with App. H's fallback
// (a failed group is retried as serial singletons) resolved on the
// device, so the host never waits for a WRITE's outcome:
//   * an injected failure (host-known) publishes nothing; the host retries;
//   * a device-detected failure (non-finite candidate, per-owner flag raised by
//     the WRITE kernels) fails the group as a whole, and its singleton retries
//     are decided here at once: a member's candidate does not depend on the
//     other members (same committed state, same evidence, same kernel), so the
//     retry of a clean member would write the very bytes already sitting in its
//     shadow slot — it is published; a flagged member's retry would fail the
//     same way — it is refused for good (v and bytes intact, its chunk's
//     evidence dropped: DESIGN.md reading xx), and a refusal record is logged.
// No payload bytes move (the dirty candidate already sits in the shadow slot),
// replacing the paper's "selective commit" copy kernel with an
// O(1)-per-owner publish.  Every member's post-commit (version, sel, seq) is
// written to pinned device-mapped host memory for the host's lazy confirmation.
//
// Checkpoint copy ("Checkpoint write", K5): a 16-byte vectorised
// device copy used when a pinned checkpoint slot must be preserved, for
// fork, and for rollback from the checkpoint pool.
#include "../internal.h"
#include "commit.cuh"

namespace ttt {
namespace {

__global__ void commit_kernel(const CommitParams p) { commit_members(p); }

// K5 (HBM-bound, 2 x slot bytes): 8 independent 16-B streaming loads per thread in flight
// (128 B x 2048 threads = 256 KB per SM), then 8 streaming stores; neither side is re-read soon.
__global__ void __launch_bounds__(512) copy_kernel(uint4 *__restrict__ dst, const uint4 *__restrict__ src,
                                                   size_t n16) {
  constexpr int U = 8;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = __ldcs(src + i + k * stride);
#pragma unroll
    for (int k = 0; k < U; ++k) __stcs(dst + i + k * stride, v[k]);
  }
  for (; i < n16; i += stride) dst[i] = src[i];
  // the decode READ may request its first ΔW batch before its PDL wait (p.early_delta): slot
  // bytes this copy wrote (rollback from the checkpoint pool, fork) must be visible at exit
  __threadfence();
}

__global__ void copy_tail_bytes(unsigned char *dst, const unsigned char *src, size_t n) {
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  __threadfence();
}

__global__ void member_upload_kernel(const __grid_constant__ MemberTable t, int n, int *dst) {
  for (int i = threadIdx.x; i < 5 * n; i += blockDim.x) {
    const int k = i / n, b = i - k * n;
    dst[k * kMaxGroup + b] = t.a[k][b];
  }
}

__global__ void set_state_kernel(int *sel, unsigned long long *version, int *mfail, int idx, int s,
                                 unsigned long long v) {
  sel[idx] = s;
  version[idx] = v;
  mfail[idx] = 0;
  __threadfence();                               // visible at exit (see copy_kernel)
}

}  // namespace

cudaError_t launch_commit(const CommitParams &p, cudaStream_t s) {
  commit_kernel<<<1, 256, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_copy(void *dst, const void *src, size_t bytes, cudaStream_t s) {
  const size_t n16 = bytes / 16;
  if (n16) {
    const int grid = device_sm_count() * 4;
    copy_kernel<<<grid, 512, 0, s>>>(static_cast<uint4 *>(dst), static_cast<const uint4 *>(src), n16);
    count_launch();
  }
  if (bytes % 16) {
    copy_tail_bytes<<<1, 32, 0, s>>>(static_cast<unsigned char *>(dst) + n16 * 16,
                                     static_cast<const unsigned char *>(src) + n16 * 16, bytes % 16);
    count_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_member_upload(const MemberTable &t, int n, int *dst, cudaStream_t s) {
  member_upload_kernel<<<1, 256, 0, s>>>(t, n, dst);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_set_state(int *sel, unsigned long long *version, int *mfail, int idx, int sel_v,
                             unsigned long long ver, cudaStream_t s) {
  set_state_kernel<<<1, 1, 0, s>>>(sel, version, mfail, idx, sel_v, ver);
  count_launch();
  return cudaGetLastError();
}

}  // namespace ttt
