// a5 — WRITE (BoundaryUpdate) on tcgen05 tensor cores: placeholder until the
// sm_100a kernel lands; write_tc_supported() gates dispatch.
#include "../internal.h"

namespace ttt {
bool write_tc_supported(int, int, int) { return false; }
cudaError_t launch_write_tc(const WriteParams &, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace ttt
