// kernel_lanesplit.cu -- placeholder until the lane-split kernel lands.
#include "kernels.cuh"

namespace b200sha3 {

bool lanesplit_supported(int, uint64_t, uint64_t) { return false; }

cudaError_t launch_hash_lanesplit(const HashArgs&, const LaunchPlan&, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace b200sha3
