// b200sha3_dropin.cpp -- link-time replacement for the reference's
// proj/core/src/batch.cpp: defines sha3::hash_batch itself on top of the GPU
// engine.  Link this file (plus batch_adapter.cpp and libb200sha3.so) instead of
// the reference's batch.cpp; callers such as bench::run_benchmark
// (proj/tools/sha3cli/runner.cpp:45,52) need no source change.
//
// Compile with -DB200SHA3_USE_REFERENCE_TYPES -I<reference>/proj/core/include to
// build against the reference's own headers, or without it to use the
// compatible declarations of include/b200sha3/batch.hpp.
#include "b200sha3/batch.hpp"

namespace sha3 {

#ifndef B200SHA3_USE_REFERENCE_TYPES
BatchResult hash_batch(const HashBatch& batch, const EngineConfig& config);
#endif

BatchResult hash_batch(const HashBatch& batch, const EngineConfig& config) {
  return b200::hash_batch(batch, config, b200::DeviceConfig{});
}

}  // namespace sha3
