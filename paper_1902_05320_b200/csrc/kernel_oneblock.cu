// kernel_oneblock.cu -- the headline kernel: equal-length single-block messages
// (cfg1 / cfg5 of BASELINE.json: SHA3-256 over 64-byte messages), one message
// per thread.
//
// Replaces hash_into (proj/core/src/batch.cpp:15-25) for batches whose
// messages are whole lanes, shorter than the rate, 16-byte aligned, with a
// digest of whole 32-bit words: no loops, no predicates -- ML 64-bit lanes in
// with 16-byte loads, pad as two immediates, one permutation, OW 32-bit words
// out.  With UNROLL = 24 ptxas also removes the work on lanes that are zero on
// entry to round 0 and the lanes nobody reads after round 23 (4186 instead of
// 4370 instructions per SHA3-256 hash).
#include "oneblock.cuh"

namespace b200sha3 {

namespace {

// SHA3-256 / SHAKE256, 64-byte messages, 32-byte digests: the tuning matrix.
template <int UNROLL>
cudaError_t launch_sha3_256_64(const HashArgs& args, const LaunchPlan& plan,
                               cudaStream_t stream) {
  switch (plan.fma_preset) {
#define B200SHA3_CASE(P) \
  case P: return launch_oneblock_instance<17, 8, 8, UNROLL, P>(args, plan, stream);
    B200SHA3_CASE(0) B200SHA3_CASE(1) B200SHA3_CASE(2) B200SHA3_CASE(3)
    B200SHA3_CASE(4) B200SHA3_CASE(5) B200SHA3_CASE(6) B200SHA3_CASE(7)
    B200SHA3_CASE(8)
#undef B200SHA3_CASE
    default: return cudaErrorNotSupported;
  }
}

}  // namespace

bool oneblock_supported(int rate_lanes, uint64_t msg_len, uint64_t digest_bytes) {
  if (msg_len == 0 || msg_len % 8 != 0 || digest_bytes == 0 || digest_bytes % 4 != 0) return false;
  if (msg_len >= 8u * static_cast<uint64_t>(rate_lanes) || digest_bytes > 8u * rate_lanes) return false;
  return oneblock_shape_exists(rate_lanes, static_cast<int>(msg_len / 8),
                               static_cast<int>(digest_bytes / 4));
}

cudaError_t launch_hash_oneblock(const HashArgs& args, const LaunchPlan& plan,
                                 cudaStream_t stream) {
  if (!oneblock_supported(plan.rate_lanes, args.fixed_len, args.digest_bytes) ||
      args.offsets || args.lengths || args.order || !args.aligned8 || args.last_mask != 0xffu) {
    return cudaErrorNotSupported;
  }
  const int ml = static_cast<int>(args.fixed_len / 8), ow = static_cast<int>(args.digest_bytes / 4);
  if (!(plan.rate_lanes == 17 && ml == 8 && ow == 8)) {
    // every other shape exists only as UNROLL 23 / ALU-only
    return launch_oneblock_shape(plan.rate_lanes, ml, ow, args, plan, stream);
  }
  switch (plan.unroll) {
    case 2: return launch_sha3_256_64<2>(args, plan, stream);
    case 4: return launch_sha3_256_64<4>(args, plan, stream);
    case 11: return launch_sha3_256_64<11>(args, plan, stream);
    case 20: return launch_sha3_256_64<20>(args, plan, stream);
    case 21: return launch_sha3_256_64<21>(args, plan, stream);
    case 23: return launch_sha3_256_64<23>(args, plan, stream);
    case 22: return launch_sha3_256_64<22>(args, plan, stream);
    case 24: return launch_sha3_256_64<24>(args, plan, stream);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace b200sha3
