// kernel_short.cu -- variable-length batches of SINGLE-BLOCK messages: every message shorter
// than the rate (hashing keys, identifiers, short records of uneven length).
//
// The generic kernel serves such a batch at ~0.93 of the ALU roofline and ncu shows why: no
// stalls, just instructions -- a rolled permutation that cannot drop the work on the capacity
// lanes (zero before the first permutation) or on the lanes nobody reads after the last one,
// the block-count loop, the processing order.  For batches without a message of a whole block
// the kernels here do the work instead (8-byte aligned starts: 8-byte loads; any other layout:
// aligned 4-byte loads + PRMT): lane loads straight into a zero state, the peeled permutation
// of the one-block kernel (1 + 7x3 + 2 rounds), OW digest words out.
#include "kernels.cuh"
#include "sponge.cuh"

namespace b200sha3 {

namespace {

// Input order, predicated "ragged" absorb (~6 ALU instructions per lane on 8-byte aligned
// starts, ~10 per lane on 4-byte loads + PRMT otherwise).  Launched by the host entries, which
// know from the lengths they read that the batch is all-short (BatchHints) and run no
// classification or ordering pass; the device entries use hash_ragged_kernel (kernel_ragged.cu),
// which carries this body -- plus the word-count-ordered jump-table form for batches at odd
// addresses -- next to the generic one.
template <int RL, int OW>
__global__ void __launch_bounds__(256)
hash_short_kernel(const HashArgs args) {
  static_assert(OW <= 2 * RL, "digest must fit one block");
  if (*args.long_flag != 0u) return;  // not an all-short batch: nothing to do here
  const bool aligned8 = *args.unaligned_flag == 0u;  // else: 4-byte loads re-assembled with PRMT
  // (A persistent grid-stride form of this kernel was measured 4 % slower on its own batches:
  // 0.921 vs 0.957 of the roofline on 2^24 x 0..135 B.  So was a tile form -- a block
  // counting-sorts 2048 consecutive messages by word count in shared memory and walks the sorted
  // tile, no ordering pass, no far gathers: 0.921 aligned / 0.891 unaligned on the same batch.)
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= args.count) return;
  const uint8_t* p = args.data + args.offsets[tid];
  const uint32_t len = static_cast<uint32_t>(args.lengths[tid]);  // < 8 * RL
  State a;
  state_zero(a);
  absorb_tail<RL>(a, p, len, args.head, aligned8, /*ragged=*/true);
  keccak_f1600<23, 0u>(a);  // peeled 1 + 7x3 + 2
  emit_block<RL>(a, args.digests + tid * (4u * OW), 4u * OW);
}

// The same for EQUAL-LENGTH batches of any length below the rate -- what the one-block kernel
// (whole lanes of 32 / 64 / 128 bytes, 16-byte aligned) does not take: the paper's own 10-byte
// messages, 20- or 100-byte records.  The length is uniform, so both tail forms
// are jump tables without divergence: whole-lane loads when every start is 8-byte aligned,
// aligned 4-byte loads + PRMT otherwise.
template <int RL, int OW>
__global__ void __launch_bounds__(256)
hash_short_fixed_kernel(const uint8_t* __restrict__ data, uint8_t* __restrict__ digests, uint64_t count,
                        uint32_t len, uint32_t head, uint32_t aligned8) {
  static_assert(OW <= 2 * RL, "digest must fit one block");
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= count) return;
  const uint8_t* p = data + tid * len;
  State a;
  state_zero(a);
  if (aligned8 != 0u) {
    absorb_tail<RL>(a, p, len, head, /*aligned8=*/true, /*ragged=*/false);
  } else {
    absorb_tail_uniform_unaligned<RL>(a, p, len, head);
  }
  keccak_f1600<23, 0u>(a);  // peeled 1 + 7x3 + 2
  emit_block<RL>(a, digests + tid * (4u * OW), 4u * OW);
}

template <int RL, int OW>
cudaError_t launch_fixed_instance(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  const int threads = plan.block_threads > 0 ? plan.block_threads : 128;
  const uint64_t blocks = (args.count + threads - 1) / threads;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  hash_short_fixed_kernel<RL, OW><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
      args.data, args.digests, args.count, static_cast<uint32_t>(args.fixed_len), args.head, args.aligned8);
  return cudaGetLastError();
}

template <int RL, int OW>
cudaError_t launch_instance(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  const int threads = plan.block_threads > 0 ? plan.block_threads : 128;
  const uint64_t blocks = (args.count + threads - 1) / threads;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  hash_short_kernel<RL, OW><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace

// The four hashes at their digest size; the two SHAKEs at 128-, 256- and 512-bit outputs.
bool short_supported(int rate_lanes, uint64_t digest_bytes) {
  switch (rate_lanes) {
    case 18: return digest_bytes == 28;
    case 17: return digest_bytes == 32 || digest_bytes == 16 || digest_bytes == 64;
    case 13: return digest_bytes == 48;
    case 9: return digest_bytes == 64;
    case 21: return digest_bytes == 16 || digest_bytes == 32 || digest_bytes == 64;
    default: return false;
  }
}

cudaError_t launch_hash_short_fixed(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  if (!short_supported(plan.rate_lanes, args.digest_bytes) || args.offsets || args.lengths || args.order ||
      args.fixed_len >= 8u * static_cast<uint64_t>(plan.rate_lanes) || args.last_mask != 0xffu) {
    return cudaErrorNotSupported;
  }
  const int ow = static_cast<int>(args.digest_bytes / 4);
#define B200SHA3_SHORT(RL, OW) \
  if (plan.rate_lanes == RL && ow == OW) return launch_fixed_instance<RL, OW>(args, plan, stream);
  B200SHA3_SHORT(18, 7) B200SHA3_SHORT(17, 8) B200SHA3_SHORT(13, 12) B200SHA3_SHORT(9, 16)
  B200SHA3_SHORT(17, 4) B200SHA3_SHORT(17, 16) B200SHA3_SHORT(21, 4) B200SHA3_SHORT(21, 8)
  B200SHA3_SHORT(21, 16)
#undef B200SHA3_SHORT
  return cudaErrorNotSupported;
}

cudaError_t launch_hash_short(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  if (!short_supported(plan.rate_lanes, args.digest_bytes) || !args.offsets || !args.lengths ||
      !args.unaligned_flag || !args.long_flag || args.order || args.last_mask != 0xffu) {
    return cudaErrorNotSupported;
  }
  const int ow = static_cast<int>(args.digest_bytes / 4);
#define B200SHA3_SHORT(RL, OW) \
  if (plan.rate_lanes == RL && ow == OW) return launch_instance<RL, OW>(args, plan, stream);
  B200SHA3_SHORT(18, 7) B200SHA3_SHORT(17, 8) B200SHA3_SHORT(13, 12) B200SHA3_SHORT(9, 16)
  B200SHA3_SHORT(17, 4) B200SHA3_SHORT(17, 16) B200SHA3_SHORT(21, 4) B200SHA3_SHORT(21, 8)
  B200SHA3_SHORT(21, 16)
#undef B200SHA3_SHORT
  return cudaErrorNotSupported;
}

}  // namespace b200sha3
