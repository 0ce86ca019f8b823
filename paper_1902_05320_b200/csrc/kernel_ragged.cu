// kernel_ragged.cu -- ONE launch for a variable-length batch whose shape is known on the device
// only: the body of hash_short_kernel (kernel_short.cu) when the classification pass found
// nothing but single-block messages, the body of hash_generic_kernel (kernel_generic.cu)
// otherwise -- a kernel-uniform branch on the "long" flag word.  In a mixed batch the warps that hold
// nothing but single-block messages (the tail of the bucketing order) take the short body as well.
//
// Before, both kernels were launched and one of them returned at once; the one that returned
// still had its whole grid dispatched (131 072 empty blocks for 2^24 messages: 70 us, 1.7 % of
// the call), side by side or not.  The price of merging is the register budget: the kernel is
// compiled for the generic body's 128 registers, so the short body runs at 16 warps per SM
// instead of 24 -- measured harmless, it is ALU bound with instruction-level parallelism to
// spare (tools/short_ragged.py).
#include "kernels.cuh"
#include "sponge.cuh"

namespace b200sha3 {

namespace {

constexpr int kRaggedUnroll = 3;  // rounds per loop body of the generic path (kernel_generic.cu)

template <int RL, int OW>
__global__ void __launch_bounds__(256, 2)
hash_ragged_kernel(const HashArgs args) {
  static_assert(OW <= 2 * RL, "digest must fit one block");
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= args.count) return;
  const bool aligned8 = *args.unaligned_flag == 0u;
  const bool all_short = *args.long_flag == 0u;
  // An all-short batch with 8-byte aligned starts is taken in input order (the scatter pass
  // returned at once and left no order); everything else walks the bucketing order.
  const bool ordered = args.order != nullptr && !(all_short && aligned8);
  const uint64_t m = ordered ? static_cast<uint64_t>(args.order[tid]) : tid;
  const uint64_t length = args.lengths[m];
  // The short body (kernel_short.cu) for a batch of single-block messages -- and, in a MIXED batch
  // (keys and records: some messages below the rate, some above), for every warp that holds
  // nothing else: the bucketing order puts the single-block messages last, sorted by word count,
  // so whole warps of them exist (4440 instead of 4755 instructions per message).  Predicated
  // absorb on 8-byte aligned starts, word-count order and the jump-table absorb otherwise.
  if (all_short || __all_sync(__activemask(), length < 8u * RL)) {
    const uint8_t* p = args.data + args.offsets[m];
    State a;
    state_zero(a);
    if (ordered && !aligned8) {
      absorb_tail_uniform_unaligned<RL>(a, p, static_cast<uint32_t>(length), args.head);
    } else {
      absorb_tail<RL>(a, p, static_cast<uint32_t>(length), args.head, aligned8, /*ragged=*/true);
    }
    keccak_f1600<23, 0u>(a);  // peeled 1 + 7x3 + 2
    emit_block<RL>(a, args.digests + m * (4u * OW), 4u * OW);
    return;
  }
  const bool ragged = *args.ragged_flag != 0u;
  // digest = 4 OW bytes, whole bytes (launch_hash_ragged checks): the static-output form
  hash_message_static_out<RL, OW, kRaggedUnroll, 0u>(args.data + args.offsets[m], length,
                                                     args.digests + m * (4u * OW), args.head, aligned8, ragged);
}

template <int RL, int OW>
cudaError_t launch_instance(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  const int threads = plan.block_threads > 0 ? plan.block_threads : 128;
  const uint64_t blocks = (args.count + threads - 1) / threads;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  hash_ragged_kernel<RL, OW><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace

// Same shapes as the short kernel (short_supported); needs offsets, lengths and the three flag
// words; args.order may be nullptr (no bucketing).
cudaError_t launch_hash_ragged(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  if (!short_supported(plan.rate_lanes, args.digest_bytes) || !args.offsets || !args.lengths ||
      !args.unaligned_flag || !args.ragged_flag || !args.long_flag || args.last_mask != 0xffu) {
    return cudaErrorNotSupported;
  }
  const int ow = static_cast<int>(args.digest_bytes / 4);
#define B200SHA3_RAGGED(RL, OW) \
  if (plan.rate_lanes == RL && ow == OW) return launch_instance<RL, OW>(args, plan, stream);
  B200SHA3_RAGGED(18, 7) B200SHA3_RAGGED(17, 8) B200SHA3_RAGGED(13, 12) B200SHA3_RAGGED(9, 16)
  B200SHA3_RAGGED(17, 4) B200SHA3_RAGGED(17, 16) B200SHA3_RAGGED(21, 4) B200SHA3_RAGGED(21, 8)
  B200SHA3_RAGGED(21, 16)
#undef B200SHA3_RAGGED
  return cudaErrorNotSupported;
}

}  // namespace b200sha3
