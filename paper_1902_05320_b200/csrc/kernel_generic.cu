// kernel_generic.cu -- the general batch kernel: one message per thread, any
// length and alignment, multi-block absorb, multi-block (XOF) squeeze.
//
// Replaces the per-message body of hash_batch's fan-out
// (proj/core/src/batch.cpp:86-109 -> hash_into :15-25) for arbitrary batches.
// Threads of a warp run the same instruction stream; they diverge only in the
// number of blocks, which the bucketing pass (kernel_aux.cu) bounds.
#include "kernels.cuh"
#include "sponge.cuh"

namespace b200sha3 {

namespace {

constexpr int kGenericUnroll = 3;  // rounds per loop body (8 iterations)

template <int RL, int UNROLL, uint32_t FMA_MASK>
__global__ void __launch_bounds__(256, 2)
hash_generic_kernel(const HashArgs args) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= args.count) return;
  if (args.skip_if_short != 0u && *args.long_flag == 0u) {
    return;  // hash_short_kernel has this batch
  }
  const uint64_t m = args.order ? static_cast<uint64_t>(args.order[tid]) : tid;
  const uint64_t off = args.offsets ? args.offsets[m] : m * args.fixed_len;
  const uint64_t len = args.lengths ? args.lengths[m] : args.fixed_len;
  const bool aligned8 =
      args.unaligned_flag ? (*args.unaligned_flag == 0u) : (args.aligned8 != 0u);
  const bool ragged = args.ragged_flag != nullptr && *args.ragged_flag != 0u;
  hash_message<RL, UNROLL, FMA_MASK>(args.data + off, len,
                                     args.digests + m * args.digest_bytes,
                                     args.digest_bytes, args.head, args.last_mask, aligned8, ragged);
}

template <int RL, int UNROLL, int PRESET>
cudaError_t launch_one(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  const int threads = plan.block_threads > 0 ? plan.block_threads : 128;
  const uint64_t blocks = (args.count + threads - 1) / threads;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  hash_generic_kernel<RL, UNROLL, kFmaPreset[PRESET]>
      <<<static_cast<unsigned>(blocks), threads, 0, stream>>>(args);
  return cudaGetLastError();
}

template <int RL>
cudaError_t launch_rl(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  // Generic kernel instantiations: plain loop, kGenericUnroll rounds per body; ALU only (the
  // default) or FMA preset 5 (every rho rotation on the FMA pipe), kept for the measured
  // comparison of DESIGN.md section 4.  SHA3-256's rate also carries the loop-shape sweep.
  if constexpr (RL == 17) {
    switch (plan.unroll) {
      case 2: return launch_one<RL, 2, 0>(args, plan, stream);
      case 4: return launch_one<RL, 4, 0>(args, plan, stream);
      case 6: return launch_one<RL, 6, 0>(args, plan, stream);
      default: break;
    }
  }
  switch (plan.fma_preset) {
    case 0: return launch_one<RL, kGenericUnroll, 0>(args, plan, stream);
    default: return launch_one<RL, kGenericUnroll, 5>(args, plan, stream);
  }
}

}  // namespace

cudaError_t launch_hash_generic(const HashArgs& args, const LaunchPlan& plan,
                                cudaStream_t stream) {
  switch (plan.rate_lanes) {
    case 9: return launch_rl<9>(args, plan, stream);
    case 13: return launch_rl<13>(args, plan, stream);
    case 17: return launch_rl<17>(args, plan, stream);
    case 18: return launch_rl<18>(args, plan, stream);
    case 21: return launch_rl<21>(args, plan, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace b200sha3
