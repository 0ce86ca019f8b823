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
#include "kernels.cuh"
#include "sponge.cuh"

namespace b200sha3 {

namespace {

template <int RL, int ML, int OW, int UNROLL, uint32_t FMA_MASK>
__global__ void __launch_bounds__(256)
hash_oneblock_kernel(const uint8_t* __restrict__ data, uint8_t* __restrict__ digests,
                     uint64_t count, uint32_t head) {
  static_assert(ML < RL, "message must leave room for the pad byte");
  static_assert(OW <= 2 * RL, "digest must fit one block");
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= count) return;
  State a;
  state_zero(a);
  const uint8_t* p = data + tid * (8u * ML);
  if constexpr (ML % 2 == 0) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
    for (int i = 0; i < ML / 2; ++i) {
      const uint4 v = __ldg(q + i);
      a.lo[2 * i] = v.x;
      a.hi[2 * i] = v.y;
      a.lo[2 * i + 1] = v.z;
      a.hi[2 * i + 1] = v.w;
    }
  } else {
    const uint2* q = reinterpret_cast<const uint2*>(p);
#pragma unroll
    for (int i = 0; i < ML; ++i) {
      const uint2 v = __ldg(q + i);
      a.lo[i] = v.x;
      a.hi[i] = v.y;
    }
  }
  a.lo[ML] ^= head;                // sponge.cpp:122-123
  a.hi[RL - 1] ^= 0x80000000u;     // sponge.cpp:124-125
  keccak_f1600<UNROLL, FMA_MASK>(a);
  uint8_t* o = digests + tid * (4u * OW);
  if constexpr (OW % 4 == 0) {
#pragma unroll
    for (int k = 0; k < OW / 4; ++k) {
      *reinterpret_cast<uint4*>(o + 16 * k) =
          make_uint4(state_word(a, 4 * k), state_word(a, 4 * k + 1), state_word(a, 4 * k + 2),
                     state_word(a, 4 * k + 3));
    }
  } else {
#pragma unroll
    for (int j = 0; j < OW; ++j) {
      *reinterpret_cast<uint32_t*>(o + 4 * j) = state_word(a, j);
    }
  }
}

template <int RL, int ML, int OW, int UNROLL, int PRESET>
cudaError_t launch_one(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  const int threads = plan.block_threads > 0 ? plan.block_threads : 128;
  const uint64_t blocks = (args.count + threads - 1) / threads;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  hash_oneblock_kernel<RL, ML, OW, UNROLL, kFmaPreset[PRESET]>
      <<<static_cast<unsigned>(blocks), threads, 0, stream>>>(args.data, args.digests,
                                                              args.count, args.head);
  return cudaGetLastError();
}

// SHA3-256 / SHAKE256, 64-byte messages, 32-byte digests: the tuning matrix.
template <int UNROLL>
cudaError_t launch_sha3_256_64(const HashArgs& args, const LaunchPlan& plan,
                               cudaStream_t stream) {
  switch (plan.fma_preset) {
#define B200SHA3_CASE(P) \
  case P: return launch_one<17, 8, 8, UNROLL, P>(args, plan, stream);
    B200SHA3_CASE(0) B200SHA3_CASE(1) B200SHA3_CASE(2) B200SHA3_CASE(3)
    B200SHA3_CASE(4) B200SHA3_CASE(5) B200SHA3_CASE(6) B200SHA3_CASE(7)
    B200SHA3_CASE(8)
#undef B200SHA3_CASE
    default: return cudaErrorNotSupported;
  }
}

}  // namespace

bool oneblock_supported(int rate_lanes, uint64_t msg_len, uint64_t digest_bytes) {
  return rate_lanes == 17 && msg_len == 64 && digest_bytes == 32;
}

cudaError_t launch_hash_oneblock(const HashArgs& args, const LaunchPlan& plan,
                                 cudaStream_t stream) {
  if (!oneblock_supported(plan.rate_lanes, args.fixed_len, args.digest_bytes) ||
      args.offsets || args.lengths || args.order || !args.aligned8) {
    return cudaErrorNotSupported;
  }
  switch (plan.unroll) {
    case 2: return launch_sha3_256_64<2>(args, plan, stream);
    case 4: return launch_sha3_256_64<4>(args, plan, stream);
    case 24: return launch_sha3_256_64<24>(args, plan, stream);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace b200sha3
