// oneblock.cuh -- the single-block kernel template (see kernel_oneblock.cu).
#pragma once
#include "kernels.cuh"
#include "sponge.cuh"

namespace b200sha3 {

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
cudaError_t launch_oneblock_instance(const HashArgs& args, const LaunchPlan& plan,
                                     cudaStream_t stream) {
  const int threads = plan.block_threads > 0 ? plan.block_threads : 128;
  const uint64_t blocks = (args.count + threads - 1) / threads;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  hash_oneblock_kernel<RL, ML, OW, UNROLL, kFmaPreset[PRESET]>
      <<<static_cast<unsigned>(blocks), threads, 0, stream>>>(args.data, args.digests,
                                                              args.count, args.head);
  return cudaGetLastError();
}

// Shapes other than the tuning-matrix one (kernel_oneblock_shapes.cu): UNROLL 23 (peeled
// 1 + 7x3 + 2, the measured best), ALU only.  Returns cudaErrorNotSupported when (rl, ml, ow) is not instantiated.
cudaError_t launch_oneblock_shape(int rl, int ml, int ow, const HashArgs& args,
                                  const LaunchPlan& plan, cudaStream_t stream);
bool oneblock_shape_exists(int rl, int ml, int ow);

}  // namespace b200sha3
