// kernel_staged.cu -- the TMA-staged variant of the general kernel (north_star "input
// staging"), kept for the measured comparison of DESIGN.md section 4.
// B200SHA3_KERNEL_STAGED selects it; AUTO never does.
//
// Same work split as hash_generic_kernel (one message per thread, bucketed order), but
// whole rate blocks reach the thread through shared memory instead of per-thread global
// loads: each thread issues ONE bulk async copy (cp.async.bulk global -> shared,
// SASS UBLKCP) per block into its private slot, double buffered, completion tracked by a
// per-warp mbarrier (32 arrivals + the copied bytes).  While block k is permuted, block
// k+1 is already in flight.  Bulk copies need 16-byte aligned sources and sizes, message
// blocks are only 8-byte aligned, so a copy starts at the block address rounded down to
// 16 and covers (p & 15) + R bytes rounded up to 16; a block is staged only when at least
// 16 more message bytes follow it (the over-read then stays inside the message).  The last
// full block, the partial block, padding and squeezing use the direct path of sponge.cuh.
//
// Staging applies when the data base is 16-byte aligned and every message start 8-byte
// aligned; otherwise all blocks take the direct path (still correct, nothing staged).
#include "kernels.cuh"
#include "sponge.cuh"

namespace b200sha3 {

namespace {

constexpr int kStagedThreads = 128;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
               ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}"
      ::"r"(bar), "r"(parity) : "memory");
}

__device__ __forceinline__ void bulk_copy_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// Orders this thread's earlier generic-proxy shared reads before later async-proxy writes.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int RL>
struct StagedLayout {
  static constexpr uint32_t R = 8u * RL;
  // slot: the block plus up to 8 leading and 8 trailing bytes, multiple of 16
  static constexpr uint32_t kSlot = (R + 16u + 15u) & ~15u;
  static constexpr uint32_t kBytes = 2u * kStagedThreads * kSlot + 2u * (kStagedThreads / 32) * 8u;
};

template <int RL>
__global__ void __launch_bounds__(kStagedThreads)
hash_staged_kernel(const HashArgs args) {
  using L = StagedLayout<RL>;
  constexpr uint32_t R = L::R;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2u * kStagedThreads * L::kSlot);
  const uint32_t bar0 = smem_addr(bars + 2 * warp), bar1 = bar0 + 8u;
  uint8_t* slot[2] = {smem + (0u * kStagedThreads + threadIdx.x) * L::kSlot,
                      smem + (1u * kStagedThreads + threadIdx.x) * L::kSlot};
  if (lane == 0) {
    mbar_init(bar0, 32u);
    mbar_init(bar1, 32u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool live = tid < args.count;
  uint64_t m = 0, len = 0;
  const uint8_t* p = args.data;
  if (live) {
    m = args.order ? static_cast<uint64_t>(args.order[tid]) : tid;
    p = args.data + (args.offsets ? args.offsets[m] : m * args.fixed_len);
    len = args.lengths ? args.lengths[m] : args.fixed_len;
  }
  // Staging needs 8-byte aligned message starts on a 16-byte aligned base; otherwise every
  // block takes the direct (generic) path below and the kernel is still correct.
  const bool aligned8 = (args.unaligned_flag ? (*args.unaligned_flag == 0u) : (args.aligned8 != 0u)) &&
                        (reinterpret_cast<uintptr_t>(args.data) & 15u) == 0u;
  // blocks this thread stages: full blocks followed by at least 16 more message bytes
  const uint64_t staged = (aligned8 && len >= R + 16u) ? (len - 16u) / R : 0u;
  uint64_t max_staged = staged;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const uint64_t other = __shfl_xor_sync(0xffffffffu, max_staged, d);
    max_staged = other > max_staged ? other : max_staged;
  }

  State a;
  state_zero(a);
  auto issue = [&](uint64_t k) {  // stage block k (or just arrive) on buffer k & 1
    const uint32_t bar = (k & 1u) ? bar1 : bar0;
    if (k < staged) {
      const uint8_t* src = p + k * R;
      const uint32_t lead = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(src)) & 15u;
      const uint32_t bytes = (lead + R + 15u) & ~15u;
      fence_proxy_async();
      mbar_arrive_expect_tx(bar, bytes);
      bulk_copy_g2s(smem_addr(slot[k & 1u]), src - lead, bytes, bar);
    } else {
      mbar_arrive(bar);
    }
  };
  if (max_staged > 0) issue(0);
  for (uint64_t k = 0; k < max_staged; ++k) {
    if (k + 1 < max_staged) issue(k + 1);
    mbar_wait((k & 1u) ? bar1 : bar0, static_cast<uint32_t>(k >> 1) & 1u);
    if (k < staged) {
      const uint32_t lead = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p + k * R)) & 15u;
      const uint2* q = reinterpret_cast<const uint2*>(slot[k & 1u] + lead);
#pragma unroll
      for (int i = 0; i < RL; ++i) {
        const uint2 v = q[i];
        a.lo[i] ^= v.x;
        a.hi[i] ^= v.y;
      }
      keccak_f1600<2, 0u>(a);
    }
  }
  if (!live) return;

  // the rest exactly like hash_message: remaining full block(s), tail + pad, squeeze
  const uint64_t nfull = len / R;
  const uint32_t rem = static_cast<uint32_t>(len - nfull * R);
  const uint8_t* q = p + staged * R;
  for (uint64_t k = staged; k < nfull; ++k) {
    if (aligned8) {
      absorb_lanes_aligned<RL>(a, q, RL);
    } else {
      absorb_words_unaligned<RL>(a, q, 2 * RL);
    }
    keccak_f1600<2, 0u>(a);
    q += R;
  }
  absorb_tail<RL>(a, q, rem, args.head, aligned8);
  uint8_t* o = args.digests + m * args.digest_bytes;
  uint64_t left = args.digest_bytes;
  for (;;) {
    keccak_f1600<2, 0u>(a);
    const uint32_t n = left < R ? static_cast<uint32_t>(left) : R;
    emit_block<RL>(a, o, n);
    o += n;
    left -= n;
    if (left == 0) break;
  }
  if (args.last_mask != 0xffu) {
    args.digests[m * args.digest_bytes + args.digest_bytes - 1u] &= static_cast<uint8_t>(args.last_mask);
  }
}

template <int RL>
cudaError_t launch_rl(const HashArgs& args, cudaStream_t stream) {
  using L = StagedLayout<RL>;
  // per device and idempotent, so simply repeated on every launch (about a microsecond)
  cudaError_t e = cudaFuncSetAttribute(hash_staged_kernel<RL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(L::kBytes));
  if (e != cudaSuccess) return e;
  const uint64_t blocks = (args.count + kStagedThreads - 1) / kStagedThreads;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  hash_staged_kernel<RL><<<static_cast<unsigned>(blocks), kStagedThreads, L::kBytes, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_hash_staged(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  switch (plan.rate_lanes) {
    case 9: return launch_rl<9>(args, stream);
    case 13: return launch_rl<13>(args, stream);
    case 17: return launch_rl<17>(args, stream);
    case 18: return launch_rl<18>(args, stream);
    case 21: return launch_rl<21>(args, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace b200sha3
