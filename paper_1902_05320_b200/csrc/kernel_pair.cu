// kernel_pair.cu -- one message per PAIR of threads: a measured experiment, selectable with
// B200SHA3_KERNEL_PAIR, never picked by KERNEL_AUTO (round 2).
//
// The question: between ~2800 messages (where the warp-per-state kernel saturates the shuffle
// unit) and ~19 000 (one warp per SMSP with one message per thread) a multi-block batch costs
// one thread's permutation latency per block, ~11 000 cycles, however idle the machine is.
// Can a layout with the SAME ALU work per message halve that latency?
//
//   thread 2k holds the LOW 32-bit halves of the 25 lanes of message k, thread 2k + 1 the HIGH
//   halves (25 registers each instead of 50).  theta's XORs, chi and iota never mix bit
//   positions, so each thread does its half of them on its own: 61 LOP3 per round instead of
//   122.  A 64-bit rotation by r needs the other half of the same lane -- one SHFL (xor 1) -- and
//   then ONE funnel shift per thread, the same instruction in both threads:
//       r < 32:  mine' = funnel_l(other, mine, r)        r > 32:  mine' = funnel_l(mine, other, r - 32)
//   so rho + the rotl-1 of theta cost 29 SHF + 29 SHFL per thread-round instead of 58 SHF:
//   2 x 90 = 180 ALU instructions per message-round, as before, plus 58 shuffles.
//
// The answer (tools/long_message_latency.py, profiles/r2_long_message_latency_pair.json): no.
// A permutation takes 9800-10 000 cycles in a pair against 10 100-10 300 in one thread, and at
// saturation the kernel is 23 % SLOWER (2^18 x 8 KiB: 154 800 vs 125 700 cycles per block step).
// A SHFL occupies the warp's issue port for ~4-5 cycles (tools/microbench/shfl_probe.cu: eight
// independent shuffles take 46 cycles from one warp), so the 29 shuffles of a thread-round cost
// the 145 cycles that the halved ALU work (90 x 2) saved, and with several warps per SMSP they
// still compete with the ALU instructions for dispatch.  Bit-exact (tests/test_gpu_warp_kernel.py).
//
// Same arithmetic as permute_1600 (proj/core/src/keccak.cpp:245-277) and the sponge of
// proj/core/src/sponge.cpp:81-143 as driven by hash_into (batch.cpp:15-25); any length,
// alignment, digest size and XOF bit count; processing order from the bucketing pass.
#include "kernels.cuh"
#include "sponge.cuh"

namespace b200sha3 {

namespace {

// This thread's 32-bit half of every lane, index x + 5y.
struct HalfState {
  uint32_t w[25];
};

// The other half of the same lane, from the partner thread.  `pair` names the two threads only:
// pairs of one warp leave the block loop at different times.
__device__ __forceinline__ uint32_t partner(uint32_t pair, uint32_t v) { return __shfl_xor_sync(pair, v, 1); }

// This thread's half of rotl64(lane, R), R a compile-time rho offset (keccak.cpp:26-32).
template <int R>
__device__ __forceinline__ uint32_t rotl_half(uint32_t pair, uint32_t mine) {
  static_assert(R >= 0 && R < 64 && R != 32, "no rho offset is 32");
  if constexpr (R == 0) {
    return mine;
  } else {
    const uint32_t other = partner(pair, mine);
    if constexpr (R < 32) {
      return __funnelshift_l(other, mine, R);
    } else {
      return __funnelshift_l(mine, other, R - 32);
    }
  }
}

#define B200SHA3_PAIR_RHOPI(SRC, ROT, DST) b[DST] = rotl_half<ROT>(pair, a.w[SRC])

// One round on this thread's halves; rc = this thread's half of the round constant.
__device__ __forceinline__ void pair_round(HalfState& a, uint32_t pair, uint32_t rc) {
  uint32_t c[5];
#pragma unroll
  for (int x = 0; x < 5; ++x) c[x] = xor3(xor3(a.w[x], a.w[x + 5], a.w[x + 10]), a.w[x + 15], a.w[x + 20]);
  uint32_t r[5];
#pragma unroll
  for (int x = 0; x < 5; ++x) r[x] = rotl_half<1>(pair, c[x]);
#pragma unroll
  for (int x = 0; x < 5; ++x) {
    const uint32_t left = c[(x + 4) % 5], right = r[(x + 1) % 5];
#pragma unroll
    for (int y = 0; y < 25; y += 5) a.w[x + y] = xor3(a.w[x + y], left, right);
  }
  uint32_t b[25];  // b[x+5y] = rotl(a[src], rho[src]), src = (x+3y)%5 + 5x   (keccak.cpp:261-267)
  B200SHA3_PAIR_RHOPI(0, 0, 0);
  B200SHA3_PAIR_RHOPI(6, 44, 1);
  B200SHA3_PAIR_RHOPI(12, 43, 2);
  B200SHA3_PAIR_RHOPI(18, 21, 3);
  B200SHA3_PAIR_RHOPI(24, 14, 4);
  B200SHA3_PAIR_RHOPI(3, 28, 5);
  B200SHA3_PAIR_RHOPI(9, 20, 6);
  B200SHA3_PAIR_RHOPI(10, 3, 7);
  B200SHA3_PAIR_RHOPI(16, 45, 8);
  B200SHA3_PAIR_RHOPI(22, 61, 9);
  B200SHA3_PAIR_RHOPI(1, 1, 10);
  B200SHA3_PAIR_RHOPI(7, 6, 11);
  B200SHA3_PAIR_RHOPI(13, 25, 12);
  B200SHA3_PAIR_RHOPI(19, 8, 13);
  B200SHA3_PAIR_RHOPI(20, 18, 14);
  B200SHA3_PAIR_RHOPI(4, 27, 15);
  B200SHA3_PAIR_RHOPI(5, 36, 16);
  B200SHA3_PAIR_RHOPI(11, 10, 17);
  B200SHA3_PAIR_RHOPI(17, 15, 18);
  B200SHA3_PAIR_RHOPI(23, 56, 19);
  B200SHA3_PAIR_RHOPI(2, 62, 20);
  B200SHA3_PAIR_RHOPI(8, 55, 21);
  B200SHA3_PAIR_RHOPI(14, 39, 22);
  B200SHA3_PAIR_RHOPI(15, 41, 23);
  B200SHA3_PAIR_RHOPI(21, 2, 24);
#pragma unroll
  for (int y = 0; y < 25; y += 5) {
#pragma unroll
    for (int x = 0; x < 5; ++x) a.w[x + y] = chi3(b[x + y], b[(x + 1) % 5 + y], b[(x + 2) % 5 + y]);
  }
  a.w[0] ^= rc;
}

#undef B200SHA3_PAIR_RHOPI

constexpr int kPairUnroll = 2;  // rounds per loop body

// 24 rounds; `half` = 0 (low halves) or 1 (high halves) picks this thread's constants.
__device__ __forceinline__ void pair_permute(HalfState& a, uint32_t pair, uint32_t half) {
#pragma unroll 1
  for (int round = 0; round < 24; round += kPairUnroll) {
#pragma unroll
    for (int u = 0; u < kPairUnroll; ++u) pair_round(a, pair, kRoundConst32[2 * (round + u) + half]);
  }
}

// Word j (32 bits) of the rate block is this thread's iff j is odd for the high-half thread:
// lane i = words 2i (low) and 2i + 1 (high).

// XORs this thread's words of one whole rate block at p into the state.
template <int RL>
__device__ __forceinline__ void absorb_block(HalfState& a, const uint8_t* p, uint32_t half) {
  const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p)) & 3u;
  if (sh == 0u) {  // 4-byte aligned starts need nothing else in this layout
    const uint32_t* q = reinterpret_cast<const uint32_t*>(p) + half;
#pragma unroll
    for (int i = 0; i < RL; ++i) a.w[i] ^= ld_u32(q + 2 * i);
  } else {  // aligned words re-assembled with PRMT; every word read holds message bytes
    const uint32_t* q = reinterpret_cast<const uint32_t*>(p - sh) + half;
    const uint32_t sel = 0x3210u + 0x1111u * sh;
#pragma unroll
    for (int i = 0; i < RL; ++i) a.w[i] ^= __byte_perm(ld_u32(q + 2 * i), ld_u32(q + 2 * i + 1), sel);
  }
}

// Final (partial) block: rem < 8 * RL message bytes at p, then the pad (sponge.cpp:113-129).
template <int RL>
__device__ __forceinline__ void absorb_final(HalfState& a, const uint8_t* p, uint32_t rem, uint32_t head,
                                             uint32_t half) {
#pragma unroll
  for (int i = 0; i < RL; ++i) {
    const uint32_t first = 8u * i + 4u * half;  // block byte of this thread's word of lane i
    uint32_t word = 0u;
    if (first + 4u <= rem && (reinterpret_cast<uintptr_t>(p + first) & 3u) == 0u) {
      word = ld_u32(reinterpret_cast<const uint32_t*>(p + first));
    } else if (first < rem) {
      const uint32_t n = rem - first < 4u ? rem - first : 4u;
      for (uint32_t k = 0; k < n; ++k) word |= ld_u8(p + first + k) << (8u * k);
    }
    if (rem >= first && rem < first + 4u) word ^= head << (8u * (rem - first));  // sponge.cpp:122-123
    a.w[i] ^= word;
  }
  if (half != 0u) a.w[RL - 1] ^= 0x80000000u;  // sponge.cpp:124-125
}

// Writes this thread's words of the first n (<= 8 * RL) bytes of the rate part to o.
template <int RL>
__device__ __forceinline__ void emit_half(const HalfState& a, uint8_t* o, uint32_t n, uint32_t half) {
#pragma unroll
  for (int i = 0; i < RL; ++i) {
    const uint32_t first = 8u * i + 4u * half;
    if (first >= n) continue;
    uint8_t* dst = o + first;
    if (first + 4u <= n && (reinterpret_cast<uintptr_t>(dst) & 3u) == 0u) {
      *reinterpret_cast<uint32_t*>(dst) = a.w[i];
    } else {
      const uint32_t k_end = n - first < 4u ? n - first : 4u;
      for (uint32_t k = 0; k < k_end; ++k) dst[k] = static_cast<uint8_t>(a.w[i] >> (8u * k));
    }
  }
}

template <int RL>
__global__ void __launch_bounds__(128, 6)
hash_pair_kernel(const HashArgs args) {
  constexpr uint32_t R = 8u * RL;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t slot = tid >> 1;
  if (slot >= args.count) return;  // both threads of a pair leave together
  if (args.skip_if_short != 0u && *args.long_flag == 0u) return;  // hash_short_kernel has this batch
  const uint32_t half = static_cast<uint32_t>(tid) & 1u;
  const uint32_t pair = 3u << (threadIdx.x & 30u);
  const uint64_t m = args.order ? static_cast<uint64_t>(args.order[slot]) : slot;
  const uint8_t* p = args.data + (args.offsets ? args.offsets[m] : m * args.fixed_len);
  const uint64_t len = args.lengths ? args.lengths[m] : args.fixed_len;
  HalfState a;
#pragma unroll
  for (int i = 0; i < 25; ++i) a.w[i] = 0u;
  // One loop over the permutations of the message (one copy of the rounds): whole blocks
  // (sponge.cpp:87-110), the partial block + pad (:113-129), extra squeeze blocks (:131-143).
  const uint64_t whole = len / R;
  const uint32_t rem = static_cast<uint32_t>(len - whole * R);
  uint8_t* o = args.digests + m * args.digest_bytes;
  uint64_t out_left = args.digest_bytes;
  for (uint64_t k = 0;; ++k) {
    if (k < whole) {
      absorb_block<RL>(a, p, half);
      p += R;
    } else if (k == whole) {
      absorb_final<RL>(a, p, rem, args.head, half);
    }
    pair_permute(a, pair, half);
    if (k < whole) continue;
    const uint32_t n = out_left < R ? static_cast<uint32_t>(out_left) : R;
    emit_half<RL>(a, o, n, half);
    out_left -= n;
    if (out_left == 0) break;
    o += n;
  }
  if (args.last_mask != 0xffu) {  // batch.cpp:22-24; the byte was stored by one of the two threads
    __syncwarp(pair);
    if (half == 0u) args.digests[m * args.digest_bytes + args.digest_bytes - 1u] &= static_cast<uint8_t>(args.last_mask);
  }
}

template <int RL>
cudaError_t launch_pair(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  const int threads = plan.block_threads > 0 ? plan.block_threads : 128;
  const uint64_t blocks = (2 * args.count + threads - 1) / threads;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull || (threads & 1)) return cudaErrorInvalidConfiguration;
  hash_pair_kernel<RL><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_hash_pair(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  if (args.digest_bytes == 0) return cudaErrorInvalidConfiguration;
  switch (plan.rate_lanes) {
    case 9: return launch_pair<9>(args, plan, stream);
    case 13: return launch_pair<13>(args, plan, stream);
    case 17: return launch_pair<17>(args, plan, stream);
    case 18: return launch_pair<18>(args, plan, stream);
    case 21: return launch_pair<21>(args, plan, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace b200sha3
