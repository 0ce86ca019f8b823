// kernel_fewblock.cu -- equal-length MULTI-block batches, one message per thread:
//   hash_fewblock_kernel<RL, ML, OW>   everything about the shape static (cfg2 lengths at or above
//                                      the rate, cfg3 outputs longer than the rate)
//   hash_manyblock_kernel<RL, OW>      the same round sequence with the message length a run-time
//                                      value (any whole number of lanes at or above the rate)
//
// hash_into (proj/core/src/batch.cpp:15-25) for a batch whose messages are ML whole lanes and whose
// digests are OW whole 32-bit words, both compile-time: NB = ML / RL full blocks are absorbed
// (sponge.cpp:87-110), then the REM = ML % RL remaining lanes with the pad (sponge.cpp:113-129), then
// NS - 1 more permutations between the NS output blocks (sponge.cpp:131-143) -- P = NB + NS
// permutations per message.  The generic kernel runs these shapes at 0.985-0.99 of the ALU
// roofline: nothing stalls, it just carries instructions a static shape does not need (offsets,
// lengths, jump tables over the tail and the digest size, a permutation that cannot drop dead
// work).  Here the 24 P rounds of a message are ONE sequence
//
//     round 0 | (8 P - 1) x [3 rounds] | rounds 22, 23 of the last permutation
//
// with the first round and the last two straight-line (ptxas drops the work on the capacity
// lanes, zero before the first permutation, and on the lanes nobody reads after the last one,
// as in the one-block kernel) and ONE rolled copy of three rounds in between, ~17 KB of code in
// all.  What happens BETWEEN permutations -- absorb the next block, absorb the final block and
// pad, or store an output block -- sits in front of the third round of every eighth loop body
// (that round is round 0 of the next permutation), behind a warp-uniform branch; lane indices
// are static everywhere, only the block's base pointer is a run-time value.
#include "kernels.cuh"
#include "sponge.cuh"

namespace b200sha3 {

namespace {

// iota constants as (lo, hi) pairs, keccak.cpp:34-43, with round 0 repeated at index 24: the
// loop body starting at round 22 ends with round 0 of the next permutation.
__constant__ uint32_t kRoundConstWrap[50] = {
    0x00000001u, 0x00000000u, 0x00008082u, 0x00000000u, 0x0000808au, 0x80000000u,
    0x80008000u, 0x80000000u, 0x0000808bu, 0x00000000u, 0x80000001u, 0x00000000u,
    0x80008081u, 0x80000000u, 0x00008009u, 0x80000000u, 0x0000008au, 0x00000000u,
    0x00000088u, 0x00000000u, 0x80008009u, 0x00000000u, 0x8000000au, 0x00000000u,
    0x8000808bu, 0x00000000u, 0x0000008bu, 0x80000000u, 0x00008089u, 0x80000000u,
    0x00008003u, 0x80000000u, 0x00008002u, 0x80000000u, 0x00000080u, 0x80000000u,
    0x0000800au, 0x00000000u, 0x8000000au, 0x80000000u, 0x80008081u, 0x80000000u,
    0x00008080u, 0x80000000u, 0x80000001u, 0x00000000u, 0x80008008u, 0x80000000u,
    0x00000001u, 0x00000000u};

// How an output block leaves the registers.  The vector stores need aligned register pairs /
// quads, and WHERE ptxas then keeps the state decides how many LOP3 / SHF of the round loop read
// three registers of one bank: 0-11 of 540 in a good allocation, 65-87 in a bad one, which runs
// 1.5-2 % under its instruction count (tools/sass_bank_census.py counts them from the SASS;
// hash_fewblock_kernel<21, 8, 128>: 87 -> 0.989 of the ALU roofline, 1 -> 1.006).  Stored straight
// from the state, the quads of a 21-lane block pin the whole state into such an allocation
// (87); stored from copies ptxas cannot coalesce (IMAD by a run-time 1: FMA pipe, next to
// free), the state is unconstrained and lands in another bad one (79).  Copying SOME lanes
// breaks the pattern: kCopyLanes was found by a search over random lane sets with that census
// (most sets give <= 2; this one gives 0 for all four multi-block-output shapes).
#ifndef B200SHA3_FEWBLOCK_COPY_LANES  // the search builds of tools/fewblock_lane_search.sh pass other sets
#define B200SHA3_FEWBLOCK_COPY_LANES 0x10b417u  // lanes 0, 1, 2, 4, 10, 12, 13, 15, 20
#endif
constexpr uint32_t kCopyLanes = B200SHA3_FEWBLOCK_COPY_LANES;
__device__ __forceinline__ uint32_t copy_reg(uint32_t v, uint32_t one) {
  uint32_t t;
  asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(t) : "r"(v), "r"(one));
  return t;
}
// lane j of the state as (lo, hi), through copies if the lane is in the set (j is a
// compile-time value after unrolling)
__device__ __forceinline__ uint2 lane_out(const State& a, int j, uint32_t one) {
  const bool c = ((kCopyLanes >> j) & 1u) != 0u;
  return make_uint2(c ? copy_reg(a.lo[j], one) : a.lo[j], c ? copy_reg(a.hi[j], one) : a.hi[j]);
}
__device__ __forceinline__ void store2(uint8_t* w, const State& a, int j, uint32_t one) {
  __stcs(reinterpret_cast<uint2*>(w), lane_out(a, j, one));
}
__device__ __forceinline__ void store4(uint8_t* w, const State& a, int j, uint32_t one) {
  const uint2 u = lane_out(a, j, one), v = lane_out(a, j + 1, one);
  __stcs(reinterpret_cast<uint4*>(w), make_uint4(u.x, u.y, v.x, v.y));
}

// Stores the first N lanes of the state to w (8-byte aligned) with 16-byte streaming stores where
// w allows: half the store instructions and half the sector writes of 8-byte ones (a thread's
// output blocks are 256 or 512 bytes apart from its neighbour's, so nothing coalesces across
// threads; 8-byte stores left the SHAKE256 shapes 1 % slower).  `off8`: w is 8 bytes past a
// 16-byte boundary (kernel-uniform).
template <int N>
__device__ __forceinline__ void store_lanes(const State& a, uint8_t* w, bool off8, uint32_t one) {
  if (!off8) {
#pragma unroll
    for (int j = 0; j + 1 < N; j += 2) store4(w + 8 * j, a, j, one);
    if (N % 2 != 0) store2(w + 8 * (N - 1), a, N - 1, one);
  } else {
    store2(w, a, 0, one);
#pragma unroll
    for (int j = 1; j + 1 < N; j += 2) store4(w + 8 * j, a, j, one);
    if (N % 2 == 0) store2(w + 8 * (N - 1), a, N - 1, one);
  }
}

template <int RL, int ML, int OW>
__global__ void __launch_bounds__(256)
hash_fewblock_kernel(const uint8_t* __restrict__ data, uint8_t* __restrict__ digests, uint64_t count,
                     uint32_t head, uint32_t one) {
  constexpr int NB = ML / RL;                       // whole blocks absorbed before the final one
  constexpr int REM = ML % RL;                      // message lanes of the final block
  constexpr int NS = (OW + 2 * RL - 1) / (2 * RL);  // output blocks
  constexpr int P = NB + NS;                        // permutations per message
  constexpr int LAST_W = OW - (NS - 1) * 2 * RL;    // 32-bit words of the last output block
  static_assert(P >= 2, "single-permutation shapes belong to the one-block kernel");
  static_assert(NS == 1 || OW % 4 == 0, "output blocks are stored with 16-byte stores into 16-byte aligned slots");
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= count) return;
  const uint2* q = reinterpret_cast<const uint2*>(data + tid * (8ull * ML));
  uint8_t* o = digests + tid * (4ull * OW);

  State a;
  state_zero(a);
  // in front of permutation 0: the first block, whole (NB >= 1) or final
#pragma unroll
  for (int j = 0; j < (NB >= 1 ? RL : REM); ++j) {
    const uint2 v = __ldg(q + j);
    a.lo[j] = v.x;
    a.hi[j] = v.y;
  }
  if constexpr (NB == 0) {
    a.lo[REM] ^= head;             // sponge.cpp:122-123
    a.hi[RL - 1] ^= 0x80000000u;   // sponge.cpp:124-125
  }
  keccak_round<0u>(a, static_cast<uint32_t>(round_constant(0)), static_cast<uint32_t>(round_constant(0) >> 32));

  uint32_t r = 1u;  // round number of the loop body's first round
  int k = 0;        // permutations started so far, minus one
#pragma unroll 1
  for (int i = 0; i < 8 * P - 1; ++i) {
    keccak_round<0u>(a, kRoundConstWrap[2u * r], kRoundConstWrap[2u * r + 1u]);
    keccak_round<0u>(a, kRoundConstWrap[2u * r + 2u], kRoundConstWrap[2u * r + 3u]);
    if (r == 22u) {  // permutation k is complete after these two rounds; the next round starts k + 1
      ++k;
      if (NB >= 2 && k < NB) {  // whole block k
        const uint2* b = q + k * RL;
#pragma unroll
        for (int j = 0; j < RL; ++j) {
          const uint2 v = __ldg(b + j);
          a.lo[j] ^= v.x;
          a.hi[j] ^= v.y;
        }
      } else if (NB >= 1 && k == NB) {  // final block: REM lanes, pad
        const uint2* b = q + NB * RL;
#pragma unroll
        for (int j = 0; j < REM; ++j) {
          const uint2 v = __ldg(b + j);
          a.lo[j] ^= v.x;
          a.hi[j] ^= v.y;
        }
        a.lo[REM] ^= head;
        a.hi[RL - 1] ^= 0x80000000u;
      } else if (NS >= 2) {  // output block k - NB - 1 is complete
        // the digest slot is 16-byte aligned and a block is 8 RL bytes: with RL odd every other
        // block starts 8 bytes off
        const uint32_t m = static_cast<uint32_t>(k - NB - 1);
        store_lanes<RL>(a, o + m * (8u * RL), RL % 2 != 0 && (m & 1u) != 0u, one);
      }
    }
    keccak_round<0u>(a, kRoundConstWrap[2u * r + 4u], kRoundConstWrap[2u * r + 5u]);
    r = r == 22u ? 1u : r + 3u;
  }
  keccak_round<0u>(a, static_cast<uint32_t>(round_constant(22)), static_cast<uint32_t>(round_constant(22) >> 32));
  keccak_round<0u>(a, static_cast<uint32_t>(round_constant(23)), static_cast<uint32_t>(round_constant(23) >> 32));
  if constexpr (NS == 1) {
    emit_words_static<RL, LAST_W, OW % 4 == 0>(a, o);
  } else {  // LAST_W is even here (OW % 4 == 0, whole lanes before it)
    store_lanes<LAST_W / 2>(a, o + (NS - 1) * (8 * RL), ((NS - 1) * 8 * RL) % 16 != 0, one);
  }
}

// (rate lanes, message lanes, output 32-bit words)
// The same round sequence with the message length a RUN-TIME value: equal-length messages of ANY
// whole number of lanes at or above the rate (200-byte records, 1000-byte rows ...), digest of OW
// words that fits one block.  nb = ml / RL whole blocks, then the final block of rem = ml % RL
// lanes through a jump table over rem (kernel-uniform, every case static), so a message costs
// the instructions of the static-shape kernel; only the zero-lane savings of round 0 need ml >= RL
// (the first block is whole), which is this kernel's precondition.
template <int RL, int REM>
__device__ __forceinline__ void absorb_final_lanes(State& a, const uint2* b, uint32_t head) {
#pragma unroll
  for (int j = 0; j < REM; ++j) {
    const uint2 v = __ldg(b + j);
    a.lo[j] ^= v.x;
    a.hi[j] ^= v.y;
  }
  a.lo[REM] ^= head;            // sponge.cpp:122-123
  a.hi[RL - 1] ^= 0x80000000u;  // sponge.cpp:124-125
}

template <int RL, int OW>
__global__ void __launch_bounds__(256)
hash_manyblock_kernel(const uint8_t* __restrict__ data, uint8_t* __restrict__ digests, uint64_t count,
                      uint32_t head, uint32_t ml) {
  static_assert(OW <= 2 * RL, "digest must fit one block");
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= count) return;
  const uint32_t nb = ml / RL, rem = ml - nb * RL;  // nb >= 1
  const uint2* q = reinterpret_cast<const uint2*>(data + tid * (8ull * ml));
  uint8_t* o = digests + tid * (4ull * OW);

  State a;
  state_zero(a);
#pragma unroll
  for (int j = 0; j < RL; ++j) {
    const uint2 v = __ldg(q + j);
    a.lo[j] = v.x;
    a.hi[j] = v.y;
  }
  keccak_round<0u>(a, static_cast<uint32_t>(round_constant(0)), static_cast<uint32_t>(round_constant(0) >> 32));

  uint32_t r = 1u, k = 0u;
  const uint32_t trips = 8u * (nb + 1u) - 1u;
#pragma unroll 1
  for (uint32_t i = 0; i < trips; ++i) {
    keccak_round<0u>(a, kRoundConstWrap[2u * r], kRoundConstWrap[2u * r + 1u]);
    keccak_round<0u>(a, kRoundConstWrap[2u * r + 2u], kRoundConstWrap[2u * r + 3u]);
    if (r == 22u) {
      ++k;
      const uint2* b = q + static_cast<uint64_t>(k) * RL;
      if (k < nb) {  // whole block k
#pragma unroll
        for (int j = 0; j < RL; ++j) {
          const uint2 v = __ldg(b + j);
          a.lo[j] ^= v.x;
          a.hi[j] ^= v.y;
        }
      } else {  // final block: rem lanes, pad
        switch (rem) {
#define B200SHA3_FINAL_CASE(R) \
  case R:                      \
    if constexpr (R < RL) absorb_final_lanes<RL, (R < RL ? R : 0)>(a, b, head); \
    break;
          B200SHA3_FINAL_CASE(0) B200SHA3_FINAL_CASE(1) B200SHA3_FINAL_CASE(2) B200SHA3_FINAL_CASE(3)
          B200SHA3_FINAL_CASE(4) B200SHA3_FINAL_CASE(5) B200SHA3_FINAL_CASE(6) B200SHA3_FINAL_CASE(7)
          B200SHA3_FINAL_CASE(8) B200SHA3_FINAL_CASE(9) B200SHA3_FINAL_CASE(10) B200SHA3_FINAL_CASE(11)
          B200SHA3_FINAL_CASE(12) B200SHA3_FINAL_CASE(13) B200SHA3_FINAL_CASE(14) B200SHA3_FINAL_CASE(15)
          B200SHA3_FINAL_CASE(16) B200SHA3_FINAL_CASE(17) B200SHA3_FINAL_CASE(18) B200SHA3_FINAL_CASE(19)
          B200SHA3_FINAL_CASE(20)
#undef B200SHA3_FINAL_CASE
          default: break;
        }
      }
    }
    keccak_round<0u>(a, kRoundConstWrap[2u * r + 4u], kRoundConstWrap[2u * r + 5u]);
    r = r == 22u ? 1u : r + 3u;
  }
  keccak_round<0u>(a, static_cast<uint32_t>(round_constant(22)), static_cast<uint32_t>(round_constant(22) >> 32));
  keccak_round<0u>(a, static_cast<uint32_t>(round_constant(23)), static_cast<uint32_t>(round_constant(23) >> 32));
  emit_words_static<RL, OW, OW % 4 == 0>(a, o);
}

// (rate lanes, output 32-bit words): the four hashes, the two SHAKEs at 128- / 256- / 512-bit outputs
#define B200SHA3_MANYBLOCK_SHAPES(X) \
  X(18, 7) X(17, 8) X(13, 12) X(9, 16) X(17, 4) X(17, 16) X(21, 4) X(21, 8) X(21, 16)

// (rate lanes, message lanes, output 32-bit words)
#define B200SHA3_FEWBLOCK_SHAPES(X)                                                               \
  X(18, 32, 7) X(18, 64, 7) X(18, 128, 7)                /* SHA3-224: 256 / 512 / 1024 B       */ \
  X(17, 32, 8) X(17, 64, 8) X(17, 128, 8)                /* SHA3-256: 256 / 512 / 1024 B       */ \
  X(13, 16, 12) X(13, 32, 12) X(13, 64, 12) X(13, 128, 12) /* SHA3-384: 128 ... 1024 B         */ \
  X(9, 16, 16) X(9, 32, 16) X(9, 64, 16) X(9, 128, 16)   /* SHA3-512: 128 ... 1024 B           */ \
  X(21, 8, 64) X(21, 8, 128)                             /* SHAKE128: 64 B -> 2048 / 4096 bits */ \
  X(17, 8, 64) X(17, 8, 128)                             /* SHAKE256: 64 B -> 2048 / 4096 bits */

}  // namespace

bool fewblock_supported(int rate_lanes, uint64_t msg_len, uint64_t digest_bytes) {
  if (msg_len % 8 != 0 || digest_bytes % 4 != 0 || msg_len > 1024 || digest_bytes > 512) return false;
  const int ml = static_cast<int>(msg_len / 8), ow = static_cast<int>(digest_bytes / 4);
#define X(RL, ML, OW) \
  if (rate_lanes == RL && ml == ML && ow == OW) return true;
  B200SHA3_FEWBLOCK_SHAPES(X)
#undef X
  return false;
}

// Equal-length, 16-byte aligned data and digests, whole-byte output (no XOF tail mask).
cudaError_t launch_hash_fewblock(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  if (!fewblock_supported(plan.rate_lanes, args.fixed_len, args.digest_bytes) || args.offsets || args.lengths ||
      args.order || !args.aligned8 || args.last_mask != 0xffu) {
    return cudaErrorNotSupported;
  }
  const int threads = plan.block_threads > 0 ? plan.block_threads : 128;  // 64 / 128 / 256 swept: tools/fewblock_sweep.py
  const uint64_t blocks = (args.count + threads - 1) / threads;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  const int ml = static_cast<int>(args.fixed_len / 8), ow = static_cast<int>(args.digest_bytes / 4);
#define X(RL, ML, OW)                                                                              \
  if (plan.rate_lanes == RL && ml == ML && ow == OW) {                                             \
    hash_fewblock_kernel<RL, ML, OW><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(       \
        args.data, args.digests, args.count, args.head, 1u);                                           \
    return cudaGetLastError();                                                                     \
  }
  B200SHA3_FEWBLOCK_SHAPES(X)
#undef X
  return cudaErrorNotSupported;
}

}  // namespace b200sha3

namespace b200sha3 {

bool manyblock_supported(int rate_lanes, uint64_t msg_len, uint64_t digest_bytes) {
  if (msg_len % 8 != 0 || digest_bytes % 4 != 0 || msg_len < 8u * static_cast<uint64_t>(rate_lanes) ||
      msg_len >= (1ull << 31)) {
    return false;
  }
  const int ow = static_cast<int>(digest_bytes / 4);
#define X(RL, OW) \
  if (rate_lanes == RL && ow == OW) return true;
  B200SHA3_MANYBLOCK_SHAPES(X)
#undef X
  return false;
}

// Equal-length messages of whole lanes, 16-byte aligned data and digests, whole-byte output.
cudaError_t launch_hash_manyblock(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  if (!manyblock_supported(plan.rate_lanes, args.fixed_len, args.digest_bytes) || args.offsets || args.lengths ||
      args.order || !args.aligned8 || args.last_mask != 0xffu) {
    return cudaErrorNotSupported;
  }
  const int threads = plan.block_threads > 0 ? plan.block_threads : 128;
  const uint64_t blocks = (args.count + threads - 1) / threads;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  const int ow = static_cast<int>(args.digest_bytes / 4);
  const uint32_t ml = static_cast<uint32_t>(args.fixed_len / 8);
#define X(RL, OW)                                                                            \
  if (plan.rate_lanes == RL && ow == OW) {                                                   \
    hash_manyblock_kernel<RL, OW><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(    \
        args.data, args.digests, args.count, args.head, ml);                                 \
    return cudaGetLastError();                                                               \
  }
  B200SHA3_MANYBLOCK_SHAPES(X)
#undef X
  return cudaErrorNotSupported;
}

}  // namespace b200sha3
