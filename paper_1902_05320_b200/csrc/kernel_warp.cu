// kernel_warp.cu -- one Keccak state per WARP, for batches of few (long) messages.
//
// The sponge is sequential per message (sponge.cpp:87-110: block k+1 is absorbed into the
// state block k left behind), so with one message per thread a batch of N messages keeps
// N / 32 warps busy and its run time is (blocks per message) x (latency of one
// permutation in one thread: ~10^4 cycles, 4174 dependent-issue ALU instructions) however
// small N is -- 1024 x 1 MiB sits at 5 % of the ALU roofline.  The only parallelism left is
// INSIDE permute_1600 (keccak.cpp:245-277), and this kernel spends a warp on it:
//
//   thread t = x + 5y (t < 25) holds lane (x, y) as two 32-bit registers; threads 25..31 idle.
//   theta   column parity C[x]: four shuffles from the other lanes of the column, two xor3;
//           C[x-1] and C[x+1]: two shuffles from the row neighbours; one xor3.
//   rho     the thread's own rotation amount (two variable funnel shifts).
//   pi+chi  thread (x, y) fetches the three rho outputs that pi moves to (x, y), (x+1, y)
//           and (x+2, y) -- three shuffles with per-thread constant sources -- and applies
//           chi; iota on lane 0 through a mask.
//   = 9 64-bit shuffles (18 SHFL) in three dependent stages + ~16 ALU instructions per round:
//   measured 3994 cycles per permutation (24 x (18 x ~4 cycles of SHFL issue + 3 x ~28 of
//   latency + the dependent ALU instructions)) against ~10 000 in one thread.
//
// Absorb is one coalesced 8 x RL-byte read per block (thread t loads lane t; the next block
// is prefetched before the rounds of the current one), squeeze one coalesced write.
// Throughput per message is far below the one-thread kernels (25 of 32 lanes, shuffle
// bound: ~1 SHFL per clock per SM), so capi.cu picks this kernel only when the batch could not
// fill the machine anyway (warp_kernel_max_count() there: 2816 messages).
#include "kernels.cuh"
#include "warp_state.cuh"

namespace b200sha3 {

namespace {

using namespace warp_state;

__global__ void __launch_bounds__(32)
hash_warp_kernel(const HashArgs args, const uint32_t rate_lanes) {
  const uint32_t t = threadIdx.x;
  const uint64_t w = blockIdx.x;
  const uint64_t m = args.order ? static_cast<uint64_t>(args.order[w]) : w;
  const uint64_t off = args.offsets ? args.offsets[m] : m * args.fixed_len;
  uint64_t left = args.lengths ? args.lengths[m] : args.fixed_len;
  const uint8_t* p = args.data + off;
  const LaneRole role = lane_role(t);
  const uint32_t R = 8u * rate_lanes;
  const bool in_rate = t < rate_lanes;

  // One loop over the permutations of the message, so that the unrolled rounds exist once:
  // floor(len / R) whole-block absorbs (sponge.cpp:87-110; the next block is in flight during
  // the rounds), then the partial block + pad (sponge.cpp:113-129), then one more permutation
  // per extra squeeze block (sponge.cpp:131-143).  Every branch is warp-uniform.
  const uint64_t whole = left / R;
  const uint32_t rem = static_cast<uint32_t>(left - whole * R);
  uint8_t* o = args.digests + m * args.digest_bytes;
  uint64_t out_left = args.digest_bytes;
  uint32_t lo = 0u, hi = 0u;
  uint2 next = make_uint2(0u, 0u);
  if (whole != 0 && in_rate) next = load_lane(p + 8u * t);
  for (uint64_t i = 0;; ++i) {
    if (i < whole) {
      lo ^= next.x;
      hi ^= next.y;
      p += R;
      next = make_uint2(0u, 0u);
      if (i + 1 < whole && in_rate) next = load_lane(p + 8u * t);
    } else if (i == whole) {
      if (8u * t + 8u <= rem) {
        const uint2 v = load_lane(p + 8u * t);
        lo ^= v.x;
        hi ^= v.y;
      } else if (8u * t < rem) {
        const uint2 v = load_lane_head(p + 8u * t, rem - 8u * t);
        lo ^= v.x;
        hi ^= v.y;
      }
      if (t == (rem >> 3)) {
        const uint32_t shift = 8u * (rem & 7u);
        if (shift < 32u) {
          lo ^= args.head << shift;
        } else {
          hi ^= args.head << (shift - 32u);
        }
      }
      if (t == rate_lanes - 1u) hi ^= 0x80000000u;
    }
    warp_permute(lo, hi, role);
    if (i < whole) continue;
    const uint32_t n = out_left < R ? static_cast<uint32_t>(out_left) : R;
    if (8u * t < n) {
      uint8_t* dst = o + 8u * t;
      const uint32_t k = n - 8u * t < 8u ? n - 8u * t : 8u;
      if (k == 8u && (reinterpret_cast<uintptr_t>(dst) & 7u) == 0u) {
        *reinterpret_cast<uint2*>(dst) = make_uint2(lo, hi);
      } else {
        for (uint32_t b = 0; b < k; ++b) {
          dst[b] = static_cast<uint8_t>((b < 4u ? lo >> (8u * b) : hi >> (8u * (b - 4u))));
        }
      }
    }
    out_left -= n;
    if (out_left == 0) break;
    o += n;
  }
  if (args.last_mask != 0xffu) {  // batch.cpp:22-24; the byte was stored by some thread of this warp
    __syncwarp();
    if (t == 0u) args.digests[m * args.digest_bytes + args.digest_bytes - 1u] &= static_cast<uint8_t>(args.last_mask);
  }
}

}  // namespace

cudaError_t launch_hash_warp(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream) {
  if (args.count == 0) return cudaSuccess;
  if (args.count > 0x7fffffffull || args.digest_bytes == 0) return cudaErrorInvalidConfiguration;
  const unsigned grid = static_cast<unsigned>(args.count);
  const uint32_t rate_lanes = static_cast<uint32_t>(plan.rate_lanes);
  hash_warp_kernel<<<grid, 32, 0, stream>>>(args, rate_lanes);
  return cudaGetLastError();
}

}  // namespace b200sha3
