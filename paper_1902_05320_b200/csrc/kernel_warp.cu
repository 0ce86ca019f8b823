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
//   = 9 64-bit shuffles (18 SHFL) in three dependent stages + ~16 ALU instructions per round,
//   so one permutation is ~24 x 3 shuffle latencies instead of ~4200 ALU issue slots.
//
// Absorb is one coalesced 8 x RL-byte read per block (thread t loads lane t; the next block
// is prefetched before the rounds of the current one), squeeze one coalesced write.
// Throughput per message is far below the one-thread kernels (25 of 32 lanes, shuffle
// bound), so capi.cu picks this kernel only when the batch could not fill the machine
// anyway (see kWarpKernelMaxCount there).
#include "kernels.cuh"
#include "sponge.cuh"

namespace b200sha3 {

namespace {

// rho offsets, index x + 5y (keccak.cpp:26-32)
__constant__ uint32_t kRhoOffset[25] = {0,  1,  62, 28, 27, 36, 44, 6,  55, 20, 3,  10, 43,
                                        25, 39, 41, 45, 15, 21, 8,  18, 2,  61, 56, 14};

// What thread t does in every round (all sources are lane ids of the same warp).
struct LaneRole {
  uint32_t column[4];  // the other four lanes of column x: (x, y+1) .. (x, y+4)
  uint32_t left;       // (x-1, y)
  uint32_t right;      // (x+1, y)
  uint32_t from[3];    // lanes whose rho output pi moves to (x, y), (x+1, y), (x+2, y)
  uint32_t rot;        // rho offset mod 32
  bool swap;           // rho offset >= 32: halves trade places before the funnel shifts
  uint32_t first;      // all ones on lane 0 (iota), else 0
  uint32_t column0;    // all ones on the five lanes of column 0
};

__device__ __forceinline__ LaneRole lane_role(uint32_t t) {
  LaneRole r;
  if (t >= 25u) {  // idle threads take part in the shuffles with themselves as source
    for (int k = 0; k < 4; ++k) r.column[k] = t;
    r.left = r.right = r.from[0] = r.from[1] = r.from[2] = t;
    r.rot = 0u;
    r.swap = false;
    r.first = r.column0 = 0u;
    return r;
  }
  const uint32_t x = t % 5u, y = t / 5u;
  for (uint32_t k = 0; k < 4u; ++k) r.column[k] = x + 5u * ((y + k + 1u) % 5u);
  r.left = (x + 4u) % 5u + 5u * y;
  r.right = (x + 1u) % 5u + 5u * y;
  for (uint32_t k = 0; k < 3u; ++k) {
    const uint32_t X = (x + k) % 5u;       // b[X + 5y] = rotl(a[src], rho[src]),
    r.from[k] = (X + 3u * y) % 5u + 5u * X;  // src = (X + 3y) % 5 + 5X   (keccak.cpp:261-267)
  }
  r.rot = kRhoOffset[t] & 31u;
  r.swap = kRhoOffset[t] >= 32u;
  r.first = t == 0u ? 0xffffffffu : 0u;
  r.column0 = x == 0u ? 0xffffffffu : 0u;
  return r;
}

constexpr unsigned kFullWarp = 0xffffffffu;

// (A REDUX form of the column parity -- redux.sync.xor over the column's five lanes -- was
// measured 16x slower: REDUX writes a warp-uniform register, so five different member masks in
// one warp run as a serialised fallback loop.  Shared memory instead of shuffles: 47 cycles
// per STS.64 + LDS.64 round trip against 33 per SHFL, tools/microbench/shfl_probe.cu.)
// One round WITHOUT its iota; `pend_*` is the round constant the previous round still owes lane
// (0, 0).  Keeping iota out of the chi -> shuffle chain takes one dependent instruction off every
// round: the shuffles send the lanes as chi left them, and while they are in flight lane 0 adds
// the constant to itself (`own`) and every lane of column 0 adds it to its share of the parity
// (`term`) -- C[0] comes out right, nobody waited.
__device__ __forceinline__ void warp_round(uint32_t& lo, uint32_t& hi, const LaneRole& r, uint32_t pend_lo,
                                           uint32_t pend_hi) {
  // theta (keccak.cpp:250-259)
  const uint32_t l1 = __shfl_sync(kFullWarp, lo, r.column[0]), h1 = __shfl_sync(kFullWarp, hi, r.column[0]);
  const uint32_t l2 = __shfl_sync(kFullWarp, lo, r.column[1]), h2 = __shfl_sync(kFullWarp, hi, r.column[1]);
  const uint32_t l3 = __shfl_sync(kFullWarp, lo, r.column[2]), h3 = __shfl_sync(kFullWarp, hi, r.column[2]);
  const uint32_t l4 = __shfl_sync(kFullWarp, lo, r.column[3]), h4 = __shfl_sync(kFullWarp, hi, r.column[3]);
  const uint32_t own_lo = lo ^ (pend_lo & r.first), own_hi = hi ^ (pend_hi & r.first);
  const uint32_t term_lo = lo ^ (pend_lo & r.column0), term_hi = hi ^ (pend_hi & r.column0);
  const uint32_t cl = xor3(xor3(term_lo, l1, l2), l3, l4), ch = xor3(xor3(term_hi, h1, h2), h3, h4);
  const uint32_t ml = __shfl_sync(kFullWarp, cl, r.left), mh = __shfl_sync(kFullWarp, ch, r.left);
  const uint32_t pl = __shfl_sync(kFullWarp, cl, r.right), ph = __shfl_sync(kFullWarp, ch, r.right);
  lo = xor3(own_lo, ml, __funnelshift_l(ph, pl, 1));
  hi = xor3(own_hi, mh, __funnelshift_l(pl, ph, 1));
  // rho (keccak.cpp:261-267), by this lane's own offset
  const uint32_t u = r.swap ? hi : lo, v = r.swap ? lo : hi;
  const uint32_t bl = __funnelshift_l(v, u, r.rot), bh = __funnelshift_l(u, v, r.rot);
  // pi + chi (keccak.cpp:261-273); iota (:275) is the next round's `pend`
  const uint32_t b0l = __shfl_sync(kFullWarp, bl, r.from[0]), b0h = __shfl_sync(kFullWarp, bh, r.from[0]);
  const uint32_t b1l = __shfl_sync(kFullWarp, bl, r.from[1]), b1h = __shfl_sync(kFullWarp, bh, r.from[1]);
  const uint32_t b2l = __shfl_sync(kFullWarp, bl, r.from[2]), b2h = __shfl_sync(kFullWarp, bh, r.from[2]);
  lo = chi3(b0l, b1l, b2l);
  hi = chi3(b0h, b1h, b2h);
}

__device__ __forceinline__ void warp_permute(uint32_t& lo, uint32_t& hi, const LaneRole& r) {
  warp_round(lo, hi, r, 0u, 0u);
#pragma unroll
  for (int round = 1; round < 24; ++round) {
    warp_round(lo, hi, r, static_cast<uint32_t>(round_constant(round - 1)),
               static_cast<uint32_t>(round_constant(round - 1) >> 32));
  }
  lo ^= static_cast<uint32_t>(round_constant(23)) & r.first;
  hi ^= static_cast<uint32_t>(round_constant(23) >> 32) & r.first;
}

// Eight message bytes at q (all inside the message), any alignment: one 8-byte load, or
// aligned 4-byte loads re-assembled with PRMT (only words that hold message bytes are read).
__device__ __forceinline__ uint2 load_lane(const uint8_t* q) {
  const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(q));
  if ((mis & 7u) == 0u) return ld_u2(reinterpret_cast<const uint2*>(q));
  const uint32_t sh = mis & 3u;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(q - sh);
  const uint32_t w0 = ld_u32(w), w1 = ld_u32(w + 1), w2 = sh ? ld_u32(w + 2) : 0u;
  const uint32_t sel = 0x3210u + 0x1111u * sh;
  return make_uint2(__byte_perm(w0, w1, sel), __byte_perm(w1, w2, sel));
}

// The first n (< 8) bytes at q, zero-extended.
__device__ __forceinline__ uint2 load_lane_head(const uint8_t* q, uint32_t n) {
  uint2 v = make_uint2(0u, 0u);
  for (uint32_t b = 0; b < n; ++b) {
    const uint32_t byte = ld_u8(q + b);
    if (b < 4u) {
      v.x |= byte << (8u * b);
    } else {
      v.y |= byte << (8u * (b - 4u));
    }
  }
  return v;
}

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
