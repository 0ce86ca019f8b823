// warp_state.cuh -- one Keccak state spread over the 25 low threads of a warp: thread
// t = x + 5y holds lane (x, y) of permute_1600's state (proj/core/src/keccak.cpp:245-277,
// index x + 5y, keccak.hpp:36-38) as two 32-bit registers; all exchange is by shuffles.
// Shared by the batch kernel (kernel_warp.cu) and the incremental one (kernel_stream_warp.cu).
#pragma once
#include "sponge.cuh"

namespace b200sha3 {
namespace warp_state {

// rho offsets, index x + 5y (keccak.cpp:26-32)
static __constant__ uint32_t kRhoOffset[25] = {0,  1,  62, 28, 27, 36, 44, 6,  55, 20, 3,  10, 43,
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

}  // namespace warp_state
}  // namespace b200sha3
