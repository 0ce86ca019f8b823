// sponge.cuh -- per-thread sponge: pad / absorb / squeeze around keccak_f1600.
//
// Replaces, for one message per thread, the reference's SpongeHasher
// (proj/core/src/sponge.cpp:71-149) as driven by hash_into
// (proj/core/src/batch.cpp:15-25):
//   update  (sponge.cpp:81-111)  -> absorb_lanes_aligned / absorb_words_unaligned
//   finish  (sponge.cpp:113-129) -> absorb_tail_* (pad head byte at `rem`,
//                                   0x80 into the last rate byte)
//   squeeze (sponge.cpp:131-143) -> emit_block
//   XOF bit mask (batch.cpp:22-24) -> hash_message epilogue
//
// RL is the rate in 64-bit lanes (9, 13, 17, 18 or 21; sha3.cpp:13-20).  All
// state indices are compile-time; runtime lengths are handled with predicated,
// fully unrolled loops so the state stays in registers.
#pragma once
#include <cstdint>

#include "keccak_f1600.cuh"

namespace b200sha3 {

__device__ __forceinline__ uint2 ld_u2(const uint2* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ld_u32(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ld_u8(const uint8_t* p) { return __ldg(p); }

// XOR `lanes` (<= RL) 64-bit words from the 8-byte aligned pointer p into the state.
template <int RL>
__device__ __forceinline__ void absorb_lanes_aligned(State& a, const uint8_t* p,
                                                     uint32_t lanes) {
  const uint2* q = reinterpret_cast<const uint2*>(p);
#pragma unroll
  for (int i = 0; i < RL; ++i) {
    if (static_cast<uint32_t>(i) < lanes) {
      const uint2 v = ld_u2(q + i);
      a.lo[i] ^= v.x;
      a.hi[i] ^= v.y;
    }
  }
}

// XOR `words` (<= 2*RL) 32-bit words from the arbitrarily aligned pointer p into
// the state: aligned 4-byte loads re-assembled with PRMT.  Only aligned words
// that contain at least one byte of [p, p + 4*words) are touched.
template <int RL>
__device__ __forceinline__ void absorb_words_unaligned(State& a, const uint8_t* p,
                                                       uint32_t words) {
  const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p)) & 3u;
  const uint32_t* q = reinterpret_cast<const uint32_t*>(p - sh);
  const uint32_t sel = 0x3210u + 0x1111u * sh;
  const uint32_t nload = words ? words + (sh ? 1u : 0u) : 0u;
  uint32_t prev = nload ? ld_u32(q) : 0u;
#pragma unroll
  for (int j = 0; j < 2 * RL; ++j) {
    const uint32_t next = (static_cast<uint32_t>(j) + 1u < nload) ? ld_u32(q + j + 1) : 0u;
    const uint32_t w = (static_cast<uint32_t>(j) < words) ? __byte_perm(prev, next, sel) : 0u;
    if (j & 1) {
      a.hi[j >> 1] ^= w;
    } else {
      a.lo[j >> 1] ^= w;
    }
    prev = next;
  }
}

// Final (partial) block: `rem` < 8*RL message bytes at p, then the pad.
//   head = suffix | 1 << suffix_bits  (0x06 / 0x1f), XORed at byte `rem`;
//   0x80 XORed at byte 8*RL - 1 (the same byte when rem == 8*RL - 1).
//
// `ragged`: the threads of a warp hold final blocks of different lengths.  The jump table
// below would then run its cases one after the other (up to RL + 1 of them, each waiting
// for its own loads); the ragged form is the same work as RL predicated 8-byte loads, two
// 4-byte loads for the partial lane (nothing is read outside the aligned 4-byte words that
// hold message bytes) and predicated XORs -- ~6 ALU instructions per lane, no divergence.
template <int RL>
__device__ __forceinline__ void absorb_tail(State& a, const uint8_t* p, uint32_t rem,
                                            uint32_t head, bool aligned8, bool ragged = false) {
  if (aligned8 && ragged) {
    const uint32_t fl = rem >> 3, rb = rem & 7u;
    const uint2* q = reinterpret_cast<const uint2*>(p);
    const uint32_t* tq = reinterpret_cast<const uint32_t*>(p + 8u * fl);
    uint32_t tlo = rb != 0u ? ld_u32(tq) : 0u;
    uint32_t thi = rb > 4u ? ld_u32(tq + 1) : 0u;
    tlo &= rb >= 4u ? 0xffffffffu : (1u << (8u * rb)) - 1u;
    thi &= rb > 4u ? (1u << (8u * (rb - 4u))) - 1u : 0u;
    if (rb < 4u) {
      tlo |= head << (8u * rb);
    } else {
      thi |= head << (8u * (rb - 4u));
    }
#pragma unroll
    for (int i = 0; i < RL; ++i) {
      uint2 v = make_uint2(0u, 0u);
      if (static_cast<uint32_t>(i) < fl) v = ld_u2(q + i);
      if (static_cast<uint32_t>(i) == fl) v = make_uint2(tlo, thi);
      a.lo[i] ^= v.x;
      a.hi[i] ^= v.y;
    }
  } else if (aligned8) {
    const uint32_t fl = rem >> 3, rb = rem & 7u;
    const uint8_t* tp = p + 8u * fl;
    uint32_t tlo = 0u, thi = 0u;
    if (rb != 0u) {  // whole-lane messages (the common case) skip the byte loads
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (static_cast<uint32_t>(b) < rb) tlo |= ld_u8(tp + b) << (8 * b);
      }
#pragma unroll
      for (int b = 4; b < 7; ++b) {
        if (static_cast<uint32_t>(b) < rb) thi |= ld_u8(tp + b) << (8 * (b - 4));
      }
    }
    if (rb < 4u) {
      tlo |= head << (8u * rb);
    } else {
      thi |= head << (8u * (rb - 4u));
    }
    // One statically indexed code path per number of whole lanes (jump table) instead of
    // 2*RL predicated instructions: equal-length batches take the same case in every thread.
    const uint2* q = reinterpret_cast<const uint2*>(p);
    switch (fl) {
#define B200SHA3_TAIL_CASE(K)                         \
  case K:                                             \
    if constexpr (K < RL) {                           \
      _Pragma("unroll") for (int i = 0; i < K; ++i) { \
        const uint2 v = ld_u2(q + i);                 \
        a.lo[i] ^= v.x;                               \
        a.hi[i] ^= v.y;                               \
      }                                               \
      a.lo[K < RL ? K : 0] ^= tlo;                    \
      a.hi[K < RL ? K : 0] ^= thi;                    \
    }                                                 \
    break;
      B200SHA3_TAIL_CASE(0) B200SHA3_TAIL_CASE(1) B200SHA3_TAIL_CASE(2) B200SHA3_TAIL_CASE(3)
      B200SHA3_TAIL_CASE(4) B200SHA3_TAIL_CASE(5) B200SHA3_TAIL_CASE(6) B200SHA3_TAIL_CASE(7)
      B200SHA3_TAIL_CASE(8) B200SHA3_TAIL_CASE(9) B200SHA3_TAIL_CASE(10) B200SHA3_TAIL_CASE(11)
      B200SHA3_TAIL_CASE(12) B200SHA3_TAIL_CASE(13) B200SHA3_TAIL_CASE(14) B200SHA3_TAIL_CASE(15)
      B200SHA3_TAIL_CASE(16) B200SHA3_TAIL_CASE(17) B200SHA3_TAIL_CASE(18) B200SHA3_TAIL_CASE(19)
      B200SHA3_TAIL_CASE(20)
#undef B200SHA3_TAIL_CASE
      default: break;
    }
  } else {
    const uint32_t fw = rem >> 2, rb = rem & 3u;
    absorb_words_unaligned<RL>(a, p, fw);
    const uint8_t* tp = p + 4u * fw;
    uint32_t t = head << (8u * rb);
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      if (static_cast<uint32_t>(b) < rb) t |= ld_u8(tp + b) << (8 * b);
    }
#pragma unroll
    for (int j = 0; j < 2 * RL; ++j) {
      if (static_cast<uint32_t>(j) == fw) {
        if (j & 1) {
          a.hi[j >> 1] ^= t;
        } else {
          a.lo[j >> 1] ^= t;
        }
      }
    }
  }
  a.hi[RL - 1] ^= 0x80000000u;
}

// Final block of an EQUAL-LENGTH batch whose messages do not start on 8-byte boundaries (the
// paper's 10-byte messages: message i starts at 10 i).  `rem` = W whole 32-bit
// words + rb bytes is the same in every thread, so a jump table over W gives each case
// statically indexed aligned 4-byte loads and PRMTs with no predicates, except on the last two
// aligned words, which hold message bytes only for some shifts `sh` (the shift differs from
// thread to thread).  Nothing is read outside the aligned words that hold message bytes.
template <int RL, int W>
__device__ __forceinline__ void absorb_tail_uniform_case(State& a, const uint32_t* q, uint32_t sel,
                                                         uint32_t sh, uint32_t rb, uint32_t head) {
  if constexpr (W < 2 * RL) {
    // aligned word k covers message bytes [4k - sh, 4k - sh + 4): k < W always holds some,
    // k = W iff rb + sh > 0 (W = 0: iff rb > 0 -- an empty message touches nothing),
    // k = W + 1 iff rb + sh > 4
    uint32_t al[W + 2];
#pragma unroll
    for (int k = 0; k < W; ++k) al[k] = ld_u32(q + k);
    al[W] = ((W == 0 ? rb : rb + sh) > 0u) ? ld_u32(q + W) : 0u;
    al[W + 1] = (rb + sh > 4u) ? ld_u32(q + W + 1) : 0u;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const uint32_t w = __byte_perm(al[j], al[j + 1], sel);
      if (j & 1) {
        a.hi[j >> 1] ^= w;
      } else {
        a.lo[j >> 1] ^= w;
      }
    }
    const uint32_t t = (__byte_perm(al[W], al[W + 1], sel) & ((1u << (8u * rb)) - 1u)) | (head << (8u * rb));
    if (W & 1) {
      a.hi[W >> 1] ^= t;
    } else {
      a.lo[W >> 1] ^= t;
    }
  }
}

template <int RL>
__device__ __forceinline__ void absorb_tail_uniform_unaligned(State& a, const uint8_t* p, uint32_t rem,
                                                              uint32_t head) {
  const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p)) & 3u;
  const uint32_t* q = reinterpret_cast<const uint32_t*>(p - sh);
  const uint32_t sel = 0x3210u + 0x1111u * sh;
  const uint32_t rb = rem & 3u;
  switch (rem >> 2) {
#define B200SHA3_UTAIL_CASE(W) \
  case W: absorb_tail_uniform_case<RL, W>(a, q, sel, sh, rb, head); break;
#define B200SHA3_UTAIL_CASES6(W)                                                    \
  B200SHA3_UTAIL_CASE(W) B200SHA3_UTAIL_CASE(W + 1) B200SHA3_UTAIL_CASE(W + 2)      \
  B200SHA3_UTAIL_CASE(W + 3) B200SHA3_UTAIL_CASE(W + 4) B200SHA3_UTAIL_CASE(W + 5)
    B200SHA3_UTAIL_CASES6(0) B200SHA3_UTAIL_CASES6(6) B200SHA3_UTAIL_CASES6(12) B200SHA3_UTAIL_CASES6(18)
    B200SHA3_UTAIL_CASES6(24) B200SHA3_UTAIL_CASES6(30) B200SHA3_UTAIL_CASES6(36)
#undef B200SHA3_UTAIL_CASES6
#undef B200SHA3_UTAIL_CASE
    default: break;
  }
  a.hi[RL - 1] ^= 0x80000000u;
}

__device__ __forceinline__ uint32_t state_word(const State& a, int j) {
  return (j & 1) ? a.hi[j >> 1] : a.lo[j >> 1];
}

// Stores the first W whole 32-bit words of the rate part to the 4-byte aligned o, W a
// compile-time constant: 16-byte stores while o is 16-byte aligned (VEC), else 4-byte.
template <int RL, int W, bool VEC>
__device__ __forceinline__ void emit_words_static(const State& a, uint8_t* o) {
  if constexpr (W <= 2 * RL) {
    constexpr int kVec = VEC ? W / 4 : 0;
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
      reinterpret_cast<uint4*>(o)[k] = make_uint4(state_word(a, 4 * k), state_word(a, 4 * k + 1),
                                                  state_word(a, 4 * k + 2), state_word(a, 4 * k + 3));
    }
#pragma unroll
    for (int j = 4 * kVec; j < W; ++j) reinterpret_cast<uint32_t*>(o)[j] = state_word(a, j);
  }
}

// Jump table over the number of whole words: digests of one batch all have the same
// length, so every thread of a warp takes the same case and no predicates are needed.
template <int RL, bool VEC>
__device__ __forceinline__ void emit_words(const State& a, uint8_t* o, uint32_t words) {
  switch (words) {
#define B200SHA3_EMIT_CASE(W) \
  case W: emit_words_static<RL, W, VEC>(a, o); break;
#define B200SHA3_EMIT_CASES4(W) \
  B200SHA3_EMIT_CASE(W) B200SHA3_EMIT_CASE(W + 1) B200SHA3_EMIT_CASE(W + 2) B200SHA3_EMIT_CASE(W + 3)
    B200SHA3_EMIT_CASES4(1) B200SHA3_EMIT_CASES4(5) B200SHA3_EMIT_CASES4(9) B200SHA3_EMIT_CASES4(13)
    B200SHA3_EMIT_CASES4(17) B200SHA3_EMIT_CASES4(21) B200SHA3_EMIT_CASES4(25) B200SHA3_EMIT_CASES4(29)
    B200SHA3_EMIT_CASES4(33) B200SHA3_EMIT_CASES4(37) B200SHA3_EMIT_CASE(41) B200SHA3_EMIT_CASE(42)
#undef B200SHA3_EMIT_CASES4
#undef B200SHA3_EMIT_CASE
    default: break;
  }
}

// Writes the first n (<= 8*RL) bytes of the rate part, little-endian, to o: whole words
// through the jump table above when o is 4-byte aligned (16-byte stores when it is
// 16-byte aligned), then the 1-3 byte tail; byte stores for any other alignment.
template <int RL>
__device__ __forceinline__ void emit_block(const State& a, uint8_t* o, uint32_t n) {
  const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(o));
  if ((mis & 3u) == 0u) {
    const uint32_t words = n >> 2, tail = n & 3u;
    if ((mis & 15u) == 0u) {
      emit_words<RL, true>(a, o, words);
    } else {
      emit_words<RL, false>(a, o, words);
    }
    if (tail != 0u) {  // XOF lengths that are not a multiple of 4 bytes
      uint32_t w = 0u;
#pragma unroll
      for (int j = 0; j < 2 * RL; ++j) {
        if (static_cast<uint32_t>(j) == words) w = state_word(a, j);
      }
      for (uint32_t b = 0; b < tail; ++b) o[4u * words + b] = static_cast<uint8_t>(w >> (8u * b));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 2 * RL; ++j) {
      const uint32_t w = state_word(a, j);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (4u * j + b < n) o[4 * j + b] = static_cast<uint8_t>(w >> (8 * b));
      }
    }
  }
}

// One whole message: the a4 -> a5 -> a6 -> a7 sequence of SURVEY.md section 8(a).
//   p/len        message bytes (any alignment unless aligned8 says otherwise)
//   out/out_len  digest slot, out_len >= 1
//   head         0x06 (SHA-3) or 0x1f (SHAKE)
//   last_mask    0xff, or (1 << bits%8) - 1 for an XOF length that is not a
//                multiple of 8 (batch.cpp:22-24)
// Three phases, each with its own copy of the (rolled) permutation so that the hot
// full-block loop carries nothing but loads, XORs and the rounds:
//   absorb   floor(len/R) whole blocks                      (sponge.cpp:81-111)
//   finish   the partial block + pad, one permutation       (sponge.cpp:113-129)
//   squeeze  out_len bytes, a permutation between blocks    (sponge.cpp:131-143)
template <int RL, int UNROLL, uint32_t FMA_MASK>
__device__ __forceinline__ void hash_message(const uint8_t* p, uint64_t len, uint8_t* out,
                                             uint64_t out_len, uint32_t head,
                                             uint32_t last_mask, bool aligned8, bool ragged = false) {
  constexpr uint32_t R = 8u * RL;
  State a;
  state_zero(a);
  uint64_t left_in = len;
  if (aligned8) {
    while (left_in >= R) {
      absorb_lanes_aligned<RL>(a, p, RL);
      keccak_f1600<UNROLL, FMA_MASK>(a);
      p += R;
      left_in -= R;
    }
  } else {
    while (left_in >= R) {
      absorb_words_unaligned<RL>(a, p, 2 * RL);
      keccak_f1600<UNROLL, FMA_MASK>(a);
      p += R;
      left_in -= R;
    }
  }
  absorb_tail<RL>(a, p, static_cast<uint32_t>(left_in), head, aligned8, ragged);
  keccak_f1600<UNROLL, FMA_MASK>(a);
  uint8_t* o = out;
  uint64_t left = out_len;
  for (;;) {
    const uint32_t n = left < R ? static_cast<uint32_t>(left) : R;
    emit_block<RL>(a, o, n);
    left -= n;
    if (left == 0) break;
    o += n;
    keccak_f1600<UNROLL, FMA_MASK>(a);
  }
  if (last_mask != 0xffu) {
    out[out_len - 1u] &= static_cast<uint8_t>(last_mask);
  }
}

// The same for a digest of OW whole 32-bit words that fits one block, OW a compile-time value
// (the four hashes; short SHAKE outputs): no squeeze loop, and the finishing permutation is the
// peeled form (1 + 7x3 + 2) followed by a static store, so ptxas drops the work of the last two
// rounds on the lanes nobody reads -- ~120 instructions per message, which is what a message of
// two or three blocks notices.
template <int RL, int OW, int UNROLL, uint32_t FMA_MASK>
__device__ __forceinline__ void hash_message_static_out(const uint8_t* p, uint64_t len, uint8_t* out,
                                                        uint32_t head, bool aligned8, bool ragged) {
  static_assert(OW <= 2 * RL, "digest must fit one block");
  constexpr uint32_t R = 8u * RL;
  State a;
  state_zero(a);
  uint64_t left_in = len;
  if (aligned8) {
    while (left_in >= R) {
      absorb_lanes_aligned<RL>(a, p, RL);
      keccak_f1600<UNROLL, FMA_MASK>(a);
      p += R;
      left_in -= R;
    }
  } else {
    while (left_in >= R) {
      absorb_words_unaligned<RL>(a, p, 2 * RL);
      keccak_f1600<UNROLL, FMA_MASK>(a);
      p += R;
      left_in -= R;
    }
  }
  absorb_tail<RL>(a, p, static_cast<uint32_t>(left_in), head, aligned8, ragged);
  keccak_f1600<23, FMA_MASK>(a);
  emit_block<RL>(a, out, 4u * OW);
}

// ---------------------------------------------------------------------------
// Byte-granular pieces for the incremental (streaming) entry points: the state
// carries a byte position like SpongeHasher::pos_ (sponge.hpp:60-63).

// Byte mask of a 32-bit word: bytes [s, e) set; s and e are clamped to [0, 4].
__device__ __forceinline__ uint32_t byte_mask(int s, int e) {
  s = s < 0 ? 0 : (s > 4 ? 4 : s);
  e = e < 0 ? 0 : (e > 4 ? 4 : e);
  if (e <= s) return 0u;
  const uint32_t hi = e == 4 ? 0xffffffffu : ((1u << (8 * e)) - 1u);
  const uint32_t lo = (1u << (8 * s)) - 1u;  // s <= 3 here
  return hi & ~lo;
}

// XORs bytes [lo, hi) of the current rate block into the state, the block being laid
// out at the virtual pointer vp (block byte k is vp[k]; only [vp+lo, vp+hi) is message
// data).  0 <= lo <= hi <= 8*RL.  Aligned 4-byte loads + PRMT; a word is loaded only if
// it holds at least one byte of the range.  This is the byte loop of
// SpongeHasher::update (sponge.cpp:100-104) for one block, done word-parallel.
template <int RL>
__device__ __forceinline__ void absorb_bytes(State& a, const uint8_t* vp, uint32_t lo,
                                             uint32_t hi) {
  const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(vp)) & 3u;
  const uint32_t* q = reinterpret_cast<const uint32_t*>(vp - sh);
  const uint32_t sel = 0x3210u + 0x1111u * sh;
  // aligned word k covers block bytes [4k - sh, 4k - sh + 4)
  auto need = [&](int k) {
    const int first = 4 * k - static_cast<int>(sh);
    return first < static_cast<int>(hi) && first + 4 > static_cast<int>(lo);
  };
  uint32_t prev = need(0) ? ld_u32(q) : 0u;
#pragma unroll
  for (int j = 0; j < 2 * RL; ++j) {
    const uint32_t next = need(j + 1) ? ld_u32(q + j + 1) : 0u;
    const uint32_t m = byte_mask(static_cast<int>(lo) - 4 * j, static_cast<int>(hi) - 4 * j);
    const uint32_t w = __byte_perm(prev, next, sel) & m;
    if (j & 1) {
      a.hi[j >> 1] ^= w;
    } else {
      a.lo[j >> 1] ^= w;
    }
    prev = next;
  }
}

// XORs `value` (one byte) into the state at byte position pos < 8*RL.
template <int RL>
__device__ __forceinline__ void xor_byte_at(State& a, uint32_t pos, uint32_t value) {
  const uint32_t word = pos >> 2, shifted = value << (8u * (pos & 3u));
#pragma unroll
  for (int j = 0; j < 2 * RL; ++j) {
    if (static_cast<uint32_t>(j) == word) {
      if (j & 1) {
        a.hi[j >> 1] ^= shifted;
      } else {
        a.lo[j >> 1] ^= shifted;
      }
    }
  }
}

// Writes bytes [lo, hi) of the rate part to o[0 .. hi-lo) with byte stores (the general
// form of SpongeHasher::squeeze's copy-out, sponge.cpp:135-141).
template <int RL>
__device__ __forceinline__ void emit_bytes(const State& a, uint8_t* o, uint32_t lo, uint32_t hi) {
#pragma unroll
  for (int j = 0; j < 2 * RL; ++j) {
    const uint32_t w = state_word(a, j);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t k = 4u * j + b;
      if (k >= lo && k < hi) o[k - lo] = static_cast<uint8_t>(w >> (8 * b));
    }
  }
}

}  // namespace b200sha3
