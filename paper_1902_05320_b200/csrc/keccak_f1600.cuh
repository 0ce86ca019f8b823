// keccak_f1600.cuh -- Keccak-f[1600] for sm_100a, one state per thread.
//
// Replaces the reference's permute_1600 (proj/core/src/keccak.cpp:245-277) and
// its two tables kRho1600 (:26-32) and kRoundConstants1600 (:34-43).
//
// Layout: the 25 64-bit lanes (index x + 5y, keccak.hpp:36-38) live in 50
// 32-bit registers as (lo, hi) halves.  All lane indices are compile-time, so
// the state never touches local memory.  Per round:
//   theta parity   20 LOP3 (xor3, LUT 0x96)
//   theta rotl 1   10 SHF   (or 15 IMAD-class ops with kFmaTheta)
//   theta apply    50 LOP3 (a ^ C[x-1] ^ rotl(C[x+1],1) in one xor3)
//   rho            48 SHF   (pi is register renaming; or IMAD-class, see below)
//   chi            50 LOP3 (LUT 0xD2 = a ^ (~b & c))
//   iota           <=2 LOP3
// = 122 LOP3 + 58 SHF on the ALU pipe, the 4320-instruction contract figure of
// SURVEY.md section 8(d).
//
// FMA-pipe offload (template mask FMA_MASK): on sm_100 LOP3/SHF issue on the
// 16-lane/SMSP ALU pipe while IMAD issues on the FMA pipe, which a pure
// LOP3/SHF kernel leaves idle.  A 64-bit rotate by r (0<r<32, after swapping
// halves for r>32) can be done with three multiplies by 2^r:
//   c0       = hi32(hi * 2^r)      (IMAD.HI: hi >> (32-r))
//   c1       = lo32(hi * 2^r)      (IMAD:    hi << r)
//   out      = lo * 2^r + {c1:c0}  (IMAD.WIDE: {lo>>(32-r) + hi<<r : lo<<r + hi>>(32-r)})
// The additions never carry because the summands occupy disjoint bits.  The
// multipliers are read from __constant__ memory so ptxas cannot strength-reduce
// them back into SHF.  Bit i of FMA_MASK moves the rho rotation of source lane
// i to the FMA pipe; bit 25 moves the five theta rotl-by-1; bits 28..29 pick
// the multiply flavour (see rotl64).
#pragma once
#include <cstdint>

namespace b200sha3 {

// 2^r multipliers for the FMA-pipe rotations (index r = 0..31).
static __constant__ uint32_t kPow2[32] = {
    1u << 0,  1u << 1,  1u << 2,  1u << 3,  1u << 4,  1u << 5,  1u << 6,  1u << 7,
    1u << 8,  1u << 9,  1u << 10, 1u << 11, 1u << 12, 1u << 13, 1u << 14, 1u << 15,
    1u << 16, 1u << 17, 1u << 18, 1u << 19, 1u << 20, 1u << 21, 1u << 22, 1u << 23,
    1u << 24, 1u << 25, 1u << 26, 1u << 27, 1u << 28, 1u << 29, 1u << 30, 1u << 31};

// iota constants as (lo, hi) pairs for the rolled loop (keccak.cpp:34-43).
static __constant__ uint32_t kRoundConst32[48] = {
    0x00000001u, 0x00000000u, 0x00008082u, 0x00000000u, 0x0000808au, 0x80000000u,
    0x80008000u, 0x80000000u, 0x0000808bu, 0x00000000u, 0x80000001u, 0x00000000u,
    0x80008081u, 0x80000000u, 0x00008009u, 0x80000000u, 0x0000008au, 0x00000000u,
    0x00000088u, 0x00000000u, 0x80008009u, 0x00000000u, 0x8000000au, 0x00000000u,
    0x8000808bu, 0x00000000u, 0x0000008bu, 0x80000000u, 0x00008089u, 0x80000000u,
    0x00008003u, 0x80000000u, 0x00008002u, 0x80000000u, 0x00000080u, 0x80000000u,
    0x0000800au, 0x00000000u, 0x8000000au, 0x80000000u, 0x80008081u, 0x80000000u,
    0x00008080u, 0x80000000u, 0x80000001u, 0x00000000u, 0x80008008u, 0x80000000u};

// Same constants as compile-time immediates for the fully unrolled form.
__host__ __device__ constexpr uint64_t round_constant(int i) {
  constexpr uint64_t rc[24] = {
      0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808aull,
      0x8000000080008000ull, 0x000000000000808bull, 0x0000000080000001ull,
      0x8000000080008081ull, 0x8000000000008009ull, 0x000000000000008aull,
      0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000aull,
      0x000000008000808bull, 0x800000000000008bull, 0x8000000000008089ull,
      0x8000000000008003ull, 0x8000000000008002ull, 0x8000000000000080ull,
      0x000000000000800aull, 0x800000008000000aull, 0x8000000080008081ull,
      0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};
  return rc[i];
}

struct State {
  uint32_t lo[25];
  uint32_t hi[25];
};

__device__ __forceinline__ void state_zero(State& a) {
#pragma unroll
  for (int i = 0; i < 25; ++i) {
    a.lo[i] = 0u;
    a.hi[i] = 0u;
  }
}

__device__ __forceinline__ uint32_t xor3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// a ^ (~b & c)
__device__ __forceinline__ uint32_t chi3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xD2;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// 64-bit rotate-left of (lo, hi) by the compile-time amount R.
// IMPL 0: two SHF funnel shifts (ALU pipe).
// IMPL 1..2: multiplies by 2^S on the FMA pipe (S = R mod 32 after swapping the
// halves for R > 32); with s = 32 - S:
//   out.lo = (l << S) + (h >> s),  out.hi = (h << S) + (l >> s)   (no carries)
//   1: W = h * m (wide);  {out.hi:out.lo} = l * m + {W.lo:W.hi}   (ptxas splits
//      the swapped 64-bit add into IMAD.WIDE + IMAD + IADD3)
//   2: out.lo = l * m + hi32(h * m);  out.hi = h * m + hi32(l * m)
//      (2 IMAD.HI + 2 IMAD, no ALU op)
// (A third flavour that produced the two halves of h * m separately, straight
// into the accumulator pair, made ptxas insert two MOVs per rotation; dropped.)
template <int R, int IMPL>
__device__ __forceinline__ void rotl64(uint32_t lo, uint32_t hi, uint32_t& olo,
                                       uint32_t& ohi) {
  static_assert(R >= 0 && R < 64, "rotation out of range");
  if constexpr (R == 0) {
    olo = lo;
    ohi = hi;
  } else if constexpr (R == 32) {
    olo = hi;
    ohi = lo;
  } else {
    const uint32_t l = (R < 32) ? lo : hi;
    const uint32_t h = (R < 32) ? hi : lo;
    constexpr int S = (R < 32) ? R : R - 32;
    if constexpr (IMPL == 0) {
      olo = __funnelshift_l(h, l, S);
      ohi = __funnelshift_l(l, h, S);
    } else if constexpr (IMPL == 2) {
      const uint32_t m = kPow2[S];
      uint32_t t0, t1;
      asm("mul.hi.u32 %0, %1, %2;" : "=r"(t0) : "r"(h), "r"(m));
      asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(olo) : "r"(l), "r"(m), "r"(t0));
      asm("mul.hi.u32 %0, %1, %2;" : "=r"(t1) : "r"(l), "r"(m));
      asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(ohi) : "r"(h), "r"(m), "r"(t1));
    } else {
      const uint32_t m = kPow2[S];
      asm("{\n\t"
          ".reg .b32 c0, c1;\n\t"
          ".reg .b64 c, w;\n\t"
          "mul.hi.u32 c0, %3, %4;\n\t"
          "mul.lo.u32 c1, %3, %4;\n\t"
          "mov.b64 c, {c0, c1};\n\t"
          "mad.wide.u32 w, %2, %4, c;\n\t"
          "mov.b64 {%0, %1}, w;\n\t"
          "}"
          : "=r"(olo), "=r"(ohi)
          : "r"(l), "r"(h), "r"(m));
    }
  }
}

#define B200SHA3_RHOPI(SRC, ROT, DST)                                              \
  rotl64<ROT, ((FMA_MASK >> (SRC)) & 1u) ? kImpl : 0>(a.lo[SRC], a.hi[SRC],       \
                                                      b.lo[DST], b.hi[DST])

// One round.  rho offsets and the pi source map follow keccak.cpp:26-32 and
// :261-267: b[x+5y] = rotl(a[src], rho[src]) with src = (x+3y)%5 + 5x.
template <uint32_t FMA_MASK>
__device__ __forceinline__ void keccak_round(State& a, uint32_t rc_lo, uint32_t rc_hi) {
  // bits 28..29 of the mask pick the FMA rotate flavour (0 -> flavour 1)
  constexpr int kImpl = ((FMA_MASK >> 28) & 3u) ? static_cast<int>((FMA_MASK >> 28) & 3u) : 1;
  uint32_t clo[5], chi[5];
#pragma unroll
  for (int x = 0; x < 5; ++x) {
    clo[x] = xor3(xor3(a.lo[x], a.lo[x + 5], a.lo[x + 10]), a.lo[x + 15], a.lo[x + 20]);
    chi[x] = xor3(xor3(a.hi[x], a.hi[x + 5], a.hi[x + 10]), a.hi[x + 15], a.hi[x + 20]);
  }
#pragma unroll
  for (int x = 0; x < 5; ++x) {
    uint32_t rl, rh;
    rotl64<1, ((FMA_MASK >> 25) & 1u) ? kImpl : 0>(clo[(x + 1) % 5], chi[(x + 1) % 5], rl, rh);
    const uint32_t pl = clo[(x + 4) % 5], ph = chi[(x + 4) % 5];
#pragma unroll
    for (int y = 0; y < 25; y += 5) {
      a.lo[x + y] = xor3(a.lo[x + y], pl, rl);
      a.hi[x + y] = xor3(a.hi[x + y], ph, rh);
    }
  }
  State b;
  B200SHA3_RHOPI(0, 0, 0);
  B200SHA3_RHOPI(6, 44, 1);
  B200SHA3_RHOPI(12, 43, 2);
  B200SHA3_RHOPI(18, 21, 3);
  B200SHA3_RHOPI(24, 14, 4);
  B200SHA3_RHOPI(3, 28, 5);
  B200SHA3_RHOPI(9, 20, 6);
  B200SHA3_RHOPI(10, 3, 7);
  B200SHA3_RHOPI(16, 45, 8);
  B200SHA3_RHOPI(22, 61, 9);
  B200SHA3_RHOPI(1, 1, 10);
  B200SHA3_RHOPI(7, 6, 11);
  B200SHA3_RHOPI(13, 25, 12);
  B200SHA3_RHOPI(19, 8, 13);
  B200SHA3_RHOPI(20, 18, 14);
  B200SHA3_RHOPI(4, 27, 15);
  B200SHA3_RHOPI(5, 36, 16);
  B200SHA3_RHOPI(11, 10, 17);
  B200SHA3_RHOPI(17, 15, 18);
  B200SHA3_RHOPI(23, 56, 19);
  B200SHA3_RHOPI(2, 62, 20);
  B200SHA3_RHOPI(8, 55, 21);
  B200SHA3_RHOPI(14, 39, 22);
  B200SHA3_RHOPI(15, 41, 23);
  B200SHA3_RHOPI(21, 2, 24);
#pragma unroll
  for (int y = 0; y < 25; y += 5) {
#pragma unroll
    for (int x = 0; x < 5; ++x) {
      a.lo[x + y] = chi3(b.lo[x + y], b.lo[(x + 1) % 5 + y], b.lo[(x + 2) % 5 + y]);
      a.hi[x + y] = chi3(b.hi[x + y], b.hi[(x + 1) % 5 + y], b.hi[(x + 2) % 5 + y]);
    }
  }
  a.lo[0] ^= rc_lo;
  a.hi[0] ^= rc_hi;
}

#undef B200SHA3_RHOPI

// HEAD straight-line rounds, ITERS iterations of BODY rounds, then the remaining rounds
// straight-line.  The straight-line head and tail let ptxas drop the work on lanes that are
// known zero on entry and on lanes nobody reads on exit, exactly as in the fully unrolled
// form, while the loop keeps the code inside the instruction cache.
template <int HEAD, int BODY, int ITERS, uint32_t FMA_MASK>
__device__ __forceinline__ void keccak_f1600_peeled(State& a) {
  constexpr int kTailStart = HEAD + BODY * ITERS;
  static_assert(kTailStart <= 24, "too many rounds");
#pragma unroll
  for (int r = 0; r < HEAD; ++r) {
    keccak_round<FMA_MASK>(a, static_cast<uint32_t>(round_constant(r)),
                           static_cast<uint32_t>(round_constant(r) >> 32));
  }
#pragma unroll 1
  for (int r = HEAD; r < kTailStart; r += BODY) {
#pragma unroll
    for (int u = 0; u < BODY; ++u) {
      keccak_round<FMA_MASK>(a, kRoundConst32[2 * (r + u)], kRoundConst32[2 * (r + u) + 1]);
    }
  }
#pragma unroll
  for (int r = kTailStart; r < 24; ++r) {
    keccak_round<FMA_MASK>(a, static_cast<uint32_t>(round_constant(r)),
                           static_cast<uint32_t>(round_constant(r) >> 32));
  }
}

// 24 rounds.
//   UNROLL = 24  straight-line code with immediates; ptxas also drops the work on lanes
//                that are known zero on entry and on lanes nobody reads on exit.
//   UNROLL = 22  "peeled": rounds 0 and 23 straight-line (so the same dead-work removal
//                applies to them), rounds 1..22 in a loop of two rounds per body that
//                stays I-cache resident (the 67 KB fully unrolled body does not).
//   UNROLL = 21, 20, 23, 11  peeled forms (see keccak_f1600_peeled): head + iterations x
//                body + tail = 1 + 3x7 + 2, 1 + 4x5 + 3, 1 + 7x3 + 2, 1 + 2x11 + 1.
//   UNROLL = 1, 2, 4  plain loop, constants from the constant bank.
template <int UNROLL, uint32_t FMA_MASK>
__device__ __forceinline__ void keccak_f1600(State& a) {
  if constexpr (UNROLL == 24) {
#pragma unroll
    for (int r = 0; r < 24; ++r) {
      keccak_round<FMA_MASK>(a, static_cast<uint32_t>(round_constant(r)),
                             static_cast<uint32_t>(round_constant(r) >> 32));
    }
  } else if constexpr (UNROLL == 22) {
    keccak_f1600_peeled<1, 2, 11, FMA_MASK>(a);  // 1 + 11 x 2 + 1, ~10 KB
  } else if constexpr (UNROLL == 21) {
    keccak_f1600_peeled<1, 7, 3, FMA_MASK>(a);   // 1 + 3 x 7 + 2, ~29 KB of code
  } else if constexpr (UNROLL == 20) {
    keccak_f1600_peeled<1, 5, 4, FMA_MASK>(a);   // 1 + 4 x 5 + 3, ~26 KB
  } else if constexpr (UNROLL == 23) {
    keccak_f1600_peeled<1, 3, 7, FMA_MASK>(a);   // 1 + 7 x 3 + 2, ~17 KB
  } else if constexpr (UNROLL == 11) {
    keccak_f1600_peeled<1, 11, 2, FMA_MASK>(a);  // 1 + 2 x 11 + 1, ~37 KB
  } else {
    static_assert(24 % UNROLL == 0, "UNROLL must divide 24");
#pragma unroll 1
    for (int r = 0; r < 24; r += UNROLL) {
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        keccak_round<FMA_MASK>(a, kRoundConst32[2 * (r + u)], kRoundConst32[2 * (r + u) + 1]);
      }
    }
  }
}

}  // namespace b200sha3
