// probe.cu -- issue-rate microbenchmarks for the integer pipes of one B200.
//
// SURVEY.md section 8(d) derives the roofline of this path from an assumption:
// LOP3 and SHF share a 16-lane/SMSP ALU pipe (64 thread-instructions per clock
// per SM), and IMAD runs on the separate FMA pipe.  These kernels measure both
// on the box the benchmark runs on, so that `roofline.peak` in bench.py is a
// measured number rather than a datasheet one.
//
// Each thread runs kChains independent dependency chains per instruction type,
// kUnroll steps per loop iteration, so the pipes (4-cycle latency) stay full
// with 16 resident warps per SMSP.
#include <cstdio>

#include "kernels.cuh"

namespace b200sha3 {

namespace {

constexpr int kIters = 512;
constexpr int kUnroll = 8;

__device__ __forceinline__ uint64_t global_timer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#define LOP(x, y, z) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(y), "r"(z))
#define SHFW(x, y) asm volatile("shf.l.wrap.b32 %0, %0, %1, 7;" : "+r"(x) : "r"(y))
#define MAD(x, m, y) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(m), "r"(y))
#define MULHI(x, m) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x) : "r"(m))
// One IMAD.WIDE (x * m -> {h:l}) followed by one IMAD (h * m + l -> x): both on
// the FMA pipe, both halves of the wide product consumed, chain through x.
#define MADWIDE(w, x, m)                                                        \
  asm volatile("{\n\t.reg .b32 l, h;\n\t.reg .b64 t;\n\t"                       \
               "mul.wide.u32 t, %0, %1;\n\tmov.b64 {l, h}, t;\n\t"              \
               "mad.lo.u32 %0, h, %1, l;\n\t}"                                  \
               : "+r"(x)                                                        \
               : "r"(m))

// Returns through out[]: per block {clock64 delta, globaltimer delta}.
template <int MIX>
__global__ void __launch_bounds__(256) probe_kernel(uint32_t seed, uint32_t mult,
                                                    uint32_t* sink, uint64_t* timing) {
  uint32_t a0 = seed + threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
  uint32_t b0 = a0 ^ 0x1234u, b1 = a1 ^ 0x77u, b2 = a2 ^ 0x99u, b3 = a3 ^ 0x4321u;
  uint32_t c0 = a0 + 11u, c1 = a1 + 13u, c2 = a2 + 17u, c3 = a3 + 19u;
  uint64_t w0 = a0, w1 = a1, w2 = a2, w3 = a3;
  uint32_t pool[12] = {a0, a1, a2, a3, b0, b1, b2, b3, c0, c1, c2, c3};
  const uint32_t y = seed * 0x9e3779b9u + 1u, z = ~seed;
  const uint32_t m = mult;  // runtime value (a power of two), opaque to ptxas
  const long long t0 = clock64();
  const uint64_t g0 = global_timer_ns();
#pragma unroll 1
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if constexpr (MIX == 0) {  // 8 LOP3
        LOP(a0, y, z); LOP(a1, y, z); LOP(a2, y, z); LOP(a3, y, z);
        LOP(b0, y, z); LOP(b1, y, z); LOP(b2, y, z); LOP(b3, y, z);
      } else if constexpr (MIX == 1) {  // 8 SHF
        SHFW(a0, y); SHFW(a1, y); SHFW(a2, y); SHFW(a3, y);
        SHFW(b0, y); SHFW(b1, y); SHFW(b2, y); SHFW(b3, y);
      } else if constexpr (MIX == 2) {  // 8 LOP3 + 4 SHF
        LOP(a0, y, z); LOP(a1, y, z); SHFW(c0, y); LOP(a2, y, z); LOP(a3, y, z); SHFW(c1, y);
        LOP(b0, y, z); LOP(b1, y, z); SHFW(c2, y); LOP(b2, y, z); LOP(b3, y, z); SHFW(c3, y);
      } else if constexpr (MIX == 3) {  // 8 IMAD
        MAD(a0, m, y); MAD(a1, m, y); MAD(a2, m, y); MAD(a3, m, y);
        MAD(b0, m, y); MAD(b1, m, y); MAD(b2, m, y); MAD(b3, m, y);
      } else if constexpr (MIX == 4) {  // 8 x (IMAD.WIDE + IMAD)
        MADWIDE(w0, a0, m); MADWIDE(w1, a1, m); MADWIDE(w2, a2, m); MADWIDE(w3, a3, m);
        MADWIDE(w0, b0, m); MADWIDE(w1, b1, m); MADWIDE(w2, b2, m); MADWIDE(w3, b3, m);
      } else if constexpr (MIX == 5) {  // 8 IMAD.HI
        MULHI(a0, m); MULHI(a1, m); MULHI(a2, m); MULHI(a3, m);
        MULHI(b0, m); MULHI(b1, m); MULHI(b2, m); MULHI(b3, m);
      } else if constexpr (MIX == 6) {  // 4 LOP3 + 4 IMAD
        LOP(a0, y, z); MAD(b0, m, y); LOP(a1, y, z); MAD(b1, m, y);
        LOP(a2, y, z); MAD(b2, m, y); LOP(a3, y, z); MAD(b3, m, y);
      } else if constexpr (MIX == 7) {  // 4 LOP3 + 4 x (IMAD.WIDE + IMAD)
        LOP(a0, y, z); MADWIDE(w0, b0, m); LOP(a1, y, z); MADWIDE(w1, b1, m);
        LOP(a2, y, z); MADWIDE(w2, b2, m); LOP(a3, y, z); MADWIDE(w3, b3, m);
      } else if constexpr (MIX == 8) {  // 4 LOP3 + 4 IMAD.HI
        LOP(a0, y, z); MULHI(b0, m); LOP(a1, y, z); MULHI(b1, m);
        LOP(a2, y, z); MULHI(b2, m); LOP(a3, y, z); MULHI(b3, m);
      } else if constexpr (MIX >= 10) {
        // Realistic operand traffic: a pool of 12 registers, every one rewritten every 12
        // steps; each LOP3 reads three distinct pool registers (like theta / chi do), and
        // the interleaved second instruction reads pool registers too.
        //   10: LOP3 only              11: LOP3 + IMAD(r,c,r) 1:1     12: LOP3 + IMAD(r,c,r) 3:1
        //   13: LOP3 + IMAD(r,c,RZ) 3:1   14: LOP3 + IMAD.HI(r,c,RZ) 3:1   15: LOP3 + SHF 2:1
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;"
                       : "=r"(pool[k])
                       : "r"(pool[(k + 1) % 12]), "r"(pool[(k + 5) % 12]), "r"(pool[(k + 8) % 12]));
          const bool second = (MIX == 11) || (MIX >= 12 && MIX <= 14 && k % 3 == 2) ||
                              (MIX == 15 && k % 2 == 1);
          if (second) {
            const int j = (k + 6) % 12;
            if constexpr (MIX == 11 || MIX == 12) {
              asm volatile("mad.lo.u32 %0, %1, %2, %3;"
                           : "=r"(pool[j]) : "r"(pool[(j + 2) % 12]), "r"(m), "r"(pool[(j + 7) % 12]));
            } else if constexpr (MIX == 13) {
              asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(pool[j]) : "r"(pool[(j + 2) % 12]), "r"(m));
            } else if constexpr (MIX == 14) {
              asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(pool[j]) : "r"(pool[(j + 2) % 12]), "r"(m));
            } else {
              asm volatile("shf.l.wrap.b32 %0, %1, %2, 7;"
                           : "=r"(pool[j]) : "r"(pool[(j + 2) % 12]), "r"(pool[(j + 7) % 12]));
            }
          }
        }
      } else {  // 9: the flavour-2 Keccak mix, 5 LOP3 : 2 IMAD : 2 IMAD.HI (+ 1 SHF per 2)
        LOP(a0, y, z); LOP(a1, y, z); MAD(b0, m, y); MULHI(c0, m); LOP(a2, y, z);
        LOP(a3, y, z); MAD(b1, m, y); MULHI(c1, m); LOP(b2, y, z);
      }
    }
  }
  const uint64_t g1 = global_timer_ns();
  const long long t1 = clock64();
  uint32_t pr = 0;
#pragma unroll
  for (int k = 0; k < 12; ++k) pr ^= pool[k];
  const uint32_t r = pr ^ a0 ^ a1 ^ a2 ^ a3 ^ b0 ^ b1 ^ b2 ^ b3 ^ c0 ^ c1 ^ c2 ^ c3 ^
                     static_cast<uint32_t>(w0 ^ w1 ^ w2 ^ w3) ^
                     static_cast<uint32_t>((w0 ^ w1 ^ w2 ^ w3) >> 32);
  if (r == 0x5a5a5a5au) sink[0] = r;  // keeps the chains alive
  if (threadIdx.x == 0) {
    timing[2 * blockIdx.x] = static_cast<uint64_t>(t1 - t0);
    timing[2 * blockIdx.x + 1] = g1 - g0;
  }
}

// MADWIDE counts as two instructions (IMAD.WIDE + IMAD).
constexpr int kProbeMixes = 16;
constexpr int kInstrPerUnroll[kProbeMixes] = {8, 8, 12, 8, 16, 8, 8, 12, 8, 9, 12, 24, 16, 16, 16, 18};

template <int MIX>
cudaError_t launch_probe(unsigned blocks, uint32_t* sink, uint64_t* timing, cudaStream_t s) {
  probe_kernel<MIX><<<blocks, 256, 0, s>>>(12345u, 1u << 7, sink, timing);
  return cudaGetLastError();
}

cudaError_t launch_mix(int mix, unsigned blocks, uint32_t* sink, uint64_t* timing,
                       cudaStream_t s) {
  switch (mix) {
    case 0: return launch_probe<0>(blocks, sink, timing, s);
    case 1: return launch_probe<1>(blocks, sink, timing, s);
    case 2: return launch_probe<2>(blocks, sink, timing, s);
    case 3: return launch_probe<3>(blocks, sink, timing, s);
    case 4: return launch_probe<4>(blocks, sink, timing, s);
    case 5: return launch_probe<5>(blocks, sink, timing, s);
    case 6: return launch_probe<6>(blocks, sink, timing, s);
    case 7: return launch_probe<7>(blocks, sink, timing, s);
    case 8: return launch_probe<8>(blocks, sink, timing, s);
    case 9: return launch_probe<9>(blocks, sink, timing, s);
    case 10: return launch_probe<10>(blocks, sink, timing, s);
    case 11: return launch_probe<11>(blocks, sink, timing, s);
    case 12: return launch_probe<12>(blocks, sink, timing, s);
    case 13: return launch_probe<13>(blocks, sink, timing, s);
    case 14: return launch_probe<14>(blocks, sink, timing, s);
    case 15: return launch_probe<15>(blocks, sink, timing, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t run_pipe_probe(int mix, double* instr_per_s, double* sm_hz, cudaStream_t stream) {
  if (mix < 0 || mix >= kProbeMixes) return cudaErrorInvalidValue;
  int dev = 0, sms = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (err != cudaSuccess) return err;
  // 8 blocks of 256 threads per SM = 64 resident warps, several waves.
  const unsigned blocks = static_cast<unsigned>(sms) * 8u * 4u;
  uint32_t* sink = nullptr;
  uint64_t* timing = nullptr;
  err = cudaMalloc(&sink, sizeof(uint32_t));
  if (err != cudaSuccess) return err;
  err = cudaMalloc(&timing, sizeof(uint64_t) * 2 * blocks);
  if (err != cudaSuccess) { cudaFree(sink); return err; }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best_ms = 0.f;
  for (int rep = 0; rep < 6 && err == cudaSuccess; ++rep) {  // first two are warm-up
    cudaEventRecord(e0, stream);
    err = launch_mix(mix, blocks, sink, timing, stream);
    cudaEventRecord(e1, stream);
    if (err == cudaSuccess) err = cudaEventSynchronize(e1);
    float ms = 0.f;
    if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, e0, e1);
    if (rep >= 2 && (best_ms == 0.f || ms < best_ms)) best_ms = ms;
  }
  double hz = 0.0;
  if (err == cudaSuccess) {
    uint64_t t[2] = {0, 0};
    err = cudaMemcpy(t, timing, sizeof t, cudaMemcpyDeviceToHost);
    if (err == cudaSuccess && t[1] > 0) hz = static_cast<double>(t[0]) / (1e-9 * t[1]);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(timing);
  cudaFree(sink);
  if (err != cudaSuccess) return err;
  const double instr = static_cast<double>(blocks) * 256.0 * kIters * kUnroll *
                       kInstrPerUnroll[mix];
  if (instr_per_s) *instr_per_s = best_ms > 0.f ? instr / (1e-3 * best_ms) : 0.0;
  if (sm_hz) *sm_hz = hz;
  return cudaSuccess;
}

}  // namespace b200sha3
