// shfl_alu_mix.cu -- can the shuffle unit carry Keccak's rotations while the ALU pipe does the
// rest?  A z-sliced layout (thread t of a warp holds bits 2t, 2t+1 of every lane for 32 messages)
// turns the 58 SHF of a round into ~52 SHFL with constant offsets and leaves 122 LOP3.  This probe
// runs that instruction mix -- per "round" NL independent LOP3 and NS independent SHFL over 50
// registers -- on every SM at full occupancy and reports SMSP cycles per round, next to the
// LOP3-only and SHFL-only rounds.  122 LOP3 alone need 244 cycles (one ALU instruction per two
// clocks per SMSP); 180 (today's round) need 360.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o shfl_alu_mix shfl_alu_mix.cu && ./shfl_alu_mix
#include <cuda_runtime.h>

#include <cstdio>

template <int NL, int NS>
__global__ void __launch_bounds__(128) mix_kernel(unsigned* out, int rounds, unsigned seed) {
  unsigned r[50];
#pragma unroll
  for (int i = 0; i < 50; ++i) r[i] = seed * (i + 1) + threadIdx.x;
  const unsigned lane = threadIdx.x & 31u;
  // source lanes (t - offset) & 31 for the 24 distinct thread offsets of the rho rotations: computed
  // once, kept in registers (computing them per shuffle would put an ALU instruction back per SHFL)
  unsigned src[24];
#pragma unroll
  for (int i = 0; i < 24; ++i) src[i] = (lane + 32u - (unsigned)(i + 1 + (seed & 1u))) & 31u;
#pragma unroll 1
  for (int it = 0; it < rounds; ++it) {
    // NS shuffles with constant offsets, one per register (round-robin)
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int i = k % 50;
      r[i] = __shfl_sync(0xffffffffu, r[i], src[k % 24]);
    }
    // NL three-input LOP3 over distinct registers
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const int i = k % 50, j = (k + 17) % 50, l = (k + 31) % 50;
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(r[j]), "r"(r[l]));
    }
  }
  unsigned acc = 0;
#pragma unroll
  for (int i = 0; i < 50; ++i) acc ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int NL, int NS>
void run(const char* what) {
  int dev = 0, sms = 0, khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
  const int blocks_per_sm = 4, threads = 128, rounds = 4000;  // 16 warps per SM = 4 per SMSP
  unsigned* out;
  cudaMalloc(&out, sizeof(unsigned) * sms * blocks_per_sm * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix_kernel<NL, NS><<<sms * blocks_per_sm, threads>>>(out, rounds, 3u);
  cudaEventRecord(e0);
  mix_kernel<NL, NS><<<sms * blocks_per_sm, threads>>>(out, rounds, 5u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  // every SMSP runs 4 warps x `rounds` rounds
  const double cycles = ms * 1e-3 * khz * 1e3;
  std::printf("%-28s LOP3 %3d SHFL %3d: %7.1f SMSP cycles per warp-round (%.3f ms at %.0f MHz)\n", what, NL, NS,
              cycles / (4.0 * rounds), ms, khz / 1e3);
  cudaFree(out);
}

int main() {
  run<180, 0>("today's round (ALU only)");
  run<122, 0>("LOP3 part alone");
  run<0, 52>("SHFL part alone");
  run<122, 52>("z-sliced round");
  run<122, 58>("z-sliced round, 58 SHFL");
  run<122, 26>("half the shuffles");
  run<140, 52>("z-sliced + transposes");
  return cudaDeviceSynchronize() != cudaSuccess;
}
