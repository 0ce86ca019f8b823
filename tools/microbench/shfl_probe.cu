// shfl_probe.cu -- what one warp pays for cross-lane exchange on sm_100a: latency of a
// dependent SHFL chain, issue interval of independent SHFLs, and the same for an
// STS + LDS round trip through shared memory.  Cycles per instruction, one warp on one SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o shfl_probe shfl_probe.cu && ./shfl_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void shfl_chain(unsigned* out, long long* cycles, int iters, int src_xor) {
  unsigned v[ILP];
  for (int k = 0; k < ILP; ++k) v[k] = threadIdx.x * 2654435761u + k;
  const int src = threadIdx.x ^ src_xor;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) v[k] = __shfl_sync(0xffffffffu, v[k], src) + 1u;
  }
  long long t1 = clock64();
  unsigned acc = 0;
  for (int k = 0; k < ILP; ++k) acc ^= v[k];
  out[threadIdx.x + blockIdx.x * blockDim.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int ILP>
__global__ void smem_chain(unsigned* out, long long* cycles, int iters, int src_xor) {
  __shared__ unsigned long long buf[ILP][32];
  unsigned long long v[ILP];
  for (int k = 0; k < ILP; ++k) v[k] = threadIdx.x * 2654435761ull + k;
  const int src = threadIdx.x ^ src_xor;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) buf[k][threadIdx.x] = v[k];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < ILP; ++k) v[k] = buf[k][src] + 1ull;
    __syncwarp();
  }
  long long t1 = clock64();
  unsigned long long acc = 0;
  for (int k = 0; k < ILP; ++k) acc ^= v[k];
  out[threadIdx.x] = (unsigned)acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int ILP>
void run(const char* what, bool smem, int warps_per_block) {
  unsigned* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 16);
  cudaMalloc(&cyc, 8 * 256);
  const int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    if (smem) smem_chain<ILP><<<1, 32>>>(out, cyc, iters, 5);
    else shfl_chain<ILP><<<1, 32 * warps_per_block>>>(out, cyc, iters, 5);
  }
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-34s ILP %2d warps %d: %7.2f cycles per %s, %7.2f per group of %d\n", what, ILP, warps_per_block,
         (double)c / iters / ILP, smem ? "STS.64+LDS.64 pair" : "SHFL", (double)c / iters, ILP);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<1>("dependent SHFL chain", false, 1);
  run<2>("2 independent SHFL chains", false, 1);
  run<4>("4 independent SHFL chains", false, 1);
  run<8>("8 independent SHFL chains", false, 1);
  run<16>("16 independent SHFL chains", false, 1);
  run<8>("8 chains, 4 warps (one per SMSP)", false, 4);
  run<8>("8 chains, 8 warps", false, 8);
  run<1>("smem round trip", true, 1);
  run<4>("smem 4 independent", true, 1);
  run<8>("smem 8 independent", true, 1);
  return cudaDeviceSynchronize() != cudaSuccess;
}
