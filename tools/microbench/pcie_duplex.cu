// pcie_duplex.cu -- what the host link can do for the e2e shape of bench.py (2 bytes in for
// every byte out): plain copies with no hashing at all.  The e2e figure of the bench line is
// read against the "duplex" row of this probe, not against a one-way copy.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pcie_duplex pcie_duplex.cu
//   ./pcie_duplex [GiB in (default 4)] [chunk MiB (default 64)]
//
// Rows (JSON on stdout):
//   h2d_pinned      one cudaMemcpyAsync of the input from cudaHostAlloc(Default) memory
//   h2d_wc          the same from cudaHostAllocWriteCombined memory
//   d2h_pinned      one copy of the output (half the input size) to pinned memory
//   duplex_whole    both at once on two streams, whole buffers
//   duplex_chunked  both at once, cut into chunks on two streams (the shape of the pipeline)
//   duplex_wc       duplex_chunked with the input in write-combined memory
//   zero_copy_read  a kernel reading the mapped input with 16-byte loads (no copy engine)
//   zero_copy_write / duplex_h2d_copy_with_zero_copy_write
//                   a kernel storing the output straight into mapped host memory, alone and
//                   while the copy engine brings the input in
// The *_gbs figures of the duplex rows are bytes over the time of the WHOLE row (both copies).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CU(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void read_kernel(const uint4* __restrict__ src, size_t n, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * size_t{blockDim.x} + threadIdx.x; i < n; i += size_t{gridDim.x} * blockDim.x) {
    const uint4 v = src[i];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) *sink = acc;
}

__global__ void write_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * size_t{blockDim.x} + threadIdx.x; i < n; i += size_t{gridDim.x} * blockDim.x) dst[i] = src[i];
}

template <class F>
static double best_of(int reps, F&& f) {
  double best = 1e30;
  for (int r = 0; r < reps; ++r) {
    CU(cudaDeviceSynchronize());
    const double t0 = now();
    f();
    CU(cudaDeviceSynchronize());
    best = std::min(best, now() - t0);
  }
  return best;
}

int main(int argc, char** argv) {
  const size_t gib_in = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 4;
  const size_t chunk_in = (argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 64) << 20;
  const size_t in_bytes = gib_in << 30, out_bytes = in_bytes / 2, chunk_out = chunk_in / 2;
  uint8_t *h_in, *h_wc, *h_out, *d_in, *d_out;
  CU(cudaHostAlloc(reinterpret_cast<void**>(&h_in), in_bytes, cudaHostAllocDefault));
  CU(cudaHostAlloc(reinterpret_cast<void**>(&h_wc), in_bytes, cudaHostAllocWriteCombined | cudaHostAllocMapped));
  CU(cudaHostAlloc(reinterpret_cast<void**>(&h_out), out_bytes, cudaHostAllocMapped));
  CU(cudaMalloc(reinterpret_cast<void**>(&d_in), in_bytes));
  CU(cudaMalloc(reinterpret_cast<void**>(&d_out), out_bytes));
  std::memset(h_in, 1, in_bytes);
  std::memset(h_wc, 2, in_bytes);
  std::memset(h_out, 3, out_bytes);
  CU(cudaMemset(d_out, 4, out_bytes));
  cudaStream_t s_in, s_out;
  CU(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));

  auto duplex_chunked = [&](const uint8_t* src) {
    for (size_t off = 0; off < in_bytes; off += chunk_in) {
      CU(cudaMemcpyAsync(d_in + off, src + off, std::min(chunk_in, in_bytes - off), cudaMemcpyHostToDevice, s_in));
      const size_t oo = off / 2;
      CU(cudaMemcpyAsync(h_out + oo, d_out + oo, std::min(chunk_out, out_bytes - oo), cudaMemcpyDeviceToHost, s_out));
    }
  };
  const int reps = 4;
  const double h2d = best_of(reps, [&] { CU(cudaMemcpyAsync(d_in, h_in, in_bytes, cudaMemcpyHostToDevice, s_in)); });
  const double h2d_wc = best_of(reps, [&] { CU(cudaMemcpyAsync(d_in, h_wc, in_bytes, cudaMemcpyHostToDevice, s_in)); });
  const double d2h = best_of(reps, [&] { CU(cudaMemcpyAsync(h_out, d_out, out_bytes, cudaMemcpyDeviceToHost, s_out)); });
  const double dup_whole = best_of(reps, [&] {
    CU(cudaMemcpyAsync(d_in, h_in, in_bytes, cudaMemcpyHostToDevice, s_in));
    CU(cudaMemcpyAsync(h_out, d_out, out_bytes, cudaMemcpyDeviceToHost, s_out));
  });
  const double dup_chunk = best_of(reps, [&] { duplex_chunked(h_in); });
  const double dup_wc = best_of(reps, [&] { duplex_chunked(h_wc); });
  uint4* sink;
  CU(cudaMalloc(reinterpret_cast<void**>(&sink), 16));
  uint8_t* mapped;
  CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&mapped), h_wc, 0));
  const double zc = best_of(reps, [&] {
    read_kernel<<<148 * 8, 256, 0, s_in>>>(reinterpret_cast<const uint4*>(mapped), in_bytes / 16, sink);
  });
  CU(cudaGetLastError());
  // the output written by a kernel straight into mapped host memory (posted writes, no copy
  // engine) while the copy engine brings the input in; and alone.  Few blocks: a hash kernel
  // would produce its digests at a trickle, not in one burst.
  uint8_t* mapped_out;
  CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&mapped_out), h_out, 0));
  const double zc_write = best_of(reps, [&] {
    write_kernel<<<148, 256, 0, s_out>>>(reinterpret_cast<uint4*>(mapped_out), reinterpret_cast<const uint4*>(d_out), out_bytes / 16);
  });
  const double dup_zc_write = best_of(reps, [&] {
    CU(cudaMemcpyAsync(d_in, h_in, in_bytes, cudaMemcpyHostToDevice, s_in));
    write_kernel<<<148, 256, 0, s_out>>>(reinterpret_cast<uint4*>(mapped_out), reinterpret_cast<const uint4*>(d_out), out_bytes / 16);
  });
  // H2D alone while NOTHING goes the other way but with the D2H done afterwards (serial)
  const double serial = best_of(reps, [&] {
    CU(cudaMemcpyAsync(d_in, h_in, in_bytes, cudaMemcpyHostToDevice, s_in));
    CU(cudaStreamSynchronize(s_in));
    CU(cudaMemcpyAsync(h_out, d_out, out_bytes, cudaMemcpyDeviceToHost, s_out));
  });
  CU(cudaGetLastError());
  auto gbs = [](size_t bytes, double s) { return bytes / s / 1e9; };
  std::printf(
      "{\"in_gib\": %zu, \"chunk_mib\": %zu, \"h2d_pinned_gbs\": %.2f, \"h2d_wc_gbs\": %.2f, \"d2h_pinned_gbs\": %.2f, "
      "\"duplex_whole\": {\"seconds\": %.4f, \"h2d_gbs\": %.2f, \"d2h_gbs\": %.2f}, "
      "\"duplex_chunked\": {\"seconds\": %.4f, \"h2d_gbs\": %.2f, \"d2h_gbs\": %.2f}, "
      "\"duplex_wc\": {\"seconds\": %.4f, \"h2d_gbs\": %.2f, \"d2h_gbs\": %.2f}, "
      "\"zero_copy_read_gbs\": %.2f, \"zero_copy_write_gbs\": %.2f, "
      "\"duplex_h2d_copy_with_zero_copy_write\": {\"seconds\": %.4f, \"h2d_gbs\": %.2f}, \"serial_h2d_then_d2h_seconds\": %.4f}\n",
      gib_in, chunk_in >> 20, gbs(in_bytes, h2d), gbs(in_bytes, h2d_wc), gbs(out_bytes, d2h), dup_whole,
      gbs(in_bytes, dup_whole), gbs(out_bytes, dup_whole), dup_chunk, gbs(in_bytes, dup_chunk),
      gbs(out_bytes, dup_chunk), dup_wc, gbs(in_bytes, dup_wc), gbs(out_bytes, dup_wc), gbs(in_bytes, zc), gbs(out_bytes, zc_write), dup_zc_write,
      gbs(in_bytes, dup_zc_write), serial);
  return 0;
}
