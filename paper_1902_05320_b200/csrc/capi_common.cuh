// capi_common.cuh -- shared host-side plumbing of the C ABI translation units
// (capi.cu, capi_host.cu, capi_stream.cu): the variant table, error reporting,
// per-call configuration, device selection and event timing.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdio>

#include "../../include/b200sha3.h"
#include "kernels.cuh"

namespace b200sha3::capi {

// Variant table (proj/core/src/sha3.cpp:13-20): rate lanes, pad head byte
// (suffix | 1 << suffix_bits, proj/core/src/sponge.cpp:122), digest bytes.
struct Variant {
  int rate_lanes;
  uint32_t head;
  uint32_t digest_bytes;  // 0 = XOF
};
constexpr Variant kVariants[6] = {
    {18, 0x06u, 28}, {17, 0x06u, 32}, {13, 0x06u, 48},
    {9, 0x06u, 64},  {21, 0x1fu, 0},  {17, 0x1fu, 0},
};

// Text behind b200sha3_last_cuda_error(), per calling thread (defined in capi.cu).
char* last_error_buffer();
constexpr size_t kLastErrorSize = 256;

inline int cuda_fail(cudaError_t err, const char* what) {
  std::snprintf(last_error_buffer(), kLastErrorSize, "%s: %s (%s)", what, cudaGetErrorName(err),
                cudaGetErrorString(err));
  return B200SHA3_ERR_CUDA;
}

inline void set_error_text(const char* text) {
  std::snprintf(last_error_buffer(), kLastErrorSize, "%s", text);
}

#define CU(call)                                                            \
  do {                                                                      \
    cudaError_t err_ = (call);                                              \
    if (err_ != cudaSuccess) return ::b200sha3::capi::cuda_fail(err_, #call); \
  } while (0)

struct Config {
  int device = -1;
  cudaStream_t stream = nullptr;
  uint32_t flags = 0;
  int kernel = B200SHA3_KERNEL_AUTO;
  int unroll = 0;
  int fma_preset = -1;
  int block_threads = 0;
  double* device_ms = nullptr;
  uint32_t* kernel_launches = nullptr;
};

// Reads only the fields the caller's struct has: struct_size is the sizeof the caller was
// built with (0 = this version), so an older, shorter struct leaves the later knobs at
// their defaults instead of having bytes past its end interpreted.
inline Config resolve(const b200sha3_config* cfg) {
  Config c;
  if (!cfg) return c;
  const size_t have = cfg->struct_size ? cfg->struct_size : sizeof(b200sha3_config);
#define B200SHA3_FIELD(name) (offsetof(b200sha3_config, name) + sizeof(cfg->name) <= have)
  if (B200SHA3_FIELD(device)) c.device = cfg->device;
  if (B200SHA3_FIELD(stream)) c.stream = static_cast<cudaStream_t>(cfg->stream);
  if (B200SHA3_FIELD(flags)) c.flags = cfg->flags;
  if (B200SHA3_FIELD(kernel)) c.kernel = cfg->kernel;
  if (B200SHA3_FIELD(unroll)) c.unroll = cfg->unroll;
  if (B200SHA3_FIELD(fma_preset)) c.fma_preset = cfg->fma_preset;
  if (B200SHA3_FIELD(block_threads)) c.block_threads = cfg->block_threads;
  if (B200SHA3_FIELD(device_ms)) c.device_ms = cfg->device_ms;
  if (B200SHA3_FIELD(kernel_launches)) c.kernel_launches = cfg->kernel_launches;
#undef B200SHA3_FIELD
  return c;
}

// Selects the device for the duration of a call and restores the previous one.
class DeviceGuard {
 public:
  cudaError_t enter(int device) {
    cudaError_t err = cudaGetDevice(&prev_);
    if (err != cudaSuccess) return err;
    if (device >= 0 && device != prev_) {
      err = cudaSetDevice(device);
      if (err != cudaSuccess) return err;
      changed_ = true;
    }
    return cudaSuccess;
  }
  ~DeviceGuard() {
    if (changed_) cudaSetDevice(prev_);
  }

 private:
  int prev_ = 0;
  bool changed_ = false;
};

// CUDA-event timer around the hashing kernels of one call (cfg->device_ms).
class Timer {
 public:
  cudaError_t start(bool enabled, cudaStream_t s) {
    enabled_ = enabled;
    if (!enabled_) return cudaSuccess;
    cudaError_t err = cudaEventCreate(&e0_);
    if (err == cudaSuccess) err = cudaEventCreate(&e1_);
    if (err == cudaSuccess) err = cudaEventRecord(e0_, s);
    return err;
  }
  cudaError_t stop(cudaStream_t s, double* ms_out) {
    if (!enabled_) return cudaSuccess;
    cudaError_t err = cudaEventRecord(e1_, s);
    if (err == cudaSuccess) err = cudaEventSynchronize(e1_);
    float ms = 0.f;
    if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, e0_, e1_);
    if (err == cudaSuccess && ms_out) *ms_out += ms;
    return err;
  }
  ~Timer() {
    if (e0_) cudaEventDestroy(e0_);
    if (e1_) cudaEventDestroy(e1_);
  }

 private:
  bool enabled_ = false;
  cudaEvent_t e0_ = nullptr, e1_ = nullptr;
};

// Stream-ordered scratch memory, returned to the pool when the scope ends -- on the error
// paths too.
class AsyncScratch {
 public:
  cudaError_t alloc(size_t bytes, cudaStream_t stream) {
    stream_ = stream;
    return cudaMallocAsync(&ptr_, bytes, stream);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(ptr_);
  }
  ~AsyncScratch() {
    if (ptr_) cudaFreeAsync(ptr_, stream_);
  }
  AsyncScratch() = default;
  AsyncScratch(const AsyncScratch&) = delete;
  AsyncScratch& operator=(const AsyncScratch&) = delete;

 private:
  void* ptr_ = nullptr;
  cudaStream_t stream_ = nullptr;
};

// Largest batch (messages / streams) KERNEL_AUTO gives to the warp-per-state kernels.
uint64_t warp_kernel_max_count();
inline bool few_enough_for_warps(uint64_t count, const Config& c) {
  return count <= warp_kernel_max_count() && (c.flags & B200SHA3_FLAG_NO_WARP_KERNEL) == 0 &&
         (c.kernel == B200SHA3_KERNEL_AUTO || c.kernel == B200SHA3_KERNEL_WARP);
}

// Keeps stream-ordered allocations cached between calls (once per process).
void tune_mempool_once();

// Validation in the reference's order (batch.cpp:64-75): bad algorithm id, then XOF
// without an output length -- before any work.  Fills *digest_bytes.
int validate(int algorithm, uint64_t xof_bits, uint64_t* digest_bytes);

inline uint32_t last_byte_mask(int algorithm, uint64_t xof_bits) {
  if (kVariants[algorithm].digest_bytes != 0 || xof_bits % 8 == 0) return 0xffu;
  return (1u << (xof_bits % 8)) - 1u;  // batch.cpp:22-24
}

inline bool is_aligned(const void* p, uintptr_t a) {
  return (reinterpret_cast<uintptr_t>(p) % a) == 0;
}

// Equal-length batch already in HBM, on the current device; asynchronous on `stream`.
// `launches` (optional) is incremented per kernel launched.
int run_fixed_device(int algorithm, const uint8_t* d_data, uint64_t msg_len, uint64_t count,
                     uint64_t xof_bits, uint64_t digest_bytes, uint8_t* d_digests,
                     const Config& c, cudaStream_t stream, uint32_t* launches);

// What a caller that has read the offsets / lengths on the HOST (the host-buffer entries)
// knows about a batch; lets run_batch_device pick the kernel without the device-side
// classification / bucketing passes.
struct BatchHints {
  bool aligned8 = false;   // every message starts at a multiple of 8 (relative to `data`)
  bool all_short = false;  // every message is shorter than the rate: single block
  bool all_equal = false;  // all lengths are equal: nothing to bucket, uniform final block
};

// Variable-length batch already in HBM: bucketing pass (unless disabled) + hash kernel per
// slice of at most 2^30 messages; asynchronous on `stream`.  `hints` may be nullptr.
int run_batch_device(int algorithm, const uint8_t* d_data, const uint64_t* d_offsets,
                     const uint64_t* d_lengths, uint64_t count, uint64_t xof_bits,
                     uint64_t digest_bytes, uint8_t* d_digests, const Config& c,
                     cudaStream_t stream, uint32_t* launches, const BatchHints* hints = nullptr);

}  // namespace b200sha3::capi
