// capi.cu -- the C ABI of include/b200sha3.h over the kernels.
//
// Host-side logic of the path: validation in the order the reference applies
// it (proj/core/src/batch.cpp:64-75), kernel selection, the bucketing pass for
// variable-length batches, and the chunked copy/compute pipeline of the
// host-buffer entries.  No CPU hashing code exists in this library: if CUDA
// is unusable every compute entry returns B200SHA3_ERR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/b200sha3.h"
#include "kernels.cuh"

namespace {

using namespace b200sha3;

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

thread_local char g_last_error[256] = "";

int cuda_fail(cudaError_t err, const char* what) {
  std::snprintf(g_last_error, sizeof g_last_error, "%s: %s (%s)", what,
                cudaGetErrorName(err), cudaGetErrorString(err));
  return B200SHA3_ERR_CUDA;
}

#define CU(call)                                          \
  do {                                                    \
    cudaError_t err_ = (call);                            \
    if (err_ != cudaSuccess) return cuda_fail(err_, #call); \
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

Config resolve(const b200sha3_config* cfg) {
  Config c;
  if (!cfg) return c;
  c.device = cfg->device;
  c.stream = static_cast<cudaStream_t>(cfg->stream);
  c.flags = cfg->flags;
  c.kernel = cfg->kernel;
  c.unroll = cfg->unroll;
  c.fma_preset = cfg->fma_preset;
  c.block_threads = cfg->block_threads;
  c.device_ms = cfg->device_ms;
  c.kernel_launches = cfg->kernel_launches;
  return c;
}

// Measured defaults.
constexpr int kDefaultUnrollOneblock = 24;
constexpr int kDefaultFmaOneblock = 0;
constexpr int kDefaultFmaGeneric = 0;

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

// Keep stream-ordered allocations cached between calls.
void tune_mempool_once() {
  static std::once_flag once;
  std::call_once(once, [] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return;
    for (int d = 0; d < n; ++d) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
        uint64_t threshold = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
      }
    }
    cudaGetLastError();
  });
}

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

int validate(int algorithm, uint64_t xof_bits, uint64_t* digest_bytes) {
  if (algorithm < 0 || algorithm > 5) {
    std::snprintf(g_last_error, sizeof g_last_error, "algorithm id %d out of range", algorithm);
    return B200SHA3_ERR_INVALID_ARGUMENT;
  }
  // batch.cpp:66-68 -- rejected before any work.
  if (kVariants[algorithm].digest_bytes == 0 && xof_bits == 0) {
    return B200SHA3_ERR_INVALID_ARGUMENT;
  }
  *digest_bytes = b200sha3_digest_bytes(algorithm, xof_bits);
  return B200SHA3_OK;
}

uint32_t last_byte_mask(int algorithm, uint64_t xof_bits) {
  if (kVariants[algorithm].digest_bytes != 0 || xof_bits % 8 == 0) return 0xffu;
  return (1u << (xof_bits % 8)) - 1u;  // batch.cpp:22-24
}

bool is_aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// Equal-length batch already in HBM, on the current device.  `launches` counts
// kernels.  Asynchronous on `stream`.
int run_fixed_device(int algorithm, const uint8_t* d_data, uint64_t msg_len, uint64_t count,
                     uint64_t xof_bits, uint64_t digest_bytes, uint8_t* d_digests,
                     const Config& c, cudaStream_t stream, uint32_t* launches) {
  const Variant& v = kVariants[algorithm];
  HashArgs args{};
  args.data = d_data;
  args.fixed_len = msg_len;
  args.count = count;
  args.digests = d_digests;
  args.digest_bytes = digest_bytes;
  args.head = v.head;
  args.last_mask = last_byte_mask(algorithm, xof_bits);
  args.aligned8 = (is_aligned(d_data, 8) && (msg_len % 8 == 0 || count <= 1)) ? 1u : 0u;

  LaunchPlan plan{};
  plan.rate_lanes = v.rate_lanes;
  plan.block_threads = c.block_threads;

  const bool fits_oneblock = oneblock_supported(v.rate_lanes, msg_len, digest_bytes) &&
                             is_aligned(d_data, 16) && is_aligned(d_digests, 16);
  int kernel = c.kernel;
  if (kernel == B200SHA3_KERNEL_AUTO) {
    kernel = fits_oneblock ? B200SHA3_KERNEL_ONEBLOCK : B200SHA3_KERNEL_GENERIC;
  }
  cudaError_t err;
  if (kernel == B200SHA3_KERNEL_ONEBLOCK) {
    if (!fits_oneblock) {
      std::snprintf(g_last_error, sizeof g_last_error, "one-block kernel does not fit this batch");
      return B200SHA3_ERR_UNSUPPORTED;
    }
    plan.unroll = c.unroll ? c.unroll : kDefaultUnrollOneblock;
    plan.fma_preset = c.fma_preset >= 0 ? c.fma_preset : kDefaultFmaOneblock;
    args.aligned8 = 1u;
    err = launch_hash_oneblock(args, plan, stream);
  } else if (kernel == B200SHA3_KERNEL_LANESPLIT) {
    if (!lanesplit_supported(v.rate_lanes, msg_len, digest_bytes) || !args.aligned8) {
      std::snprintf(g_last_error, sizeof g_last_error, "lane-split kernel does not fit this batch");
      return B200SHA3_ERR_UNSUPPORTED;
    }
    err = launch_hash_lanesplit(args, plan, stream);
  } else {
    plan.unroll = 2;
    plan.fma_preset = c.fma_preset >= 0 ? c.fma_preset : kDefaultFmaGeneric;
    err = launch_hash_generic(args, plan, stream);
  }
  if (err == cudaErrorNotSupported) {
    cudaGetLastError();
    std::snprintf(g_last_error, sizeof g_last_error, "no kernel instantiation for this selection");
    return B200SHA3_ERR_UNSUPPORTED;
  }
  if (err != cudaSuccess) return cuda_fail(err, "hash kernel launch");
  if (launches) *launches += 1;
  return B200SHA3_OK;
}

// Variable-length batch already in HBM.  Slices of at most 2^30 messages; each
// slice is bucketed by block count (unless disabled) and hashed with one launch.
int run_batch_device(int algorithm, const uint8_t* d_data, const uint64_t* d_offsets,
                     const uint64_t* d_lengths, uint64_t count, uint64_t xof_bits,
                     uint64_t digest_bytes, uint8_t* d_digests, const Config& c,
                     cudaStream_t stream, uint32_t* launches) {
  const Variant& v = kVariants[algorithm];
  tune_mempool_once();
  const uint64_t kSlice = 1ull << 30;
  const bool bucketing = (c.flags & B200SHA3_FLAG_NO_BUCKETING) == 0;
  for (uint64_t first = 0; first < count; first += kSlice) {
    const uint32_t n = static_cast<uint32_t>(std::min<uint64_t>(kSlice, count - first));
    uint32_t* scratch = nullptr;  // [0] unaligned flag, then bucket scratch, then order
    const size_t words = 8 + kBucketScratchWords + (bucketing ? static_cast<size_t>(n) : 0);
    CU(cudaMallocAsync(&scratch, words * sizeof(uint32_t), stream));
    uint32_t* flag = scratch;
    uint32_t* bucket_scratch = scratch + 8;
    uint32_t* order = bucketing ? scratch + 8 + kBucketScratchWords : nullptr;
    CU(cudaMemsetAsync(flag, 0, 8 * sizeof(uint32_t), stream));
    if (bucketing) {
      CU(launch_bucket_order(d_offsets + first, d_lengths + first, n, 8u * v.rate_lanes, order,
                             bucket_scratch, flag, stream));
      if (launches) *launches += 3;
    } else {
      CU(launch_alignment_check(d_offsets + first, n, flag, stream));
      if (launches) *launches += 1;
    }
    HashArgs args{};
    args.data = d_data;
    args.offsets = d_offsets + first;
    args.lengths = d_lengths + first;
    args.count = n;
    args.order = order;
    args.unaligned_flag = is_aligned(d_data, 8) ? flag : nullptr;
    args.aligned8 = 0u;  // used only when the base pointer itself is misaligned
    args.digests = d_digests + first * digest_bytes;
    args.digest_bytes = digest_bytes;
    args.head = v.head;
    args.last_mask = last_byte_mask(algorithm, xof_bits);
    LaunchPlan plan{};
    plan.rate_lanes = v.rate_lanes;
    plan.unroll = 2;
    plan.fma_preset = c.fma_preset >= 0 ? c.fma_preset : kDefaultFmaGeneric;
    plan.block_threads = c.block_threads;
    cudaError_t err = launch_hash_generic(args, plan, stream);
    if (err != cudaSuccess) {
      cudaFreeAsync(scratch, stream);
      return cuda_fail(err, "hash kernel launch");
    }
    if (launches) *launches += 1;
    CU(cudaFreeAsync(scratch, stream));
  }
  return B200SHA3_OK;
}

}  // namespace

extern "C" {

uint64_t b200sha3_digest_bytes(int algorithm, uint64_t xof_output_bits) {
  if (algorithm < 0 || algorithm > 5) return 0;
  const uint32_t fixed = kVariants[algorithm].digest_bytes;
  return fixed ? fixed : (xof_output_bits + 7) / 8;
}

uint32_t b200sha3_rate_bytes(int algorithm) {
  if (algorithm < 0 || algorithm > 5) return 0;
  return 8u * static_cast<uint32_t>(kVariants[algorithm].rate_lanes);
}

uint64_t b200sha3_permutations(int algorithm, uint64_t msg_len, uint64_t xof_output_bits) {
  const uint64_t rate = b200sha3_rate_bytes(algorithm);
  if (rate == 0) return 0;
  const uint64_t out = b200sha3_digest_bytes(algorithm, xof_output_bits);
  return msg_len / rate + 1 + (out > rate ? (out - 1) / rate : 0);
}

const char* b200sha3_strerror(int status) {
  switch (status) {
    case B200SHA3_OK: return "ok";
    case B200SHA3_ERR_INVALID_ARGUMENT: return "invalid argument";
    case B200SHA3_ERR_CUDA: return "CUDA error";
    case B200SHA3_ERR_UNSUPPORTED: return "unsupported batch shape or kernel selection";
    case B200SHA3_ERR_STATE: return "incremental API used out of order";
    default: return "unknown status";
  }
}

const char* b200sha3_last_cuda_error(void) { return g_last_error; }

const char* b200sha3_version(void) { return "b200sha3 0.1 (sm_100a)"; }

int b200sha3_hash_fixed_device(int algorithm, const uint8_t* d_data, uint64_t msg_len,
                               uint64_t count, uint64_t xof_output_bits, uint8_t* d_digests,
                               const b200sha3_config* cfg) {
  uint64_t digest_bytes = 0;
  if (int rc = validate(algorithm, xof_output_bits, &digest_bytes)) return rc;
  const Config c = resolve(cfg);
  if (c.device_ms) *c.device_ms = 0.0;
  if (c.kernel_launches) *c.kernel_launches = 0;
  if (count == 0) return B200SHA3_OK;  // empty batch, empty result (test_batch.cpp:113-117)
  if (!d_digests || (!d_data && msg_len != 0)) return B200SHA3_ERR_INVALID_ARGUMENT;
  DeviceGuard guard;
  CU(guard.enter(c.device));
  Timer timer;
  CU(timer.start(c.device_ms != nullptr, c.stream));
  if (int rc = run_fixed_device(algorithm, d_data, msg_len, count, xof_output_bits, digest_bytes,
                                d_digests, c, c.stream, c.kernel_launches)) {
    return rc;
  }
  CU(timer.stop(c.stream, c.device_ms));
  return B200SHA3_OK;
}

int b200sha3_hash_batch_device(int algorithm, const uint8_t* d_data, const uint64_t* d_offsets,
                               const uint64_t* d_lengths, uint64_t count,
                               uint64_t xof_output_bits, uint8_t* d_digests,
                               const b200sha3_config* cfg) {
  uint64_t digest_bytes = 0;
  if (int rc = validate(algorithm, xof_output_bits, &digest_bytes)) return rc;
  const Config c = resolve(cfg);
  if (c.device_ms) *c.device_ms = 0.0;
  if (c.kernel_launches) *c.kernel_launches = 0;
  if (count == 0) return B200SHA3_OK;
  if (!d_digests || !d_offsets || !d_lengths || !d_data) return B200SHA3_ERR_INVALID_ARGUMENT;
  DeviceGuard guard;
  CU(guard.enter(c.device));
  Timer timer;
  CU(timer.start(c.device_ms != nullptr, c.stream));
  if (int rc = run_batch_device(algorithm, d_data, d_offsets, d_lengths, count, xof_output_bits,
                                digest_bytes, d_digests, c, c.stream, c.kernel_launches)) {
    return rc;
  }
  CU(timer.stop(c.stream, c.device_ms));
  return B200SHA3_OK;
}

// Host entry, equal-length messages: chunks of ~64 MiB of input cycle through
// three slots, each with its own stream, so that (with pinned host memory) the
// H2D copy of chunk k+1, the kernel of chunk k and the D2H copy of chunk k-1
// overlap.
int b200sha3_hash_fixed(int algorithm, const uint8_t* data, uint64_t msg_len, uint64_t count,
                        uint64_t xof_output_bits, uint8_t* digests,
                        const b200sha3_config* cfg) {
  uint64_t digest_bytes = 0;
  if (int rc = validate(algorithm, xof_output_bits, &digest_bytes)) return rc;
  const Config c = resolve(cfg);
  if (c.device_ms) *c.device_ms = 0.0;
  if (c.kernel_launches) *c.kernel_launches = 0;
  if (count == 0) return B200SHA3_OK;
  if (!digests || (!data && msg_len != 0)) return B200SHA3_ERR_INVALID_ARGUMENT;
  DeviceGuard guard;
  CU(guard.enter(c.device));
  tune_mempool_once();
  if (c.stream) CU(cudaStreamSynchronize(c.stream));

  constexpr int kSlots = 3;
  const bool pipeline = (c.flags & B200SHA3_FLAG_NO_PIPELINE) == 0;
  const uint64_t per_msg = std::max<uint64_t>(1, msg_len + digest_bytes);
  uint64_t chunk = pipeline ? std::max<uint64_t>(1, (64ull << 20) / per_msg) : count;
  chunk = std::min(chunk, count);
  // keep every chunk start 16-byte aligned in both buffers
  if (chunk < count) chunk = std::max<uint64_t>(16, chunk & ~15ull);
  const int slots = chunk < count ? kSlots : 1;

  cudaStream_t streams[kSlots] = {};
  uint8_t* d_in[kSlots] = {};
  uint8_t* d_out[kSlots] = {};
  cudaEvent_t ev0[kSlots] = {}, ev1[kSlots] = {};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed;
  int rc = B200SHA3_OK;
  auto fail = [&](cudaError_t e, const char* what) { rc = cuda_fail(e, what); };
  for (int s = 0; s < slots && rc == B200SHA3_OK; ++s) {
    cudaError_t e = cudaStreamCreateWithFlags(&streams[s], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_in[s], std::max<uint64_t>(16, chunk * msg_len), streams[s]);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_out[s], chunk * digest_bytes, streams[s]);
    if (e == cudaSuccess && c.device_ms) {
      e = cudaEventCreate(&ev0[s]);
      if (e == cudaSuccess) e = cudaEventCreate(&ev1[s]);
    }
    if (e != cudaSuccess) fail(e, "pipeline setup");
  }
  double kernel_ms = 0.0;
  uint32_t launches = 0;
  uint64_t done = 0;
  for (uint64_t k = 0; done < count && rc == B200SHA3_OK; ++k) {
    const int s = static_cast<int>(k % slots);
    const uint64_t n = std::min(chunk, count - done);
    cudaError_t e = cudaSuccess;
    if (c.device_ms && k >= static_cast<uint64_t>(slots)) {
      // the slot's previous events are about to be reused: harvest them first
      e = cudaEventSynchronize(ev1[s]);
      float ms = 0.f;
      if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, ev0[s], ev1[s]);
      kernel_ms += ms;
    }
    if (e == cudaSuccess && msg_len)
      e = cudaMemcpyAsync(d_in[s], data + done * msg_len, n * msg_len, cudaMemcpyHostToDevice,
                          streams[s]);
    if (e == cudaSuccess && c.device_ms) e = cudaEventRecord(ev0[s], streams[s]);
    if (e != cudaSuccess) { fail(e, "H2D copy"); break; }
    rc = run_fixed_device(algorithm, d_in[s], msg_len, n, xof_output_bits, digest_bytes, d_out[s],
                          c, streams[s], &launches);
    if (rc != B200SHA3_OK) break;
    if (c.device_ms) e = cudaEventRecord(ev1[s], streams[s]);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(digests + done * digest_bytes, d_out[s], n * digest_bytes,
                          cudaMemcpyDeviceToHost, streams[s]);
    if (e != cudaSuccess) { fail(e, "D2H copy"); break; }
    done += n;
  }
  for (int s = 0; s < slots; ++s) {
    if (!streams[s]) continue;
    cudaError_t e = cudaStreamSynchronize(streams[s]);
    if (e != cudaSuccess && rc == B200SHA3_OK) fail(e, "pipeline drain");
    if (rc == B200SHA3_OK && c.device_ms && ev1[s] &&
        static_cast<uint64_t>(s) < (count + chunk - 1) / chunk) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ev0[s], ev1[s]) == cudaSuccess) kernel_ms += ms;
    }
    if (d_in[s]) cudaFreeAsync(d_in[s], streams[s]);
    if (d_out[s]) cudaFreeAsync(d_out[s], streams[s]);
    cudaStreamSynchronize(streams[s]);
    if (ev0[s]) cudaEventDestroy(ev0[s]);
    if (ev1[s]) cudaEventDestroy(ev1[s]);
    cudaStreamDestroy(streams[s]);
  }
  if (rc != B200SHA3_OK) {
    cudaGetLastError();
    return rc;
  }
  if (c.device_ms) *c.device_ms = kernel_ms;
  if (c.kernel_launches) *c.kernel_launches = launches;
  return B200SHA3_OK;
}

}  // extern "C"

// Host entry, variable-length messages.
//
// Packed batches (offsets non-decreasing, messages not overlapping -- what the C++
// adapter and every sane caller produce) are cut into chunks of ~64 MiB of message bytes
// that cycle through three slots, each with its own stream, so that (with pinned host
// memory) the H2D copy of chunk k+1, the bucketing + hash kernels of chunk k and the D2H
// copy of chunk k-1 overlap.  Anything else takes one copy of the byte range the batch
// touches, one device pass, one copy back.
namespace {

struct HostChunk {
  uint64_t first, count;  // message range
  uint64_t lo, hi;        // byte range of `data` (lo is 16-byte aligned)
};

// Returns false when the batch is not packed in order (caller falls back to one shot).
bool plan_host_chunks(const uint64_t* offsets, const uint64_t* lengths, uint64_t count,
                      uint64_t target_bytes, std::vector<HostChunk>* chunks) {
  uint64_t prev_end = 0;
  HostChunk cur{0, 0, 0, 0};
  for (uint64_t i = 0; i < count; ++i) {
    if (offsets[i] < prev_end) return false;
    const uint64_t end = offsets[i] + lengths[i];
    if (end < offsets[i]) return false;  // overflow
    if (cur.count == 0) {
      cur.first = i;
      cur.lo = offsets[i] & ~15ull;
    }
    cur.count += 1;
    cur.hi = end;
    prev_end = end;
    if (cur.hi - cur.lo >= target_bytes || cur.count >= (1ull << 22)) {
      chunks->push_back(cur);
      cur = HostChunk{0, 0, 0, 0};
    }
  }
  if (cur.count) chunks->push_back(cur);
  return true;
}

int hash_batch_host_single(int algorithm, const uint8_t* data, const uint64_t* offsets,
                           const uint64_t* lengths, uint64_t count, uint64_t xof_output_bits,
                           uint64_t digest_bytes, uint8_t* digests, const Config& c) {
  // Byte range [lo, hi) of `data` that the batch reads.
  uint64_t lo = ~0ull, hi = 0;
  for (uint64_t i = 0; i < count; ++i) {
    if (lengths[i] == 0) continue;
    lo = std::min(lo, offsets[i]);
    hi = std::max(hi, offsets[i] + lengths[i]);
  }
  if (hi == 0) lo = 0;
  if (hi > lo && !data) return B200SHA3_ERR_INVALID_ARGUMENT;
  lo &= ~15ull;  // keep the device copy congruent to the host buffer modulo 16
  cudaStream_t s = nullptr;
  CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  uint8_t* d_data = nullptr;
  uint64_t* d_meta = nullptr;
  uint8_t* d_out = nullptr;
  int rc = B200SHA3_OK;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  uint32_t launches = 0;
  do {
    cudaError_t e = cudaMallocAsync(&d_data, std::max<uint64_t>(16, hi - lo), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_meta, 2 * count * sizeof(uint64_t), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_out, count * digest_bytes, s);
    if (e == cudaSuccess && hi > lo)
      e = cudaMemcpyAsync(d_data, data + lo, hi - lo, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d_meta, offsets, count * sizeof(uint64_t), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d_meta + count, lengths, count * sizeof(uint64_t),
                          cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && c.device_ms) {
      e = cudaEventCreate(&e0);
      if (e == cudaSuccess) e = cudaEventCreate(&e1);
      if (e == cudaSuccess) e = cudaEventRecord(e0, s);
    }
    if (e != cudaSuccess) { rc = cuda_fail(e, "batch upload"); break; }
    // offsets are relative to `data`; the device copy starts at data + lo
    rc = run_batch_device(algorithm, d_data - lo, d_meta, d_meta + count, count, xof_output_bits,
                          digest_bytes, d_out, c, s, &launches);
    if (rc != B200SHA3_OK) break;
    if (c.device_ms) e = cudaEventRecord(e1, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(digests, d_out, count * digest_bytes, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess && c.device_ms) {
      float ms = 0.f;
      e = cudaEventElapsedTime(&ms, e0, e1);
      *c.device_ms = ms;
    }
    if (e != cudaSuccess) rc = cuda_fail(e, "batch download");
  } while (false);
  if (d_data) cudaFreeAsync(d_data, s);
  if (d_meta) cudaFreeAsync(d_meta, s);
  if (d_out) cudaFreeAsync(d_out, s);
  cudaStreamSynchronize(s);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaStreamDestroy(s);
  if (rc != B200SHA3_OK) {
    cudaGetLastError();
    return rc;
  }
  if (c.kernel_launches) *c.kernel_launches = launches;
  return B200SHA3_OK;
}

int hash_batch_host_pipelined(int algorithm, const uint8_t* data, const uint64_t* offsets,
                              const uint64_t* lengths, uint64_t xof_output_bits,
                              uint64_t digest_bytes, uint8_t* digests, const Config& c,
                              const std::vector<HostChunk>& chunks) {
  constexpr int kSlots = 3;
  uint64_t max_span = 16, max_count = 1;
  for (const HostChunk& ch : chunks) {
    max_span = std::max(max_span, ch.hi - ch.lo);
    max_count = std::max(max_count, ch.count);
  }
  const int slots = static_cast<int>(std::min<size_t>(kSlots, chunks.size()));
  cudaStream_t streams[kSlots] = {};
  uint8_t* d_data[kSlots] = {};
  uint64_t* d_meta[kSlots] = {};
  uint8_t* d_out[kSlots] = {};
  cudaEvent_t ev0[kSlots] = {}, ev1[kSlots] = {};
  int rc = B200SHA3_OK;
  for (int s = 0; s < slots && rc == B200SHA3_OK; ++s) {
    cudaError_t e = cudaStreamCreateWithFlags(&streams[s], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_data[s], max_span, streams[s]);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_meta[s], 2 * max_count * sizeof(uint64_t), streams[s]);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_out[s], max_count * digest_bytes, streams[s]);
    if (e == cudaSuccess && c.device_ms) {
      e = cudaEventCreate(&ev0[s]);
      if (e == cudaSuccess) e = cudaEventCreate(&ev1[s]);
    }
    if (e != cudaSuccess) rc = cuda_fail(e, "pipeline setup");
  }
  double kernel_ms = 0.0;
  uint32_t launches = 0;
  for (size_t k = 0; k < chunks.size() && rc == B200SHA3_OK; ++k) {
    const int s = static_cast<int>(k % slots);
    const HostChunk& ch = chunks[k];
    cudaError_t e = cudaSuccess;
    if (c.device_ms && k >= static_cast<size_t>(slots)) {
      e = cudaEventSynchronize(ev1[s]);
      float ms = 0.f;
      if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, ev0[s], ev1[s]);
      kernel_ms += ms;
    }
    if (e == cudaSuccess && ch.hi > ch.lo)
      e = cudaMemcpyAsync(d_data[s], data + ch.lo, ch.hi - ch.lo, cudaMemcpyHostToDevice, streams[s]);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d_meta[s], offsets + ch.first, ch.count * sizeof(uint64_t),
                          cudaMemcpyHostToDevice, streams[s]);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d_meta[s] + max_count, lengths + ch.first, ch.count * sizeof(uint64_t),
                          cudaMemcpyHostToDevice, streams[s]);
    if (e == cudaSuccess && c.device_ms) e = cudaEventRecord(ev0[s], streams[s]);
    if (e != cudaSuccess) { rc = cuda_fail(e, "H2D copy"); break; }
    rc = run_batch_device(algorithm, d_data[s] - ch.lo, d_meta[s], d_meta[s] + max_count, ch.count,
                          xof_output_bits, digest_bytes, d_out[s], c, streams[s], &launches);
    if (rc != B200SHA3_OK) break;
    if (c.device_ms) e = cudaEventRecord(ev1[s], streams[s]);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(digests + ch.first * digest_bytes, d_out[s], ch.count * digest_bytes,
                          cudaMemcpyDeviceToHost, streams[s]);
    if (e != cudaSuccess) { rc = cuda_fail(e, "D2H copy"); break; }
  }
  for (int s = 0; s < slots; ++s) {
    if (!streams[s]) continue;
    cudaError_t e = cudaStreamSynchronize(streams[s]);
    if (e != cudaSuccess && rc == B200SHA3_OK) rc = cuda_fail(e, "pipeline drain");
    if (rc == B200SHA3_OK && c.device_ms && ev1[s]) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ev0[s], ev1[s]) == cudaSuccess) kernel_ms += ms;
    }
    if (d_data[s]) cudaFreeAsync(d_data[s], streams[s]);
    if (d_meta[s]) cudaFreeAsync(d_meta[s], streams[s]);
    if (d_out[s]) cudaFreeAsync(d_out[s], streams[s]);
    cudaStreamSynchronize(streams[s]);
    if (ev0[s]) cudaEventDestroy(ev0[s]);
    if (ev1[s]) cudaEventDestroy(ev1[s]);
    cudaStreamDestroy(streams[s]);
  }
  if (rc != B200SHA3_OK) {
    cudaGetLastError();
    return rc;
  }
  if (c.device_ms) *c.device_ms = kernel_ms;
  if (c.kernel_launches) *c.kernel_launches = launches;
  return B200SHA3_OK;
}

}  // namespace

extern "C" {

int b200sha3_hash_batch(int algorithm, const uint8_t* data, const uint64_t* offsets,
                        const uint64_t* lengths, uint64_t count, uint64_t xof_output_bits,
                        uint8_t* digests, const b200sha3_config* cfg) {
  uint64_t digest_bytes = 0;
  if (int rc = validate(algorithm, xof_output_bits, &digest_bytes)) return rc;
  const Config c = resolve(cfg);
  if (c.device_ms) *c.device_ms = 0.0;
  if (c.kernel_launches) *c.kernel_launches = 0;
  if (count == 0) return B200SHA3_OK;
  if (!digests || !offsets || !lengths) return B200SHA3_ERR_INVALID_ARGUMENT;
  DeviceGuard guard;
  CU(guard.enter(c.device));
  tune_mempool_once();
  if (c.stream) CU(cudaStreamSynchronize(c.stream));
  std::vector<HostChunk> chunks;
  const bool pipeline = (c.flags & B200SHA3_FLAG_NO_PIPELINE) == 0 && data != nullptr &&
                        plan_host_chunks(offsets, lengths, count, 64ull << 20, &chunks) &&
                        chunks.size() > 1;
  if (pipeline) {
    return hash_batch_host_pipelined(algorithm, data, offsets, lengths, xof_output_bits,
                                     digest_bytes, digests, c, chunks);
  }
  return hash_batch_host_single(algorithm, data, offsets, lengths, count, xof_output_bits,
                                digest_bytes, digests, c);
}

// Page-locked host memory for callers that want the copy/compute pipeline at full PCIe
// speed (the C++ adapter packs into it).
int b200sha3_pinned_alloc(uint64_t bytes, void** out) {
  if (!out) return B200SHA3_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (bytes == 0) return B200SHA3_OK;
  CU(cudaHostAlloc(out, bytes, cudaHostAllocPortable));
  return B200SHA3_OK;
}

int b200sha3_pinned_free(void* ptr) {
  if (!ptr) return B200SHA3_OK;
  CU(cudaFreeHost(ptr));
  return B200SHA3_OK;
}

int b200sha3_generate_workload_device(uint64_t seed, uint64_t total_bytes, uint64_t message_size,
                                      uint64_t first_message, uint64_t count, uint8_t* d_out,
                                      const b200sha3_config* cfg) {
  if (message_size == 0 || total_bytes < message_size) return B200SHA3_ERR_INVALID_ARGUMENT;
  if (count == 0) return B200SHA3_OK;
  if (!d_out) return B200SHA3_ERR_INVALID_ARGUMENT;
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(c.device));
  // workload.cpp:34 -- one generator stream per (seed, total) pair
  const uint64_t stream_seed = seed ^ (total_bytes * 0x9e3779b97f4a7c15ull);
  CU(launch_generate_workload(stream_seed, message_size, first_message, count, d_out, c.stream));
  return B200SHA3_OK;
}

int b200sha3_generate_lengths_device(uint64_t seed_len, uint64_t min_len, uint64_t max_len,
                                     uint64_t first_message, uint64_t count, uint64_t* d_lengths,
                                     const b200sha3_config* cfg) {
  if (max_len < min_len) return B200SHA3_ERR_INVALID_ARGUMENT;
  if (count == 0) return B200SHA3_OK;
  if (!d_lengths) return B200SHA3_ERR_INVALID_ARGUMENT;
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(c.device));
  CU(launch_generate_lengths(seed_len, min_len, max_len, first_message, count, d_lengths,
                             c.stream));
  return B200SHA3_OK;
}

int b200sha3_fill_messages_device(uint64_t seed, uint64_t first_message, uint64_t count,
                                  const uint64_t* d_offsets, const uint64_t* d_lengths,
                                  uint8_t* d_data, const b200sha3_config* cfg) {
  if (count == 0) return B200SHA3_OK;
  if (!d_offsets || !d_lengths || !d_data) return B200SHA3_ERR_INVALID_ARGUMENT;
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(c.device));
  CU(launch_fill_messages(seed, first_message, count, d_offsets, d_lengths, d_data, c.stream));
  return B200SHA3_OK;
}

int b200sha3_permute_device(uint64_t* d_states, uint64_t count, const b200sha3_config* cfg) {
  if (count == 0) return B200SHA3_OK;
  if (!d_states) return B200SHA3_ERR_INVALID_ARGUMENT;
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(c.device));
  CU(launch_permute(d_states, count, c.stream));
  return B200SHA3_OK;
}

int b200sha3_bucket_order_device(int algorithm, const uint64_t* d_lengths, uint64_t count,
                                 uint32_t* d_order, const b200sha3_config* cfg) {
  if (algorithm < 0 || algorithm > 5) return B200SHA3_ERR_INVALID_ARGUMENT;
  if (count == 0) return B200SHA3_OK;
  if (count >= (1ull << 32)) return B200SHA3_ERR_UNSUPPORTED;
  if (!d_lengths || !d_order) return B200SHA3_ERR_INVALID_ARGUMENT;
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(c.device));
  tune_mempool_once();
  uint32_t* scratch = nullptr;
  CU(cudaMallocAsync(&scratch, (8 + kBucketScratchWords) * sizeof(uint32_t), c.stream));
  CU(cudaMemsetAsync(scratch, 0, 8 * sizeof(uint32_t), c.stream));
  // lengths double as "offsets" here: only their low bits feed the alignment flag
  CU(launch_bucket_order(d_lengths, d_lengths, static_cast<uint32_t>(count),
                         8u * kVariants[algorithm].rate_lanes, d_order, scratch + 8, scratch,
                         c.stream));
  CU(cudaFreeAsync(scratch, c.stream));
  return B200SHA3_OK;
}

// ---- batched incremental hashing -------------------------------------------------------
}  // extern "C"

struct b200sha3_states {
  int algorithm;
  int device;
  uint64_t count;
  void* lanes;      // 25 * count uint2, structure of arrays
  uint32_t* pos;    // count words
  bool finished;
};

extern "C" {

int b200sha3_states_create(int algorithm, uint64_t count, const b200sha3_config* cfg,
                           b200sha3_states** out) {
  if (!out) return B200SHA3_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (algorithm < 0 || algorithm > 5) return B200SHA3_ERR_INVALID_ARGUMENT;
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(c.device));
  int dev = 0;
  CU(cudaGetDevice(&dev));
  b200sha3_states* st = new (std::nothrow) b200sha3_states{algorithm, dev, count, nullptr, nullptr, false};
  if (!st) return B200SHA3_ERR_CUDA;
  const size_t n = static_cast<size_t>(std::max<uint64_t>(count, 1));
  cudaError_t e = cudaMalloc(&st->lanes, n * 25 * sizeof(uint2));
  if (e == cudaSuccess) e = cudaMalloc(&st->pos, n * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemsetAsync(st->lanes, 0, n * 25 * sizeof(uint2), c.stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(st->pos, 0, n * sizeof(uint32_t), c.stream);
  if (e != cudaSuccess) {
    cudaFree(st->lanes);
    cudaFree(st->pos);
    delete st;
    return cuda_fail(e, "states allocation");
  }
  *out = st;
  return B200SHA3_OK;
}

int b200sha3_states_destroy(b200sha3_states* st) {
  if (!st) return B200SHA3_OK;
  DeviceGuard guard;
  CU(guard.enter(st->device));
  cudaFree(st->lanes);
  cudaFree(st->pos);
  delete st;
  return B200SHA3_OK;
}

int b200sha3_states_reset(b200sha3_states* st, const b200sha3_config* cfg) {
  if (!st) return B200SHA3_ERR_INVALID_ARGUMENT;
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(st->device));
  const size_t n = static_cast<size_t>(std::max<uint64_t>(st->count, 1));
  CU(cudaMemsetAsync(st->lanes, 0, n * 25 * sizeof(uint2), c.stream));
  CU(cudaMemsetAsync(st->pos, 0, n * sizeof(uint32_t), c.stream));
  st->finished = false;
  return B200SHA3_OK;
}

static int states_update(b200sha3_states* st, const uint8_t* d_data, const uint64_t* d_offsets,
                         const uint64_t* d_lengths, uint64_t fixed_len,
                         const b200sha3_config* cfg) {
  if (!st) return B200SHA3_ERR_INVALID_ARGUMENT;
  if (st->finished) return B200SHA3_ERR_STATE;  // sponge.cpp:82-84
  if (st->count == 0) return B200SHA3_OK;
  if (!d_data && (d_lengths || fixed_len)) return B200SHA3_ERR_INVALID_ARGUMENT;
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(st->device));
  CU(launch_states_update(kVariants[st->algorithm].rate_lanes, st->lanes, st->pos, st->count,
                          d_data, d_offsets, d_lengths, fixed_len, c.stream));
  if (c.kernel_launches) *c.kernel_launches = 1;
  return B200SHA3_OK;
}

int b200sha3_states_update_device(b200sha3_states* st, const uint8_t* d_data,
                                  const uint64_t* d_offsets, const uint64_t* d_lengths,
                                  const b200sha3_config* cfg) {
  if (!d_offsets || !d_lengths) return B200SHA3_ERR_INVALID_ARGUMENT;
  return states_update(st, d_data, d_offsets, d_lengths, 0, cfg);
}

int b200sha3_states_update_fixed_device(b200sha3_states* st, const uint8_t* d_data,
                                        uint64_t chunk_len, const b200sha3_config* cfg) {
  return states_update(st, d_data, nullptr, nullptr, chunk_len, cfg);
}

int b200sha3_states_finish_device(b200sha3_states* st, uint64_t xof_output_bits,
                                  uint8_t* d_digests, const b200sha3_config* cfg) {
  if (!st) return B200SHA3_ERR_INVALID_ARGUMENT;
  if (st->finished) return B200SHA3_ERR_STATE;  // sponge.cpp:114-116
  const Variant& v = kVariants[st->algorithm];
  const uint64_t out_len = v.digest_bytes ? v.digest_bytes : (xof_output_bits + 7) / 8;
  if (out_len != 0 && !d_digests && st->count != 0) return B200SHA3_ERR_INVALID_ARGUMENT;
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(st->device));
  CU(launch_states_finish(v.rate_lanes, st->lanes, st->pos, st->count, v.head, d_digests, out_len,
                          last_byte_mask(st->algorithm, xof_output_bits), c.stream));
  st->finished = true;
  if (c.kernel_launches) *c.kernel_launches = st->count ? 1 : 0;
  return B200SHA3_OK;
}

int b200sha3_states_squeeze_device(b200sha3_states* st, uint64_t out_bytes, uint8_t* d_out,
                                   const b200sha3_config* cfg) {
  if (!st) return B200SHA3_ERR_INVALID_ARGUMENT;
  // read() is for XOF variants, after finish() (sha3.cpp:117-126, sponge.cpp:132-134)
  if (!st->finished || kVariants[st->algorithm].digest_bytes != 0) return B200SHA3_ERR_STATE;
  if (out_bytes == 0 || st->count == 0) return B200SHA3_OK;
  if (!d_out) return B200SHA3_ERR_INVALID_ARGUMENT;
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(st->device));
  CU(launch_states_squeeze(kVariants[st->algorithm].rate_lanes, st->lanes, st->pos, st->count,
                           d_out, out_bytes, c.stream));
  if (c.kernel_launches) *c.kernel_launches = 1;
  return B200SHA3_OK;
}

int b200sha3_probe_pipe(int mix, double* instr_per_s, double* sm_hz,
                        const b200sha3_config* cfg) {
  if (mix < 0 || mix > 15) return B200SHA3_ERR_INVALID_ARGUMENT;
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(c.device));
  CU(run_pipe_probe(mix, instr_per_s, sm_hz, c.stream));
  return B200SHA3_OK;
}

}  // extern "C"
