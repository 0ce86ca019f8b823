// capi.cu -- the C ABI of include/b200sha3.h: queries, device-buffer entries, harness
// helpers.  (Host-buffer entries: capi_host.cu; incremental hashing: capi_stream.cu.)
//
// Host-side logic of the path: validation in the order the reference applies it
// (proj/core/src/batch.cpp:64-75), kernel selection, the bucketing pass for
// variable-length batches.  No CPU hashing code exists in this library: if CUDA is
// unusable every compute entry returns B200SHA3_ERR_CUDA.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "capi_common.cuh"

namespace b200sha3::capi {

namespace {
thread_local char g_last_error[kLastErrorSize] = "";

// Measured defaults ("What was tried and what was kept").
constexpr int kDefaultUnrollOneblock = 23;  // peeled 1 + 7x3 + 2 (17 KB): 4.43 vs 4.37 G hash/s for 24
constexpr int kDefaultFmaOneblock = 0;
constexpr int kDefaultFmaGeneric = 0;

}  // namespace

char* last_error_buffer() { return g_last_error; }

// Batches of at most this many messages go to the warp-per-state kernel (kernel_warp.cu) when
// they are multi-block: one warp per message then finishes a permutation in 0.4x the time one
// thread needs, and the machine has warps to spare (592 SMSPs).  Above it the shuffle unit
// saturates and one message per thread is faster again (DESIGN.md section 3.3c,
// tools/long_message_latency.py).  B200SHA3_WARP_KERNEL_MAX overrides it for experiments.
uint64_t warp_kernel_max_count() {
  static const uint64_t value = [] {
    const char* env = std::getenv("B200SHA3_WARP_KERNEL_MAX");
    return env ? std::strtoull(env, nullptr, 10) : 2816ull;
  }();
  return value;
}


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

int validate(int algorithm, uint64_t xof_bits, uint64_t* digest_bytes) {
  if (algorithm < 0 || algorithm > 5) {
    std::snprintf(last_error_buffer(), kLastErrorSize, "algorithm id %d out of range", algorithm);
    return B200SHA3_ERR_INVALID_ARGUMENT;
  }
  // batch.cpp:66-68 -- rejected before any work.
  if (kVariants[algorithm].digest_bytes == 0 && xof_bits == 0) {
    return B200SHA3_ERR_INVALID_ARGUMENT;
  }
  *digest_bytes = b200sha3_digest_bytes(algorithm, xof_bits);
  return B200SHA3_OK;
}

namespace {

// One launch: at most 2^30 equal-length messages.
int run_fixed_slice(int algorithm, const uint8_t* d_data, uint64_t msg_len, uint64_t count,
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

  // The one-block and lane-split kernels write whole words and never see last_mask: an XOF
  // length that is not a whole number of bytes (batch.cpp:22-24) goes to the generic kernel.
  const bool whole_bytes = args.last_mask == 0xffu;
  const bool fits_oneblock = whole_bytes && oneblock_supported(v.rate_lanes, msg_len, digest_bytes) &&
                             is_aligned(d_data, 16) && is_aligned(d_digests, 16);
  // multi-block shapes of cfg2 / cfg3 with a static-shape instantiation (kernel_fewblock.cu)
  const bool aligned16 = is_aligned(d_data, 16) && is_aligned(d_digests, 16);
  const bool fits_static = whole_bytes && aligned16 && fewblock_supported(v.rate_lanes, msg_len, digest_bytes);
  // ... or any other whole number of lanes at or above the rate, through the run-time-length form
  const bool fits_fewblock = fits_static ||
                             (whole_bytes && aligned16 && manyblock_supported(v.rate_lanes, msg_len, digest_bytes));
  // single-block lengths the one-block kernel has no shape for (10, 20, 100 bytes ...)
  const bool fits_short = !fits_oneblock && !fits_fewblock && c.kernel == B200SHA3_KERNEL_AUTO &&
                          msg_len < 8u * static_cast<uint64_t>(v.rate_lanes) &&
                          args.last_mask == 0xffu && short_supported(v.rate_lanes, digest_bytes);
  int kernel = c.kernel;
  if (kernel == B200SHA3_KERNEL_AUTO) {
    kernel = fits_oneblock   ? B200SHA3_KERNEL_ONEBLOCK
             : fits_fewblock ? B200SHA3_KERNEL_FEWBLOCK
                             : B200SHA3_KERNEL_GENERIC;
    // few multi-block messages: latency of the sponge chain is all there is
    if (count <= warp_kernel_max_count() && (c.flags & B200SHA3_FLAG_NO_WARP_KERNEL) == 0 &&
        b200sha3_permutations(algorithm, msg_len, xof_bits) >= 2) {
      kernel = B200SHA3_KERNEL_WARP;
    }
  }
  cudaError_t err;
  if (kernel == B200SHA3_KERNEL_WARP) {
    err = launch_hash_warp(args, plan, stream);
  } else if (kernel == B200SHA3_KERNEL_PAIR) {
    err = launch_hash_pair(args, plan, stream);
  } else if (fits_short) {
    err = launch_hash_short_fixed(args, plan, stream);
  } else if (kernel == B200SHA3_KERNEL_ONEBLOCK) {
    if (!fits_oneblock) {
      set_error_text("one-block kernel does not fit this batch");
      return B200SHA3_ERR_UNSUPPORTED;
    }
    plan.unroll = c.unroll ? c.unroll : kDefaultUnrollOneblock;
    plan.fma_preset = c.fma_preset >= 0 ? c.fma_preset : kDefaultFmaOneblock;
    args.aligned8 = 1u;
    err = launch_hash_oneblock(args, plan, stream);
  } else if (kernel == B200SHA3_KERNEL_FEWBLOCK) {
    if (!fits_fewblock) {
      set_error_text("few-block kernel has no instantiation for this batch");
      return B200SHA3_ERR_UNSUPPORTED;
    }
    args.aligned8 = 1u;
    err = fits_static ? launch_hash_fewblock(args, plan, stream) : launch_hash_manyblock(args, plan, stream);
  } else if (kernel == B200SHA3_KERNEL_LANESPLIT) {
    if (!whole_bytes || !lanesplit_supported(v.rate_lanes, msg_len, digest_bytes) || !args.aligned8) {
      set_error_text("lane-split kernel does not fit this batch");
      return B200SHA3_ERR_UNSUPPORTED;
    }
    err = launch_hash_lanesplit(args, plan, stream);
  } else if (kernel == B200SHA3_KERNEL_STAGED) {
    err = launch_hash_staged(args, plan, stream);
  } else {
    plan.unroll = c.unroll;  // 0 = the kernel's default loop shape
    plan.fma_preset = c.fma_preset >= 0 ? c.fma_preset : kDefaultFmaGeneric;
    err = launch_hash_generic(args, plan, stream);
  }
  if (err == cudaErrorNotSupported) {
    cudaGetLastError();
    set_error_text("no kernel instantiation for this selection");
    return B200SHA3_ERR_UNSUPPORTED;
  }
  if (err != cudaSuccess) return cuda_fail(err, "hash kernel launch");
  if (launches) *launches += 1;
  return B200SHA3_OK;
}

}  // namespace

// Equal-length batch already in HBM, on the current device; one launch per slice of 2^30
// messages (the grid is 32-bit).  `launches` counts kernels.  Asynchronous on `stream`.
int run_fixed_device(int algorithm, const uint8_t* d_data, uint64_t msg_len, uint64_t count,
                     uint64_t xof_bits, uint64_t digest_bytes, uint8_t* d_digests,
                     const Config& c, cudaStream_t stream, uint32_t* launches) {
  constexpr uint64_t kSlice = 1ull << 30;
  for (uint64_t first = 0; first < count; first += kSlice) {
    const uint64_t n = std::min<uint64_t>(kSlice, count - first);
    if (int rc = run_fixed_slice(algorithm, d_data + first * msg_len, msg_len, n, xof_bits,
                                 digest_bytes, d_digests + first * digest_bytes, c, stream, launches)) {
      return rc;
    }
  }
  return B200SHA3_OK;
}

// Variable-length batch already in HBM.  Slices of at most 2^30 messages; each
// slice is bucketed by block count (unless disabled) and hashed with one launch.
int run_batch_device(int algorithm, const uint8_t* d_data, const uint64_t* d_offsets,
                     const uint64_t* d_lengths, uint64_t count, uint64_t xof_bits,
                     uint64_t digest_bytes, uint8_t* d_digests, const Config& c,
                     cudaStream_t stream, uint32_t* launches, const BatchHints* hints) {
  const Variant& v = kVariants[algorithm];
  // Few messages: one warp each, every warp resident at once -- no classification, no order.
  if (c.kernel == B200SHA3_KERNEL_WARP ||
      (c.kernel == B200SHA3_KERNEL_AUTO && count <= warp_kernel_max_count() &&
       (c.flags & B200SHA3_FLAG_NO_WARP_KERNEL) == 0 && !(hints && hints->all_short))) {
    if (count > 0x7fffffffull) {
      set_error_text("warp-per-state kernel: too many messages for one launch");
      return B200SHA3_ERR_UNSUPPORTED;
    }
    HashArgs args{};
    args.data = d_data;
    args.offsets = d_offsets;
    args.lengths = d_lengths;
    args.count = count;
    args.digests = d_digests;
    args.digest_bytes = digest_bytes;
    args.head = v.head;
    args.last_mask = last_byte_mask(algorithm, xof_bits);
    LaunchPlan plan{};
    plan.rate_lanes = v.rate_lanes;
    const cudaError_t err = launch_hash_warp(args, plan, stream);
    if (err != cudaSuccess) return cuda_fail(err, "hash kernel launch");
    if (launches) *launches += 1;
    return B200SHA3_OK;
  }
  tune_mempool_once();
  const uint64_t kSlice = 1ull << 30;
  const bool short_shape = c.kernel == B200SHA3_KERNEL_AUTO && is_aligned(d_data, 8) &&
                           last_byte_mask(algorithm, xof_bits) == 0xffu &&
                           short_supported(v.rate_lanes, digest_bytes);
  // With host knowledge of the batch: all-short aligned batches go straight to the short
  // kernel, equal-length ones straight to the generic kernel -- no classification, no order.
  const bool host_short = hints && hints->all_short && short_shape;
  const bool host_plain = hints && !host_short && hints->all_equal && c.kernel != B200SHA3_KERNEL_STAGED;
  const bool bucketing = (c.flags & B200SHA3_FLAG_NO_BUCKETING) == 0 && !host_short && !host_plain;
  for (uint64_t first = 0; first < count; first += kSlice) {
    const uint32_t n = static_cast<uint32_t>(std::min<uint64_t>(kSlice, count - first));
    // [0] unaligned flag, [1] ragged flag, [2] long flag, then bucket scratch, then order
    const size_t words = 8 + kBucketScratchWords + (bucketing ? static_cast<size_t>(n) : 0);
    AsyncScratch scratch_memory;
    CU(scratch_memory.alloc(words * sizeof(uint32_t), stream));
    uint32_t* scratch = scratch_memory.as<uint32_t>();
    uint32_t* flag = scratch;
    uint32_t* bucket_scratch = scratch + 8;
    uint32_t* order = bucketing ? scratch + 8 + kBucketScratchWords : nullptr;
    // flag words, and right behind them the histogram / cursor words of the bucketing pass
    CU(cudaMemsetAsync(flag, 0, (8 + (bucketing ? kBucketScratchWords : 0)) * sizeof(uint32_t), stream));
    // Batches of single-block messages only have their own kernel body (kernel_short.cu).  Without
    // host knowledge, whether this is one is known on the device only (flag words): the merged
    // kernel of kernel_ragged.cu carries both bodies and branches on the flag.
    const bool try_short = hints ? host_short : short_shape;
    if (host_short) {  // "nothing long" (word 2 stays zero); word 0 says whether the starts are aligned
      if (!hints->aligned8) CU(cudaMemsetAsync(flag, 1, sizeof(uint32_t), stream));
    } else if (host_plain) {
      if (!hints->aligned8) CU(cudaMemsetAsync(flag, 1, sizeof(uint32_t), stream));  // nonzero = unaligned
    } else if (bucketing) {
      CU(launch_bucket_order(d_offsets + first, d_lengths + first, n, 8u * v.rate_lanes, order,
                             bucket_scratch, flag, stream, try_short));
      if (launches) *launches += 2;
    } else {
      CU(launch_alignment_check(d_offsets + first, d_lengths + first, n, 8u * v.rate_lanes, flag, stream));
      if (launches) *launches += 1;
    }
    HashArgs args{};
    args.data = d_data;
    args.offsets = d_offsets + first;
    args.lengths = d_lengths + first;
    args.count = n;
    args.order = order;
    args.unaligned_flag = is_aligned(d_data, 8) ? flag : nullptr;
    args.ragged_flag = flag + 1;
    args.long_flag = flag + 2;
    args.skip_if_short = 0u;
    args.aligned8 = 0u;  // used only when the base pointer itself is misaligned
    args.digests = d_digests + first * digest_bytes;
    args.digest_bytes = digest_bytes;
    args.head = v.head;
    args.last_mask = last_byte_mask(algorithm, xof_bits);
    LaunchPlan plan{};
    plan.rate_lanes = v.rate_lanes;
    plan.unroll = c.unroll;  // 0 = the kernel's default loop shape
    plan.fma_preset = c.fma_preset >= 0 ? c.fma_preset : kDefaultFmaGeneric;
    plan.block_threads = c.block_threads;
    cudaError_t err = cudaSuccess;
    if (try_short && !host_short) {
      // Short or generic, decided by the flag words on the device: one launch with both bodies
      // (kernel_ragged.cu).  Launching both kernels and letting one return at once cost the
      // dispatch of its whole grid -- 70 us for 2^24 messages, side by side or not.
      err = launch_hash_ragged(args, plan, stream);
      if (err == cudaSuccess && launches) *launches += 1;
    } else if (host_short) {
      err = launch_hash_short(args, plan, stream);
      if (err == cudaSuccess && launches) *launches += 1;
    } else {
      err = c.kernel == B200SHA3_KERNEL_STAGED ? launch_hash_staged(args, plan, stream)
            : c.kernel == B200SHA3_KERNEL_PAIR ? launch_hash_pair(args, plan, stream)
                                               : launch_hash_generic(args, plan, stream);
      if (err == cudaSuccess && launches) *launches += 1;
    }
    if (err != cudaSuccess) return cuda_fail(err, "hash kernel launch");
  }
  return B200SHA3_OK;
}

}  // namespace b200sha3::capi

using namespace b200sha3;
using namespace b200sha3::capi;

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

const char* b200sha3_selected_kernel(int algorithm, uint64_t msg_len, uint64_t count,
                                     uint64_t xof_output_bits) {
  if (algorithm < 0 || algorithm > 5) return "";
  const Variant& v = kVariants[algorithm];
  const uint64_t digest_bytes = b200sha3_digest_bytes(algorithm, xof_output_bits);
  const bool whole_bytes = last_byte_mask(algorithm, xof_output_bits) == 0xffu;
  thread_local char name[96];
  const bool few = count <= warp_kernel_max_count();
  if (few && (msg_len == UINT64_MAX || b200sha3_permutations(algorithm, msg_len, xof_output_bits) >= 2)) {
    std::snprintf(name, sizeof name, "hash_warp_kernel");  // run_fixed_slice / run_batch_device
  } else if (msg_len == UINT64_MAX) {  // run_batch_device: classification on the device
    if (whole_bytes && short_supported(v.rate_lanes, digest_bytes)) {
      std::snprintf(name, sizeof name, "bucket_order + hash_ragged_kernel<%d,%d>", v.rate_lanes,
                    static_cast<int>(digest_bytes / 4));
    } else {
      std::snprintf(name, sizeof name, "bucket_order + hash_generic_kernel<%d>", v.rate_lanes);
    }
  } else if (whole_bytes && oneblock_supported(v.rate_lanes, msg_len, digest_bytes)) {  // run_fixed_slice
    std::snprintf(name, sizeof name, "hash_oneblock_kernel<%d,%d,%d>", v.rate_lanes,
                  static_cast<int>(msg_len / 8), static_cast<int>(digest_bytes / 4));
  } else if (whole_bytes && fewblock_supported(v.rate_lanes, msg_len, digest_bytes)) {
    std::snprintf(name, sizeof name, "hash_fewblock_kernel<%d,%d,%d>", v.rate_lanes,
                  static_cast<int>(msg_len / 8), static_cast<int>(digest_bytes / 4));
  } else if (whole_bytes && manyblock_supported(v.rate_lanes, msg_len, digest_bytes)) {
    std::snprintf(name, sizeof name, "hash_manyblock_kernel<%d,%d>", v.rate_lanes, static_cast<int>(digest_bytes / 4));
  } else if (whole_bytes && msg_len < 8u * static_cast<uint64_t>(v.rate_lanes) &&
             short_supported(v.rate_lanes, digest_bytes)) {
    std::snprintf(name, sizeof name, "hash_short_fixed_kernel<%d,%d>", v.rate_lanes,
                  static_cast<int>(digest_bytes / 4));
  } else {
    std::snprintf(name, sizeof name, "hash_generic_kernel<%d>", v.rate_lanes);
  }
  return name;
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

const char* b200sha3_last_cuda_error(void) { return last_error_buffer(); }

int b200sha3_current_device(void) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return dev;
}

int b200sha3_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

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
  AsyncScratch scratch_memory;
  CU(scratch_memory.alloc((8 + kBucketScratchWords) * sizeof(uint32_t), c.stream));
  uint32_t* scratch = scratch_memory.as<uint32_t>();
  CU(cudaMemsetAsync(scratch, 0, (8 + kBucketScratchWords) * sizeof(uint32_t), c.stream));
  // lengths double as "offsets" here: only their low bits feed the alignment flag
  CU(launch_bucket_order(d_lengths, d_lengths, static_cast<uint32_t>(count),
                         8u * kVariants[algorithm].rate_lanes, d_order, scratch + 8, scratch,
                         c.stream));
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
