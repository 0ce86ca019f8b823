// batch_adapter.cpp -- sha3::b200::hash_batch: pack -> C ABI -> unpack.
//
// Host-side mirror of the reference's hash_batch (proj/core/src/batch.cpp:64-135).
// The only computation here is memcpy; every digest comes from libb200sha3.so.
#include "b200sha3/batch.hpp"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>

#if defined(__linux__)
#include <sys/mman.h>
#endif
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

namespace sha3::b200 {

namespace {

unsigned pack_workers(const EngineConfig& config) {  // like resolve_workers, batch.cpp:38-44
  if (config.backend == Backend::sequential) return 1;  // the caller's thread only (batch.cpp:86-89)
  if (config.workers > 0) return config.workers;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? hw : 1;
}

// Runs fn(begin, end) over [0, n) split into contiguous ranges, one per worker
// (the caller participates, like batch.cpp:126).
template <class Fn>
void parallel_ranges(std::size_t n, unsigned workers, std::uint64_t bytes, Fn fn) {
  if (workers <= 1 || n < 2 || bytes < (8u << 20)) {
    fn(std::size_t{0}, n);
    return;
  }
  workers = static_cast<unsigned>(std::min<std::size_t>(workers, n));
  std::vector<std::thread> pool;
  pool.reserve(workers - 1);
  for (unsigned w = 1; w < workers; ++w) {
    pool.emplace_back(fn, n * w / workers, n * (w + 1) / workers);
  }
  fn(std::size_t{0}, n / workers);
  for (auto& t : pool) t.join();
}

[[noreturn]] void raise(int status) {
  if (status == B200SHA3_ERR_INVALID_ARGUMENT) {
    // same message as the reference (batch.cpp:67)
    throw std::invalid_argument("hash_batch: XOF variants need xof_output_bits");
  }
  throw DeviceError(status, std::string("b200sha3: ") + b200sha3_strerror(status) + ": " +
                                b200sha3_last_cuda_error());
}

// Page-locked staging memory for the packed batch and the packed digests, cached per
// calling thread (grow-only, at most kKeepBytes retained) so repeated hash_batch calls --
// run_benchmark does 4+ per size (runner.cpp:45-58) -- do not pay the pinning cost again.
// Falls back to pageable memory if pinning fails; the C ABI call reports the real error.
class StagingBuffer {
 public:
  ~StagingBuffer() { release(); }
  std::uint8_t* reserve(std::uint64_t bytes) {
    if (bytes <= capacity_) return ptr_;
    release();
    void* p = nullptr;
    if (b200sha3_pinned_alloc(bytes, &p) == B200SHA3_OK && p) {
      ptr_ = static_cast<std::uint8_t*>(p);
      pinned_ = true;
    } else {
      ptr_ = static_cast<std::uint8_t*>(std::malloc(bytes));
      pinned_ = false;
      if (!ptr_) throw std::bad_alloc();
    }
    capacity_ = bytes;
    return ptr_;
  }
  void trim(std::uint64_t keep_bytes) {
    if (capacity_ > keep_bytes) release();
  }

 private:
  void release() {
    if (ptr_) {
      if (pinned_) {
        b200sha3_pinned_free(ptr_);
      } else {
        std::free(ptr_);
      }
    }
    ptr_ = nullptr;
    capacity_ = 0;
  }
  std::uint8_t* ptr_ = nullptr;
  std::uint64_t capacity_ = 0;
  bool pinned_ = false;
};

constexpr std::uint64_t kKeepBytes = 2ull << 30;
thread_local StagingBuffer t_data_staging, t_digest_staging;

// Asks for transparent huge pages on the whole pages inside [p, p + bytes): a hint on memory
// the caller owns, ignored where the kernel has THP off.
void advise_huge_pages(void* p, std::size_t bytes) {
#if defined(__linux__) && defined(MADV_HUGEPAGE)
  constexpr std::uintptr_t kHuge = std::uintptr_t{2} << 20;
  static const bool off = std::getenv("B200SHA3_ADAPTER_NO_THP") != nullptr;  // experiment knob
  if (bytes < 2 * kHuge || off) return;
  const std::uintptr_t lo = (reinterpret_cast<std::uintptr_t>(p) + kHuge - 1) & ~(kHuge - 1);
  const std::uintptr_t hi = (reinterpret_cast<std::uintptr_t>(p) + bytes) & ~(kHuge - 1);
  if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
#else
  (void)p;
  (void)bytes;
#endif
}

b200sha3_config make_config(const DeviceConfig& device, double* ms) {
  b200sha3_config cfg{};
  cfg.struct_size = sizeof cfg;
  cfg.device = device.device;
  cfg.stream = device.stream;
  cfg.flags = device.flags;
  cfg.kernel = device.kernel;
  cfg.fma_preset = -1;
  cfg.device_ms = ms;
  return cfg;
}

}  // namespace

DeviceConfig DeviceConfig::all_devices() {
  DeviceConfig cfg;
  const int n = b200sha3_device_count();
  for (int d = 0; d < n; ++d) cfg.devices.push_back(d);
  return cfg;
}

std::vector<std::uint8_t> hash_packed(Algorithm algorithm, const std::uint8_t* data,
                                      const std::uint64_t* offsets,
                                      const std::uint64_t* lengths, std::uint64_t count,
                                      std::uint64_t xof_output_bits, const DeviceConfig& device,
                                      double* elapsed_seconds) {
  const int alg = static_cast<int>(algorithm);
  double ms = 0.0;
  b200sha3_config cfg = make_config(device, &ms);
  std::vector<std::uint8_t> out(count * b200sha3_digest_bytes(alg, xof_output_bits));
  const int rc = b200sha3_hash_batch(alg, data, offsets, lengths, count, xof_output_bits,
                                     out.data(), &cfg);
  if (rc != B200SHA3_OK) raise(rc);
  if (elapsed_seconds) *elapsed_seconds = ms * 1e-3;
  return out;
}

// memcpy into the pinned staging ring.  The ring is written once by the CPU and read once by
// the copy engine, so WHOLE cache lines go out with streaming stores: no read-for-ownership of
// the destination lines, no cache pollution (the call is bound by host memory traffic).  Only
// whole lines: a streaming store next to an ordinary store into the same line forces partial
// write-combining flushes -- streaming the 16-byte aligned body of every message made packing
// short ragged messages 4x slower.  So: messages that are whole aligned lines (64, 128, 4096
// bytes ...) and the line-aligned body of long ones; memcpy for the rest.  Callers issue
// stream_fence() before publishing.
inline void copy_to_staging(std::uint8_t* dst, const std::uint8_t* src, std::size_t n) {
#if defined(__SSE2__)
  static const bool streaming = std::getenv("B200SHA3_ADAPTER_NO_STREAMING_STORES") == nullptr;
  const std::size_t head = (64 - reinterpret_cast<std::uintptr_t>(dst) % 64) % 64;
  if (streaming && (n >= 1024 || (head == 0 && n % 64 == 0 && n != 0))) {
    if (head) std::memcpy(dst, src, head);
    const std::size_t body = (n - head) & ~std::size_t{63};
    for (std::size_t b = 0; b < body; b += 16) {
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + head + b),
                       _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + head + b)));
    }
    if (head + body < n) std::memcpy(dst + head + body, src + head + body, n - head - body);
    return;
  }
#endif
  std::memcpy(dst, src, n);
}

inline void stream_fence() {
#if defined(__SSE2__)
  _mm_sfence();
#endif
}

// ---------------------------------------------------------------------------------------
// hash_batch as a software pipeline.
//
// The reference's call is "allocate the digest slots, then hash" (batch.cpp:77-133).  On the
// GPU the hashing itself is a few percent of the call; the rest is moving bytes between
// vector<vector<uint8_t>> and the packed buffers of the C ABI.  So the call is cut into
//   scan    sizes of all messages -> equal-length or ragged, byte totals per block of messages
//   tasks   ~1 MiB each: pack (messages -> pinned staging) and unpack (pinned digests -> slots)
//   chunks  ~32 MiB each: one C-ABI call (H2D, kernels, D2H) per chunk, as soon as it is packed
// and run by `workers` threads (batch.hpp:15-19; the caller takes part, batch.cpp:126) that pull
// work from one scheduler: device calls first, then packing, then unpacking, so copies and
// kernels of chunk k overlap the packing of chunk k+1 and the unpacking of chunk k-1.  The
// value-initialisation of the outer digest vector -- inherently one thread -- is one more task
// that overlaps the packing.  With several devices, chunk k goes to device k mod n, each device
// driven by its own host thread; digests land in message order whatever the schedule.
class BatchPipeline {
 public:
  BatchPipeline(const HashBatch& batch, const EngineConfig& config, const DeviceConfig& device,
                std::uint64_t digest_bytes, BatchResult& result)
      : batch_(batch), device_(device), alg_(static_cast<int>(batch.algorithm)),
        digest_bytes_(digest_bytes), workers_(pack_workers(config)), result_(result),
        count_(batch.messages.size()) {}

  void run() {
    const auto t0 = clock::now();
    block_msgs_ = std::max<std::size_t>(1, std::min<std::size_t>(256, count_ / 1024));
    nblocks_ = (count_ + block_msgs_ - 1) / block_msgs_;
    first_len_ = batch_.messages[0].size();
    nsteps_ = (count_ + kResizeStep - 1) / kResizeStep;
    step_state_.reset(new std::atomic<std::uint8_t>[nsteps_]);
    for (std::size_t i = 0; i < nsteps_; ++i) step_state_[i].store(kStepUntouched);
    // Large batches whose sampled sizes all agree are taken as equal-length without reading
    // every size first: the pack tasks check as they copy, and a mismatch restarts the call on
    // the ragged layout.  (generate_workload batches, workload.cpp:34-45, never restart.)
    speculative_ = count_ >= kParallelScanMin && sample_is_fixed();
    if (!speculative_) scan();
    plan();
    double scan_s = since(t0);
    run_threads();
    if (mismatch_.load() && !failed_) {
      const auto t2 = clock::now();
      speculative_ = false;
      mismatch_.store(false);
      scan();
      plan();
      scan_s += since(t2);
      run_threads();
    }
    t_data_staging.trim(failed_ ? 0 : kKeepBytes);
    t_digest_staging.trim(failed_ ? 0 : kKeepBytes);
    if (error_) std::rethrow_exception(error_);  // first failure wins (batch.cpp:111-130)
    // Kernel-only device time (StageTimes::kernels): lanes of one device are added up (their
    // kernels share that GPU), devices run side by side.
    double ms = 0.0;
    for (std::size_t a = 0; a < device_ms_.size(); ++a) {
      double on_device = 0.0;
      for (std::size_t b = 0; b < device_ms_.size(); ++b) {
        if (lanes_[b] == lanes_[a]) on_device += device_ms_[b];
      }
      ms = std::max(ms, on_device);
    }
    // BatchResult::elapsed is what the reference defines it as: the wall time of the hashing
    // phase as the caller sees it (batch.cpp:84, :133) -- here scan, pack, copies, kernels and
    // unpack.  The reference's runner derives throughput from it (runner.cpp:53, :71), so a
    // kernel-only figure in this field would overstate a like-for-like run by ~20x.
    result_.elapsed = std::chrono::duration<double>(since(t0));
    if (StageTimes* st = device_.stages) {
      st->scan = scan_s;
      st->pipeline = since(t0) - scan_s;
      st->resize = resize_s_;
      st->device_calls = device_calls_s_;
      st->pack_cpu = pack_cpu_s_;
      st->unpack_cpu = unpack_cpu_s_;
      st->kernels = ms * 1e-3;
      st->threads = threads_;
      st->chunks = static_cast<unsigned>(nchunks_);
      st->tasks = static_cast<unsigned>(ntasks_);
    }
  }

 private:
  using clock = std::chrono::steady_clock;
  static double since(clock::time_point t) {
    return std::chrono::duration<double>(clock::now() - t).count();
  }
  static std::uint64_t pad8(std::uint64_t n) { return (n + 7) & ~std::uint64_t{7}; }

  // Plan granularity.  The sanitizer build of tests/cpp shrinks it (-DB200SHA3_ADAPTER_TEST_SCALE=n
  // divides every size by 2^n) so that ring wrap-around, multi-step resizes, the parallel scan and
  // the speculative restart all happen on batches small enough for a CPU test.
#ifndef B200SHA3_ADAPTER_TEST_SCALE
#define B200SHA3_ADAPTER_TEST_SCALE 0
#endif
  static constexpr int kScale = B200SHA3_ADAPTER_TEST_SCALE;
  static constexpr std::uint64_t kTaskBytes = (1ull << 20) >> kScale;     // input + output per task
  static constexpr std::uint64_t kChunkBytes = (32ull << 20) >> kScale;   // input + output per device call ...
  static constexpr std::uint64_t kMinChunkBytes = (2ull << 20) >> kScale; // ... at least this ...
  static constexpr std::uint64_t kMinChunks = 8;                          // ... aiming at this many chunks
  static constexpr std::uint64_t kChunkMinMessages = (1u << 11) >> kScale;  // ... grown to hold this many messages
  static constexpr std::uint64_t kMaxChunkBytes = (1ull << 30) >> kScale;   // ... up to this
  static constexpr std::uint64_t kPoolMinBytes = (4ull << 20) >> kScale;  // below: the caller works alone
  static constexpr std::size_t kParallelScanMin = (1u << 18) >> kScale;   // messages
  static constexpr std::size_t kArenaGrowBytes = 120u << 10;              // < glibc's 128 KiB trim threshold
  static constexpr int kLanesPerDevice = 2;                               // host threads issuing device calls
  static constexpr std::size_t kRingChunks = 12;                          // pinned staging: chunks in flight
  static constexpr std::uint64_t kRingBytes = (1ull << 30) >> kScale;     // ... and their bytes, at most
  static constexpr std::size_t kResizeStep = (1u << 17) >> kScale;        // digest slots per published step
  static constexpr std::uint8_t kStepUntouched = 0, kStepTouching = 1, kStepBuilt = 2;

  bool sample_is_fixed() const {
    const std::size_t head = std::min<std::size_t>(count_, 256), stride = count_ / 256;
    for (std::size_t i = 0; i < head; ++i) {
      if (batch_.messages[i].size() != first_len_) return false;
      if (batch_.messages[i * stride].size() != first_len_) return false;
    }
    return batch_.messages[count_ - 1].size() == first_len_;
  }

  // Sizes of all messages, per block of block_msgs_ messages: padded byte total and whether
  // every length equals the first message's.
  void scan() {
    block_base_.reset(new std::uint64_t[nblocks_ + 1]);
    std::unique_ptr<bool[]> block_fixed(new bool[nblocks_]);
    const auto scan_blocks = [&](std::size_t begin, std::size_t end) {
      for (std::size_t b = begin; b < end; ++b) {
        const std::size_t lo = b * block_msgs_, hi = std::min(count_, lo + block_msgs_);
        std::uint64_t bytes = 0;
        bool same = true;
        for (std::size_t i = lo; i < hi; ++i) {
          const std::uint64_t len = batch_.messages[i].size();
          same = same && len == first_len_;
          bytes += pad8(len);
        }
        block_base_[b + 1] = bytes;
        block_fixed[b] = same;
      }
    };
    parallel_ranges(nblocks_, count_ >= kParallelScanMin ? workers_ : 1, ~std::uint64_t{0}, scan_blocks);
    fixed_ = true;
    block_base_[0] = 0;
    for (std::size_t b = 0; b < nblocks_; ++b) {
      fixed_ = fixed_ && block_fixed[b];
      block_base_[b + 1] += block_base_[b];  // exclusive prefix: where block b starts (ragged layout)
    }
  }

  // Equal-length batches (what generate_workload builds, workload.cpp:34-45) go back to back
  // and take the fixed-length entry: no offset table, no bucketing pass.  Ragged batches get
  // 8-byte aligned offsets so the device can use aligned 64-bit loads.
  void plan() {
    if (speculative_) fixed_ = true;
    total_in_ = fixed_ ? count_ * first_len_ : block_base_[nblocks_];
    const std::uint64_t total = total_in_ + count_ * digest_bytes_;
    const std::uint64_t block_bytes = std::max<std::uint64_t>(1, total / nblocks_);
    task_blocks_ = std::max<std::size_t>(1, std::min<std::uint64_t>(kTaskBytes / block_bytes, nblocks_));
    ntasks_ = (nblocks_ + task_blocks_ - 1) / task_blocks_;
    // Device lanes: two host threads per device issue its C-ABI calls (chunk k -> lane k mod
    // lanes), so the H2D copy of one chunk overlaps the kernels / D2H of the previous one, and
    // the kernels of two chunks of few long messages share the GPU.
    lanes_.clear();
    static const int lanes_per_device = [] {  // B200SHA3_ADAPTER_LANES: experiment knob
      const char* env = std::getenv("B200SHA3_ADAPTER_LANES");
      const int n = env ? std::atoi(env) : 0;
      return n >= 1 && n <= 8 ? n : kLanesPerDevice;
    }();
    const int reps = workers_ == 1 ? 1 : lanes_per_device;  // one worker: no second thread at all
    for (int rep = 0; rep < reps; ++rep) {
      if (device_.devices.empty()) lanes_.push_back(device_.device);
      for (int d : device_.devices) lanes_.push_back(d);
    }
    const std::size_t ndev = std::max<std::size_t>(1, device_.devices.size());
    // A chunk is one kernel launch with one thread per message: long messages get larger
    // chunks so that a launch still carries ~2^11 of them (warp-per-state kernel territory: a
    // chunk's hashing then takes about as long as its copy up to ~64 KiB per message).
    static const std::uint64_t min_chunks = [] {  // B200SHA3_ADAPTER_MIN_CHUNKS: experiment knob
      const char* env = std::getenv("B200SHA3_ADAPTER_MIN_CHUNKS");
      const long n = env ? std::atol(env) : 0;
      return static_cast<std::uint64_t>(n >= 1 ? n : kMinChunks);
    }();
    // ... and mid-size batches get smaller ones, so that there is a pipeline at all
    const std::uint64_t base_bytes = std::min(kChunkBytes, std::max(kMinChunkBytes, total / min_chunks));
    const std::uint64_t chunk_bytes =
        std::min(kMaxChunkBytes, std::max(base_bytes, total / count_ * kChunkMinMessages));
    std::size_t want = static_cast<std::size_t>((total + chunk_bytes / 2) / chunk_bytes);  // nearest
    want = std::min(ntasks_, std::max(want, ndev));
    chunk_tasks_ = (ntasks_ + want - 1) / want;
    nchunks_ = (ntasks_ + chunk_tasks_ - 1) / chunk_tasks_;
    devices_used_ = static_cast<unsigned>(std::min(lanes_.size(), nchunks_));
    if (devices_used_ > 1 && lanes_[0] < 0) {  // "current device" is the CALLER's: name it for the lane threads
      const int current = b200sha3_current_device();
      for (int& d : lanes_) d = current;
    }
    threads_ = total < kPoolMinBytes ? 1u : static_cast<unsigned>(std::min<std::size_t>(workers_, ntasks_));
    threads_ = std::max(threads_, devices_used_);

    // Pinned staging is a ring of kRingChunks chunk buffers, not a copy of the batch: chunk k
    // packs into buffer k mod ring once chunk k - ring has been unpacked.
    ring_ = std::min(nchunks_, kRingChunks);
    chunk_in_cap_ = chunk_out_cap_ = 0;
    for (std::size_t k = 0; k < nchunks_; ++k) {
      const std::size_t lo = chunk_first(k), hi = chunk_first(k + 1);
      const std::uint64_t in = fixed_ ? (hi - lo) * first_len_ : chunk_base(k + 1) - chunk_base(k);
      chunk_in_cap_ = std::max(chunk_in_cap_, (in + 63) & ~std::uint64_t{63});
      chunk_out_cap_ = std::max(chunk_out_cap_, ((hi - lo) * digest_bytes_ + 63) & ~std::uint64_t{63});
    }
    const std::uint64_t fit = kRingBytes / std::max<std::uint64_t>(1, chunk_in_cap_ + chunk_out_cap_);
    ring_ = std::max<std::size_t>(devices_used_, std::min<std::uint64_t>(ring_, fit));  // odd chunks: stay bounded
    data_ = t_data_staging.reserve(std::max<std::uint64_t>(ring_ * chunk_in_cap_, 16));
    packed_ = t_digest_staging.reserve(std::max<std::uint64_t>(ring_ * chunk_out_cap_, 16));
    if (!fixed_) {  // filled by the pack tasks
      offsets_.reset(new std::uint64_t[count_]);
      lengths_.reset(new std::uint64_t[count_]);
    }
    next_pack_ = next_unpack_ = 0;
    pack_left_.assign(nchunks_, 0);
    for (std::size_t t = 0; t < ntasks_; ++t) pack_left_[t / chunk_tasks_] += 1;
    unpack_left_ = pack_left_;
    chunk_hashed_.assign(nchunks_, 0);
    device_ms_.assign(devices_used_, 0.0);
  }

  void run_threads() {
    std::vector<std::thread> pool;
    pool.reserve(threads_ - 1);
    for (unsigned t = 1; t < threads_; ++t) {
      pool.emplace_back([this, t] { thread_main(t < devices_used_ ? static_cast<int>(t) : -1); });
    }
    thread_main(0);  // the caller drives the first device (batch.cpp:126)
    for (auto& t : pool) t.join();
  }

  std::size_t task_first(std::size_t task) const {  // first message of a task
    return std::min(count_, task * task_blocks_ * block_msgs_);
  }
  std::size_t chunk_first(std::size_t chunk) const {  // first message of a chunk
    return task_first(std::min(ntasks_, chunk * chunk_tasks_));
  }
  std::uint64_t chunk_base(std::size_t chunk) const {  // ragged layout: first byte of a chunk
    return block_base_[std::min(nblocks_, chunk * chunk_tasks_ * task_blocks_)];
  }
  std::uint8_t* chunk_in(std::size_t chunk) const { return data_ + (chunk % ring_) * chunk_in_cap_; }
  std::uint8_t* chunk_out(std::size_t chunk) const { return packed_ + (chunk % ring_) * chunk_out_cap_; }

  void pack_task(std::size_t task) {
    const std::size_t lo = task_first(task), hi = task_first(task + 1);
    const std::size_t chunk = task / chunk_tasks_;
    if (fixed_) {
      std::uint8_t* dst = chunk_in(chunk) + (lo - chunk_first(chunk)) * first_len_;
      for (std::size_t i = lo; i < hi; ++i, dst += first_len_) {
        const auto& m = batch_.messages[i];
        if (m.size() != first_len_) {  // only a speculative plan can get here
          mismatch_.store(true);
          break;
        }
        if (first_len_) copy_to_staging(dst, m.data(), first_len_);
      }
      stream_fence();  // streaming stores are visible before the task is reported packed
      return;
    }
    std::uint8_t* base = chunk_in(chunk);
    std::uint64_t off = block_base_[task * task_blocks_] - chunk_base(chunk);  // within the chunk buffer
    for (std::size_t i = lo; i < hi; ++i) {
      const auto& m = batch_.messages[i];
      offsets_[i] = off;
      lengths_[i] = m.size();
      if (!m.empty()) copy_to_staging(base + off, m.data(), m.size());
      off += pad8(m.size());
    }
    stream_fence();
  }

  void unpack_task(std::size_t task) {
    const std::size_t lo = task_first(task), hi = task_first(task + 1);
    const std::size_t chunk = task / chunk_tasks_;
    const std::uint8_t* d = chunk_out(chunk) + (lo - chunk_first(chunk)) * digest_bytes_;
    // One heap allocation per digest is the result type's price.  glibc grows a thread's arena
    // one page (~85 digests) per mprotect(), and mprotect() takes the process's mmap lock for
    // writing -- with 16 threads unpacking, that lock is what they queue on.  Allocating and
    // freeing a block just under the trim threshold first makes the arena grow by that much in
    // one step; the small allocations that follow are carved from it.  (Any other allocator
    // just sees a malloc/free pair.)
    const std::size_t per_grow = std::max<std::size_t>(1, kArenaGrowBytes / (digest_bytes_ + 32));
    for (std::size_t i = lo; i < hi; ++i, d += digest_bytes_) {
      if ((i - lo) % per_grow == 0 && digest_bytes_ < kArenaGrowBytes / 4) std::free(std::malloc(kArenaGrowBytes));
      slots_[i].assign(d, d + digest_bytes_);
    }
  }

  // One C-ABI call for the messages of chunk `chunk` on device slot `slot`.
  void device_call(std::size_t chunk, int slot) {
    const std::size_t first = chunk_first(chunk), n = chunk_first(chunk + 1) - first;
    double ms = 0.0;
    b200sha3_config cfg = make_config(device_, &ms);
    cfg.device = lanes_[slot];
    if (device_.devices.size() > 1) cfg.stream = nullptr;
    std::uint8_t* out = chunk_out(chunk);
    const int rc =
        fixed_ ? b200sha3_hash_fixed(alg_, chunk_in(chunk), first_len_, n, batch_.xof_output_bits, out, &cfg)
               : b200sha3_hash_batch(alg_, chunk_in(chunk), offsets_.get() + first, lengths_.get() + first,
                                     n, batch_.xof_output_bits, out, &cfg);
    if (rc == B200SHA3_ERR_INVALID_ARGUMENT) raise(rc);
    if (rc != B200SHA3_OK) {
      std::string where;
      if (device_.devices.size() > 1) where = " on device " + std::to_string(lanes_[slot]);
      throw DeviceError(rc, std::string("b200sha3: ") + b200sha3_strerror(rc) + where + ": " +
                                b200sha3_last_cuda_error());  // thread-local text: read it here
    }
    device_ms_[slot] += ms;  // only this slot's thread writes it
  }

  // Outer digest vector: `count` empty slots, 24 B each -- value-initialised by one thread
  // (std::vector offers nothing else) and page-fault bound on fresh memory.  So: the storage
  // is reserved once (transparent huge pages requested), which means growing the vector in
  // steps never moves a slot; the other threads fault the pages of later steps in ahead of
  // the builder (prefault_step); and after every step the slots built so far are published,
  // so the unpack tasks below that mark run while the rest is still being built.  Stops early
  // (to be resumed) when the pipeline is restarting.
  void resize_result() {
    if (result_.digests.capacity() < count_) {
      result_.digests.reserve(count_);
      advise_huge_pages(result_.digests.data(), count_ * sizeof(result_.digests[0]));
      std::lock_guard<std::mutex> guard(mutex_);
      slots_ = result_.digests.data();
    }
    for (std::size_t done = result_.digests.size(); done < count_ && !mismatch_.load();) {
      const std::size_t step = done / kResizeStep;
      std::uint8_t untouched = kStepUntouched;
      if (!step_state_[step].compare_exchange_strong(untouched, kStepBuilt)) {
        while (step_state_[step].load(std::memory_order_acquire) != kStepBuilt) std::this_thread::yield();
      }
      done = std::min(count_, (step + 1) * kResizeStep);
      result_.digests.resize(done);
      {
        std::lock_guard<std::mutex> guard(mutex_);
        slots_ready_ = done;
      }
      cv_.notify_all();
    }
  }

  // Faults in the pages under the slots of one resize step that the builder has not reached.
  // Only bytes of that step are written (zeros, into raw reserved storage), and the builder
  // waits for a step being touched, so a slot is never written after it was constructed.
  void prefault_step(std::size_t step) {
    std::uint8_t untouched = kStepUntouched;
    if (!step_state_[step].compare_exchange_strong(untouched, kStepTouching)) return;
    auto* base = reinterpret_cast<volatile char*>(slots_);
    const std::size_t lo = step * kResizeStep * sizeof(result_.digests[0]);
    const std::size_t hi = std::min(count_, (step + 1) * kResizeStep) * sizeof(result_.digests[0]);
    for (std::size_t b = lo; b < hi; b += 4096) base[b] = 0;
    step_state_[step].store(kStepBuilt, std::memory_order_release);
  }

  // Runs f() with the scheduler lock released; a throw marks the pipeline failed (the first
  // exception is kept, the other threads drain; batch.cpp:95-117).  Returns the seconds f took.
  template <class F>
  double unlocked(std::unique_lock<std::mutex>& lock, F f) {
    lock.unlock();
    const auto t0 = clock::now();
    try {
      f();
    } catch (...) {
      lock.lock();
      if (!failed_) {
        failed_ = true;
        error_ = std::current_exception();
      }
      cv_.notify_all();
      return since(t0);
    }
    const double s = since(t0);
    lock.lock();
    return s;
  }

  bool ring_slot_free(std::size_t chunk) const {  // under mutex_
    return chunk < ring_ || unpack_left_[chunk - ring_] == 0;
  }

  // slot >= 0: this thread also issues the device calls of chunks slot, slot + n, ...
  void thread_main(int slot) {
    std::unique_lock<std::mutex> lock(mutex_);
    std::size_t my_chunk = slot >= 0 ? static_cast<std::size_t>(slot) : nchunks_;
    for (;;) {
      if (failed_ || mismatch_.load()) {
        cv_.notify_all();
        return;
      }
      if (my_chunk < nchunks_ && pack_left_[my_chunk] == 0) {
        const std::size_t k = my_chunk;
        device_calls_s_ += unlocked(lock, [&] { device_call(k, slot); });
        chunk_hashed_[k] = 1;
        my_chunk += devices_used_;
        cv_.notify_all();
      } else if (!resize_taken_ && slots_ready_ < count_ &&
                 (slot < 0 || threads_ == devices_used_)) {  // a pure worker, if there is one
        resize_taken_ = true;
        resize_s_ += unlocked(lock, [&] { resize_result(); });
        resize_taken_ = false;
        cv_.notify_all();
      } else if (slots_ && next_prefault_ < nsteps_) {
        const std::size_t step = next_prefault_++;
        unlocked(lock, [&] { prefault_step(step); });
      } else if (next_pack_ < ntasks_ && ring_slot_free(next_pack_ / chunk_tasks_)) {
        const std::size_t t = next_pack_++;
        pack_cpu_s_ += unlocked(lock, [&] { pack_task(t); });
        if (--pack_left_[t / chunk_tasks_] == 0) cv_.notify_all();
      } else if (next_unpack_ < ntasks_ && task_first(next_unpack_ + 1) <= slots_ready_ &&
                 chunk_hashed_[next_unpack_ / chunk_tasks_]) {
        const std::size_t t = next_unpack_++;
        unpack_cpu_s_ += unlocked(lock, [&] { unpack_task(t); });
        if (--unpack_left_[t / chunk_tasks_] == 0) cv_.notify_all();  // its ring buffers are free
      } else if (next_unpack_ == ntasks_ && my_chunk >= nchunks_) {
        return;  // nothing left to take; tasks still running finish before the join
      } else {
        cv_.wait(lock);
      }
    }
  }

  const HashBatch& batch_;
  const DeviceConfig& device_;
  const int alg_;
  const std::uint64_t digest_bytes_;
  const unsigned workers_;
  BatchResult& result_;
  const std::size_t count_;

  // plan
  std::size_t block_msgs_ = 1, nblocks_ = 0, task_blocks_ = 1, ntasks_ = 0, chunk_tasks_ = 1, nchunks_ = 0;
  std::unique_ptr<std::uint64_t[]> block_base_, offsets_, lengths_;
  std::uint64_t first_len_ = 0, total_in_ = 0;
  bool fixed_ = true, speculative_ = false;
  unsigned threads_ = 1, devices_used_ = 1;  // devices_used_: device lanes in use
  std::vector<int> lanes_;                   // CUDA ordinal per lane
  std::size_t ring_ = 1;
  std::uint64_t chunk_in_cap_ = 0, chunk_out_cap_ = 0;
  std::uint8_t* data_ = nullptr;    // ring_ x chunk_in_cap_ bytes, pinned
  std::uint8_t* packed_ = nullptr;  // ring_ x chunk_out_cap_ bytes, pinned

  // scheduler state, under mutex_
  std::mutex mutex_;
  std::condition_variable cv_;
  std::size_t next_pack_ = 0, next_unpack_ = 0, slots_ready_ = 0, next_prefault_ = 1, nsteps_ = 0;
  std::unique_ptr<std::atomic<std::uint8_t>[]> step_state_;
  std::vector<std::uint8_t>* slots_ = nullptr;
  std::vector<std::size_t> pack_left_, unpack_left_;
  std::vector<char> chunk_hashed_;
  bool resize_taken_ = false, failed_ = false;
  std::atomic<bool> mismatch_{false};
  std::exception_ptr error_;
  std::vector<double> device_ms_;
  double resize_s_ = 0, device_calls_s_ = 0, pack_cpu_s_ = 0, unpack_cpu_s_ = 0;
};

BatchResult hash_batch(const HashBatch& batch, const EngineConfig& config,
                       const DeviceConfig& device) {
  const int alg = static_cast<int>(batch.algorithm);
  // Validation first, before any allocation or copy (batch.cpp:66-68).
  const bool is_xof = alg == B200SHA3_SHAKE128 || alg == B200SHA3_SHAKE256;
  if (alg < 0 || alg > 5) throw std::invalid_argument("hash_batch: unknown algorithm");
  if (is_xof && batch.xof_output_bits == 0) raise(B200SHA3_ERR_INVALID_ARGUMENT);

  BatchResult result;
  if (batch.messages.empty()) return result;  // test_batch.cpp:113-117
  BatchPipeline(batch, config, device, b200sha3_digest_bytes(alg, batch.xof_output_bits), result).run();
  return result;
}

// ---------------------------------------------------------------------------------------
// BatchHasher: sha3::Hasher for `count` streams at once, over the b200sha3_states_* entries.

BatchHasher::BatchHasher(Algorithm algorithm, std::size_t count, const DeviceConfig& device)
    : algorithm_(algorithm), count_(count), device_(device) {
  const int alg = static_cast<int>(algorithm);
  if (alg < 0 || alg > 5) throw std::invalid_argument("BatchHasher: unknown algorithm");
  device_.stages = nullptr;
  b200sha3_config cfg = make_config(device_, nullptr);
  if (!device_.devices.empty()) cfg.device = device_.devices[0];
  check(b200sha3_states_create(alg, count, &cfg, &states_));
}

BatchHasher::~BatchHasher() {
  if (states_) b200sha3_states_destroy(states_);
}

BatchHasher::BatchHasher(BatchHasher&& other) noexcept
    : algorithm_(other.algorithm_), count_(other.count_), device_(std::move(other.device_)),
      states_(other.states_) {
  other.states_ = nullptr;
}

BatchHasher& BatchHasher::operator=(BatchHasher&& other) noexcept {
  if (this != &other) {
    if (states_) b200sha3_states_destroy(states_);
    algorithm_ = other.algorithm_;
    count_ = other.count_;
    device_ = std::move(other.device_);
    states_ = other.states_;
    other.states_ = nullptr;
  }
  return *this;
}

void BatchHasher::check(int status) const {
  if (status == B200SHA3_OK) return;
  if (status == B200SHA3_ERR_STATE) {  // the reference's std::logic_error (sponge.cpp:82-84, :114-116, :132-134)
    throw std::logic_error("BatchHasher: call out of order (update after finish, finish twice, or read before finish)");
  }
  if (status == B200SHA3_ERR_INVALID_ARGUMENT) throw std::invalid_argument("BatchHasher: invalid argument");
  throw DeviceError(status, std::string("b200sha3: ") + b200sha3_strerror(status) + ": " +
                                b200sha3_last_cuda_error());
}

void BatchHasher::update(const std::uint8_t* data, const std::uint64_t* offsets,
                         const std::uint64_t* lengths) {
  b200sha3_config cfg = make_config(device_, nullptr);
  check(b200sha3_states_update(states_, data, offsets, lengths, &cfg));
}

void BatchHasher::update_fixed(const std::uint8_t* data, std::uint64_t chunk_len) {
  b200sha3_config cfg = make_config(device_, nullptr);
  check(b200sha3_states_update_fixed(states_, data, chunk_len, &cfg));
}

void BatchHasher::update(const std::vector<std::vector<std::uint8_t>>& chunks) {
  if (chunks.size() != count_) throw std::invalid_argument("BatchHasher: one chunk per stream expected");
  std::vector<std::uint64_t> offsets(count_), lengths(count_);
  std::uint64_t total = 0;
  for (std::size_t i = 0; i < count_; ++i) {
    offsets[i] = total;
    lengths[i] = chunks[i].size();
    total += lengths[i];
  }
  std::uint8_t* data = t_data_staging.reserve(std::max<std::uint64_t>(total, 16));
  parallel_ranges(count_, pack_workers(EngineConfig{}), total, [&](std::size_t begin, std::size_t end) {
    for (std::size_t i = begin; i < end; ++i) {
      if (lengths[i]) copy_to_staging(data + offsets[i], chunks[i].data(), lengths[i]);
    }
    stream_fence();
  });
  update(data, offsets.data(), lengths.data());
  t_data_staging.trim(kKeepBytes);
}

std::vector<std::vector<std::uint8_t>> BatchHasher::split(const std::vector<std::uint8_t>& packed,
                                                          std::size_t each) const {
  std::vector<std::vector<std::uint8_t>> out(count_);
  for (std::size_t i = 0; i < count_; ++i) {
    out[i].assign(packed.begin() + i * each, packed.begin() + (i + 1) * each);
  }
  return out;
}

std::vector<std::vector<std::uint8_t>> BatchHasher::digest() {
  const int alg = static_cast<int>(algorithm_);
  if (alg >= 4) {  // sha3.cpp:103-106
    throw std::logic_error("Hasher: digest() is for fixed-output variants; use finish()/read()");
  }
  const std::size_t each = b200sha3_digest_bytes(alg, 0);
  std::vector<std::uint8_t> packed(std::max<std::size_t>(count_ * each, 1));
  b200sha3_config cfg = make_config(device_, nullptr);
  check(b200sha3_states_finish(states_, 0, packed.data(), &cfg));
  return split(packed, each);
}

void BatchHasher::finish() {
  if (static_cast<int>(algorithm_) < 4) {  // sha3.cpp:111-114
    throw std::logic_error("Hasher: finish()/read() is for XOF variants; use digest()");
  }
  b200sha3_config cfg = make_config(device_, nullptr);
  check(b200sha3_states_finish(states_, 0, nullptr, &cfg));
}

std::vector<std::vector<std::uint8_t>> BatchHasher::read(std::size_t nbytes) {
  if (static_cast<int>(algorithm_) < 4) {  // sha3.cpp:119-122
    throw std::logic_error("Hasher: finish()/read() is for XOF variants; use digest()");
  }
  std::vector<std::uint8_t> packed(std::max<std::size_t>(count_ * nbytes, 1));
  b200sha3_config cfg = make_config(device_, nullptr);
  check(b200sha3_states_squeeze(states_, nbytes, packed.data(), &cfg));
  return split(packed, nbytes);
}

void BatchHasher::reset() {
  b200sha3_config cfg = make_config(device_, nullptr);
  check(b200sha3_states_reset(states_, &cfg));
}

}  // namespace sha3::b200
