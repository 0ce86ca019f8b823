// host_io.cuh -- host <-> device copies of the host-buffer entries (capi_host.cu,
// capi_stream.cu): straight cudaMemcpyAsync for pinned memory, a pinned bounce ring fed by
// helper threads for pageable memory.
#pragma once
#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include "capi_common.cuh"

namespace b200sha3::capi {

// memcpy whose destination is written once here and read once by a copy engine (a pinned
// bounce block): whole cache lines go out with streaming stores -- no read-for-ownership.
inline void copy_for_dma(uint8_t* dst, const uint8_t* src, size_t n) {
#if defined(__SSE2__)
  const size_t head = (64 - reinterpret_cast<uintptr_t>(dst) % 64) % 64;
  if (n >= 4096 && head < n) {
    if (head) std::memcpy(dst, src, head);
    const size_t body = (n - head) & ~size_t{63};
    for (size_t b = 0; b < body; b += 16) {
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + head + b),
                       _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + head + b)));
    }
    if (head + body < n) std::memcpy(dst + head + body, src + head + body, n - head - body);
    _mm_sfence();
    return;
  }
#endif
  std::memcpy(dst, src, n);
}

// ---- pageable host memory ----------------------------------------------------------------
// cudaMemcpyAsync on pageable memory is staged by the driver through one thread: 8-10 GB/s
// measured on the B200 boxes against 50-55 GB/s from pinned memory, and synchronous.  A caller
// of the C ABI that holds its batch in ordinary malloc/std::vector memory (INTEGRATION.md,
// binding 1) would spend 5x longer in copies than the link needs.  So the host entries stage
// pageable buffers themselves: helper threads memcpy 8 MiB blocks into a small ring of pinned
// bounce buffers (cached per calling thread) and the copy engines take it from there; digests
// come back the same way.  Pinned callers (b200sha3_pinned_alloc, cudaHostRegister) skip all this.

// Experiment / test knobs: B200SHA3_NO_BOUNCE=1 leaves pageable memory to the driver;
// B200SHA3_BOUNCE_MIN_KIB and B200SHA3_BOUNCE_BLOCK_KIB shrink the threshold and the block so
// that small randomized batches (tests/fuzz_parity.py) wrap the ring many times.
inline uint64_t env_kib(const char* name, uint64_t fallback_bytes) {
  const char* env = std::getenv(name);
  if (!env) return fallback_bytes;
  const long long kib = std::atoll(env);
  return kib < 0 ? fallback_bytes : static_cast<uint64_t>(kib) << 10;
}

inline bool is_pageable(const void* p) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return attr.type == cudaMemoryTypeUnregistered;
}

// Helper threads that live for one call; copy() is a parallel memcpy that returns when done.
class CopyPool {
 public:
  CopyPool(unsigned helpers, size_t min_parallel_bytes) : min_parallel_(min_parallel_bytes) {
    for (unsigned i = 0; i < helpers; ++i) threads_.emplace_back([this, i] { worker(i + 1); });
  }
  CopyPool(const CopyPool&) = delete;
  CopyPool& operator=(const CopyPool&) = delete;
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++generation_;
    }
    wake_.notify_all();
    for (auto& t : threads_) t.join();
  }

  // `for_dma`: dst is a pinned block the copy engine reads next (streaming stores)
  void copy(void* dst, const void* src, size_t bytes, bool for_dma = false) {
    if (threads_.empty() || bytes < min_parallel_) {
      if (for_dma) {
        copy_for_dma(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), bytes);
      } else {
        std::memcpy(dst, src, bytes);
      }
      return;
    }
    {
      std::lock_guard<std::mutex> g(m_);
      dst_ = static_cast<uint8_t*>(dst);
      src_ = static_cast<const uint8_t*>(src);
      bytes_ = bytes;
      for_dma_ = for_dma;
      const size_t parts = threads_.size() + 1;
      piece_ = ((bytes + parts - 1) / parts + 4095) & ~size_t{4095};
      pending_ = threads_.size();
      ++generation_;
    }
    wake_.notify_all();
    copy_piece(0);
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void copy_piece(size_t index) {
    const size_t lo = std::min(bytes_, index * piece_), hi = std::min(bytes_, lo + piece_);
    if (hi <= lo) return;
    if (for_dma_) {
      copy_for_dma(dst_ + lo, src_ + lo, hi - lo);
    } else {
      std::memcpy(dst_ + lo, src_ + lo, hi - lo);
    }
  }
  void worker(size_t index) {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(m_);
    for (;;) {
      wake_.wait(lk, [&] { return generation_ != seen; });
      seen = generation_;
      if (stop_) return;
      lk.unlock();
      copy_piece(index);
      lk.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }

  const size_t min_parallel_;
  std::vector<std::thread> threads_;
  std::mutex m_;
  std::condition_variable wake_, done_;
  uint64_t generation_ = 0;
  bool stop_ = false;
  uint8_t* dst_ = nullptr;
  const uint8_t* src_ = nullptr;
  size_t bytes_ = 0, piece_ = 0, pending_ = 0;
  bool for_dma_ = false;
};

// The pinned bounce ring of one calling thread: kSlots blocks of kBlock bytes, used round-robin
// by both directions.  A slot is reused once the copy engine is done with it (its event) and,
// for a digest block, once it has been copied out to the caller's buffer.
class BounceRing {
 public:
  static constexpr int kSlots = 8;

  ~BounceRing() {
    for (cudaEvent_t e : events_) {
      if (e) cudaEventDestroy(e);
    }
    if (base_) cudaFreeHost(base_);
  }

  cudaError_t init() {
    if (base_) return cudaSuccess;
    static const size_t block = std::max<uint64_t>(512, env_kib("B200SHA3_BOUNCE_BLOCK_KIB", 8u << 20));
    kBlock = block;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&base_), kBlock * kSlots, cudaHostAllocPortable);
    for (int i = 0; e == cudaSuccess && i < kSlots; ++i) {
      e = cudaEventCreateWithFlags(&events_[i], cudaEventDisableTiming);
    }
    return e;
  }

  // dst (device) <- src (pageable host), asynchronous on `stream` once the bytes are staged.
  cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t stream, CopyPool& pool) {
    for (size_t off = 0; off < bytes; off += kBlock) {
      const size_t n = std::min(kBlock, bytes - off);
      int slot = 0;
      cudaError_t e = acquire(&slot, pool);
      if (e != cudaSuccess) return e;
      pool.copy(block(slot), static_cast<const uint8_t*>(src) + off, n, /*for_dma=*/true);
      e = cudaMemcpyAsync(static_cast<uint8_t*>(dst) + off, block(slot), n, cudaMemcpyHostToDevice, stream);
      if (e == cudaSuccess) e = cudaEventRecord(events_[slot], stream);
      if (e != cudaSuccess) return e;
      busy_[slot] = true;
    }
    return cudaSuccess;
  }

  // dst (pageable host) <- src (device): the DMA into the ring is enqueued now, the copy out to
  // `dst` happens when the slot comes round again or at flush().
  cudaError_t d2h(void* dst, const void* src, size_t bytes, cudaStream_t stream, CopyPool& pool) {
    for (size_t off = 0; off < bytes; off += kBlock) {
      const size_t n = std::min(kBlock, bytes - off);
      int slot = 0;
      cudaError_t e = acquire(&slot, pool);
      if (e != cudaSuccess) return e;
      e = cudaMemcpyAsync(block(slot), static_cast<const uint8_t*>(src) + off, n, cudaMemcpyDeviceToHost, stream);
      if (e == cudaSuccess) e = cudaEventRecord(events_[slot], stream);
      if (e != cudaSuccess) return e;
      busy_[slot] = true;
      out_dst_[slot] = static_cast<uint8_t*>(dst) + off;
      out_bytes_[slot] = n;
    }
    return cudaSuccess;
  }

  // Waits for every slot and delivers the digest blocks still in the ring.
  cudaError_t flush(CopyPool& pool) {
    cudaError_t first = cudaSuccess;
    for (int i = 0; i < kSlots; ++i) {
      const cudaError_t e = release((next_ + i) % kSlots, pool);
      if (e != cudaSuccess && first == cudaSuccess) first = e;
    }
    return first;
  }

  size_t block_bytes() const { return kBlock; }

  // After a failed call: forget what was in flight (the streams have been synchronised).
  void abandon() {
    for (int i = 0; i < kSlots; ++i) {
      busy_[i] = false;
      out_bytes_[i] = 0;
    }
  }

 private:
  uint8_t* block(int slot) const { return base_ + static_cast<size_t>(slot) * kBlock; }
  cudaError_t release(int slot, CopyPool& pool) {
    if (!busy_[slot]) return cudaSuccess;
    const cudaError_t e = cudaEventSynchronize(events_[slot]);
    if (e == cudaSuccess && out_bytes_[slot]) pool.copy(out_dst_[slot], block(slot), out_bytes_[slot]);
    busy_[slot] = false;
    out_bytes_[slot] = 0;
    return e;
  }
  cudaError_t acquire(int* slot, CopyPool& pool) {
    *slot = next_;
    next_ = (next_ + 1) % kSlots;
    return release(*slot, pool);
  }

  size_t kBlock = 8u << 20;  // bytes per slot
  uint8_t* base_ = nullptr;
  cudaEvent_t events_[kSlots] = {};
  bool busy_[kSlots] = {};
  uint8_t* out_dst_[kSlots] = {};
  size_t out_bytes_[kSlots] = {};
  int next_ = 0;
};

struct BounceCache {  // one ring per (calling thread, device): pinned memory is per context
  std::vector<std::unique_ptr<BounceRing>> per_device;
};
inline thread_local BounceCache t_bounce;

// Host <-> device copies of one call: straight cudaMemcpyAsync for pinned memory, through the
// bounce ring for pageable memory that is large enough to matter.
class HostIo {
 public:
  // `*_bytes`: what the call will move in total per buffer (decides whether staging pays).
  // `meta` is the offset / length tables of the variable-length entry (one allocation or two:
  // the first one's kind is taken for both).
  cudaError_t init(const void* in, uint64_t in_bytes, const void* out, uint64_t out_bytes,
                   const void* meta = nullptr, uint64_t meta_bytes = 0) {
    static const bool disabled = std::getenv("B200SHA3_NO_BOUNCE") != nullptr;
    static const uint64_t kBounceMinBytes = std::max<uint64_t>(1, env_kib("B200SHA3_BOUNCE_MIN_KIB", 4u << 20));
    bounce_in_ = !disabled && in && in_bytes >= kBounceMinBytes && is_pageable(in);
    bounce_out_ = !disabled && out && out_bytes >= kBounceMinBytes && is_pageable(out);
    bounce_meta_ = !disabled && meta && meta_bytes >= kBounceMinBytes && is_pageable(meta);
    if (!bounce_in_ && !bounce_out_ && !bounce_meta_) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= static_cast<int>(t_bounce.per_device.size())) t_bounce.per_device.resize(dev + 1);
    if (!t_bounce.per_device[dev]) t_bounce.per_device[dev] = std::make_unique<BounceRing>();
    ring_ = t_bounce.per_device[dev].get();
    e = ring_->init();
    if (e != cudaSuccess) {  // no pinned memory to be had: fall back to the driver's staging
      cudaGetLastError();
      t_bounce.per_device[dev].reset();
      ring_ = nullptr;
      bounce_in_ = bounce_out_ = bounce_meta_ = false;
      return cudaSuccess;
    }
    const unsigned hw = std::thread::hardware_concurrency();  // helpers + the caller: half the cores, <= 8
    pool_ = std::make_unique<CopyPool>(hw >= 4 ? std::min(7u, hw / 2 - 1) : 0u,
                                       std::min<size_t>(1u << 20, ring_->block_bytes()));
    return cudaSuccess;
  }

  cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
    if (!bounce_in_) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream);
    return ring_->h2d(dst, src, bytes, stream, *pool_);
  }
  cudaError_t h2d_meta(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
    if (!bounce_meta_) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream);
    return ring_->h2d(dst, src, bytes, stream, *pool_);
  }
  cudaError_t d2h(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
    if (!bounce_out_) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream);
    return ring_->d2h(dst, src, bytes, stream, *pool_);
  }
  // After the streams have drained: deliver what is still in the ring.
  cudaError_t finish(bool ok) {
    if (!ring_) return cudaSuccess;
    if (!ok) {
      ring_->abandon();
      return cudaSuccess;
    }
    return ring_->flush(*pool_);
  }

 private:
  bool bounce_in_ = false, bounce_out_ = false, bounce_meta_ = false;
  BounceRing* ring_ = nullptr;
  std::unique_ptr<CopyPool> pool_;
};

}  // namespace b200sha3::capi
