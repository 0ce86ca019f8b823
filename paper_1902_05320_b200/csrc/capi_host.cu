// capi_host.cu -- the host-buffer entries of the C ABI (the hash_batch drop-in proper):
// chunked copy / compute pipelines over the device paths of capi.cu, and the pinned
// staging allocator.
#include <algorithm>
#include <cstdlib>
#include <utility>
#include <vector>

#include "capi_common.cuh"

using namespace b200sha3;
using namespace b200sha3::capi;

// Host entry, variable-length messages.
//
// Packed batches (offsets non-decreasing, messages not overlapping -- what the C++
// adapter and every sane caller produce) are cut into chunks of ~64 MiB of message bytes
// that cycle through three slots, each with its own stream, so that (with pinned host
// memory) the H2D copy of chunk k+1, the bucketing + hash kernels of chunk k and the D2H
// copy of chunk k-1 overlap.  Anything else takes one copy of the byte range the batch
// touches, one device pass, one copy back.
namespace {

// Pipeline chunk size (bytes of input + output per chunk).  64 MiB measured best on the
// B200 boxes; B200SHA3_CHUNK_MIB overrides it for experiments.
// Streams of the copy/compute pipeline, created once per (calling thread, device) and
// reused: creating and destroying three streams per call costs more than hashing a small
// batch.  A thread's streams are only ever used by that thread, so calls stay reentrant.
constexpr int kPipelineSlots = 3;

class StreamCache {
 public:
  cudaError_t get(int slot, cudaStream_t* out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= static_cast<int>(per_device_.size())) per_device_.resize(dev + 1);
    cudaStream_t& s = per_device_[dev].streams[slot];
    if (!s) {
      e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (e != cudaSuccess) return e;
    }
    *out = s;
    return cudaSuccess;
  }
  ~StreamCache() {
    for (auto& d : per_device_) {
      for (cudaStream_t s : d.streams) {
        if (s) cudaStreamDestroy(s);  // harmless error if the context is already gone
      }
    }
  }

 private:
  struct Entry {
    cudaStream_t streams[kPipelineSlots] = {};
  };
  std::vector<Entry> per_device_;
};

thread_local StreamCache t_streams;

uint64_t chunk_target_bytes() {
  static const uint64_t value = [] {
    const char* env = std::getenv("B200SHA3_CHUNK_MIB");
    const long mib = env ? std::atol(env) : 0;
    return static_cast<uint64_t>(mib > 0 ? mib : 64) << 20;
  }();
  return value;
}

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
  CU(t_streams.get(0, &s));
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
  constexpr int kSlots = kPipelineSlots;
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
    cudaError_t e = t_streams.get(s, &streams[s]);
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

  constexpr int kSlots = kPipelineSlots;
  const bool pipeline = (c.flags & B200SHA3_FLAG_NO_PIPELINE) == 0;
  const uint64_t per_msg = std::max<uint64_t>(1, msg_len + digest_bytes);
  uint64_t chunk = pipeline ? std::max<uint64_t>(1, chunk_target_bytes() / per_msg) : count;
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
    cudaError_t e = t_streams.get(s, &streams[s]);
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
  }
  if (rc != B200SHA3_OK) {
    cudaGetLastError();
    return rc;
  }
  if (c.device_ms) *c.device_ms = kernel_ms;
  if (c.kernel_launches) *c.kernel_launches = launches;
  return B200SHA3_OK;
}

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
                        plan_host_chunks(offsets, lengths, count, chunk_target_bytes(), &chunks) &&
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

}  // extern "C"
