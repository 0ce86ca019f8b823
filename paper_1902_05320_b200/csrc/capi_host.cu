// capi_host.cu -- the host-buffer entries of the C ABI (the hash_batch drop-in proper):
// chunked copy / compute pipelines over the device paths of capi.cu, and the pinned
// staging allocator.
#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

#include "capi_common.cuh"
#include "host_io.cuh"

using namespace b200sha3;
using namespace b200sha3::capi;

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

// A chunk must also carry enough MESSAGES: for long messages the byte target grows until a chunk
// holds ~2^11 of them, up to 1 GiB (three slots of that are still < 2 % of the HBM).  2^11, not
// more: a chunk of a few thousand multi-block messages runs on the warp-per-state kernel at
// ~2-4 us per block, which is about what its copy takes up to ~64 KiB per message (so copy and
// hashing of consecutive chunks overlap); round 1 grew chunks to 2^16 messages for the
// one-message-per-thread kernel and 2^14 x 64 KiB went through as ONE chunk, copy then hash.
// Beyond ~64 KiB per message a chunk is latency bound whatever it holds, and the 1 GiB cap
// (or hash_fixed_in_pieces below, for a whole batch of few long messages) applies.
uint64_t chunk_target_bytes(uint64_t avg_message_bytes) {
  static const long env_mib = [] {
    const char* env = std::getenv("B200SHA3_CHUNK_MIB");
    return env ? std::atol(env) : 0L;
  }();
  if (env_mib > 0) return static_cast<uint64_t>(env_mib) << 20;
  const uint64_t base = 64ull << 20, cap = 1ull << 30;
  const uint64_t want = avg_message_bytes > (cap >> 11) ? cap : avg_message_bytes << 11;
  return std::min(std::max(want, base), cap);
}

// Three pipeline slots, each a stream plus the device buffers of the chunk it currently
// carries.  Work of one chunk is enqueued on one slot's stream (H2D copy, kernels, D2H copy);
// consecutive chunks use different slots, so with pinned host memory the H2D copy of chunk
// k+1, the kernels of chunk k and the D2H copy of chunk k-1 overlap.  Stream order makes a
// slot's buffers safe to reuse without extra synchronisation.
class SlotPipeline {
 public:
  SlotPipeline(int slots, bool timed) : slots_(slots), timed_(timed) {}
  SlotPipeline(const SlotPipeline&) = delete;
  SlotPipeline& operator=(const SlotPipeline&) = delete;

  ~SlotPipeline() {
    for (int s = 0; s < slots_; ++s) {
      if (!streams_[s]) continue;
      for (void* p : buffers_[s]) cudaFreeAsync(p, streams_[s]);
      cudaStreamSynchronize(streams_[s]);
      if (start_[s]) cudaEventDestroy(start_[s]);
      if (stop_[s]) cudaEventDestroy(stop_[s]);
    }
  }

  cudaError_t init() {
    for (int s = 0; s < slots_; ++s) {
      cudaError_t e = t_streams.get(s, &streams_[s]);
      if (e == cudaSuccess && timed_) {
        e = cudaEventCreate(&start_[s]);
        if (e == cudaSuccess) e = cudaEventCreate(&stop_[s]);
      }
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }

  int slots() const { return slots_; }
  cudaStream_t stream(int s) const { return streams_[s]; }

  // Stream-ordered device buffer owned by slot s until the pipeline is destroyed.
  template <class T>
  cudaError_t alloc(int s, T** out, uint64_t bytes) {
    void* p = nullptr;
    // whole 16-byte units: the kernels read the aligned 4-byte words that hold message bytes
    cudaError_t e = cudaMallocAsync(&p, (std::max<uint64_t>(bytes, 16) + 15) & ~uint64_t{15}, streams_[s]);
    if (e == cudaSuccess) buffers_[s].push_back(p);
    *out = static_cast<T*>(p);
    return e;
  }

  // Bracket the hashing kernels of the chunk on slot s (cfg->device_ms accounting: copies
  // are outside, like slot allocation is outside the reference's timed region).
  cudaError_t begin_kernels(int s) {
    if (!timed_) return cudaSuccess;
    if (pending_[s]) {  // the events are about to be reused: collect the previous chunk first
      cudaError_t e = harvest(s);
      if (e != cudaSuccess) return e;
    }
    return cudaEventRecord(start_[s], streams_[s]);
  }
  cudaError_t end_kernels(int s) {
    if (!timed_) return cudaSuccess;
    pending_[s] = true;
    return cudaEventRecord(stop_[s], streams_[s]);
  }

  // Waits for everything enqueued; returns the summed kernel time through *kernel_ms.
  cudaError_t drain(double* kernel_ms) {
    cudaError_t first = cudaSuccess;
    for (int s = 0; s < slots_; ++s) {
      if (!streams_[s]) continue;
      cudaError_t e = cudaStreamSynchronize(streams_[s]);
      if (e == cudaSuccess && pending_[s]) e = harvest(s);
      if (e != cudaSuccess && first == cudaSuccess) first = e;
    }
    if (kernel_ms) *kernel_ms = kernel_ms_;
    return first;
  }

 private:
  cudaError_t harvest(int s) {
    cudaError_t e = cudaEventSynchronize(stop_[s]);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, start_[s], stop_[s]);
    if (e == cudaSuccess) kernel_ms_ += ms;
    pending_[s] = false;
    return e;
  }

  int slots_;
  bool timed_;
  cudaStream_t streams_[kPipelineSlots] = {};
  cudaEvent_t start_[kPipelineSlots] = {}, stop_[kPipelineSlots] = {};
  bool pending_[kPipelineSlots] = {};
  std::vector<void*> buffers_[kPipelineSlots];
  double kernel_ms_ = 0.0;
};



struct HostChunk {
  uint64_t first, count;  // message range
  uint64_t lo, hi;        // byte range of `data` the chunk reads (lo is 16-byte aligned)
  BatchHints hints;       // what the planner saw while reading the chunk's offsets / lengths
};

// One chunk holding the whole batch: the byte range [lo, hi) that its messages touch.
HostChunk whole_batch_chunk(const uint64_t* offsets, const uint64_t* lengths, uint64_t count,
                            uint64_t rate_bytes) {
  uint64_t lo = ~0ull, hi = 0, misaligned = 0, max_len = 0;
  bool equal = true;
  for (uint64_t i = 0; i < count; ++i) {
    misaligned |= offsets[i];
    max_len = std::max(max_len, lengths[i]);
    equal = equal && lengths[i] == lengths[0];
    if (lengths[i] == 0) continue;
    lo = std::min(lo, offsets[i]);
    hi = std::max(hi, offsets[i] + lengths[i]);
  }
  if (hi == 0) lo = 0;
  HostChunk ch{0, count, lo & ~15ull, hi, {}};  // device copy congruent to the host buffer mod 16
  ch.hints.aligned8 = (misaligned & 7u) == 0;
  ch.hints.all_short = max_len < rate_bytes;
  ch.hints.all_equal = equal;
  return ch;
}

// Chunks of a packed batch, planned one at a time while the previous ones are already in
// flight (reading 16 bytes of offsets / lengths per message for the whole batch first would
// cost a 2^24-message call ~30 ms before its first copy).  Messages in order and not
// overlapping -- what the C++ adapter and every sane caller produce -- are cut at
// `target_bytes`; from the first message that breaks the order on, the rest of the batch is
// one chunk (one copy of the byte range it touches).
class ChunkPlanner {
 public:
  ChunkPlanner(const uint64_t* offsets, const uint64_t* lengths, uint64_t count, uint64_t target_bytes,
               uint64_t rate_bytes, bool pipelined)
      : offsets_(offsets), lengths_(lengths), count_(count), target_(target_bytes), rate_(rate_bytes),
        pipelined_(pipelined) {}

  bool next(HostChunk* out) {
    if (next_ >= count_) return false;
    if (!pipelined_) return rest(out);
    HostChunk cur{next_, 0, 0, 0, {}};
    uint64_t misaligned = 0, max_len = 0;
    const uint64_t first_len = lengths_[next_];
    bool equal = true;
    const auto close = [&](uint64_t resume_at) {
      cur.hints.aligned8 = (misaligned & 7u) == 0;
      cur.hints.all_short = max_len < rate_;
      cur.hints.all_equal = equal;
      *out = cur;
      next_ = resume_at;
      return true;
    };
    // Strips of kStrip messages: the in-order test and the statistics of a strip are plain
    // reductions without early exits (this loop reads 16 bytes per message and, for 2^24 short
    // messages, is what the copy engines wait for).  A strip that is not in order, holds an
    // empty message (whose offset means nothing and must not widen the byte range) or would
    // overshoot the byte target (long messages) is walked message by message instead.
    bool have_bytes = false;
    uint64_t i = next_;
    while (i < count_) {
      const uint64_t n = std::min<uint64_t>(kStrip, count_ - i);
      const uint64_t* off = offsets_ + i;
      const uint64_t* len = lengths_ + i;
      uint64_t bad = (off[0] < prev_end_) | (off[0] + len[0] < off[0]) | (len[0] == 0);
      uint64_t strip_or = off[0], strip_max = len[0], strip_ne = len[0] ^ first_len;
      for (uint64_t k = 1; k < n; ++k) {
        const uint64_t end_before = off[k - 1] + len[k - 1];
        bad |= (off[k] < end_before) | (off[k] + len[k] < off[k]) | (len[k] == 0);
        strip_or |= off[k];
        strip_max = std::max(strip_max, len[k]);
        strip_ne |= len[k] ^ first_len;
      }
      if (!bad) {
        const uint64_t lo = have_bytes ? cur.lo : off[0] & ~15ull;
        bad = off[n - 1] + len[n - 1] - lo > target_ + target_ / 4;  // close inside the strip
      }
      if (!bad) {
        if (!have_bytes) cur.lo = off[0] & ~15ull;
        have_bytes = true;
        cur.count += n;
        cur.hi = off[n - 1] + len[n - 1];
        prev_end_ = cur.hi;
        misaligned |= strip_or;
        max_len = std::max(max_len, strip_max);
        equal = equal && strip_ne == 0;
        i += n;
      } else {
        for (const uint64_t strip_end = i + n; i < strip_end; ++i) {
          const uint64_t length = lengths_[i], end = offsets_[i] + length;
          equal = equal && length == first_len;
          if (length == 0) {  // belongs to the chunk, touches no byte of `data`
            cur.count += 1;
            continue;
          }
          if (offsets_[i] < prev_end_ || end < offsets_[i]) {  // out of order (or wrapping)
            if (cur.count == 0) return rest(out);
            return close(i);  // close the chunk in progress; the next call takes the rest
          }
          if (!have_bytes) cur.lo = offsets_[i] & ~15ull;
          have_bytes = true;
          cur.count += 1;
          cur.hi = end;
          prev_end_ = end;
          misaligned |= offsets_[i];
          max_len = std::max(max_len, length);
          if (cur.hi - cur.lo >= target_) return close(i + 1);
        }
      }
      if ((have_bytes && cur.hi - cur.lo >= target_) || cur.count >= (1ull << 22)) return close(i);
    }
    return close(count_);
  }

 private:
  bool rest(HostChunk* out) {
    *out = whole_batch_chunk(offsets_ + next_, lengths_ + next_, count_ - next_, rate_);
    out->first = next_;
    next_ = count_;
    return true;
  }
  const uint64_t* offsets_;
  const uint64_t* lengths_;
  static constexpr uint64_t kStrip = 1024;
  uint64_t count_, target_, rate_;
  bool pipelined_;
  uint64_t next_ = 0, prev_end_ = 0;
};

int finish_call(int rc, SlotPipeline& pipe, HostIo& io, const Config& c, uint32_t launches) {
  double kernel_ms = 0.0;
  cudaError_t e = pipe.drain(&kernel_ms);
  if (rc == B200SHA3_OK && e != cudaSuccess) rc = cuda_fail(e, "pipeline drain");
  e = io.finish(rc == B200SHA3_OK);
  if (rc == B200SHA3_OK && e != cudaSuccess) rc = cuda_fail(e, "digest delivery");
  if (rc != B200SHA3_OK) {
    cudaGetLastError();
    return rc;
  }
  if (c.device_ms) *c.device_ms = kernel_ms;
  if (c.kernel_launches) *c.kernel_launches = launches;
  return B200SHA3_OK;
}

// Few LONG equal-length messages from pinned host memory: the batch is latency bound (a sponge is
// sequential per message; the warp-per-state kernels need ~2 us per block whatever the count),
// so cutting it into chunks of MESSAGES only lines the chunks' latencies up behind one another.
// Cut every message into PIECES instead: piece k of all messages is one strided copy
// (cudaMemcpy2DAsync: pitch = message length), absorbed into device-resident sponge states by
// the incremental warp kernel (kernel_stream_warp.cu) while piece k + 1 is on the link.  The call
// then costs max(copy, hashing) + one piece instead of copy + hashing (1024 x 1 MiB: 36 -> 22 ms).
// Pieces are whole rate blocks, so every update leaves the byte position at 0.
int hash_fixed_in_pieces(int algorithm, const uint8_t* data, uint64_t msg_len, uint64_t count,
                         uint64_t xof_output_bits, uint64_t digest_bytes, uint8_t* digests, const Config& c) {
  const Variant& v = kVariants[algorithm];
  const uint64_t rate = 8u * static_cast<uint64_t>(v.rate_lanes);
  // ~16 pieces per message, at least 64 KiB each (a piece is one launch: >= ~1 ms of hashing), at
  // most 256 MiB per piece of the whole batch (three device buffers of that size)
  uint64_t piece = std::max<uint64_t>(64u << 10, msg_len / 16);
  if (count * piece > (256ull << 20)) piece = std::max<uint64_t>(64u << 10, (256ull << 20) / count);
  piece = std::max<uint64_t>(rate, piece / rate * rate);
  const uint64_t pieces = (msg_len + piece - 1) / piece;
  SlotPipeline pipe(kPipelineSlots, /*timed=*/false);  // (kernel time: own events, below)
  CU(pipe.init());
  HostIo io;
  CU(io.init(nullptr, 0, digests, count * digest_bytes));
  uint8_t* d_piece[kPipelineSlots] = {};
  for (int s = 0; s < pipe.slots(); ++s) CU(pipe.alloc(s, &d_piece[s], count * piece));
  uint2* lanes = nullptr;
  uint32_t* pos = nullptr;
  uint8_t* d_out = nullptr;
  CU(pipe.alloc(0, &lanes, 25 * count * sizeof(uint2)));
  CU(pipe.alloc(0, &pos, count * sizeof(uint32_t)));
  CU(pipe.alloc(0, &d_out, count * digest_bytes));
  CU(cudaMemsetAsync(lanes, 0, 25 * count * sizeof(uint2), pipe.stream(0)));
  CU(cudaMemsetAsync(pos, 0, count * sizeof(uint32_t), pipe.stream(0)));
  // updates run in piece order: each waits for the event of the one before it.  Kernel time
  // (cfg->device_ms) is bracketed per piece with its own event pair, collected after the drain:
  // the slots' shared pairs would make the host wait for piece k - 3 before it may enqueue piece k.
  // (Beyond 512 pieces one pair brackets the whole run of updates instead: copy waits included.)
  const bool timed = c.device_ms != nullptr;
  const bool per_piece = timed && pieces <= 512;
  const uint64_t brackets = !timed ? 0 : per_piece ? pieces + 1 : 1;
  std::vector<cudaEvent_t> events(pipe.slots() + 2 * brackets, nullptr);
  struct EventGuard {
    std::vector<cudaEvent_t>& e;
    ~EventGuard() {
      for (cudaEvent_t ev : e) {
        if (ev) cudaEventDestroy(ev);
      }
    }
  } guard{events};
  for (size_t i = 0; i < events.size(); ++i) {
    CU(cudaEventCreateWithFlags(&events[i], i < static_cast<size_t>(pipe.slots()) ? cudaEventDisableTiming : cudaEventDefault));
  }
  cudaEvent_t* hashed = events.data();
  cudaEvent_t* bracket = events.data() + pipe.slots();
  CU(cudaEventRecord(hashed[pipe.slots() - 1], pipe.stream(0)));  // "piece -1": the states are zeroed
  int rc = B200SHA3_OK;
  uint32_t launches = 0;
  int last = 0;
  for (uint64_t k = 0; k < pieces && rc == B200SHA3_OK; ++k) {
    const int s = static_cast<int>(k % pipe.slots());
    const int before = static_cast<int>((k + pipe.slots() - 1) % pipe.slots());
    const uint64_t width = std::min(piece, msg_len - k * piece);
    cudaStream_t stream = pipe.stream(s);
    cudaError_t e = cudaMemcpy2DAsync(d_piece[s], width, data + k * piece, msg_len, width, count,
                                      cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, hashed[before], 0);
    if (e == cudaSuccess && (per_piece || (timed && k == 0))) e = cudaEventRecord(bracket[per_piece ? 2 * k : 0], stream);
    if (e == cudaSuccess) {
      e = launch_states_update_warp(v.rate_lanes, lanes, pos, count, d_piece[s], nullptr, nullptr, width, stream);
    }
    if (e == cudaSuccess && per_piece) e = cudaEventRecord(bracket[2 * k + 1], stream);
    if (e == cudaSuccess) e = cudaEventRecord(hashed[s], stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "piece pipeline");
    launches += 1;
    last = s;
  }
  if (rc == B200SHA3_OK) {
    cudaStream_t stream = pipe.stream(last);
    cudaError_t e = per_piece ? cudaEventRecord(bracket[2 * pieces], stream) : cudaSuccess;
    if (e == cudaSuccess) {
      e = launch_states_finish_warp(v.rate_lanes, lanes, pos, count, v.head, d_out, digest_bytes,
                                    last_byte_mask(algorithm, xof_output_bits), stream);
    }
    if (e == cudaSuccess && timed) e = cudaEventRecord(bracket[per_piece ? 2 * pieces + 1 : 1], stream);
    if (e == cudaSuccess) e = io.d2h(digests, d_out, count * digest_bytes, stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "piece pipeline");
    launches += 1;
  }
  rc = finish_call(rc, pipe, io, c, launches);  // drains the streams
  if (rc == B200SHA3_OK && timed) {
    double kernel_ms = 0.0;
    for (uint64_t k = 0; k < brackets; ++k) {
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, bracket[2 * k], bracket[2 * k + 1]));
      kernel_ms += ms;
    }
    *c.device_ms = kernel_ms;
  }
  return rc;
}

}  // namespace

extern "C" {

// Host entry, equal-length messages: chunks of ~64 MiB (input + output) through the slots.
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

  const bool pipelined = (c.flags & B200SHA3_FLAG_NO_PIPELINE) == 0;
  // few long messages (warp-per-state territory) from pinned memory: pipeline over PIECES of
  // the messages instead of over message ranges
  if (pipelined && few_enough_for_warps(count, c) && c.kernel == B200SHA3_KERNEL_AUTO && count >= 2 &&
      msg_len >= (256u << 10) && msg_len < (1ull << 31) && count * msg_len >= (64ull << 20) &&
      !is_pageable(data)) {
    return hash_fixed_in_pieces(algorithm, data, msg_len, count, xof_output_bits, digest_bytes, digests, c);
  }
  const uint64_t unit = std::max<uint64_t>(1, msg_len + digest_bytes);
  uint64_t chunk = pipelined ? chunk_target_bytes(unit) / unit : count;
  chunk = std::min(std::max<uint64_t>(chunk, 16), count);
  const uint64_t nchunks = (count + chunk - 1) / chunk;
  chunk = (count + nchunks - 1) / nchunks;  // equal chunks: no straggler of a few messages
  SlotPipeline pipe(chunk < count ? kPipelineSlots : 1, c.device_ms != nullptr);
  CU(pipe.init());
  HostIo io;
  CU(io.init(data, count * msg_len, digests, count * digest_bytes));
  uint8_t* d_in[kPipelineSlots] = {};
  uint8_t* d_out[kPipelineSlots] = {};
  for (int s = 0; s < pipe.slots(); ++s) {
    CU(pipe.alloc(s, &d_in[s], chunk * msg_len));
    CU(pipe.alloc(s, &d_out[s], chunk * digest_bytes));
  }
  int rc = B200SHA3_OK;
  uint32_t launches = 0;
  uint64_t done = 0;
  for (uint64_t k = 0; done < count && rc == B200SHA3_OK; ++k) {
    const int s = static_cast<int>(k % pipe.slots());
    const uint64_t n = std::min(chunk, count - done);
    cudaError_t e = cudaSuccess;
    if (msg_len) {
      e = io.h2d(d_in[s], data + done * msg_len, n * msg_len, pipe.stream(s));
    }
    if (e == cudaSuccess) e = pipe.begin_kernels(s);
    if (e != cudaSuccess) { rc = cuda_fail(e, "H2D copy"); break; }
    rc = run_fixed_device(algorithm, d_in[s], msg_len, n, xof_output_bits, digest_bytes, d_out[s],
                          c, pipe.stream(s), &launches);
    if (rc != B200SHA3_OK) break;
    e = pipe.end_kernels(s);
    if (e == cudaSuccess) {
      e = io.d2h(digests + done * digest_bytes, d_out[s], n * digest_bytes, pipe.stream(s));
    }
    if (e != cudaSuccess) { rc = cuda_fail(e, "D2H copy"); break; }
    done += n;
  }
  return finish_call(rc, pipe, io, c, launches);
}

// Host entry, variable-length messages.  A packed batch is cut into chunks of ~64 MiB of
// message bytes (each bucketed and hashed on its own); any other layout is one chunk: one
// copy of the byte range the batch touches, one device pass, one copy back.
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
  if (!data) {  // fine only if every message is empty; checked before any work
    for (uint64_t i = 0; i < count; ++i) {
      if (lengths[i] != 0) return B200SHA3_ERR_INVALID_ARGUMENT;
    }
  }

  // average message size of a packed batch: the span from the first to the last message
  const uint64_t span = offsets[count - 1] + lengths[count - 1] - std::min(offsets[0], offsets[count - 1]);
  const bool pipelined = (c.flags & B200SHA3_FLAG_NO_PIPELINE) == 0;
  ChunkPlanner planner(offsets, lengths, count, chunk_target_bytes(span / count + digest_bytes),
                       8u * kVariants[algorithm].rate_lanes, pipelined);

  DeviceGuard guard;
  CU(guard.enter(c.device));
  tune_mempool_once();
  if (c.stream) CU(cudaStreamSynchronize(c.stream));
  SlotPipeline pipe(pipelined ? kPipelineSlots : 1, c.device_ms != nullptr);
  CU(pipe.init());
  HostIo io;
  CU(io.init(data, span, digests, count * digest_bytes, offsets, 2 * count * sizeof(uint64_t)));
  // per-slot device buffers, grown when a chunk needs more (chunks are near-equal, so this
  // happens once per slot unless one message is huge)
  uint8_t* d_data[kPipelineSlots] = {};
  uint64_t* d_meta[kPipelineSlots] = {};  // offsets, then lengths
  uint8_t* d_out[kPipelineSlots] = {};
  uint64_t cap_data[kPipelineSlots] = {}, cap_count[kPipelineSlots] = {};
  int rc = B200SHA3_OK;
  uint32_t launches = 0;
  HostChunk ch{};
  for (size_t k = 0; rc == B200SHA3_OK && planner.next(&ch); ++k) {
    const int s = static_cast<int>(k % pipe.slots());
    cudaStream_t stream = pipe.stream(s);
    cudaError_t e = cudaSuccess;
    if (ch.hi - ch.lo > cap_data[s] || !d_data[s]) {
      cap_data[s] = (ch.hi - ch.lo) + (ch.hi - ch.lo) / 8;
      e = pipe.alloc(s, &d_data[s], cap_data[s]);
    }
    if (e == cudaSuccess && (ch.count > cap_count[s] || !d_meta[s])) {
      cap_count[s] = ch.count + ch.count / 8;
      e = pipe.alloc(s, &d_meta[s], 2 * cap_count[s] * sizeof(uint64_t));
      if (e == cudaSuccess) e = pipe.alloc(s, &d_out[s], cap_count[s] * digest_bytes);
    }
    if (e != cudaSuccess) { rc = cuda_fail(e, "device staging allocation"); break; }
    if (ch.hi > ch.lo) {
      e = io.h2d(d_data[s], data + ch.lo, ch.hi - ch.lo, stream);
    }
    if (e == cudaSuccess) {
      e = io.h2d_meta(d_meta[s], offsets + ch.first, ch.count * sizeof(uint64_t), stream);
    }
    if (e == cudaSuccess) {
      e = io.h2d_meta(d_meta[s] + ch.count, lengths + ch.first, ch.count * sizeof(uint64_t), stream);
    }
    if (e == cudaSuccess) e = pipe.begin_kernels(s);
    if (e != cudaSuccess) { rc = cuda_fail(e, "H2D copy"); break; }
    // offsets are relative to `data`; the device copy starts at data + ch.lo
    rc = run_batch_device(algorithm, d_data[s] - ch.lo, d_meta[s], d_meta[s] + ch.count, ch.count,
                          xof_output_bits, digest_bytes, d_out[s], c, stream, &launches, &ch.hints);
    if (rc != B200SHA3_OK) break;
    e = pipe.end_kernels(s);
    if (e == cudaSuccess) {
      e = io.d2h(digests + ch.first * digest_bytes, d_out[s], ch.count * digest_bytes, stream);
    }
    if (e != cudaSuccess) { rc = cuda_fail(e, "D2H copy"); break; }
  }
  return finish_call(rc, pipe, io, c, launches);
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
