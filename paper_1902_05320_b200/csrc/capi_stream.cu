// capi_stream.cu -- batched incremental hashing entries of the C ABI (b200sha3_states_*):
// handle management and the state machine of sha3::Hasher / SpongeHasher
// (proj/core/src/sha3.cpp:95-130, proj/core/src/sponge.cpp:81-143) over kernel_stream.cu.
#include <algorithm>
#include <new>
#include <vector>

#include "capi_common.cuh"
#include "host_io.cuh"

using namespace b200sha3;
using namespace b200sha3::capi;

struct b200sha3_states {
  int algorithm;
  int device;
  uint64_t count;
  void* lanes;      // 25 * count uint2, structure of arrays
  uint32_t* pos;    // count words
  bool finished;
};

// ---- host-buffer forms ---------------------------------------------------------------
// What a caller of sha3::Hasher holds is host memory.  These entries stage the chunk bytes
// (pinned: straight DMA; pageable: the bounce ring of host_io.cuh) into a stream-ordered
// scratch buffer, run the device form and return when the host buffers are free again
// (update) or filled (finish / squeeze).  One copy per call: the calls themselves are the
// chunking.

namespace {

// Device scratch of one call, returned to the stream-ordered pool at scope exit.
struct Scratch {
  cudaStream_t stream = nullptr;
  std::vector<void*> buffers;
  template <class T>
  cudaError_t alloc(T** out, uint64_t bytes) {
    void* p = nullptr;
    const cudaError_t e = cudaMallocAsync(&p, (std::max<uint64_t>(bytes, 16) + 15) & ~uint64_t{15}, stream);
    if (e == cudaSuccess) buffers.push_back(p);
    *out = static_cast<T*>(p);
    return e;
  }
  ~Scratch() {
    for (void* p : buffers) cudaFreeAsync(p, stream);
  }
};

int finish_host_call(int rc, cudaError_t e, const char* what, HostIo& io, cudaStream_t stream) {
  if (rc == B200SHA3_OK && e != cudaSuccess) rc = cuda_fail(e, what);
  const cudaError_t s = cudaStreamSynchronize(stream);
  if (rc == B200SHA3_OK && s != cudaSuccess) rc = cuda_fail(s, "stream synchronize");
  const cudaError_t f = io.finish(rc == B200SHA3_OK);
  if (rc == B200SHA3_OK && f != cudaSuccess) rc = cuda_fail(f, "digest delivery");
  if (rc != B200SHA3_OK) cudaGetLastError();
  return rc;
}

}  // namespace

// Shared tail of finish / squeeze on host buffers: run `device_form(d_out)`, bring out_len bytes
// per stream back to `out`.
template <class F>
static int states_output_host(b200sha3_states* st, uint64_t out_len, uint8_t* out,
                              const b200sha3_config* cfg, F device_form) {
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(st->device));
  tune_mempool_once();
  Scratch scratch;
  scratch.stream = c.stream;
  const uint64_t bytes = st->count * out_len;
  HostIo io;
  CU(io.init(nullptr, 0, out, bytes));
  uint8_t* d_out = nullptr;
  cudaError_t e = bytes ? scratch.alloc(&d_out, bytes) : cudaSuccess;
  int rc = B200SHA3_OK;
  if (e == cudaSuccess) {
    b200sha3_config inner = cfg ? *cfg : b200sha3_config{};
    inner.device = st->device;
    inner.device_ms = nullptr;
    rc = device_form(d_out, &inner);
    if (rc == B200SHA3_OK && bytes) e = io.d2h(out, d_out, bytes, c.stream);
  }
  return finish_host_call(rc, e, "states output (host)", io, c.stream);
}

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
  // few streams: one warp each (kernel_stream_warp.cu); the state layout is the same
  CU((few_enough_for_warps(st->count, c) ? launch_states_update_warp : launch_states_update)(
      kVariants[st->algorithm].rate_lanes, st->lanes, st->pos, st->count, d_data, d_offsets, d_lengths,
      fixed_len, c.stream));
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
  CU((few_enough_for_warps(st->count, c) ? launch_states_finish_warp : launch_states_finish)(
      v.rate_lanes, st->lanes, st->pos, st->count, v.head, d_digests, out_len,
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
  CU((few_enough_for_warps(st->count, c) ? launch_states_squeeze_warp : launch_states_squeeze)(
      kVariants[st->algorithm].rate_lanes, st->lanes, st->pos, st->count, d_out, out_bytes, c.stream));
  if (c.kernel_launches) *c.kernel_launches = 1;
  return B200SHA3_OK;
}


int b200sha3_states_update(b200sha3_states* st, const uint8_t* data, const uint64_t* offsets,
                           const uint64_t* lengths, const b200sha3_config* cfg) {
  if (!st || !offsets || !lengths) return B200SHA3_ERR_INVALID_ARGUMENT;
  if (st->finished) return B200SHA3_ERR_STATE;
  if (st->count == 0) return B200SHA3_OK;
  uint64_t lo = ~0ull, hi = 0;  // the byte range of `data` this round touches
  for (uint64_t i = 0; i < st->count; ++i) {
    if (lengths[i] == 0) continue;
    lo = std::min(lo, offsets[i]);
    hi = std::max(hi, offsets[i] + lengths[i]);
  }
  if (hi == 0) return B200SHA3_OK;  // every chunk is empty
  if (!data) return B200SHA3_ERR_INVALID_ARGUMENT;
  lo &= ~15ull;  // device copy congruent to the host buffer mod 16
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(st->device));
  tune_mempool_once();
  Scratch scratch;
  scratch.stream = c.stream;
  HostIo io;
  CU(io.init(data + lo, hi - lo, nullptr, 0, offsets, 2 * st->count * sizeof(uint64_t)));
  uint8_t* d_data = nullptr;
  uint64_t* d_meta = nullptr;
  cudaError_t e = scratch.alloc(&d_data, hi - lo);
  if (e == cudaSuccess) e = scratch.alloc(&d_meta, 2 * st->count * sizeof(uint64_t));
  if (e == cudaSuccess) e = io.h2d(d_data, data + lo, hi - lo, c.stream);
  if (e == cudaSuccess) e = io.h2d_meta(d_meta, offsets, st->count * sizeof(uint64_t), c.stream);
  if (e == cudaSuccess) e = io.h2d_meta(d_meta + st->count, lengths, st->count * sizeof(uint64_t), c.stream);
  int rc = B200SHA3_OK;
  if (e == cudaSuccess) {
    b200sha3_config inner = cfg ? *cfg : b200sha3_config{};
    inner.device = st->device;
    inner.device_ms = nullptr;
    rc = b200sha3_states_update_device(st, d_data - lo, d_meta, d_meta + st->count, &inner);
  }
  return finish_host_call(rc, e, "states update (host)", io, c.stream);
}

int b200sha3_states_update_fixed(b200sha3_states* st, const uint8_t* data, uint64_t chunk_len,
                                 const b200sha3_config* cfg) {
  if (!st) return B200SHA3_ERR_INVALID_ARGUMENT;
  if (st->finished) return B200SHA3_ERR_STATE;
  if (st->count == 0 || chunk_len == 0) return B200SHA3_OK;
  if (!data) return B200SHA3_ERR_INVALID_ARGUMENT;
  const Config c = resolve(cfg);
  DeviceGuard guard;
  CU(guard.enter(st->device));
  tune_mempool_once();
  Scratch scratch;
  scratch.stream = c.stream;
  const uint64_t bytes = st->count * chunk_len;
  HostIo io;
  CU(io.init(data, bytes, nullptr, 0));
  uint8_t* d_data = nullptr;
  cudaError_t e = scratch.alloc(&d_data, bytes);
  if (e == cudaSuccess) e = io.h2d(d_data, data, bytes, c.stream);
  int rc = B200SHA3_OK;
  if (e == cudaSuccess) {
    b200sha3_config inner = cfg ? *cfg : b200sha3_config{};
    inner.device = st->device;
    inner.device_ms = nullptr;
    rc = b200sha3_states_update_fixed_device(st, d_data, chunk_len, &inner);
  }
  return finish_host_call(rc, e, "states update (host)", io, c.stream);
}

int b200sha3_states_finish(b200sha3_states* st, uint64_t xof_output_bits, uint8_t* digests,
                           const b200sha3_config* cfg) {
  if (!st) return B200SHA3_ERR_INVALID_ARGUMENT;
  if (st->finished) return B200SHA3_ERR_STATE;
  const Variant& v = kVariants[st->algorithm];
  const uint64_t out_len = v.digest_bytes ? v.digest_bytes : (xof_output_bits + 7) / 8;
  if (out_len != 0 && !digests && st->count != 0) return B200SHA3_ERR_INVALID_ARGUMENT;
  return states_output_host(st, out_len, digests, cfg, [&](uint8_t* d_out, const b200sha3_config* inner) {
    return b200sha3_states_finish_device(st, xof_output_bits, d_out, inner);
  });
}

int b200sha3_states_squeeze(b200sha3_states* st, uint64_t out_bytes, uint8_t* out,
                            const b200sha3_config* cfg) {
  if (!st) return B200SHA3_ERR_INVALID_ARGUMENT;
  if (!st->finished || kVariants[st->algorithm].digest_bytes != 0) return B200SHA3_ERR_STATE;
  if (out_bytes == 0 || st->count == 0) return B200SHA3_OK;
  if (!out) return B200SHA3_ERR_INVALID_ARGUMENT;
  return states_output_host(st, out_bytes, out, cfg, [&](uint8_t* d_out, const b200sha3_config* inner) {
    return b200sha3_states_squeeze_device(st, out_bytes, d_out, inner);
  });
}

}  // extern "C"
