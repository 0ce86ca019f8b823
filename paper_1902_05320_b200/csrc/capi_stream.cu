// capi_stream.cu -- batched incremental hashing entries of the C ABI (b200sha3_states_*):
// handle management and the state machine of sha3::Hasher / SpongeHasher
// (proj/core/src/sha3.cpp:95-130, proj/core/src/sponge.cpp:81-143) over kernel_stream.cu.
#include <algorithm>
#include <new>

#include "capi_common.cuh"

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

}  // extern "C"
