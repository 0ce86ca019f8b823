// tests/cpp/fake_device_capi.cpp -- TEST DOUBLE for libb200sha3.so.  NOT part of the product
// and never linked into it: it exists so that the HOST-side scheduling of the C++ adapter
// (host/batch_adapter.cpp: scan, chunk plan, pinned ring, pack / device-call / unpack tasks,
// restart, error propagation) can run under ThreadSanitizer / AddressSanitizer on a machine
// without a GPU.  Every "device call" is answered by the CPU oracle (oracle/liboracle.so),
// which only test code may link.  Built only by tests/cpp/Makefile into fuzz_batch_adapter_san.
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "b200sha3.h"

extern "C" int ko_hash_one(int algorithm, std::uint64_t xof_bits, const std::uint8_t* msg,
                           std::uint64_t len, std::uint8_t* out);
extern "C" std::uint64_t ko_digest_bytes(int algorithm, std::uint64_t xof_bits);
extern "C" unsigned ko_rate_bytes(int algorithm);

namespace {
std::atomic<long> g_calls{0};
std::atomic<long> g_fail_at{-1};  // the n-th compute call fails with ERR_CUDA (fault injection)

int fake_device_ok(const b200sha3_config* cfg) {
  if (cfg && cfg->device > 7) return B200SHA3_ERR_CUDA;  // "no such device"
  const long n = g_calls.fetch_add(1);
  return n == g_fail_at.load() ? B200SHA3_ERR_CUDA : B200SHA3_OK;
}
}  // namespace

extern "C" {

void fake_device_fail_at(long nth_call_from_now) {
  g_fail_at.store(nth_call_from_now < 0 ? -1 : g_calls.load() + nth_call_from_now);
}

uint64_t b200sha3_digest_bytes(int algorithm, uint64_t xof_output_bits) {
  return algorithm < 0 || algorithm > 5 ? 0 : ko_digest_bytes(algorithm, xof_output_bits);
}
uint32_t b200sha3_rate_bytes(int algorithm) {
  return algorithm < 0 || algorithm > 5 ? 0 : ko_rate_bytes(algorithm);
}
const char* b200sha3_strerror(int status) { return status == B200SHA3_OK ? "ok" : "fake device error"; }
const char* b200sha3_last_cuda_error(void) { return "injected"; }
int b200sha3_device_count(void) { return 1; }
int b200sha3_current_device(void) { return 0; }

int b200sha3_pinned_alloc(uint64_t bytes, void** out) {
  *out = std::malloc(bytes ? bytes : 1);  // fresh, unaligned-to-page memory: ASan sees overruns
  return *out ? B200SHA3_OK : B200SHA3_ERR_CUDA;
}
int b200sha3_pinned_free(void* ptr) {
  std::free(ptr);
  return B200SHA3_OK;
}

// The incremental entries are not part of what the sanitizer build exercises.
int b200sha3_states_create(int, uint64_t, const b200sha3_config*, b200sha3_states** out) {
  if (out) *out = nullptr;
  return B200SHA3_ERR_CUDA;
}
int b200sha3_states_destroy(b200sha3_states*) { return B200SHA3_OK; }
int b200sha3_states_reset(b200sha3_states*, const b200sha3_config*) { return B200SHA3_ERR_CUDA; }
int b200sha3_states_update(b200sha3_states*, const uint8_t*, const uint64_t*, const uint64_t*,
                           const b200sha3_config*) { return B200SHA3_ERR_CUDA; }
int b200sha3_states_update_fixed(b200sha3_states*, const uint8_t*, uint64_t, const b200sha3_config*) {
  return B200SHA3_ERR_CUDA;
}
int b200sha3_states_finish(b200sha3_states*, uint64_t, uint8_t*, const b200sha3_config*) {
  return B200SHA3_ERR_CUDA;
}
int b200sha3_states_squeeze(b200sha3_states*, uint64_t, uint8_t*, const b200sha3_config*) {
  return B200SHA3_ERR_CUDA;
}

int b200sha3_hash_fixed(int algorithm, const uint8_t* data, uint64_t msg_len, uint64_t count,
                        uint64_t xof_output_bits, uint8_t* digests, const b200sha3_config* cfg) {
  if (const int rc = fake_device_ok(cfg)) return rc;
  const uint64_t db = b200sha3_digest_bytes(algorithm, xof_output_bits);
  const uint8_t none = 0;
  for (uint64_t i = 0; i < count; ++i) {
    ko_hash_one(algorithm, xof_output_bits, msg_len ? data + i * msg_len : &none, msg_len, digests + i * db);
  }
  if (cfg && cfg->device_ms) *cfg->device_ms = 0.001;
  return B200SHA3_OK;
}

int b200sha3_hash_batch(int algorithm, const uint8_t* data, const uint64_t* offsets,
                        const uint64_t* lengths, uint64_t count, uint64_t xof_output_bits,
                        uint8_t* digests, const b200sha3_config* cfg) {
  if (const int rc = fake_device_ok(cfg)) return rc;
  const uint64_t db = b200sha3_digest_bytes(algorithm, xof_output_bits);
  const uint8_t none = 0;
  for (uint64_t i = 0; i < count; ++i) {
    ko_hash_one(algorithm, xof_output_bits, lengths[i] ? data + offsets[i] : &none, lengths[i],
                digests + i * db);
  }
  if (cfg && cfg->device_ms) *cfg->device_ms = 0.001;
  return B200SHA3_OK;
}

}  // extern "C"
