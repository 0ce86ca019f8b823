// oracle/ref_shim.cpp -- C entry points over the compiled reference library.
//
// TEST INFRASTRUCTURE ONLY (see oracle/keccak_oracle.c header).  Built by
// oracle/Makefile into oracle/_ref/libsha3kit_ref.so together with the
// reference's own translation units, compiled from /root/reference where they
// lie.  Used (a) to validate the C restatement in keccak_oracle.c, and (b) as
// the CPU baseline (`cpu_baseline.kind = "reference"`) in bench.py.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <new>
#include <stdexcept>
#include <vector>

#include "sha3/batch.hpp"
#include "sha3/keccak.hpp"
#include "sha3/sha3.hpp"
#include "workload.hpp"

#ifndef REF_HASH_INTO  // (the hash_into build replaces the call instead, see ref_prelude.hpp)
namespace sha3 {
// The function batch.cpp:108 expects (see ref_prelude.hpp).  It is the
// reference's one-shot path, which performs the same update/finish/squeeze
// sequence as hash_into (batch.cpp:15-25).
std::vector<std::uint8_t> hash_one(const HashBatch& batch,
                                   const std::vector<std::uint8_t>& message) {
  if (variant_info(batch.algorithm).is_xof()) {
    return shake(batch.algorithm, message, batch.xof_output_bits);
  }
  return sha3_digest(batch.algorithm, message);
}
}  // namespace sha3
#endif

namespace {

sha3::HashBatch* make_batch(int algorithm, const std::uint8_t* data,
                            const std::uint64_t* offsets, const std::uint64_t* lengths,
                            std::uint64_t fixed_len, std::uint64_t count,
                            std::uint64_t xof_bits) {
  auto* batch = new sha3::HashBatch;
  batch->algorithm = static_cast<sha3::Algorithm>(algorithm);
  batch->xof_output_bits = xof_bits;
  batch->messages.resize(count);
  for (std::uint64_t i = 0; i < count; ++i) {
    const std::uint64_t off = offsets ? offsets[i] : i * fixed_len;
    const std::uint64_t len = lengths ? lengths[i] : fixed_len;
    batch->messages[i].assign(data + off, data + off + len);
  }
  return batch;
}

int run_batch(const sha3::HashBatch& batch, int backend, unsigned workers,
              std::uint64_t chunk, std::uint8_t* out, double* elapsed) {
  try {
    sha3::EngineConfig cfg;
    cfg.backend = backend == 0 ? sha3::Backend::sequential : sha3::Backend::parallel;
    cfg.workers = workers;
    cfg.chunk_size = chunk;
    const sha3::BatchResult res = sha3::hash_batch(batch, cfg);
    if (elapsed) *elapsed = res.elapsed.count();
    if (out) {
      std::uint8_t* p = out;
      for (const auto& d : res.digests) {
        std::memcpy(p, d.data(), d.size());
        p += d.size();
      }
    }
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (...) {
    return 2;
  }
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) void* ref_batch_create(
    int algorithm, const std::uint8_t* data, const std::uint64_t* offsets,
    const std::uint64_t* lengths, std::uint64_t fixed_len, std::uint64_t count,
    std::uint64_t xof_bits) {
  try {
    return make_batch(algorithm, data, offsets, lengths, fixed_len, count, xof_bits);
  } catch (...) {
    return nullptr;
  }
}

__attribute__((visibility("default"))) int ref_batch_run(void* handle, int backend,
                                                         unsigned workers,
                                                         std::uint64_t chunk,
                                                         std::uint8_t* out,
                                                         double* elapsed) {
  if (!handle) return 2;
  return run_batch(*static_cast<sha3::HashBatch*>(handle), backend, workers, chunk, out,
                   elapsed);
}

// Wall clock of the reference's hash_batch call alone (slot allocation, batch.cpp:77-81,
// included; the result's destruction excluded) next to BatchResult::elapsed.
__attribute__((visibility("default"))) int ref_batch_run_wall(void* handle, unsigned workers,
                                                              double* call_wall,
                                                              double* elapsed) {
  if (!handle) return 2;
  try {
    sha3::EngineConfig cfg;
    cfg.backend = sha3::Backend::parallel;
    cfg.workers = workers;
    const auto t0 = std::chrono::steady_clock::now();
    const sha3::BatchResult res = sha3::hash_batch(*static_cast<sha3::HashBatch*>(handle), cfg);
    if (call_wall) {
      *call_wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    if (elapsed) *elapsed = res.elapsed.count();
    return 0;
  } catch (...) {
    return 2;
  }
}

__attribute__((visibility("default"))) void ref_batch_destroy(void* handle) {
  delete static_cast<sha3::HashBatch*>(handle);
}

// 0 ok, 1 std::invalid_argument, 2 anything else.
__attribute__((visibility("default"))) int ref_hash_batch(
    int algorithm, const std::uint8_t* data, const std::uint64_t* offsets,
    const std::uint64_t* lengths, std::uint64_t fixed_len, std::uint64_t count,
    std::uint64_t xof_bits, std::uint8_t* out, int backend, unsigned workers,
    std::uint64_t chunk, double* elapsed) {
  sha3::HashBatch* batch = nullptr;
  try {
    batch = make_batch(algorithm, data, offsets, lengths, fixed_len, count, xof_bits);
  } catch (...) {
    return 2;
  }
  const int rc = run_batch(*batch, backend, workers, chunk, out, elapsed);
  delete batch;
  return rc;
}

__attribute__((visibility("default"))) int ref_one_shot(int algorithm,
                                                        const std::uint8_t* msg,
                                                        std::uint64_t len,
                                                        std::uint64_t xof_bits,
                                                        std::uint8_t* out) {
  try {
    const auto a = static_cast<sha3::Algorithm>(algorithm);
    const std::span<const std::uint8_t> m(msg, len);
    const std::vector<std::uint8_t> d =
        sha3::variant_info(a).is_xof() ? sha3::shake(a, m, xof_bits) : sha3::sha3_digest(a, m);
    std::memcpy(out, d.data(), d.size());
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (...) {
    return 2;
  }
}

__attribute__((visibility("default"))) void ref_permute_1600(std::uint64_t* lanes) {
  std::array<std::uint64_t, 25> a;
  std::memcpy(a.data(), lanes, sizeof a);
  sha3::permute_1600(a, sha3::round_constants_1600());
  std::memcpy(lanes, a.data(), sizeof a);
}

__attribute__((visibility("default"))) std::uint64_t ref_generate_workload(
    std::uint64_t seed, std::uint64_t total_bytes, std::uint64_t message_size,
    std::uint8_t* out) {
  try {
    sha3::bench::WorkloadSpec spec;
    spec.message_size = message_size;
    spec.seed = seed;
    const sha3::HashBatch batch = sha3::bench::generate_workload(spec, total_bytes);
    std::uint8_t* p = out;
    for (const auto& m : batch.messages) {
      std::memcpy(p, m.data(), m.size());
      p += m.size();
    }
    return batch.messages.size();
  } catch (...) {
    return 0;
  }
}

__attribute__((visibility("default"))) unsigned ref_hardware_workers() {
  return sha3::resolve_workers(sha3::EngineConfig{});
}

}  // extern "C"
