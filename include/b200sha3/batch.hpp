// b200sha3/batch.hpp -- C++ adapter: the reference's batch interface over the
// B200 engine.
//
// Mirrors proj/core/include/sha3/batch.hpp:13-65 of the reference: the same
// HashBatch / BatchResult / EngineConfig shapes, the same contract for
// hash_batch (order preserved, digests[i] belongs to messages[i], XOF without a
// length throws std::invalid_argument before any work, empty batch -> empty
// result, blocking and reentrant).  What differs is where the work happens:
// messages are packed into one buffer, hashed by libb200sha3.so on the GPU
// through the C ABI (include/b200sha3.h), and unpacked.
//
// Two ways to use it:
//   * next to the reference's headers: define B200SHA3_USE_REFERENCE_TYPES
//     before including this file; it then includes the reference's own
//     "sha3/batch.hpp" and adds sha3::b200::hash_batch on those types;
//   * instead of them: the types below are layout- and name-compatible
//     declarations, and linking b200sha3_dropin.cpp (host/) provides
//     sha3::hash_batch itself, replacing proj/core/src/batch.cpp at link time.
#pragma once

#include <chrono>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "../b200sha3.h"

#ifdef B200SHA3_USE_REFERENCE_TYPES
#include "sha3/batch.hpp"
#else
namespace sha3 {

// Enum order is the C ABI's algorithm id (proj/core/include/sha3/sha3.hpp:15-22).
enum class Algorithm { sha3_224, sha3_256, sha3_384, sha3_512, shake128, shake256 };

enum class Backend { sequential, parallel };

// proj/core/include/sha3/batch.hpp:15-19.  On the GPU engine `workers` sizes the
// host-side pack/unpack thread pool (0 = one per hardware thread) and
// Backend::sequential keeps all host work on the calling thread; `chunk_size`
// has no device meaning and is accepted for compatibility.
struct EngineConfig {
  Backend backend = Backend::parallel;
  unsigned workers = 0;
  std::size_t chunk_size = 0;
};

// proj/core/include/sha3/batch.hpp:23-27
struct HashBatch {
  Algorithm algorithm = Algorithm::sha3_256;
  std::vector<std::vector<std::uint8_t>> messages;
  std::uint64_t xof_output_bits = 0;  // required for XOF variants
};

// proj/core/include/sha3/batch.hpp:29-34
struct BatchResult {
  std::vector<std::vector<std::uint8_t>> digests;  // digests[i] is the digest of messages[i]
  std::chrono::duration<double> elapsed{0};        // hashing phase only
};

}  // namespace sha3
#endif  // B200SHA3_USE_REFERENCE_TYPES

namespace sha3::b200 {

// Raised for CUDA failures and unsupported shapes (the C ABI's ERR_CUDA /
// ERR_UNSUPPORTED).  Invalid arguments raise std::invalid_argument like the
// reference (proj/core/src/batch.cpp:66-68).
class DeviceError : public std::runtime_error {
 public:
  DeviceError(int status, const std::string& what) : std::runtime_error(what), status_(status) {}
  int status() const { return status_; }

 private:
  int status_;
};

// Where the wall clock of one hash_batch call went (optional, see DeviceConfig::stages).
// The call is a software pipeline (host/batch_adapter.cpp): `scan` (message sizes, plan,
// staging) runs first, then pack tasks, C-ABI calls (H2D + kernels + D2H, one per ~32 MiB
// chunk) and unpack tasks overlap for `pipeline` seconds; `resize` is the value-initialisation
// of the outer digest vector (one thread, overlapped with packing).  `*_cpu` are summed over
// the threads that ran the tasks, `device_calls` over the chunks.  `kernels` is the CUDA-event
// time of the hashing kernels alone (per device: summed over its chunks; devices side by side).
struct StageTimes {
  double scan = 0, pipeline = 0, resize = 0, device_calls = 0, pack_cpu = 0, unpack_cpu = 0;
  double kernels = 0;
  unsigned threads = 0, chunks = 0, tasks = 0;
};

// Device-side knobs that EngineConfig has no field for.
struct DeviceConfig {
  int device = -1;           // CUDA ordinal, -1 = current
  void* stream = nullptr;    // cudaStream_t
  std::uint32_t flags = 0;   // B200SHA3_FLAG_*
  int kernel = 0;            // B200SHA3_KERNEL_*
  // More than one entry: the chunks of the call's pipeline (contiguous message ranges) are
  // dealt round-robin to the listed devices, each driven by its own host thread --
  // plan_partition (batch.cpp:46-62) one level up; no inter-device traffic, digests land
  // in message order.  `device` and `stream` are then ignored.
  std::vector<int> devices;
  StageTimes* stages = nullptr;  // filled when non-null (profiling aid)

  // Every CUDA device visible to the process.
  static DeviceConfig all_devices();
};

// Drop-in for sha3::hash_batch (proj/core/src/batch.cpp:64-135).
// BatchResult::elapsed is the wall time of the hashing phase as the caller sees it
// (batch.cpp:84, :133): scan, pack, host<->device copies, kernels and unpack -- the
// number the reference's runner turns into throughput (runner.cpp:53, :71).  The
// kernel-only device time is StageTimes::kernels (DeviceConfig::stages).
BatchResult hash_batch(const HashBatch& batch, const EngineConfig& config = {},
                       const DeviceConfig& device = {});

// The same call on an already packed batch (what the adapter does internally):
// message i is data[offsets[i], offsets[i] + lengths[i]).  Returns
// count * digest_bytes bytes in message order.
std::vector<std::uint8_t> hash_packed(Algorithm algorithm, const std::uint8_t* data,
                                      const std::uint64_t* offsets,
                                      const std::uint64_t* lengths, std::uint64_t count,
                                      std::uint64_t xof_output_bits = 0,
                                      const DeviceConfig& device = {},
                                      double* elapsed_seconds = nullptr);

// `count` incremental hashers on the device: the batch form of sha3::Hasher
// (proj/core/include/sha3/sha3.hpp:66-86, proj/core/src/sha3.cpp:95-130).  update() feeds
// chunk i to stream i (any chunking gives the one-shot digest, proj/tests/test_sponge.cpp:114-132);
// digest() finalises the hash variants; finish() + read() stream XOF output
// (proj/tests/test_sponge.cpp:134-150).  Misuse throws std::logic_error with the reference's
// messages (sha3.cpp:103-126, sponge.cpp:82-84, :114-116, :132-134).  Single owner; movable.
class BatchHasher {
 public:
  BatchHasher(Algorithm algorithm, std::size_t count, const DeviceConfig& device = {});
  ~BatchHasher();
  BatchHasher(BatchHasher&& other) noexcept;
  BatchHasher& operator=(BatchHasher&& other) noexcept;
  BatchHasher(const BatchHasher&) = delete;
  BatchHasher& operator=(const BatchHasher&) = delete;

  // chunks.size() must equal count(); chunks[i] may be empty.
  void update(const std::vector<std::vector<std::uint8_t>>& chunks);
  // The same on a packed buffer: chunk i is data[offsets[i], offsets[i] + lengths[i]).
  void update(const std::uint8_t* data, const std::uint64_t* offsets, const std::uint64_t* lengths);
  // Equal-length chunks back to back: chunk i is data[i * chunk_len, (i + 1) * chunk_len).
  void update_fixed(const std::uint8_t* data, std::uint64_t chunk_len);

  std::vector<std::vector<std::uint8_t>> digest();                   // hash variants only
  void finish();                                                     // XOF variants only
  std::vector<std::vector<std::uint8_t>> read(std::size_t nbytes);   // XOF, after finish()

  Algorithm algorithm() const { return algorithm_; }
  std::size_t count() const { return count_; }
  void reset();

 private:
  void check(int status) const;
  std::vector<std::vector<std::uint8_t>> split(const std::vector<std::uint8_t>& packed, std::size_t each) const;
  Algorithm algorithm_;
  std::size_t count_;
  DeviceConfig device_;
  b200sha3_states* states_ = nullptr;
};

}  // namespace sha3::b200
