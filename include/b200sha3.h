/*
 * b200sha3.h -- C ABI of the B200-native batch SHA-3 / SHAKE engine.
 *
 * This is the drop-in boundary for the one path this project accelerates: the
 * reference's
 *
 *     sha3::BatchResult sha3::hash_batch(const sha3::HashBatch&, const sha3::EngineConfig&)
 *                                         (proj/core/include/sha3/batch.hpp:65,
 *                                          proj/core/src/batch.cpp:64-135)
 *
 * The reference has no FFI of its own (it is a C++ static library); the
 * functions below are what a `Backend::cuda` branch in batch.cpp, or the C++
 * adapter in include/b200sha3/batch.hpp, binds to.  INTEGRATION.md shows both.
 *
 * Conventions
 *  - plain C types only; the library never throws across this boundary and
 *    never takes ownership of a caller buffer;
 *  - `algorithm` uses the reference's enum order
 *    (proj/core/include/sha3/sha3.hpp:15-22):
 *        0 sha3_224, 1 sha3_256, 2 sha3_384, 3 sha3_512, 4 shake128, 5 shake256;
 *  - messages live in one packed byte buffer `data`; message i is
 *    data[offsets[i] .. offsets[i] + lengths[i]) (any byte length incl. 0, any
 *    alignment).  The `_fixed` entries take equal-length messages back to back
 *    (offset i*msg_len) -- the layout of the reference's workload generator
 *    (proj/tools/sha3cli/workload.cpp:16-47);
 *  - digests are written packed in message order: digest i at
 *    digests[i*digest_bytes .. (i+1)*digest_bytes), digest_bytes =
 *    b200sha3_digest_bytes(algorithm, xof_output_bits)   (batch.cpp:74-75);
 *  - `xof_output_bits` is required (>0) for SHAKE and ignored for the hashes
 *    (batch.cpp:66-75); a bit count that is not a multiple of 8 keeps the low
 *    bits of the last byte (batch.cpp:22-24);
 *  - every entry is thread-safe and reentrant (batch.hpp:61-64);
 *  - there is NO CPU fallback: without a usable CUDA device every compute
 *    entry returns B200SHA3_ERR_CUDA.
 */
#ifndef B200SHA3_H_
#define B200SHA3_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define B200SHA3_API __attribute__((visibility("default")))
#else
#define B200SHA3_API
#endif

/* Status codes. */
enum {
  B200SHA3_OK = 0,
  /* Bad enum value, XOF without output length, NULL where data is required.
   * Maps to std::invalid_argument in the C++ adapter (batch.cpp:66-68). */
  B200SHA3_ERR_INVALID_ARGUMENT = 1,
  /* Any CUDA runtime failure (no device, out of memory, launch failure). */
  B200SHA3_ERR_CUDA = 2,
  /* Batch shape the engine cannot take (e.g. a single digest > 4 GiB). */
  B200SHA3_ERR_UNSUPPORTED = 3,
  /* Incremental API used out of order: update after finish, finish twice, squeeze before
   * finish or on a fixed-output variant.  Maps to std::logic_error
   * (proj/core/src/sponge.cpp:82-84, :114-116, :132-134; proj/core/src/sha3.cpp:103-126). */
  B200SHA3_ERR_STATE = 4
};

/* Algorithm ids, reference enum order (sha3.hpp:15-22). */
enum {
  B200SHA3_SHA3_224 = 0,
  B200SHA3_SHA3_256 = 1,
  B200SHA3_SHA3_384 = 2,
  B200SHA3_SHA3_512 = 3,
  B200SHA3_SHAKE128 = 4,
  B200SHA3_SHAKE256 = 5
};

/* Config flags. */
enum {
  /* Variable-length batches: skip the device-side bucketing by block count
   * (messages are then hashed in input order, one per thread). */
  B200SHA3_FLAG_NO_BUCKETING = 1u << 0,
  /* Host-buffer entries: do not chunk/overlap copies with compute. */
  B200SHA3_FLAG_NO_PIPELINE = 1u << 1,
  /* KERNEL_AUTO: never pick the warp-per-state kernel, however few the messages
   * (small batches then take the same kernels as large ones). */
  B200SHA3_FLAG_NO_WARP_KERNEL = 1u << 2
};

/* Kernel selection for experiments; 0 picks the measured default. */
enum {
  B200SHA3_KERNEL_AUTO = 0,
  B200SHA3_KERNEL_GENERIC = 1,   /* rolled rounds, any length / alignment        */
  B200SHA3_KERNEL_ONEBLOCK = 2,  /* specialised single-block kernel when it fits  */
  B200SHA3_KERNEL_LANESPLIT = 3, /* 5 threads per state + warp shuffles (kept for
                                    the measured comparison in DESIGN.md)         */
  B200SHA3_KERNEL_STAGED = 4,    /* generic kernel with rate blocks staged through
                                    shared memory by bulk async copies (TMA); also
                                    kept for the measured comparison               */
  B200SHA3_KERNEL_WARP = 5,      /* one message per warp (25 lanes over 25 threads,
                                    shuffles): AUTO picks it for batches of few
                                    multi-block messages                           */
  B200SHA3_KERNEL_PAIR = 6,      /* one message per pair of threads (low / high halves
                                    of every lane, one shuffle per rotation): kept
                                    for the measured comparison, never AUTO         */
  B200SHA3_KERNEL_FEWBLOCK = 7   /* equal-length multi-block batches as one round
                                    sequence per message: static-shape instantiations
                                    (cfg2 / cfg3 lengths) or the run-time-length form
                                    (any whole number of lanes at or above the rate);
                                    AUTO picks it when one fits                       */
};

/* Optional per-call configuration; NULL means all defaults.  The analogue of
 * the reference's EngineConfig (batch.hpp:15-19): `workers`/`chunk_size` have
 * no meaning on a GPU and are replaced by device / stream / kernel knobs. */
typedef struct b200sha3_config {
  uint32_t struct_size;    /* sizeof(b200sha3_config) the caller was built with; 0 = this
                              version.  Fields beyond it are not read (ABI growth).      */
  int32_t device;          /* CUDA device ordinal; -1 = current device              */
  void* stream;            /* cudaStream_t to enqueue on; NULL = the default stream */
  uint32_t flags;          /* B200SHA3_FLAG_*                                        */
  int32_t kernel;          /* B200SHA3_KERNEL_*                                      */
  int32_t unroll;          /* one-block kernel: 0 = default; 2, 4 rolled; 11, 20..23 peeled; 24 full */
  int32_t fma_preset;      /* -1 = default; 0..8 = FMA-pipe rotation offload preset  */
  int32_t block_threads;   /* 0 = default                                            */
  /* If non-NULL receives the device time of the hashing phase in milliseconds
   * (CUDA events around the kernels; copies excluded) -- the adapter's
   * StageTimes::kernels.  Forces the call to wait for completion. */
  double* device_ms;
  /* If non-NULL receives how many kernels this call launched. */
  uint32_t* kernel_launches;
} b200sha3_config;

/* ---- queries ------------------------------------------------------------ */

/* Digest size in bytes: ceil(xof_output_bits/8) for SHAKE, 28/32/48/64 for the
 * hashes; 0 for a bad algorithm id.  (batch.cpp:74-75) */
B200SHA3_API uint64_t b200sha3_digest_bytes(int algorithm, uint64_t xof_output_bits);

/* Sponge rate in bytes (144/136/104/72/168/136); 0 for a bad id. (sha3.hpp:40) */
B200SHA3_API uint32_t b200sha3_rate_bytes(int algorithm);

/* Keccak-f[1600] calls one message costs: floor(len/rate) + 1 absorb
 * permutations plus max(0, ceil(digest_bytes/rate) - 1) squeeze permutations. */
B200SHA3_API uint64_t b200sha3_permutations(int algorithm, uint64_t msg_len,
                                            uint64_t xof_output_bits);

/* Which kernel B200SHA3_KERNEL_AUTO runs for a batch of this shape on 16-byte aligned
 * buffers: `count` equal-length messages of `msg_len` bytes, or a variable-length batch when
 * msg_len == UINT64_MAX.  A static string such as "hash_oneblock_kernel<17,8,8>"; ""
 * for a bad id.  Introspection for reports (bench.py); never needed to hash. */
B200SHA3_API const char* b200sha3_selected_kernel(int algorithm, uint64_t msg_len, uint64_t count,
                                                  uint64_t xof_output_bits);

B200SHA3_API const char* b200sha3_strerror(int status);

/* Text of the last CUDA error seen by the calling thread ("" if none). */
B200SHA3_API const char* b200sha3_last_cuda_error(void);

B200SHA3_API const char* b200sha3_version(void);

/* Number of CUDA devices visible to the process (0 if CUDA is unusable). */
B200SHA3_API int b200sha3_device_count(void);

/* The calling thread's current CUDA device (what `device = -1` resolves to), -1 if CUDA is
 * unusable.  Lets a host layer hand the caller's device to helper threads it starts. */
B200SHA3_API int b200sha3_current_device(void);

/* ---- host-buffer entries (the hash_batch drop-in) ------------------------
 * All pointers are HOST pointers.  The call copies the batch to the device
 * (chunked and overlapped with compute when the host memory is pinned), hashes
 * it and copies the digests back; it returns when `digests` is complete.
 * Replaces hash_batch (batch.cpp:64-135) for a caller holding host memory. */
B200SHA3_API int b200sha3_hash_batch(int algorithm, const uint8_t* data,
                                     const uint64_t* offsets, const uint64_t* lengths,
                                     uint64_t count, uint64_t xof_output_bits,
                                     uint8_t* digests, const b200sha3_config* cfg);

B200SHA3_API int b200sha3_hash_fixed(int algorithm, const uint8_t* data, uint64_t msg_len,
                                     uint64_t count, uint64_t xof_output_bits,
                                     uint8_t* digests, const b200sha3_config* cfg);

/* Page-locked (pinned, portable) host memory: buffers obtained here let the host entries
 * above overlap their copies with compute at full PCIe speed; pageable memory works too,
 * more slowly.  The C++ adapter packs into such buffers. */
B200SHA3_API int b200sha3_pinned_alloc(uint64_t bytes, void** out);
B200SHA3_API int b200sha3_pinned_free(void* ptr);

/* ---- device-buffer entries ----------------------------------------------
 * All pointers are DEVICE pointers on cfg->device.  Work is enqueued on
 * cfg->stream and the call returns without waiting (unless cfg->device_ms is
 * set); digests stay resident in HBM. */
B200SHA3_API int b200sha3_hash_batch_device(int algorithm, const uint8_t* d_data,
                                            const uint64_t* d_offsets,
                                            const uint64_t* d_lengths, uint64_t count,
                                            uint64_t xof_output_bits, uint8_t* d_digests,
                                            const b200sha3_config* cfg);

B200SHA3_API int b200sha3_hash_fixed_device(int algorithm, const uint8_t* d_data,
                                            uint64_t msg_len, uint64_t count,
                                            uint64_t xof_output_bits, uint8_t* d_digests,
                                            const b200sha3_config* cfg);

/* ---- harness helpers (device) --------------------------------------------
 * Bit-identical device version of the reference's synthetic workload
 * (proj/tools/sha3cli/workload.cpp:16-47): `count` messages of `message_size`
 * bytes starting at global message index `first_message`, generator seeded
 * with seed ^ total_bytes*0x9e3779b97f4a7c15.  Counter-based, so any shard of
 * the stream can be produced on any GPU. */
B200SHA3_API int b200sha3_generate_workload_device(uint64_t seed, uint64_t total_bytes,
                                                   uint64_t message_size,
                                                   uint64_t first_message, uint64_t count,
                                                   uint8_t* d_out,
                                                   const b200sha3_config* cfg);

/* Variable-length synthetic workload (ours; the reference has none, SURVEY.md
 * section 8(d) cfg4): lengths[i] = min_len + splitmix64_at(seed_len, i) %
 * (max_len - min_len + 1) for global message index first_message + i. */
B200SHA3_API int b200sha3_generate_lengths_device(uint64_t seed_len, uint64_t min_len,
                                                  uint64_t max_len, uint64_t first_message,
                                                  uint64_t count, uint64_t* d_lengths,
                                                  const b200sha3_config* cfg);

/* Fills message i (at d_offsets[i], d_lengths[i] bytes) with the splitmix64
 * stream of key seed ^ (first_message + i): word k = mix(key + (k+1)*gamma). */
B200SHA3_API int b200sha3_fill_messages_device(uint64_t seed, uint64_t first_message,
                                               uint64_t count, const uint64_t* d_offsets,
                                               const uint64_t* d_lengths, uint8_t* d_data,
                                               const b200sha3_config* cfg);

/* Applies Keccak-f[1600] to `count` 200-byte states in place (25 little-endian
 * 64-bit lanes each).  Test hook for the permutation alone
 * (permute_1600, proj/core/src/keccak.cpp:245-277). */
B200SHA3_API int b200sha3_permute_device(uint64_t* d_states, uint64_t count,
                                         const b200sha3_config* cfg);

/* Device-side bucketing on its own (test hook): writes the processing order
 * of a variable-length batch (a permutation of 0..count-1, heaviest block count
 * first) to d_order (uint32, count entries; count < 2^32). */
B200SHA3_API int b200sha3_bucket_order_device(int algorithm, const uint64_t* d_lengths,
                                              uint64_t count, uint32_t* d_order,
                                              const b200sha3_config* cfg);

/* ---- batched incremental hashing (device) --------------------------------
 * `count` independent sponge states resident in HBM, fed chunk by chunk: the batch
 * analogue of sha3::Hasher (proj/core/include/sha3/sha3.hpp:66-86) over SpongeHasher
 * (proj/core/include/sha3/sponge.hpp:38-64).  For inputs that do not fit one buffer or
 * arrive in pieces.  Feeding a message in any chunking gives the one-shot digest
 * (proj/tests/test_sponge.cpp:114-132); squeezing an XOF in pieces gives the one-shot
 * output (proj/tests/test_sponge.cpp:134-150).  All pointers are device pointers; calls
 * are asynchronous on cfg->stream.  A handle is single-owner (not for concurrent calls),
 * like the reference's Hasher. */
typedef struct b200sha3_states b200sha3_states;

B200SHA3_API int b200sha3_states_create(int algorithm, uint64_t count,
                                        const b200sha3_config* cfg, b200sha3_states** out);
B200SHA3_API int b200sha3_states_destroy(b200sha3_states* states);
/* Hasher::reset (sha3.cpp:128-130). */
B200SHA3_API int b200sha3_states_reset(b200sha3_states* states, const b200sha3_config* cfg);
/* Hasher::update: chunk i = d_data[d_offsets[i], +d_lengths[i]) goes to stream i
 * (lengths may be 0). */
B200SHA3_API int b200sha3_states_update_device(b200sha3_states* states, const uint8_t* d_data,
                                               const uint64_t* d_offsets,
                                               const uint64_t* d_lengths,
                                               const b200sha3_config* cfg);
/* Same with equal-length chunks back to back. */
B200SHA3_API int b200sha3_states_update_fixed_device(b200sha3_states* states,
                                                     const uint8_t* d_data, uint64_t chunk_len,
                                                     const b200sha3_config* cfg);
/* Hasher::digest (hash variants: d_digests required) / Hasher::finish + first read (XOF:
 * xof_output_bits may be 0 to only close the input; otherwise ceil(bits/8) bytes per stream
 * are written, last byte masked like batch.cpp:22-24). */
B200SHA3_API int b200sha3_states_finish_device(b200sha3_states* states, uint64_t xof_output_bits,
                                               uint8_t* d_digests, const b200sha3_config* cfg);
/* Hasher::read: the next out_bytes bytes of every XOF stream, packed count x out_bytes. */
B200SHA3_API int b200sha3_states_squeeze_device(b200sha3_states* states, uint64_t out_bytes,
                                                uint8_t* d_out, const b200sha3_config* cfg);

/* The same four steps on HOST buffers (what a caller of sha3::Hasher holds): the chunk bytes are
 * staged to the device (pinned memory: straight DMA; pageable memory: through the library's
 * bounce ring), the device form runs on cfg->stream, and the call returns when the host
 * buffers are free again (update) or filled (finish / squeeze). */
B200SHA3_API int b200sha3_states_update(b200sha3_states* states, const uint8_t* data,
                                        const uint64_t* offsets, const uint64_t* lengths,
                                        const b200sha3_config* cfg);
B200SHA3_API int b200sha3_states_update_fixed(b200sha3_states* states, const uint8_t* data,
                                              uint64_t chunk_len, const b200sha3_config* cfg);
B200SHA3_API int b200sha3_states_finish(b200sha3_states* states, uint64_t xof_output_bits,
                                        uint8_t* digests, const b200sha3_config* cfg);
B200SHA3_API int b200sha3_states_squeeze(b200sha3_states* states, uint64_t out_bytes, uint8_t* out,
                                         const b200sha3_config* cfg);

/* ---- pipe microbenchmark ---------------------------------------------------
 * Measures the issue rate of one instruction mix on the current device:
 * returns thread-instructions per second through *instr_per_s, and the SM
 * clock seen (cycles of clock64 per second of globaltimer) through *sm_hz.
 * mix: 0 LOP3, 1 SHF, 2 LOP3+SHF 2:1 (the Keccak ALU mix), 3 IMAD, 4 IMAD.WIDE,
 *      5 IMAD.HI, 6 LOP3+IMAD 1:1, 7 LOP3+IMAD.WIDE 1:1, 8 LOP3+IMAD.HI 1:1,
 *      9 the flavour-2 Keccak mix (5 LOP3 : 2 IMAD : 2 IMAD.HI);
 *      10..15 the same with realistic operand traffic (three distinct registers per
 *      LOP3): 10 LOP3, 11 LOP3+IMAD 1:1, 12 LOP3+IMAD 3:1, 13 LOP3+IMAD(1 reg) 3:1,
 *      14 LOP3+IMAD.HI 3:1, 15 LOP3+SHF 2:1. */
B200SHA3_API int b200sha3_probe_pipe(int mix, double* instr_per_s, double* sm_hz,
                                     const b200sha3_config* cfg);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* B200SHA3_H_ */
