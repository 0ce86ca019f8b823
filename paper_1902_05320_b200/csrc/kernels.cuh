// kernels.cuh -- kernel declarations shared by the translation units of
// libb200sha3.so.  One message per thread unless stated otherwise.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace b200sha3 {

// Arguments of the batch kernels (passed by value in the parameter bank).
struct HashArgs {
  const uint8_t* data;       // packed message bytes
  const uint64_t* offsets;   // per-message byte offset, or nullptr: i * fixed_len
  const uint64_t* lengths;   // per-message byte length, or nullptr: fixed_len
  uint64_t fixed_len;
  uint64_t count;
  const uint32_t* order;     // processing order (bucketed), or nullptr: identity
  const uint32_t* unaligned_flag;  // device word, nonzero if any message start is not
                                   // 8-byte aligned; nullptr: use `aligned8`
  const uint32_t* ragged_flag;     // device word, nonzero if the final (partial) blocks of the
                                   // batch differ in length; nullptr: they are all alike
  const uint32_t* long_flag;       // device word, nonzero if some message fills a whole rate block
                                   // (>= rate bytes); nullptr: unknown
  uint32_t skip_if_short;          // generic / pair kernel: return at once when the batch is
                                   // all-short (the flag above says so); for callers that launch
                                   // hash_short_kernel next to it (none does by default)
  uint8_t* digests;          // count * digest_bytes, message order
  uint64_t digest_bytes;
  uint32_t head;             // pad head byte: 0x06 / 0x1f
  uint32_t last_mask;        // 0xff or the XOF partial-byte mask
  uint32_t aligned8;         // host-known alignment of every message start
};

// FMA-pipe rotation presets (see keccak_f1600.cuh): bit i = rho rotation of
// source lane i on the FMA pipe, bit 25 = theta rotl-1.
constexpr uint32_t kRhoAll = 0x1fffffeu;    // all 24 rotating rho lanes
constexpr uint32_t kRhoOdd = 0x0aaaaaau;    // 12 of them
constexpr uint32_t kTheta = 0x2000000u;
constexpr uint32_t kFlavour(int f) { return static_cast<uint32_t>(f) << 28; }
constexpr int kFmaPresets = 9;
constexpr uint32_t kFmaPreset[kFmaPresets] = {
    0u,                                   // 0: ALU only (LOP3 + SHF)
    kRhoAll | kTheta | kFlavour(1),       // 1: everything, flavour 1
    kRhoAll | kFlavour(1),                // 2: all rho, flavour 1
    kRhoOdd | kFlavour(1),                // 3: 12 rho, flavour 1
    kRhoAll | kTheta | kFlavour(2),       // 4: everything, flavour 2
    kRhoAll | kFlavour(2),                // 5: all rho, flavour 2
    (kRhoOdd | 0x0000554u) | kFlavour(2), // 6: 17 rho, flavour 2
    kRhoOdd | kFlavour(2),                // 7: 12 rho, flavour 2
    0x0888888u | kFlavour(2),             // 8: 6 rho, flavour 2
};

struct LaunchPlan {
  int rate_lanes;     // 9, 13, 17, 18, 21
  int unroll;         // 1, 2, 4, 24 (availability depends on the kernel)
  int fma_preset;     // 0..kFmaPresets-1
  int block_threads;
};

// Generic kernel: any length, any alignment, multi-block absorb and squeeze.
cudaError_t launch_hash_generic(const HashArgs& args, const LaunchPlan& plan,
                                cudaStream_t stream);

// Specialised kernel: equal-length, 16-byte aligned, single-block messages of
// whole lanes with a digest of whole 32-bit words that fits one block.  Returns
// cudaErrorNotSupported when no instantiation matches.
cudaError_t launch_hash_oneblock(const HashArgs& args, const LaunchPlan& plan,
                                 cudaStream_t stream);
bool oneblock_supported(int rate_lanes, uint64_t msg_len, uint64_t digest_bytes);

// Equal-length multi-block shapes with everything static (kernel_fewblock.cu): messages of whole
// lanes at or above the rate, or outputs longer than the rate, for the shapes of BASELINE.json
// cfg2 / cfg3; 16-byte aligned buffers, whole-byte output.  cudaErrorNotSupported otherwise.
cudaError_t launch_hash_fewblock(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream);
bool fewblock_supported(int rate_lanes, uint64_t msg_len, uint64_t digest_bytes);
// The same round sequence with the message length a run-time value (same file): equal-length
// messages of any whole number of lanes at or above the rate, digest within one block.
cudaError_t launch_hash_manyblock(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream);
bool manyblock_supported(int rate_lanes, uint64_t msg_len, uint64_t digest_bytes);

// Variable-length batches made of single-block messages only (kernel_short.cu), input order; for
// callers that KNOW the batch is all-short (the host entries).  Returns at once if the "long" flag
// word says otherwise.  cudaErrorNotSupported when no instantiation matches.
cudaError_t launch_hash_short(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream);
bool short_supported(int rate_lanes, uint64_t digest_bytes);
// Equal-length form: any length below the rate (args.fixed_len), any alignment (args.aligned8).
cudaError_t launch_hash_short_fixed(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream);

// One launch for a variable-length batch classified on the device (kernel_ragged.cu): the short
// kernel's body if the flag words say "nothing as long as the rate", the generic kernel's body
// otherwise.  Same shapes as short_supported; cudaErrorNotSupported otherwise.
cudaError_t launch_hash_ragged(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream);

// Lane-split kernel (5 threads per state, warp shuffles); equal-length,
// 8-byte aligned, single-block messages.
cudaError_t launch_hash_lanesplit(const HashArgs& args, const LaunchPlan& plan,
                                  cudaStream_t stream);
bool lanesplit_supported(int rate_lanes, uint64_t msg_len, uint64_t digest_bytes);

// Warp-per-state kernel (kernel_warp.cu): one message per WARP, the 25 lanes spread over 25
// threads and exchanged with shuffles -- ~4x lower latency per permutation, for batches too
// small to fill the machine with one message per thread.  Any length / alignment / digest
// size; args.order may be nullptr.
cudaError_t launch_hash_warp(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream);

// Pair-split kernel (kernel_pair.cu): one message per PAIR of threads (low / high 32-bit halves
// of every lane, one shuffle per rotation).  A measured experiment (no faster than one message
// per thread: the shuffles cost the issue slots the halved ALU work frees); forced selection
// only.  Honours order / skip_if_short like the generic kernel.
cudaError_t launch_hash_pair(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream);

// TMA-staged variant of the generic kernel (kernel_staged.cu); blocks are staged when the
// data base is 16-byte aligned and message starts are 8-byte aligned (else direct loads).
cudaError_t launch_hash_staged(const HashArgs& args, const LaunchPlan& plan, cudaStream_t stream);

// Keccak-f[1600] on raw 200-byte states (test hook).
cudaError_t launch_permute(uint64_t* states, uint64_t count, cudaStream_t stream);

// Bucketing: writes a processing order -- by block count, heaviest first, single-block
// messages by their number of whole 32-bit words -- sets *unaligned_flag if any offset is not
// a multiple of 8, unaligned_flag[1] (the "ragged" word) if the messages do not all leave the
// same number of bytes for the final block and unaligned_flag[2] (the "long" word) if some
// message is at least one rate block long.  With `short_kernel_next` (hash_short_kernel is
// launched after this pass) the order is left unwritten for a batch of single-block messages
// with 8-byte aligned starts: that kernel takes those in input order.
// `scratch` needs kBucketScratchWords 32-bit words; the caller zeroes them and the three flag
// words (one memset when they are adjacent).
constexpr int kBucketBins = 512;
constexpr int kBucketScratchWords = 2 * kBucketBins + 8;
cudaError_t launch_bucket_order(const uint64_t* offsets, const uint64_t* lengths,
                                uint32_t count, uint32_t rate_bytes, uint32_t* order,
                                uint32_t* scratch, uint32_t* unaligned_flag,
                                cudaStream_t stream, bool short_kernel_next = false);
// The two flag words only (no ordering).
cudaError_t launch_alignment_check(const uint64_t* offsets, const uint64_t* lengths, uint64_t count,
                                   uint32_t rate_bytes, uint32_t* unaligned_flag, cudaStream_t stream);

// Synthetic workloads.
cudaError_t launch_generate_workload(uint64_t stream_seed, uint64_t message_size,
                                     uint64_t first_message, uint64_t count, uint8_t* out,
                                     cudaStream_t stream);
cudaError_t launch_generate_lengths(uint64_t seed_len, uint64_t min_len, uint64_t max_len,
                                    uint64_t first_message, uint64_t count,
                                    uint64_t* lengths, cudaStream_t stream);
cudaError_t launch_fill_messages(uint64_t seed, uint64_t first_message, uint64_t count,
                                 const uint64_t* offsets, const uint64_t* lengths,
                                 uint8_t* data, cudaStream_t stream);

// Batched incremental hashing (kernel_stream.cu): `lanes` is 25 * count uint2 (structure
// of arrays), `pos` is count words.
cudaError_t launch_states_update(int rate_lanes, void* lanes, uint32_t* pos, uint64_t count,
                                 const uint8_t* data, const uint64_t* offsets,
                                 const uint64_t* lengths, uint64_t fixed_len, cudaStream_t stream);
cudaError_t launch_states_finish(int rate_lanes, void* lanes, uint32_t* pos, uint64_t count,
                                 uint32_t head, uint8_t* out, uint64_t out_len, uint32_t last_mask,
                                 cudaStream_t stream);
cudaError_t launch_states_squeeze(int rate_lanes, void* lanes, uint32_t* pos, uint64_t count,
                                  uint8_t* out, uint64_t out_len, cudaStream_t stream);

// The same three steps with one stream per WARP (kernel_stream_warp.cu): same state layout, for
// few streams.
cudaError_t launch_states_update_warp(int rate_lanes, void* lanes, uint32_t* pos, uint64_t count,
                                      const uint8_t* data, const uint64_t* offsets,
                                      const uint64_t* lengths, uint64_t fixed_len, cudaStream_t stream);
cudaError_t launch_states_finish_warp(int rate_lanes, void* lanes, uint32_t* pos, uint64_t count,
                                      uint32_t head, uint8_t* out, uint64_t out_len, uint32_t last_mask,
                                      cudaStream_t stream);
cudaError_t launch_states_squeeze_warp(int rate_lanes, void* lanes, uint32_t* pos, uint64_t count,
                                       uint8_t* out, uint64_t out_len, cudaStream_t stream);

// Pipe microbenchmark; see b200sha3_probe_pipe.
cudaError_t run_pipe_probe(int mix, double* instr_per_s, double* sm_hz, cudaStream_t stream);

}  // namespace b200sha3
