// kernel_aux.cu -- everything around the hash kernels: device-side bucketing of
// variable-length batches, the synthetic workload generators, and the raw
// permutation test hook.
#include <algorithm>

#include "kernels.cuh"
#include "keccak_f1600.cuh"

namespace b200sha3 {

namespace {

// ---------------------------------------------------------------------------
// Keccak-f[1600] on raw states: permute_1600 (proj/core/src/keccak.cpp:245-277)
// with nothing around it; pins the device permutation against the 200-byte KAT
// of proj/tests/test_keccak.cpp:456-466.
__global__ void __launch_bounds__(128) permute_kernel(uint64_t* states, uint64_t count) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid >= count) return;
  uint2* s = reinterpret_cast<uint2*>(states + 25 * tid);
  State a;
#pragma unroll
  for (int i = 0; i < 25; ++i) {
    const uint2 v = s[i];
    a.lo[i] = v.x;
    a.hi[i] = v.y;
  }
  keccak_f1600<2, 0u>(a);
#pragma unroll
  for (int i = 0; i < 25; ++i) s[i] = make_uint2(a.lo[i], a.hi[i]);
}

// ---------------------------------------------------------------------------
// Bucketing.  The reference balances uneven messages by handing small chunks
// to a thread pool (plan_partition, proj/core/src/batch.cpp:46-62).  On the
// GPU the cost of an uneven batch is warp divergence: 32 threads run as long
// as the longest message among them.  We therefore process messages in order
// of their absorb-block count, heaviest first, so that the threads of a warp
// run (nearly) the same number of permutations.
//
// Single-block messages (len < rate) are ordered too -- by their number of whole 32-bit
// words: their cost does not differ, but a warp whose threads hold the SAME number of words
// absorbs the final block through a jump table of statically indexed loads instead of
// 2 x RL predicated ones (sponge.cuh: absorb_tail / absorb_tail_uniform_unaligned), which is
// the difference between 0.90 and ~0.97 of the ALU roofline on short ragged batches.
//
// Key, 512 values, stored inverted so that key 0 is the heaviest bin:
//   one block    its word count len >> 2                      (0 .. 41)
//   2 .. 128     40 + block count: every bin one block count   (42 .. 168)
//   >= 129       16 sub-bins per power of two (<= 6.25 % spread inside a bin), clamped at 2^28 blocks
// RATE is a template argument: the block count is a division by a compile-time constant
// (multiply + shift) -- with a run-time divisor the two 64-bit divisions per message made
// these passes compute bound (84 us for 2^24 messages against 45 us of memory traffic).
template <uint32_t RATE>
__device__ __forceinline__ uint64_t whole_blocks(uint64_t len) {
  return (len >> 32) == 0 ? static_cast<uint64_t>(static_cast<uint32_t>(len) / RATE) : len / RATE;
}

template <uint32_t RATE>
__device__ __forceinline__ uint32_t bucket_key(uint64_t len) {
  const uint64_t blocks = whole_blocks<RATE>(len) + 1u;
  uint32_t key;
  if (blocks == 1u) {
    key = static_cast<uint32_t>(len) >> 2;  // < 42: the largest rate is 168 bytes
  } else if (blocks <= 128u) {
    key = 40u + static_cast<uint32_t>(blocks);
  } else {
    const int e = 63 - __clzll(static_cast<long long>(blocks));  // >= 7
    const uint32_t frac = static_cast<uint32_t>(blocks >> (e - 4)) & 15u;
    key = 169u + static_cast<uint32_t>(e - 7) * 16u + frac;
    if (key > kBucketBins - 1u) key = kBucketBins - 1u;
  }
  return (kBucketBins - 1u) - key;
}

// Sets flags[0] / [1] / [2] if any thread of the warp saw a misaligned start / a different tail
// length / a message of a whole block.  The words only ever go from 0 to 1, so a warp looks
// before it writes: in a ragged batch EVERY warp has something to report, and 65536 atomics on
// one address (2^24 messages) cost more than reading the batch (116 us against 45).
__device__ __forceinline__ void raise_flags(uint32_t* flags, uint32_t misaligned, uint32_t ragged,
                                            uint32_t has_long) {
  const bool report[3] = {__any_sync(0xffffffffu, misaligned != 0u) != 0, __any_sync(0xffffffffu, ragged != 0u) != 0,
                          __any_sync(0xffffffffu, has_long != 0u) != 0};
  if ((threadIdx.x & 31) != 0) return;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (report[k] && *reinterpret_cast<volatile uint32_t*>(flags + k) == 0u) atomicOr(flags + k, 1u);
  }
}

constexpr int kBucketThreads = kBucketBins;
constexpr int kBucketItems = 4;  // messages per thread
static_assert(kBucketThreads == kBucketBins, "one thread per bin in the block-level steps");

// scratch layout: [0, kBucketBins) histogram, [kBucketBins, 2 kBucketBins) running cursor.
template <uint32_t RATE>
__global__ void __launch_bounds__(kBucketThreads)
bucket_histogram_kernel(const uint64_t* __restrict__ offsets,
                        const uint64_t* __restrict__ lengths, uint32_t count,
                        uint32_t* __restrict__ hist, uint32_t* __restrict__ unaligned_flag) {
  __shared__ uint32_t local[kBucketBins];
  local[threadIdx.x] = 0u;
  __syncthreads();
  const uint64_t len0 = lengths[0];
  const uint32_t first_tail = static_cast<uint32_t>(len0 - whole_blocks<RATE>(len0) * RATE);
  uint32_t misaligned = 0u, ragged = 0u, has_long = 0u;
  // A block walks several tiles and flushes its counters once: the flush is one global atomic
  // per bin and block, all blocks on the same few addresses.
  constexpr uint32_t kTile = kBucketThreads * kBucketItems;
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTile; base < count;
       base += static_cast<uint64_t>(gridDim.x) * kTile) {
#pragma unroll
    for (int k = 0; k < kBucketItems; ++k) {
      const uint64_t i = base + k * kBucketThreads + threadIdx.x;
      if (i < count) {
        const uint64_t len = lengths[i];
        atomicAdd(&local[bucket_key<RATE>(len)], 1u);
        misaligned |= static_cast<uint32_t>(offsets[i]) & 7u;
        ragged |= static_cast<uint32_t>(len - whole_blocks<RATE>(len) * RATE) ^ first_tail;
        has_long |= len >= RATE ? 1u : 0u;
      }
    }
  }
  raise_flags(unaligned_flag, misaligned, ragged, has_long);
  __syncthreads();
  if (local[threadIdx.x]) atomicAdd(&hist[threadIdx.x], local[threadIdx.x]);
}

// Exclusive scan of kBucketBins values held one per thread (whole block of kBucketBins threads):
// shuffle scans inside the warps, one more over the warp totals; two barriers.  `warp_sums` holds
// kBucketBins / 32 words.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t mine, uint32_t* warp_sums) {
  constexpr int kWarps = kBucketBins / 32;
  static_assert(kWarps <= 32, "the warp totals are scanned by one warp");
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t v = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t up = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= static_cast<uint32_t>(d)) v += up;
  }
  if (lane == 31u) warp_sums[warp] = v;
  __syncthreads();
  if (warp == 0u) {
    const uint32_t own = lane < kWarps ? warp_sums[lane] : 0u;
    uint32_t s = own;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t up = __shfl_up_sync(0xffffffffu, s, d);
      if (lane >= static_cast<uint32_t>(d)) s += up;
    }
    if (lane < kWarps) warp_sums[lane] = s - own;
  }
  __syncthreads();
  return v - mine + warp_sums[warp];
}

// A block ranks its 2048 messages inside their bins (shared-memory counters), reserves a run
// of every bin it touches (one global atomic per bin), lays the message indices out bin by bin
// in shared memory and writes them from there: consecutive threads then write consecutive
// entries of `order`.  (Writing order[base + rank] straight from the ranking loop sent the 32
// stores of a warp to up to 32 different bins: 105 us for 2^24 messages.)
template <uint32_t RATE>
__global__ void __launch_bounds__(kBucketThreads)
bucket_scatter_kernel(const uint64_t* __restrict__ lengths, uint32_t count,
                      const uint32_t* __restrict__ hist, uint32_t* __restrict__ cursor,
                      uint32_t* __restrict__ order, const uint32_t* __restrict__ flags) {
  // `flags` is given when hash_short_kernel is launched next: an all-short batch whose
  // messages start on 8-byte boundaries is hashed there in input order (predicated 8-byte lane
  // loads: 0.97 of the roofline; ordering it costs more in gathered loads than the uniform
  // absorb saves), so no order is needed.
  if (flags != nullptr && flags[2] == 0u && flags[0] == 0u) return;
  constexpr int kTile = kBucketThreads * kBucketItems;
  __shared__ uint32_t local[kBucketBins];     // per-block count of the bin
  __shared__ uint32_t warp_sums[2][kBucketBins / 32];
  __shared__ uint32_t tile_index[kTile];      // message index, bin by bin
  __shared__ uint32_t tile_target[kTile];     // where it goes in `order`
  local[threadIdx.x] = 0u;
  __syncthreads();
  const uint32_t base = blockIdx.x * kTile;
  uint32_t key[kBucketItems], rank[kBucketItems];
#pragma unroll
  for (int k = 0; k < kBucketItems; ++k) {
    const uint32_t i = base + k * kBucketThreads + threadIdx.x;
    if (i < count) {
      key[k] = bucket_key<RATE>(lengths[i]);
      rank[k] = atomicAdd(&local[key[k]], 1u);
    }
  }
  __syncthreads();
  const uint32_t n = local[threadIdx.x];
  // where the bin starts in `order` (every block scans the 512 totals of the histogram pass
  // itself: cheaper than one more launch) and where this block's part of it starts in the tile
  const uint32_t bin_base = block_exclusive_scan(hist[threadIdx.x], warp_sums[0]);
  const uint32_t in_tile = block_exclusive_scan(n, warp_sums[1]);
  const uint32_t in_order = n ? bin_base + atomicAdd(&cursor[threadIdx.x], n) : 0u;
  __shared__ uint32_t tile_start[kBucketBins], order_start[kBucketBins];
  tile_start[threadIdx.x] = in_tile;
  order_start[threadIdx.x] = in_order;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kBucketItems; ++k) {
    const uint32_t i = base + k * kBucketThreads + threadIdx.x;
    if (i < count) {
      const uint32_t q = tile_start[key[k]] + rank[k];
      tile_index[q] = i;
      tile_target[q] = order_start[key[k]] + rank[k];
    }
  }
  __syncthreads();
  const uint32_t tile_count = count - base < static_cast<uint32_t>(kTile) ? count - base : kTile;
  for (uint32_t q = threadIdx.x; q < tile_count; q += kBucketThreads) order[tile_target[q]] = tile_index[q];
}

template <uint32_t RATE>
__global__ void __launch_bounds__(256)
alignment_check_kernel(const uint64_t* __restrict__ offsets, const uint64_t* __restrict__ lengths,
                       uint64_t count, uint32_t* __restrict__ unaligned_flag) {
  const uint64_t len0 = lengths[0];
  const uint32_t first_tail = static_cast<uint32_t>(len0 - whole_blocks<RATE>(len0) * RATE);
  uint32_t misaligned = 0u, ragged = 0u, has_long = 0u;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t len = lengths[i];
    misaligned |= static_cast<uint32_t>(offsets[i]) & 7u;
    ragged |= static_cast<uint32_t>(len - whole_blocks<RATE>(len) * RATE) ^ first_tail;
    has_long |= len >= RATE ? 1u : 0u;
  }
  raise_flags(unaligned_flag, misaligned, ragged, has_long);
}

// ---------------------------------------------------------------------------
// Workloads.  splitmix64 is counter-based: output number n (1-based) of a
// generator seeded with s is mix(s + n * gamma)
// (proj/tools/sha3cli/workload.hpp:25-36), so any slice of the reference's
// stream can be produced independently.
__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t n) {
  uint64_t z = seed + n * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void store_word_bytes(uint8_t* dst, uint64_t word, uint32_t nbytes) {
  if (nbytes == 8u && (reinterpret_cast<uintptr_t>(dst) & 7u) == 0u) {
    *reinterpret_cast<uint64_t*>(dst) = word;
  } else {
    for (uint32_t b = 0; b < nbytes; ++b) dst[b] = static_cast<uint8_t>(word >> (8u * b));
  }
}

// generate_workload (proj/tools/sha3cli/workload.cpp:34-45): message i draws
// ceil(size/8) consecutive words; surplus bytes of its last word are dropped.
__global__ void __launch_bounds__(256)
generate_workload_kernel(uint64_t stream_seed, uint64_t message_size, uint64_t words_per_msg,
                         uint64_t first_message, uint64_t total_words, uint8_t* out) {
  for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
       w < total_words; w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = w / words_per_msg;
    const uint64_t k = w - i * words_per_msg;
    const uint64_t n = (first_message + i) * words_per_msg + k + 1u;
    const uint64_t left = message_size - 8u * k;
    store_word_bytes(out + i * message_size + 8u * k, splitmix_at(stream_seed, n),
                     left < 8u ? static_cast<uint32_t>(left) : 8u);
  }
}

__global__ void __launch_bounds__(256)
generate_lengths_kernel(uint64_t seed_len, uint64_t min_len, uint64_t span,
                        uint64_t first_message, uint64_t count, uint64_t* lengths) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    lengths[i] = min_len + splitmix_at(seed_len, first_message + i + 1u) % span;
  }
}

// One warp per message; lane k strides over the message's words.
__global__ void __launch_bounds__(256)
fill_messages_kernel(uint64_t seed, uint64_t first_message, uint64_t count,
                     const uint64_t* __restrict__ offsets,
                     const uint64_t* __restrict__ lengths, uint8_t* data) {
  const uint64_t warps_per_grid = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  const uint32_t lane = threadIdx.x & 31u;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       i < count; i += warps_per_grid) {
    const uint64_t key = seed ^ ((first_message + i) * 0xd1342543de82ef95ull);
    const uint64_t len = lengths[i];
    uint8_t* dst = data + offsets[i];
    const uint64_t words = (len + 7u) / 8u;
    for (uint64_t k = lane; k < words; k += 32u) {
      const uint64_t left = len - 8u * k;
      store_word_bytes(dst + 8u * k, splitmix_at(key, k + 1u),
                       left < 8u ? static_cast<uint32_t>(left) : 8u);
    }
  }
}

unsigned grid_for(uint64_t items, unsigned threads, unsigned cap = 148u * 32u) {
  const uint64_t blocks = (items + threads - 1) / threads;
  return static_cast<unsigned>(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

}  // namespace

cudaError_t launch_permute(uint64_t* states, uint64_t count, cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  const uint64_t blocks = (count + 127) / 128;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  permute_kernel<<<static_cast<unsigned>(blocks), 128, 0, stream>>>(states, count);
  return cudaGetLastError();
}

namespace {

template <uint32_t RATE>
cudaError_t bucket_order_for_rate(const uint64_t* offsets, const uint64_t* lengths, uint32_t count,
                                  uint32_t* order, uint32_t* scratch, uint32_t* unaligned_flag,
                                  cudaStream_t stream, bool short_kernel_next) {
  uint32_t* hist = scratch;             // zeroed by the caller, like the flag words
  uint32_t* cursor = scratch + kBucketBins;
  const unsigned per_block = kBucketThreads * kBucketItems;
  const unsigned blocks = (count + per_block - 1) / per_block;
  bucket_histogram_kernel<RATE><<<std::min(blocks, 148u * 8u), kBucketThreads, 0, stream>>>(offsets, lengths, count,
                                                                                          hist, unaligned_flag);
  bucket_scatter_kernel<RATE><<<blocks, kBucketThreads, 0, stream>>>(
      lengths, count, hist, cursor, order, short_kernel_next ? unaligned_flag : nullptr);
  return cudaGetLastError();
}

}  // namespace

// One instantiation per sponge rate (sha3.cpp:13-20).
#define B200SHA3_FOR_RATE(RATE_BYTES, CALL)      \
  switch (RATE_BYTES) {                          \
    case 72u: return CALL(72u);                  \
    case 104u: return CALL(104u);                \
    case 136u: return CALL(136u);                \
    case 144u: return CALL(144u);                \
    case 168u: return CALL(168u);                \
    default: return cudaErrorInvalidValue;       \
  }

cudaError_t launch_bucket_order(const uint64_t* offsets, const uint64_t* lengths,
                                uint32_t count, uint32_t rate_bytes, uint32_t* order,
                                uint32_t* scratch, uint32_t* unaligned_flag,
                                cudaStream_t stream, bool short_kernel_next) {
  if (count == 0) return cudaSuccess;
#define B200SHA3_CALL(R) \
  bucket_order_for_rate<R>(offsets, lengths, count, order, scratch, unaligned_flag, stream, short_kernel_next)
  B200SHA3_FOR_RATE(rate_bytes, B200SHA3_CALL)
#undef B200SHA3_CALL
}

namespace {
template <uint32_t RATE>
cudaError_t alignment_check_for_rate(const uint64_t* offsets, const uint64_t* lengths, uint64_t count,
                                     uint32_t* unaligned_flag, cudaStream_t stream) {
  alignment_check_kernel<RATE><<<grid_for(count, 256), 256, 0, stream>>>(offsets, lengths, count, unaligned_flag);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_alignment_check(const uint64_t* offsets, const uint64_t* lengths, uint64_t count,
                                   uint32_t rate_bytes, uint32_t* unaligned_flag, cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
#define B200SHA3_CALL(R) alignment_check_for_rate<R>(offsets, lengths, count, unaligned_flag, stream)
  B200SHA3_FOR_RATE(rate_bytes, B200SHA3_CALL)
#undef B200SHA3_CALL
}

cudaError_t launch_generate_workload(uint64_t stream_seed, uint64_t message_size,
                                     uint64_t first_message, uint64_t count, uint8_t* out,
                                     cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  const uint64_t wpm = (message_size + 7) / 8;
  const uint64_t total_words = wpm * count;
  generate_workload_kernel<<<grid_for(total_words, 256), 256, 0, stream>>>(
      stream_seed, message_size, wpm, first_message, total_words, out);
  return cudaGetLastError();
}

cudaError_t launch_generate_lengths(uint64_t seed_len, uint64_t min_len, uint64_t max_len,
                                    uint64_t first_message, uint64_t count,
                                    uint64_t* lengths, cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  generate_lengths_kernel<<<grid_for(count, 256), 256, 0, stream>>>(
      seed_len, min_len, max_len - min_len + 1, first_message, count, lengths);
  return cudaGetLastError();
}

cudaError_t launch_fill_messages(uint64_t seed, uint64_t first_message, uint64_t count,
                                 const uint64_t* offsets, const uint64_t* lengths,
                                 uint8_t* data, cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  fill_messages_kernel<<<grid_for(count * 32, 256, 148u * 64u), 256, 0, stream>>>(
      seed, first_message, count, offsets, lengths, data);
  return cudaGetLastError();
}

}  // namespace b200sha3
