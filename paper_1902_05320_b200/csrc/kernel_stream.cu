// kernel_stream.cu -- batched incremental hashing: N independent sponge states resident
// in HBM, fed chunk by chunk.
//
// The batch analogue of the reference's SpongeHasher (proj/core/include/sha3/sponge.hpp:38-64,
// proj/core/src/sponge.cpp:81-143) and Hasher (proj/core/include/sha3/sha3.hpp:66-86):
//   states_update_kernel   = update():  XOR bytes at the running position, permute at
//                            every block boundary, keep the position      (sponge.cpp:81-111)
//   states_finish_kernel   = finish():  pad at the position, permute      (sponge.cpp:113-129)
//                            followed by the first squeeze()
//   states_squeeze_kernel  = squeeze(): continue the output stream        (sponge.cpp:131-143)
// State layout (structure of arrays, so a warp's loads are coalesced): lane l of stream i
// at lanes[l * count + i] as (lo, hi); pos[i] = byte position in the current block;
// bit 31 of pos[i] set once the stream is finished (squeezing_).
#include <type_traits>

#include "kernels.cuh"
#include "sponge.cuh"

namespace b200sha3 {

namespace {

constexpr uint32_t kFinishedBit = 0x80000000u;

__device__ __forceinline__ void load_state(State& a, const uint2* lanes, uint64_t count, uint64_t i) {
#pragma unroll
  for (int l = 0; l < 25; ++l) {
    const uint2 v = lanes[l * count + i];
    a.lo[l] = v.x;
    a.hi[l] = v.y;
  }
}

__device__ __forceinline__ void store_state(const State& a, uint2* lanes, uint64_t count, uint64_t i) {
#pragma unroll
  for (int l = 0; l < 25; ++l) lanes[l * count + i] = make_uint2(a.lo[l], a.hi[l]);
}

template <int RL>
__global__ void __launch_bounds__(128)
states_update_kernel(uint2* lanes, uint32_t* pos_arr, uint64_t count, const uint8_t* data,
                     const uint64_t* offsets, const uint64_t* lengths, uint64_t fixed_len) {
  constexpr uint32_t R = 8u * RL;
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  uint64_t len = lengths ? lengths[i] : fixed_len;
  if (len == 0) return;
  const uint8_t* p = data + (offsets ? offsets[i] : i * fixed_len);
  uint32_t pos = pos_arr[i];
  State a;
  load_state(a, lanes, count, i);
  if (pos != 0u) {  // complete the block in progress
    const uint32_t n = len < R - pos ? static_cast<uint32_t>(len) : R - pos;
    absorb_bytes<RL>(a, p - pos, pos, pos + n);
    pos += n;
    p += n;
    len -= n;
    if (pos == R) {
      keccak_f1600<2, 0u>(a);
      pos = 0u;
    }
  }
  while (len >= R) {  // whole blocks (pos == 0 here)
    absorb_words_unaligned<RL>(a, p, 2 * RL);
    keccak_f1600<2, 0u>(a);
    p += R;
    len -= R;
  }
  if (len != 0u) {  // start of the next block
    absorb_bytes<RL>(a, p, 0u, static_cast<uint32_t>(len));
    pos = static_cast<uint32_t>(len);
  }
  store_state(a, lanes, count, i);
  pos_arr[i] = pos;
}

// Continues the output stream of finished states: `out_len` more bytes per stream.
template <int RL>
__device__ __forceinline__ uint32_t squeeze_from(State& a, uint32_t pos, uint8_t* o, uint64_t left) {
  constexpr uint32_t R = 8u * RL;
  while (left != 0u) {
    if (pos == R) {
      keccak_f1600<2, 0u>(a);
      pos = 0u;
    }
    const uint32_t n = left < R - pos ? static_cast<uint32_t>(left) : R - pos;
    if (pos == 0u) {
      emit_block<RL>(a, o, n);
    } else {
      emit_bytes<RL>(a, o, pos, pos + n);
    }
    pos += n;
    o += n;
    left -= n;
  }
  return pos;
}

template <int RL>
__global__ void __launch_bounds__(128)
states_finish_kernel(uint2* lanes, uint32_t* pos_arr, uint64_t count, uint32_t head,
                     uint8_t* out, uint64_t out_len, uint32_t last_mask) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  State a;
  load_state(a, lanes, count, i);
  xor_byte_at<RL>(a, pos_arr[i], head);   // sponge.cpp:122-123
  a.hi[RL - 1] ^= 0x80000000u;            // sponge.cpp:124-125
  keccak_f1600<2, 0u>(a);
  uint32_t pos = 0u;
  if (out != nullptr && out_len != 0u) {
    uint8_t* o = out + i * out_len;
    pos = squeeze_from<RL>(a, 0u, o, out_len);
    if (last_mask != 0xffu) o[out_len - 1u] &= static_cast<uint8_t>(last_mask);
  }
  store_state(a, lanes, count, i);
  pos_arr[i] = pos | kFinishedBit;
}

template <int RL>
__global__ void __launch_bounds__(128)
states_squeeze_kernel(uint2* lanes, uint32_t* pos_arr, uint64_t count, uint8_t* out,
                      uint64_t out_len) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  State a;
  load_state(a, lanes, count, i);
  const uint32_t pos = squeeze_from<RL>(a, pos_arr[i] & ~kFinishedBit, out + i * out_len, out_len);
  store_state(a, lanes, count, i);
  pos_arr[i] = pos | kFinishedBit;
}

template <class F>
cudaError_t dispatch_rate(int rate_lanes, F&& f) {
  switch (rate_lanes) {
    case 9: return f(std::integral_constant<int, 9>{});
    case 13: return f(std::integral_constant<int, 13>{});
    case 17: return f(std::integral_constant<int, 17>{});
    case 18: return f(std::integral_constant<int, 18>{});
    case 21: return f(std::integral_constant<int, 21>{});
    default: return cudaErrorInvalidValue;
  }
}

unsigned blocks_for(uint64_t count) { return static_cast<unsigned>((count + 127) / 128); }

}  // namespace

cudaError_t launch_states_update(int rate_lanes, void* lanes, uint32_t* pos, uint64_t count,
                                 const uint8_t* data, const uint64_t* offsets,
                                 const uint64_t* lengths, uint64_t fixed_len, cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  if (count > (0x7fffffffull * 128)) return cudaErrorInvalidConfiguration;
  return dispatch_rate(rate_lanes, [&](auto rl) {
    states_update_kernel<decltype(rl)::value><<<blocks_for(count), 128, 0, stream>>>(
        static_cast<uint2*>(lanes), pos, count, data, offsets, lengths, fixed_len);
    return cudaGetLastError();
  });
}

cudaError_t launch_states_finish(int rate_lanes, void* lanes, uint32_t* pos, uint64_t count,
                                 uint32_t head, uint8_t* out, uint64_t out_len, uint32_t last_mask,
                                 cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  if (count > (0x7fffffffull * 128)) return cudaErrorInvalidConfiguration;
  return dispatch_rate(rate_lanes, [&](auto rl) {
    states_finish_kernel<decltype(rl)::value><<<blocks_for(count), 128, 0, stream>>>(
        static_cast<uint2*>(lanes), pos, count, head, out, out_len, last_mask);
    return cudaGetLastError();
  });
}

cudaError_t launch_states_squeeze(int rate_lanes, void* lanes, uint32_t* pos, uint64_t count,
                                  uint8_t* out, uint64_t out_len, cudaStream_t stream) {
  if (count == 0 || out_len == 0) return cudaSuccess;
  if (count > (0x7fffffffull * 128)) return cudaErrorInvalidConfiguration;
  return dispatch_rate(rate_lanes, [&](auto rl) {
    states_squeeze_kernel<decltype(rl)::value><<<blocks_for(count), 128, 0, stream>>>(
        static_cast<uint2*>(lanes), pos, count, out, out_len);
    return cudaGetLastError();
  });
}

}  // namespace b200sha3
