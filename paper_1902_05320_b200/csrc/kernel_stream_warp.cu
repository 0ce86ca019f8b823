// kernel_stream_warp.cu -- batched incremental hashing, one stream per WARP: the
// warp-per-state form (warp_state.cuh, kernel_warp.cu) of the three kernels of kernel_stream.cu,
// for few streams -- the usual way the incremental API is used (one big input fed in pieces:
// sha3::Hasher, proj/core/include/sha3/sha3.hpp:66-86; `b200sha3cli hash FILE`).  A stream's
// chunk is absorbed block after block by one warp at ~2.0 us per permutation instead of ~5.1 us
// on one thread.  Same state layout in HBM as the one-thread kernels (lane l of stream i at
// lanes[l * count + i], pos[i] with bit 31 = finished), so the two forms can be mixed freely on
// one set of states; capi_stream.cu picks this one below warp_kernel_max_count() streams.
//
//   states_update_warp_kernel   update():  sponge.cpp:81-111
//   states_finish_warp_kernel   finish() + first squeeze(): sponge.cpp:113-143
//   states_squeeze_warp_kernel  squeeze(): sponge.cpp:131-143
#include "kernels.cuh"
#include "warp_state.cuh"

namespace b200sha3 {

namespace {

using namespace warp_state;

constexpr uint32_t kFinishedBit = 0x80000000u;

struct WarpLane {
  uint32_t lo = 0u, hi = 0u;
};

__device__ __forceinline__ WarpLane load_warp_state(const uint2* lanes, uint64_t count, uint64_t i, uint32_t t) {
  WarpLane s;
  if (t < 25u) {
    const uint2 v = lanes[t * count + i];
    s.lo = v.x;
    s.hi = v.y;
  }
  return s;
}

__device__ __forceinline__ void store_warp_state(const WarpLane& s, uint2* lanes, uint64_t count, uint64_t i,
                                                 uint32_t t) {
  if (t < 25u) lanes[t * count + i] = make_uint2(s.lo, s.hi);
}

// XORs bytes [from, to) of the current rate block into the state; block byte k is vp[k] (only
// [vp + from, vp + to) is message data).  Thread t owns block bytes [8t, 8t + 8).
__device__ __forceinline__ void absorb_range(WarpLane& s, const uint8_t* vp, uint32_t from, uint32_t to,
                                             uint32_t t) {
  const uint32_t b = from > 8u * t ? from : 8u * t;
  const uint32_t e = to < 8u * t + 8u ? to : 8u * t + 8u;
  if (b >= e) return;
  uint2 v = make_uint2(0u, 0u);
  if (e - b == 8u) {
    v = load_lane(vp + 8u * t);
  } else {
    for (uint32_t k = b; k < e; ++k) {
      const uint32_t byte = ld_u8(vp + k), shift = 8u * (k - 8u * t);
      if (shift < 32u) {
        v.x |= byte << shift;
      } else {
        v.y |= byte << (shift - 32u);
      }
    }
  }
  s.lo ^= v.x;
  s.hi ^= v.y;
}

// Writes block bytes [from, to) of the rate part to o[0 .. to - from).
__device__ __forceinline__ void emit_range(const WarpLane& s, uint8_t* o, uint32_t from, uint32_t to, uint32_t t) {
  const uint32_t b = from > 8u * t ? from : 8u * t;
  const uint32_t e = to < 8u * t + 8u ? to : 8u * t + 8u;
  if (b >= e) return;
  uint8_t* dst = o + (b - from);
  if (e - b == 8u && (reinterpret_cast<uintptr_t>(dst) & 7u) == 0u) {
    *reinterpret_cast<uint2*>(dst) = make_uint2(s.lo, s.hi);
    return;
  }
  for (uint32_t k = b; k < e; ++k) {
    const uint32_t shift = 8u * (k - 8u * t);
    dst[k - b] = static_cast<uint8_t>(shift < 32u ? s.lo >> shift : s.hi >> (shift - 32u));
  }
}

__global__ void __launch_bounds__(32)
states_update_warp_kernel(uint2* lanes, uint32_t* pos_arr, uint64_t count, const uint8_t* data,
                          const uint64_t* offsets, const uint64_t* lengths, uint64_t fixed_len,
                          uint32_t rate_lanes) {
  const uint32_t t = threadIdx.x;
  const uint64_t i = blockIdx.x;
  uint64_t len = lengths ? lengths[i] : fixed_len;
  if (len == 0) return;
  const uint8_t* p = data + (offsets ? offsets[i] : i * fixed_len);
  const uint32_t R = 8u * rate_lanes;
  const LaneRole role = lane_role(t);
  uint32_t pos = pos_arr[i];
  WarpLane s = load_warp_state(lanes, count, i, t);
  // The block in progress first (sponge.cpp:100-109), then whole blocks with the next one in
  // flight during the rounds, then the start of the next block -- one loop, one copy of the rounds.
  uint32_t head = 0u;  // bytes that complete the block in progress
  if (pos != 0u) {
    head = len < R - pos ? static_cast<uint32_t>(len) : R - pos;
    absorb_range(s, p - pos, pos, pos + head, t);
    pos += head;
    p += head;
    len -= head;
  }
  const bool close_head = pos == R;
  const uint64_t whole = (pos == 0u || close_head) ? len / R : 0;
  const bool in_rate = t < rate_lanes;
  uint2 next = make_uint2(0u, 0u);
  if (!close_head && whole != 0 && in_rate) next = load_lane(p + 8u * t);
  const uint64_t rounds = whole + (close_head ? 1u : 0u);
  for (uint64_t k = 0; k < rounds; ++k) {
    if (!(close_head && k == 0)) {  // a whole block straight from the message
      s.lo ^= next.x;
      s.hi ^= next.y;
      p += R;
    }
    next = make_uint2(0u, 0u);
    if (k + 1 < rounds && in_rate) next = load_lane(p + 8u * t);
    warp_permute(s.lo, s.hi, role);
  }
  if (rounds != 0) {
    pos = 0u;
    len -= whole * R;
  }
  if (len != 0 && pos == 0u) {  // start of the next block
    absorb_range(s, p, 0u, static_cast<uint32_t>(len), t);
    pos = static_cast<uint32_t>(len);
  }
  store_warp_state(s, lanes, count, i, t);
  if (t == 0u) pos_arr[i] = pos;
}

// Continues the output stream: `left` more bytes to o, permuting at block boundaries.
__device__ __forceinline__ uint32_t squeeze_from(WarpLane& s, uint32_t pos, uint8_t* o, uint64_t left,
                                                 uint32_t R, const LaneRole& role, uint32_t t) {
  while (left != 0u) {
    if (pos == R) {
      warp_permute(s.lo, s.hi, role);
      pos = 0u;
    }
    const uint32_t n = left < R - pos ? static_cast<uint32_t>(left) : R - pos;
    emit_range(s, o, pos, pos + n, t);
    pos += n;
    o += n;
    left -= n;
  }
  return pos;
}

__global__ void __launch_bounds__(32)
states_finish_warp_kernel(uint2* lanes, uint32_t* pos_arr, uint64_t count, uint32_t head, uint8_t* out,
                          uint64_t out_len, uint32_t last_mask, uint32_t rate_lanes) {
  const uint32_t t = threadIdx.x;
  const uint64_t i = blockIdx.x;
  const uint32_t R = 8u * rate_lanes;
  const LaneRole role = lane_role(t);
  WarpLane s = load_warp_state(lanes, count, i, t);
  const uint32_t at = pos_arr[i];
  if (t == (at >> 3)) {  // sponge.cpp:122-123
    const uint32_t shift = 8u * (at & 7u);
    if (shift < 32u) {
      s.lo ^= head << shift;
    } else {
      s.hi ^= head << (shift - 32u);
    }
  }
  if (t == rate_lanes - 1u) s.hi ^= 0x80000000u;  // sponge.cpp:124-125
  // (pos == R triggers the permutation inside squeeze_from: finish()'s own permute, sponge.cpp:126)
  uint32_t pos = R;
  if (out != nullptr && out_len != 0u) {
    uint8_t* o = out + i * out_len;
    pos = squeeze_from(s, pos, o, out_len, R, role, t);
    if (last_mask != 0xffu) {
      __syncwarp();
      if (t == 0u) o[out_len - 1u] &= static_cast<uint8_t>(last_mask);
    }
  } else {
    warp_permute(s.lo, s.hi, role);
    pos = 0u;
  }
  store_warp_state(s, lanes, count, i, t);
  if (t == 0u) pos_arr[i] = pos | kFinishedBit;
}

__global__ void __launch_bounds__(32)
states_squeeze_warp_kernel(uint2* lanes, uint32_t* pos_arr, uint64_t count, uint8_t* out, uint64_t out_len,
                           uint32_t rate_lanes) {
  const uint32_t t = threadIdx.x;
  const uint64_t i = blockIdx.x;
  const LaneRole role = lane_role(t);
  WarpLane s = load_warp_state(lanes, count, i, t);
  const uint32_t pos =
      squeeze_from(s, pos_arr[i] & ~kFinishedBit, out + i * out_len, out_len, 8u * rate_lanes, role, t);
  store_warp_state(s, lanes, count, i, t);
  __syncwarp();
  if (t == 0u) pos_arr[i] = pos | kFinishedBit;
}

}  // namespace

cudaError_t launch_states_update_warp(int rate_lanes, void* lanes, uint32_t* pos, uint64_t count,
                                      const uint8_t* data, const uint64_t* offsets, const uint64_t* lengths,
                                      uint64_t fixed_len, cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  if (count > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  states_update_warp_kernel<<<static_cast<unsigned>(count), 32, 0, stream>>>(
      static_cast<uint2*>(lanes), pos, count, data, offsets, lengths, fixed_len, static_cast<uint32_t>(rate_lanes));
  return cudaGetLastError();
}

cudaError_t launch_states_finish_warp(int rate_lanes, void* lanes, uint32_t* pos, uint64_t count, uint32_t head,
                                      uint8_t* out, uint64_t out_len, uint32_t last_mask, cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  if (count > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  states_finish_warp_kernel<<<static_cast<unsigned>(count), 32, 0, stream>>>(
      static_cast<uint2*>(lanes), pos, count, head, out, out_len, last_mask, static_cast<uint32_t>(rate_lanes));
  return cudaGetLastError();
}

cudaError_t launch_states_squeeze_warp(int rate_lanes, void* lanes, uint32_t* pos, uint64_t count, uint8_t* out,
                                       uint64_t out_len, cudaStream_t stream) {
  if (count == 0 || out_len == 0) return cudaSuccess;
  if (count > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  states_squeeze_warp_kernel<<<static_cast<unsigned>(count), 32, 0, stream>>>(
      static_cast<uint2*>(lanes), pos, count, out, out_len, static_cast<uint32_t>(rate_lanes));
  return cudaGetLastError();
}

}  // namespace b200sha3
