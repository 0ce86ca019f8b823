// kernel_lanesplit.cu -- the lane-split layout of BASELINE.json's north_star,
// kept for the measured comparison against one-message-per-thread (DESIGN.md
// section 8); B200SHA3_KERNEL_LANESPLIT selects it, AUTO never does.
//
// Five threads share one Keccak state: thread x (0..4) of a group holds the
// column a[x][0..4] (5 lanes = 10 registers instead of 50).  A warp carries six
// groups (lanes 30, 31 idle).  Per round:
//   theta  column parity C[x] is thread-local; C[x-1] and C[x+1] come from the
//          neighbouring threads with four __shfl_sync;
//   rho    thread-local, per-thread rotation amounts (variable funnel shifts);
//   pi     moves 4 of every 5 lanes to another thread: done through a 200-byte
//          shared-memory tile per state (scatter to pi positions, __syncwarp);
//   chi    needs b[x], b[x+1], b[x+2] of every row: three shared loads per lane;
//   iota   thread 0 of the group.
// Same arithmetic as permute_1600 (proj/core/src/keccak.cpp:245-277); single
// block, whole-lane, equal-length messages only (the cfg1 / cfg5 shape).
#include "kernels.cuh"
#include "keccak_f1600.cuh"

namespace b200sha3 {

namespace {

// rho offsets, index x + 5y (keccak.cpp:26-32)
__constant__ uint32_t kRho[25] = {0,  1,  62, 28, 27, 36, 44, 6,  55, 20, 3,  10, 43,
                                  25, 39, 41, 45, 15, 21, 8,  18, 2,  61, 56, 14};

__device__ __forceinline__ uint2 rotl64_var(uint2 v, uint32_t n) {
  // n in [0, 63]; funnel shifts take n mod 32, halves swap for n >= 32
  const uint32_t lo = __funnelshift_l(v.y, v.x, n);
  const uint32_t hi = __funnelshift_l(v.x, v.y, n);
  return (n & 32u) ? make_uint2(hi, lo) : make_uint2(lo, hi);
}

constexpr int kGroupsPerWarp = 6;
constexpr int kWarpsPerBlock = 4;

__global__ void __launch_bounds__(32 * kWarpsPerBlock)
hash_lanesplit_kernel(const uint8_t* __restrict__ data, uint8_t* __restrict__ digests,
                      uint64_t count, uint32_t msg_lanes, uint32_t rate_lanes,
                      uint32_t out_lanes, uint32_t head) {
  __shared__ uint2 tile[kWarpsPerBlock][kGroupsPerWarp][25];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t group = lane / 5u, x = lane % 5u;
  const bool active_lane = lane < 30u;
  const uint64_t m = (static_cast<uint64_t>(blockIdx.x) * kWarpsPerBlock + warp) * kGroupsPerWarp + group;
  const bool live = active_lane && m < count;
  const uint32_t base = group * 5u;                 // first lane of this group in the warp
  const uint32_t left = base + (x + 4u) % 5u, right = base + (x + 1u) % 5u;

  uint2 a[5];
  uint32_t rho[5], dest[5];
#pragma unroll
  for (int y = 0; y < 5; ++y) {
    const uint32_t i = x + 5u * y;
    rho[y] = kRho[i];
    dest[y] = y + 5u * ((2u * x + 3u * y) % 5u);    // pi: (x, y) -> (y, 2x + 3y)
    uint2 v = make_uint2(0u, 0u);
    if (live && i < msg_lanes) {
      v = __ldg(reinterpret_cast<const uint2*>(data + m * (8ull * msg_lanes)) + i);
    }
    if (i == msg_lanes) v.x ^= head;                // sponge.cpp:122-123
    if (i == rate_lanes - 1u) v.y ^= 0x80000000u;   // sponge.cpp:124-125
    a[y] = v;
  }
  uint2* t = tile[warp][active_lane ? group : 0];

#pragma unroll 1
  for (int round = 0; round < 24; ++round) {
    uint2 c;
    c.x = xor3(xor3(a[0].x, a[1].x, a[2].x), a[3].x, a[4].x);
    c.y = xor3(xor3(a[0].y, a[1].y, a[2].y), a[3].y, a[4].y);
    uint2 cm, cp;
    cm.x = __shfl_sync(0xffffffffu, c.x, left);
    cm.y = __shfl_sync(0xffffffffu, c.y, left);
    cp.x = __shfl_sync(0xffffffffu, c.x, right);
    cp.y = __shfl_sync(0xffffffffu, c.y, right);
    const uint32_t rl = __funnelshift_l(cp.y, cp.x, 1), rh = __funnelshift_l(cp.x, cp.y, 1);
#pragma unroll
    for (int y = 0; y < 5; ++y) {
      a[y].x = xor3(a[y].x, cm.x, rl);
      a[y].y = xor3(a[y].y, cm.y, rh);
      if (active_lane) t[dest[y]] = rotl64_var(a[y], rho[y]);
    }
    __syncwarp();
#pragma unroll
    for (int y = 0; y < 5; ++y) {
      const uint2 b0 = t[x + 5u * y], b1 = t[(x + 1u) % 5u + 5u * y], b2 = t[(x + 2u) % 5u + 5u * y];
      a[y].x = chi3(b0.x, b1.x, b2.x);
      a[y].y = chi3(b0.y, b1.y, b2.y);
    }
    if (x == 0u) {
      a[0].x ^= kRoundConst32[2 * round];
      a[0].y ^= kRoundConst32[2 * round + 1];
    }
    __syncwarp();
  }
#pragma unroll
  for (int y = 0; y < 5; ++y) {
    const uint32_t i = x + 5u * y;
    if (live && i < out_lanes) {
      reinterpret_cast<uint2*>(digests + m * (8ull * out_lanes))[i] = a[y];
    }
  }
}

}  // namespace

bool lanesplit_supported(int rate_lanes, uint64_t msg_len, uint64_t digest_bytes) {
  return msg_len % 8 == 0 && msg_len < 8u * static_cast<uint64_t>(rate_lanes) &&
         digest_bytes % 8 == 0 && digest_bytes != 0 && digest_bytes <= 8u * rate_lanes;
}

cudaError_t launch_hash_lanesplit(const HashArgs& args, const LaunchPlan& plan,
                                  cudaStream_t stream) {
  if (!lanesplit_supported(plan.rate_lanes, args.fixed_len, args.digest_bytes) || args.offsets ||
      args.lengths || args.order || !args.aligned8 || args.last_mask != 0xffu) {
    return cudaErrorNotSupported;
  }
  const uint64_t per_block = static_cast<uint64_t>(kWarpsPerBlock) * kGroupsPerWarp;
  const uint64_t blocks = (args.count + per_block - 1) / per_block;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  hash_lanesplit_kernel<<<static_cast<unsigned>(blocks), 32 * kWarpsPerBlock, 0, stream>>>(
      args.data, args.digests, args.count, static_cast<uint32_t>(args.fixed_len / 8),
      static_cast<uint32_t>(plan.rate_lanes), static_cast<uint32_t>(args.digest_bytes / 8),
      args.head);
  return cudaGetLastError();
}

}  // namespace b200sha3
