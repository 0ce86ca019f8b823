// tests/integration/dropin_wall.cpp -- wall clock of the WHOLE sha3::hash_batch call on the
// reference's own types (vector<vector<uint8_t>> in, vector<vector<uint8_t>> out), the GPU
// drop-in (sha3::b200::hash_batch, pack + H2D + kernels + D2H + unpack) beside the compiled
// reference (oracle/_ref/libsha3kit_ref.so, Backend::parallel on every host core; its wall
// includes the digest-slot allocation of batch.cpp:77-81).  Measurement aid for DESIGN.md
// section 9 (row f-3); the reference side is loaded with dlopen and is optional.
//
//   dropin_wall [log2_count=20] [message_bytes=64 | 0 = ragged 0..300] [repeats=5]
//               [reference library | none] [workers=0 (all host threads)]
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "b200sha3/batch.hpp"

namespace {

struct SplitMix {
  std::uint64_t s;
  std::uint64_t next() {
    std::uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
};

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

using ref_create_fn = void* (*)(int, const std::uint8_t*, const std::uint64_t*, const std::uint64_t*,
                                std::uint64_t, std::uint64_t, std::uint64_t);
using ref_run_fn = int (*)(void*, int, unsigned, std::uint64_t, std::uint8_t*, double*);
using ref_destroy_fn = void (*)(void*);
using ref_wall_fn = int (*)(void*, unsigned, double*, double*);

}  // namespace

int main(int argc, char** argv) {
  const int log2_count = argc > 1 ? std::atoi(argv[1]) : 20;
  const std::uint64_t msg_bytes = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 64;
  const int repeats = argc > 3 ? std::atoi(argv[3]) : 5;
  const std::size_t count = std::size_t{1} << log2_count;

  sha3::HashBatch batch;
  batch.algorithm = sha3::Algorithm::sha3_256;
  batch.messages.resize(count);
  SplitMix rng{1};
  std::uint64_t total = 0;
  std::vector<std::uint64_t> offsets(count), lengths(count);
  for (std::size_t i = 0; i < count; ++i) {
    const std::uint64_t len = msg_bytes ? msg_bytes : rng.next() % 301;
    auto& m = batch.messages[i];
    m.resize(len);
    for (std::uint64_t k = 0; k < len; k += 8) {
      const std::uint64_t w = rng.next();
      std::memcpy(m.data() + k, &w, std::min<std::uint64_t>(8, len - k));
    }
    offsets[i] = total;
    lengths[i] = len;
    total += len;
  }

  // --- the GPU drop-in ---
  sha3::b200::StageTimes st;
  sha3::b200::DeviceConfig dev;
  dev.stages = &st;
  sha3::EngineConfig engine;
  engine.workers = argc > 5 ? static_cast<unsigned>(std::atoi(argv[5])) : 0;
  sha3::BatchResult ours = sha3::b200::hash_batch(batch, engine, dev);  // warm-up (context, pinning)
  std::vector<double> wall, scan, pipe, resize, call, pack, unpack, kern, elapsed_field;
  sha3::BatchResult prev;
  for (int r = 0; r < repeats; ++r) {
    prev = std::move(ours);  // keep the old digests alive: their destruction is not part of the call
    const double t0 = now_s();
    ours = sha3::b200::hash_batch(batch, engine, dev);
    wall.push_back(now_s() - t0);
    prev = {};
    scan.push_back(st.scan);
    pipe.push_back(st.pipeline);
    resize.push_back(st.resize);
    call.push_back(st.device_calls);
    pack.push_back(st.pack_cpu);
    unpack.push_back(st.unpack_cpu);
    kern.push_back(st.kernels);
    elapsed_field.push_back(ours.elapsed.count());
  }
  const double w = median(wall);
  std::printf("{\"count\": %zu, \"message_bytes\": \"%s\", \"total_bytes\": %llu, \"host_threads\": %u,\n"
              " \"b200_dropin\": {\"wall_s\": %.6f, \"hashes_per_s\": %.4g, \"scan_s\": %.6f, "
              "\"pipeline_s\": %.6f, \"resize_s\": %.6f, \"device_calls_s\": %.6f, \"pack_cpu_s\": %.6f, "
              "\"unpack_cpu_s\": %.6f, \"kernel_s\": %.6f, \"elapsed_field_s\": %.6f, \"threads\": %u, \"chunks\": %u, \"tasks\": %u}",
              count, msg_bytes ? std::to_string(msg_bytes).c_str() : "ragged 0..300",
              static_cast<unsigned long long>(total), std::thread::hardware_concurrency(), w,
              count / w, median(scan), median(pipe), median(resize), median(call), median(pack),
              median(unpack), median(kern), median(elapsed_field), st.threads, st.chunks, st.tasks);

  // --- the compiled reference, if present ---
  std::string lib = argc > 4 ? argv[4] : "oracle/_ref/libsha3kit_ref.so";
  if (void* h = dlopen(lib.c_str(), RTLD_NOW | RTLD_LOCAL)) {
    auto create = reinterpret_cast<ref_create_fn>(dlsym(h, "ref_batch_create"));
    auto run = reinterpret_cast<ref_run_fn>(dlsym(h, "ref_batch_run"));
    auto destroy = reinterpret_cast<ref_destroy_fn>(dlsym(h, "ref_batch_destroy"));
    auto run_wall = reinterpret_cast<ref_wall_fn>(dlsym(h, "ref_batch_run_wall"));
    if (create && run && destroy && run_wall) {
      std::vector<std::uint8_t> flat(total + 8);
      for (std::size_t i = 0; i < count; ++i) {
        if (lengths[i]) std::memcpy(flat.data() + offsets[i], batch.messages[i].data(), lengths[i]);
      }
      void* rb = create(1, flat.data(), offsets.data(), lengths.data(), 0, count, 0);
      std::vector<std::uint8_t> ref_out(count * 32);
      double elapsed = 0;
      run(rb, 1, 0, 0, ref_out.data(), &elapsed);  // warm-up + digests for the cross-check
      std::size_t bad = 0;
      for (std::size_t i = 0; i < count; ++i) {
        bad += std::memcmp(ours.digests[i].data(), ref_out.data() + i * 32, 32) != 0;
      }
      std::vector<double> rwall, rel;
      for (int r = 0; r < std::min(repeats, 3); ++r) {
        double call_wall = 0;
        run_wall(rb, 0, &call_wall, &elapsed);
        rwall.push_back(call_wall);
        rel.push_back(elapsed);
      }
      destroy(rb);
      const double rw = median(rwall);
      std::printf(",\n \"reference_parallel\": {\"wall_s\": %.6f, \"hashes_per_s\": %.4g, \"elapsed_s\": %.6f},\n"
                  " \"wall_speedup\": %.2f, \"digest_mismatches\": %zu",
                  rw, count / rw, median(rel), rw / w, bad);
    }
  }
  std::printf("}\n");
  return 0;
}
