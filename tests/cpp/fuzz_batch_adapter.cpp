// tests/cpp/fuzz_batch_adapter.cpp -- randomized stress of sha3::b200::hash_batch (the pipelined
// C++ adapter) against the CPU oracle: random batch shapes (equal-length, ragged, "equal but
// for one message" -- the speculative plan's restart --, a few long messages among short ones,
// all-empty), all six algorithms, odd XOF bit counts, worker counts, one or several device
// entries, concurrent callers.  Linked against libb200sha3.so it exercises the real device;
// linked against fake_device_capi.cpp (+ -fsanitize=thread/address) it checks the host-side
// scheduling alone and adds fault injection.
//
//   fuzz_batch_adapter [seconds=10] [seed=1] [max_log2_count=17]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "b200sha3/batch.hpp"

extern "C" int ko_hash_one(int algorithm, std::uint64_t xof_bits, const std::uint8_t* msg,
                           std::uint64_t len, std::uint8_t* out);
extern "C" std::uint64_t ko_digest_bytes(int algorithm, std::uint64_t xof_bits);
#ifdef B200SHA3_FAKE_DEVICE
extern "C" void fake_device_fail_at(long nth_call_from_now);
#endif

namespace {

struct Rng {
  std::uint64_t s;
  std::uint64_t next() {
    std::uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  std::uint64_t below(std::uint64_t n) { return n ? next() % n : 0; }
};

void fill(std::vector<std::uint8_t>& m, std::size_t len, Rng& rng) {
  m.resize(len);
  for (std::size_t k = 0; k < len; k += 8) {
    const std::uint64_t w = rng.next();
    std::memcpy(m.data() + k, &w, std::min<std::size_t>(8, len - k));
  }
}

struct Case {
  sha3::HashBatch batch;
  sha3::EngineConfig engine;
  sha3::b200::DeviceConfig device;
  std::string shape;
};

Case make_case(Rng& rng, int max_log2) {
  Case c;
  const int alg = static_cast<int>(rng.below(6));
  c.batch.algorithm = static_cast<sha3::Algorithm>(alg);
  if (alg >= 4) c.batch.xof_output_bits = 1 + rng.below(rng.below(4) ? 600 : 3000);
  const int lg = static_cast<int>(rng.below(max_log2 + 1));
  std::size_t count = (std::size_t{1} << lg) + rng.below(std::size_t{1} << lg) - (rng.below(2) ? 1 : 0);
  const int shape = static_cast<int>(rng.below(6));
  const std::size_t base = rng.below(3) ? rng.below(200) : rng.below(1500);
  // keep the oracle side affordable
  while (count > 64 && count * (base + 200) > (48u << 20)) count /= 2;
  c.batch.messages.resize(count);
  const std::size_t odd = rng.below(count ? count : 1);
  for (std::size_t i = 0; i < count; ++i) {
    std::size_t len = base;
    switch (shape) {
      case 0: break;                                                     // equal length
      case 1: len = rng.below(2 * base + 2); break;                      // ragged
      case 2: if (i == odd) len = base + 1 + rng.below(300); break;      // equal but for one
      case 3: if (rng.below(4096) == 0) len = 20000 + rng.below(60000); else len = rng.below(base + 1); break;
      case 4: len = 0; break;                                            // all empty
      default: if (i == count - 1) len = base ? base - 1 : 1; break;     // odd one last
    }
    fill(c.batch.messages[i], len, rng);
  }
  static const char* names[] = {"equal", "ragged", "equal-but-one", "few-long", "all-empty", "odd-last"};
  c.shape = names[shape];
  const unsigned workers[] = {0, 1, 2, 3, 5, 16};
  c.engine.workers = workers[rng.below(6)];
  switch (rng.below(4)) {
    case 0: c.device.devices = {0}; break;
    case 1: c.device.devices = {0, 0}; break;
    case 2: c.device.devices = {0, 0, 0}; break;
    default: break;
  }
  return c;
}

// Number of digests that differ from the oracle's (checked by `threads` threads).
std::size_t mismatches(const sha3::HashBatch& batch, const sha3::BatchResult& res, unsigned threads) {
  const std::size_t n = batch.messages.size();
  if (res.digests.size() != n) return n + 1;
  const int alg = static_cast<int>(batch.algorithm);
  const std::uint64_t db = ko_digest_bytes(alg, batch.xof_output_bits);
  std::vector<std::size_t> bad(threads, 0);
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      std::vector<std::uint8_t> e(db);
      const std::uint8_t none = 0;
      for (std::size_t i = n * t / threads; i < n * (t + 1) / threads; ++i) {
        const auto& m = batch.messages[i];
        ko_hash_one(alg, batch.xof_output_bits, m.empty() ? &none : m.data(), m.size(), e.data());
        bad[t] += res.digests[i] != e;
      }
    });
  }
  for (auto& t : pool) t.join();
  std::size_t total = 0;
  for (std::size_t b : bad) total += b;
  return total;
}

}  // namespace

int main(int argc, char** argv) {
  const double seconds = argc > 1 ? std::atof(argv[1]) : 10.0;
  Rng rng{argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1};
  const int max_log2 = argc > 3 ? std::atoi(argv[3]) : 17;
  const unsigned check_threads = std::max(2u, std::thread::hardware_concurrency());
  const auto t0 = std::chrono::steady_clock::now();
  const auto elapsed = [&] {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  std::size_t batches = 0, messages = 0, failures = 0, injected = 0;
  while (elapsed() < seconds) {
    Case c = make_case(rng, max_log2);
    sha3::b200::StageTimes st;
    c.device.stages = &st;
    std::size_t bad = 0;
    if (rng.below(8) == 0 && c.batch.messages.size() < 5000) {  // three concurrent callers
      std::vector<std::size_t> each(3, 0);
      std::vector<std::thread> callers;
      for (int k = 0; k < 3; ++k) {
        callers.emplace_back([&, k] {
          sha3::b200::DeviceConfig dev = c.device;
          dev.stages = nullptr;
          each[k] = mismatches(c.batch, sha3::b200::hash_batch(c.batch, c.engine, dev), 2);
        });
      }
      for (auto& t : callers) t.join();
      bad = each[0] + each[1] + each[2];
    } else {
      bad = mismatches(c.batch, sha3::b200::hash_batch(c.batch, c.engine, c.device), check_threads);
    }
#ifdef B200SHA3_FAKE_DEVICE
    if (rng.below(4) == 0 && !c.batch.messages.empty()) {  // a device call fails mid-pipeline
      fake_device_fail_at(static_cast<long>(rng.below(st.chunks ? st.chunks : 1)));
      bool threw = false;
      try {
        sha3::b200::hash_batch(c.batch, c.engine, c.device);
      } catch (const sha3::b200::DeviceError&) {
        threw = true;
      }
      fake_device_fail_at(-1);
      bad += threw ? 0 : 1;
      ++injected;
      // and the adapter is healthy afterwards
      bad += mismatches(c.batch, sha3::b200::hash_batch(c.batch, c.engine, c.device), check_threads);
    }
#endif
    if (bad) {
      ++failures;
      std::fprintf(stderr, "FAIL batch %zu: shape %s alg %d count %zu workers %u devices %zu: %zu bad\n",
                   batches, c.shape.c_str(), static_cast<int>(c.batch.algorithm), c.batch.messages.size(),
                   c.engine.workers, c.device.devices.size(), bad);
    }
    ++batches;
    messages += c.batch.messages.size();
  }
  std::printf("{\"seconds\": %.1f, \"batches\": %zu, \"messages\": %zu, \"injected_failures\": %zu, "
              "\"mismatching_batches\": %zu}\n", elapsed(), batches, messages, injected, failures);
  return failures ? 1 : 0;
}
