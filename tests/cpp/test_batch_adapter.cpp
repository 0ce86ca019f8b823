// tests/cpp/test_batch_adapter.cpp -- the hash_batch cases of the reference's
// proj/tests/test_batch.cpp:101-197 and proj/tests/acceptance.cpp:254-273,
// restated against the C++ adapter (sha3::b200::hash_batch and the
// sha3::hash_batch drop-in).  Expected digests come from the CPU oracle
// (oracle/liboracle.so, ko_hash_one) -- this file is test code, the only kind
// allowed to link it.
//
//   test_batch_adapter            all cases (needs a GPU)
//   test_batch_adapter --cpu-only the cases that must work without a device
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "b200sha3/batch.hpp"

extern "C" int ko_hash_one(int algorithm, std::uint64_t xof_bits, const std::uint8_t* msg,
                           std::uint64_t len, std::uint8_t* out);
extern "C" std::uint64_t ko_digest_bytes(int algorithm, std::uint64_t xof_bits);

namespace sha3 {
BatchResult hash_batch(const HashBatch& batch, const EngineConfig& config);  // the drop-in
}

namespace {

int g_failures = 0;
int g_checks = 0;

#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_failures;                                                        \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)

// testutil::Rng (proj/tests/test_util.hpp:14-35)
struct Rng {
  std::uint64_t state;
  explicit Rng(std::uint64_t seed) : state(seed) {}
  std::uint64_t next() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  std::uint64_t below(std::uint64_t n) { return next() % n; }
};

std::vector<std::uint8_t> random_bytes(Rng& rng, std::size_t n) {
  std::vector<std::uint8_t> out(n);
  for (auto& b : out) b = static_cast<std::uint8_t>(rng.next());
  return out;
}

sha3::HashBatch random_batch(Rng& rng, std::size_t count, std::size_t max_len = 300) {
  sha3::HashBatch batch;
  batch.messages.reserve(count);
  for (std::size_t i = 0; i < count; ++i) {
    batch.messages.push_back(random_bytes(rng, rng.below(max_len + 1)));
  }
  return batch;
}

std::vector<std::uint8_t> expect(sha3::Algorithm a, const std::vector<std::uint8_t>& m,
                                 std::uint64_t bits = 0) {
  const int alg = static_cast<int>(a);
  std::vector<std::uint8_t> out(ko_digest_bytes(alg, bits));
  const std::uint8_t dummy = 0;
  ko_hash_one(alg, bits, m.empty() ? &dummy : m.data(), m.size(), out.data());
  return out;
}

bool matches_oracle(const sha3::HashBatch& batch, const sha3::BatchResult& res) {
  if (res.digests.size() != batch.messages.size()) return false;
  for (std::size_t i = 0; i < batch.messages.size(); ++i) {
    if (res.digests[i] != expect(batch.algorithm, batch.messages[i], batch.xof_output_bits)) {
      return false;
    }
  }
  return true;
}

void cpu_only_cases() {
  using namespace sha3;
  {  // "XOF without an output length is rejected up front" (test_batch.cpp:162-167)
    HashBatch batch;
    batch.algorithm = Algorithm::shake256;
    batch.messages = {{1}};
    bool threw = false;
    try {
      hash_batch(batch, {});
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()) == "hash_batch: XOF variants need xof_output_bits";
    }
    CHECK(threw);
    threw = false;
    try {
      b200::hash_batch(batch);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // "empty batch yields an empty result" (test_batch.cpp:113-117)
    const BatchResult res = hash_batch(HashBatch{}, {});
    CHECK(res.digests.empty());
    CHECK(res.elapsed.count() < 0.5);
    HashBatch xof;
    xof.algorithm = Algorithm::shake128;
    xof.xof_output_bits = 328;
    CHECK(hash_batch(xof, {}).digests.empty());
  }
}

void gpu_cases() {
  using namespace sha3;
  {  // "a hundred copies of one message" (test_batch.cpp:102-111)
    HashBatch batch;
    batch.messages.assign(100, std::vector<std::uint8_t>(10, 0x42));
    const BatchResult res = hash_batch(batch, {});
    CHECK(res.digests.size() == 100);
    const auto e = expect(Algorithm::sha3_256, batch.messages[0]);
    for (const auto& d : res.digests) CHECK(d == e);
    CHECK(res.elapsed.count() > 0.0);
  }
  {  // "parallel equals sequential on random batches" (test_batch.cpp:119-135):
     // here every EngineConfig must give the oracle's digests
    Rng rng(52);
    for (std::size_t count : {0u, 1u, 7u, 100u, 2000u}) {
      const HashBatch batch = random_batch(rng, count);
      EngineConfig seq;
      seq.backend = Backend::sequential;
      const BatchResult first = hash_batch(batch, seq);
      CHECK(matches_oracle(batch, first));
      for (unsigned workers : {2u, 3u, 8u}) {
        EngineConfig par;
        par.backend = Backend::parallel;
        par.workers = workers;
        par.chunk_size = 1 + rng.below(17);
        CHECK(hash_batch(batch, par).digests == first.digests);
      }
    }
  }
  {  // "order is preserved" (test_batch.cpp:137-148)
    Rng rng(53);
    const HashBatch batch = random_batch(rng, 500, 40);
    EngineConfig cfg;
    cfg.workers = 4;
    cfg.chunk_size = 7;
    CHECK(matches_oracle(batch, hash_batch(batch, cfg)));
  }
  {  // "XOF batches carry the requested output length" (test_batch.cpp:150-160)
    HashBatch batch;
    batch.algorithm = Algorithm::shake128;
    batch.xof_output_bits = 328;
    batch.messages = {{1, 2, 3}, {}, {9, 9, 9, 9}};
    const BatchResult res = hash_batch(batch, {});
    CHECK(res.digests.size() == 3);
    for (const auto& d : res.digests) CHECK(d.size() == 41);
    CHECK(matches_oracle(batch, res));
  }
  {  // "variable-length messages are fine" (test_batch.cpp:169-176)
    HashBatch batch;
    batch.messages = {{}, std::vector<std::uint8_t>(1000, 1), {5}, std::vector<std::uint8_t>(137, 2)};
    CHECK(matches_oracle(batch, hash_batch(batch, {})));
  }
  {  // "reentrant from multiple callers" (test_batch.cpp:178-196)
    Rng rng(54);
    const HashBatch batch = random_batch(rng, 200, 30);
    const BatchResult e = hash_batch(batch, {});
    CHECK(matches_oracle(batch, e));
    std::array<bool, 3> ok{};
    {
      std::vector<std::thread> callers;
      for (int t = 0; t < 3; ++t) {
        callers.emplace_back([&, t] {
          EngineConfig cfg;
          cfg.workers = 2;
          ok[t] = hash_batch(batch, cfg).digests == e.digests;
        });
      }
      for (auto& c : callers) c.join();
    }
    for (bool b : ok) CHECK(b);
  }
  {  // acceptance criterion 5 (acceptance.cpp:254-273), all six variants
    Rng rng(0xe9);
    for (const std::size_t count : {0, 1, 7, 100, 10000}) {
      HashBatch batch;
      batch.messages.reserve(count);
      for (std::size_t i = 0; i < count; ++i) {
        batch.messages.push_back(random_bytes(rng, rng.below(200)));
      }
      for (int a = 0; a < 6; ++a) {
        batch.algorithm = static_cast<Algorithm>(a);
        batch.xof_output_bits = a >= 4 ? 4099 : 0;
        CHECK(matches_oracle(batch, hash_batch(batch, {})));
      }
    }
  }
  {  // equal-length batch large enough for the pipelined fixed-length entry and
     // the pack/unpack thread pool
    Rng rng(77);
    HashBatch batch;
    const std::size_t count = 300000;
    batch.messages.resize(count);
    for (auto& m : batch.messages) {
      m.resize(64);
      for (std::size_t i = 0; i < 64; i += 8) {
        const std::uint64_t w = rng.next();
        std::memcpy(m.data() + i, &w, 8);
      }
    }
    const BatchResult res = hash_batch(batch, {});
    bool ok = res.digests.size() == count;
    for (std::size_t i = 0; ok && i < count; i += 997) {
      ok = res.digests[i] == expect(batch.algorithm, batch.messages[i]);
    }
    CHECK(ok);
  }
  {  // a large batch that LOOKS equal-length (every sampled size agrees) but is not: the
     // adapter starts on the fixed-length layout, a pack task finds the odd message and the
     // call restarts on the ragged layout.  Also the all-empty batch (length 0 everywhere).
    Rng rng(78);
    HashBatch batch;
    const std::size_t count = (1u << 18) + 4321;
    batch.messages.resize(count);
    for (auto& m : batch.messages) {
      m.resize(24);
      for (std::size_t i = 0; i < 24; i += 8) {
        const std::uint64_t w = rng.next();
        std::memcpy(m.data() + i, &w, 8);
      }
    }
    for (const std::size_t odd : {count / 2 + 3, count - 2}) {
      HashBatch ragged = batch;
      ragged.messages[odd].resize(odd % 2 ? 200 : 0, 0x5a);
      b200::StageTimes st;
      b200::DeviceConfig dev;
      dev.stages = &st;
      const BatchResult res = b200::hash_batch(ragged, {}, dev);
      bool ok = res.digests.size() == count;
      for (std::size_t i = 0; ok && i < count; i += 1009) {
        ok = res.digests[i] == expect(ragged.algorithm, ragged.messages[i]);
      }
      for (std::size_t i = odd - 2; ok && i < std::min(count, odd + 3); ++i) {
        ok = res.digests[i] == expect(ragged.algorithm, ragged.messages[i]);
      }
      CHECK(ok);
      CHECK(st.threads >= 1 && st.chunks >= 1);
    }
    HashBatch empties;
    empties.algorithm = Algorithm::sha3_512;
    empties.messages.resize(count);
    const BatchResult res = hash_batch(empties, {});
    const auto e = expect(Algorithm::sha3_512, {});
    bool ok = res.digests.size() == count;
    for (std::size_t i = 0; ok && i < count; i += 511) ok = res.digests[i] == e;
    CHECK(ok && res.digests.back() == e);
  }
  {  // several devices: chunks dealt round-robin, one host thread per device.  The box has
     // one GPU, so the same ordinal is listed three times -- the sharding, threading and
     // in-order digest placement are what is under test.
    Rng rng(91);
    HashBatch batch = random_batch(rng, 5000, 700);
    b200::DeviceConfig dev;
    dev.devices = {0, 0, 0};
    for (int a : {1, 4}) {
      batch.algorithm = static_cast<Algorithm>(a);
      batch.xof_output_bits = a >= 4 ? 1352 : 0;
      CHECK(matches_oracle(batch, b200::hash_batch(batch, {}, dev)));
    }
    HashBatch fixed_batch;
    fixed_batch.messages.assign(10007, std::vector<std::uint8_t>(64, 0));
    for (std::size_t i = 0; i < fixed_batch.messages.size(); ++i) {
      fixed_batch.messages[i][i % 64] = static_cast<std::uint8_t>(i);
    }
    CHECK(matches_oracle(fixed_batch, b200::hash_batch(fixed_batch, {}, dev)));
    HashBatch tiny;
    tiny.messages = {{1, 2, 3}};
    CHECK(matches_oracle(tiny, b200::hash_batch(tiny, {}, dev)));   // fewer messages than devices
    CHECK(b200::DeviceConfig::all_devices().devices.size() >= 1);
    dev.devices = {0, 99};                                          // a device that does not exist
    bool threw = false;
    try {
      b200::hash_batch(batch, {}, dev);
    } catch (const b200::DeviceError& e) {
      threw = std::string(e.what()).find("device 99") != std::string::npos;
    }
    CHECK(threw);
  }
  {  // BatchHasher: sha3::Hasher for N streams at once on HOST buffers.  Restates
     // proj/tests/test_sponge.cpp:114-150 (any chunking == one shot; XOF output read in pieces ==
     // one shot) and proj/tests/test_sha3.cpp:205-246 (digest / finish / read misuse throws
     // std::logic_error, reset gives fresh states).
    Rng rng(61);
    const std::size_t n = 300;
    for (int a = 0; a < 6; ++a) {
      const Algorithm alg = static_cast<Algorithm>(a);
      std::vector<std::vector<std::uint8_t>> whole(n);
      for (auto& m : whole) m = random_bytes(rng, rng.below(700));
      whole[0].clear();
      b200::BatchHasher h(alg, n);
      CHECK(h.count() == n && h.algorithm() == alg);
      for (int round = 0; round < 3; ++round) {  // message i arrives in three pieces, some empty
        std::vector<std::vector<std::uint8_t>> chunks(n);
        for (std::size_t i = 0; i < n; ++i) {
          const std::size_t len = whole[i].size();
          const std::size_t c1 = len ? (i * 7 + 3) % (len + 1) : 0, c2 = c1 + (len - c1) / 2;
          const std::size_t lo = round == 0 ? 0 : (round == 1 ? c1 : c2);
          const std::size_t hi = round == 0 ? c1 : (round == 1 ? c2 : len);
          chunks[i].assign(whole[i].begin() + lo, whole[i].begin() + hi);
        }
        h.update(chunks);
      }
      bool ok = true;
      if (a < 4) {
        const auto got = h.digest();
        for (std::size_t i = 0; i < n; ++i) ok = ok && got[i] == expect(alg, whole[i]);
        bool threw = false;
        try { h.update(whole); } catch (const std::logic_error&) { threw = true; }   // update after digest
        CHECK(threw);
        threw = false;
        try { h.finish(); } catch (const std::logic_error&) { threw = true; }        // finish() on a hash variant
        CHECK(threw);
      } else {
        bool threw = false;
        try { h.read(8); } catch (const std::logic_error&) { threw = true; }         // read before finish
        CHECK(threw);
        threw = false;
        try { h.digest(); } catch (const std::logic_error&) { threw = true; }        // digest() on an XOF
        CHECK(threw);
        h.finish();
        threw = false;
        try { h.finish(); } catch (const std::logic_error&) { threw = true; }        // finish twice
        CHECK(threw);
        const auto p1 = h.read(5), p2 = h.read(200), p3 = h.read(295);               // 500 bytes in pieces
        for (std::size_t i = 0; i < n; ++i) {
          std::vector<std::uint8_t> all = p1[i];
          all.insert(all.end(), p2[i].begin(), p2[i].end());
          all.insert(all.end(), p3[i].begin(), p3[i].end());
          ok = ok && all == expect(alg, whole[i], 4000);
        }
      }
      CHECK(ok);
      h.reset();                                                                     // Hasher::reset
      std::vector<std::uint8_t> flat(n * 24);
      for (auto& b : flat) b = static_cast<std::uint8_t>(rng.next());
      h.update_fixed(flat.data(), 24);
      b200::BatchHasher moved = std::move(h);
      ok = true;
      if (a < 4) {
        const auto got = moved.digest();
        for (std::size_t i = 0; i < n; ++i) {
          ok = ok && got[i] == expect(alg, std::vector<std::uint8_t>(flat.begin() + 24 * i, flat.begin() + 24 * (i + 1)));
        }
      } else {
        moved.finish();
        const auto got = moved.read(17);
        for (std::size_t i = 0; i < n; ++i) {
          ok = ok && got[i] == expect(alg, std::vector<std::uint8_t>(flat.begin() + 24 * i, flat.begin() + 24 * (i + 1)), 136);
        }
      }
      CHECK(ok);
    }
    {  // one long input fed in 1 MiB pieces to 64 streams (each its own 3 MiB message)
      const std::size_t streams = 64, piece = 1u << 20;
      std::vector<std::vector<std::uint8_t>> whole(streams);
      b200::BatchHasher h(Algorithm::sha3_256, streams);
      for (int k = 0; k < 3; ++k) {
        std::vector<std::uint8_t> flat(streams * piece);
        for (std::size_t i = 0; i < flat.size(); i += 8) {
          const std::uint64_t w = rng.next();
          std::memcpy(flat.data() + i, &w, 8);
        }
        for (std::size_t i = 0; i < streams; ++i) {
          whole[i].insert(whole[i].end(), flat.begin() + i * piece, flat.begin() + (i + 1) * piece);
        }
        h.update_fixed(flat.data(), piece);   // pageable memory, 64 MiB: the bounce ring
      }
      const auto got = h.digest();
      bool ok = true;
      for (std::size_t i = 0; i < streams; i += 9) ok = ok && got[i] == expect(Algorithm::sha3_256, whole[i]);
      CHECK(ok);
    }
  }
  {  // hash_packed on caller-packed buffers with odd offsets
    const std::vector<std::uint8_t> data = {9, 9, 9, 'a', 'b', 'c', 7, 7, 1, 2, 3, 4, 5};
    const std::uint64_t offsets[] = {3, 8, 0}, lengths[] = {3, 5, 0};
    const auto out = b200::hash_packed(Algorithm::sha3_256, data.data(), offsets, lengths, 3);
    CHECK(out.size() == 96);
    CHECK(std::vector<std::uint8_t>(out.begin(), out.begin() + 32) ==
          expect(Algorithm::sha3_256, {'a', 'b', 'c'}));
    CHECK(std::vector<std::uint8_t>(out.begin() + 32, out.begin() + 64) ==
          expect(Algorithm::sha3_256, {1, 2, 3, 4, 5}));
    CHECK(std::vector<std::uint8_t>(out.begin() + 64, out.end()) == expect(Algorithm::sha3_256, {}));
  }
}

}  // namespace

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::string(argv[1]) == "--cpu-only";
  cpu_only_cases();
  if (!cpu_only) gpu_cases();
  std::printf("%d checks, %d failures%s\n", g_checks, g_failures, cpu_only ? " (cpu-only)" : "");
  return g_failures == 0 ? 0 : 1;
}
