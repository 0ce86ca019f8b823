// b200sha3cli.cpp -- command-line callers of the hot path on the GPU backend
// (f-4 for `hash`).  Same sub-commands, option
// names, exit codes and CSV columns as the reference's sha3cli
// (proj/tools/sha3cli/main.cpp:21-24, :176-207; report.cpp:15-16), so rows and scripts
// carry over; the work itself goes through the packed C ABI.
//
//   b200sha3cli vectors --file F.rsp [--algo A]
//       A response file is read straight into the packed batch layout (rsp_reader.hpp)
//       and verified with ONE b200sha3_hash_batch call per output length.
//   b200sha3cli bench [--algo A] [--message-size N] [--sizes a,b,c] [--bits B] [--repeats R]
//                     [--seed S] [--workers W] [--layout vectors|packed] [--csv FILE]
//       Throughput sweep over total-byte targets.  Methodology contract of the reference's
//       runner (runner.hpp:30-36): one untimed pass, then at least R (>= 3) timed passes and
//       at least 1 ms of timed work, median reported; generation is outside the timed region.
//       --layout vectors times sha3::b200::hash_batch on vector<vector<uint8_t>> (the
//       reference's call shape; time = BatchResult::elapsed); --layout packed times
//       b200sha3_hash_fixed on pinned packed buffers (the C ABI's own shape).
//   b200sha3cli hash [--algo A] [--bits B] [FILE|-]
//       Digest of one file or stdin, streamed through the device-resident incremental
//       hasher (b200sha3_states_*), lowercase hex.
//
// Exit codes: 0 ok, 1 verification failed, 2 usage, 3 I/O or device error.
#include <algorithm>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "b200sha3/batch.hpp"
#include "rsp_reader.hpp"

namespace {

namespace rsp = b200sha3::rsp;

enum ExitCode { kOk = 0, kVerifyFailed = 1, kUsage = 2, kIo = 3 };

// Canonical names in C-ABI id order (the variant table, proj/core/src/sha3.cpp:13-20).
constexpr const char* kAlgorithmNames[6] = {"sha3-224", "sha3-256", "sha3-384", "sha3-512", "shake128", "shake256"};

// Name -> id; case-insensitive, '-' and '_' optional ("SHA3_256", "shake-128"); -1 unknown.
int algorithm_id(const std::string& name) {
  const auto squash = [](const std::string& s) {
    std::string out;
    for (const char c : s) {
      if (c != '-' && c != '_') out.push_back(static_cast<char>(std::tolower(static_cast<unsigned char>(c))));
    }
    return out;
  };
  const std::string want = squash(name);
  for (int id = 0; id < 6; ++id) {
    if (want == squash(kAlgorithmNames[id])) return id;
  }
  return -1;
}

bool is_xof(int id) { return id >= B200SHA3_SHAKE128; }

struct UsageError {
  std::string text;
};

// ---------------------------------------------------------------------------------------
// vectors

int run_vectors(const std::string& path, const std::string& algo_name) {
  const int algorithm = algo_name.empty() ? rsp::algorithm_in_filename(path) : algorithm_id(algo_name);
  if (algorithm < 0) {
    if (algo_name.empty()) throw UsageError{"no algorithm in the file name '" + path + "'; pass --algo"};
    throw UsageError{"unknown algorithm '" + algo_name + "'"};
  }
  rsp::PackedVectors file;
  try {
    file = rsp::load(path);
  } catch (const rsp::SyntaxError& e) {
    std::cerr << "b200sha3cli: " << path << ": " << e.what() << "\n";
    return kIo;
  }

  // Batches by output length: one for the hash variants and for XOF files with an
  // [Outputlen] header; otherwise one per distinct digest length in the file.  Every batch
  // reads the same message arena through its own offsets / lengths.
  std::map<std::uint64_t, std::vector<std::size_t>> by_bits;
  for (std::size_t i = 0; i < file.size(); ++i) by_bits[is_xof(algorithm) ? file.xof_bits(i) : 0].push_back(i);

  std::size_t passed = 0;
  for (const auto& [bits, members] : by_bits) {
    std::vector<std::uint64_t> offsets(members.size()), lengths(members.size());
    for (std::size_t k = 0; k < members.size(); ++k) {
      offsets[k] = file.offsets[members[k]];
      lengths[k] = file.lengths[members[k]];
    }
    const std::uint64_t each = b200sha3_digest_bytes(algorithm, bits);
    std::vector<std::uint8_t> digests(members.size() * each + 1);
    const int rc = b200sha3_hash_batch(algorithm, file.messages.data(), offsets.data(), lengths.data(),
                                       members.size(), bits, digests.data(), nullptr);
    if (rc != B200SHA3_OK) {
      std::cerr << "b200sha3cli: " << b200sha3_strerror(rc) << ": " << b200sha3_last_cuda_error() << "\n";
      return kIo;
    }
    for (std::size_t k = 0; k < members.size(); ++k) {
      const std::size_t i = members[k];
      const std::uint8_t* want = file.expected.data() + file.expected_offsets[i];
      const std::uint8_t* got = digests.data() + k * each;
      if (file.expected_lengths[i] == each && std::memcmp(want, got, each) == 0) {
        ++passed;
        continue;
      }
      std::cout << "FAIL line " << file.source_line[i] << " (Len = " << file.message_bits[i] << ")\n"
                << "  expected " << rsp::hex(want, file.expected_lengths[i]) << "\n"
                << "  actual   " << rsp::hex(got, each) << "\n";
    }
  }
  std::cout << passed << "/" << file.size() << " vectors passed (" << kAlgorithmNames[algorithm] << ", cuda)\n";
  return passed == file.size() ? kOk : kVerifyFailed;
}

// ---------------------------------------------------------------------------------------
// bench

// The reference's synthetic message stream (byte-stream contract of
// proj/tools/sha3cli/workload.cpp:16-47): splitmix64 seeded with
// seed ^ total_bytes * golden, ceil(size / 8) draws per message, bytes little-endian, the
// surplus of the last draw dropped.  splitmix64 is a counter generator -- draw n (from 1)
// is mix(seed + n * golden) -- so any message can be produced on its own, by any thread.
class MessageStream {
 public:
  MessageStream(std::uint64_t seed, std::uint64_t total_bytes, std::size_t message_size)
      : base_(seed ^ (total_bytes * kGolden)), size_(message_size), draws_((message_size + 7) / 8) {}

  void write(std::uint64_t message, std::uint8_t* dst) const {
    std::uint64_t counter = base_ + (message * draws_ + 1) * kGolden;
    for (std::size_t at = 0; at < size_; at += 8, counter += kGolden) {
      const std::uint64_t word = mix(counter);  // little-endian host (x86-64 / aarch64)
      std::memcpy(dst + at, &word, std::min<std::size_t>(8, size_ - at));
    }
  }

 private:
  static constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ull;
  static std::uint64_t mix(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  std::uint64_t base_;
  std::size_t size_, draws_;
};

template <class Fn>
void for_each_range(std::uint64_t n, Fn fn) {  // fn(first, last) on hardware threads
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned parts = static_cast<unsigned>(std::min<std::uint64_t>(hw, std::max<std::uint64_t>(1, n >> 14)));
  std::vector<std::thread> pool;
  for (unsigned p = 1; p < parts; ++p) pool.emplace_back(fn, n * p / parts, n * (p + 1) / parts);
  fn(std::uint64_t{0}, n / parts);
  for (auto& t : pool) t.join();
}

struct Pass {
  double seconds = 0;  // what the row reports
  double kernels = 0;  // CUDA-event time of the hashing kernels inside it
};

struct Row {
  std::uint64_t hashed_bytes = 0;
  std::size_t message_size = 0;
  std::uint64_t messages = 0;
  double seconds = 0, kernels = 0;
  unsigned passes = 0;
};

double middle(std::vector<double>& v) {  // median; reorders v
  const std::size_t half = v.size() / 2;
  std::nth_element(v.begin(), v.begin() + half, v.end());
  double m = v[half];
  if (v.size() % 2 == 0) m = 0.5 * (m + *std::max_element(v.begin(), v.begin() + half));
  return m;
}

// One untimed pass (context, pinned staging, memory pools), then timed passes until there
// are `min_passes` of them AND a millisecond of timed work, so no row reports a zero time.
template <class OnePass>
void measure(unsigned min_passes, OnePass one_pass, Row& row) {
  constexpr double kMinTimedSeconds = 1e-3;
  constexpr std::size_t kPassLimit = std::size_t{1} << 20;  // a clock that never advances
  one_pass();
  std::vector<double> seconds, kernels;
  double timed = 0;
  do {
    const Pass p = one_pass();
    seconds.push_back(p.seconds);
    kernels.push_back(p.kernels);
    timed += p.seconds;
  } while ((seconds.size() < min_passes || timed < kMinTimedSeconds) && seconds.size() < kPassLimit);
  row.passes = static_cast<unsigned>(seconds.size());
  row.seconds = middle(seconds);
  if (!(row.seconds > 0)) row.seconds = timed / row.passes;
  row.kernels = middle(kernels);
}

struct BenchOptions {
  int algorithm = B200SHA3_SHA3_256;
  std::uint64_t xof_bits = 0;
  std::size_t message_size = 10;
  // default sweep: the total-byte targets of the paper's Table 3 (workload.hpp:16-18)
  std::vector<std::uint64_t> totals = {1202, 4652, 9302, 18602, 37202, 74402, 148802, 297602, 595202, 1190402};
  std::uint64_t seed = 1;
  unsigned repeats = 3, workers = 0;
  bool packed = false;
  std::string csv;
};

Row bench_vectors(const BenchOptions& o, std::uint64_t total) {
  sha3::HashBatch batch;
  batch.algorithm = static_cast<sha3::Algorithm>(o.algorithm);
  batch.xof_output_bits = o.xof_bits;
  batch.messages.assign(total / o.message_size, std::vector<std::uint8_t>(o.message_size));
  const MessageStream stream(o.seed, total, o.message_size);
  for_each_range(batch.messages.size(), [&](std::uint64_t first, std::uint64_t last) {
    for (std::uint64_t i = first; i < last; ++i) stream.write(i, batch.messages[i].data());
  });
  sha3::EngineConfig engine;
  engine.workers = o.workers;
  sha3::b200::StageTimes stages;
  sha3::b200::DeviceConfig device;
  device.stages = &stages;
  Row row{batch.messages.size() * o.message_size, o.message_size, batch.messages.size()};
  measure(o.repeats, [&] {
    const sha3::BatchResult result = sha3::b200::hash_batch(batch, engine, device);
    return Pass{result.elapsed.count(), stages.kernels};
  }, row);
  return row;
}

Row bench_packed(const BenchOptions& o, std::uint64_t total) {
  const std::uint64_t count = total / o.message_size;
  const std::uint64_t each = b200sha3_digest_bytes(o.algorithm, o.xof_bits);
  void *in = nullptr, *out = nullptr;
  if (b200sha3_pinned_alloc(count * o.message_size + 16, &in) != B200SHA3_OK ||
      b200sha3_pinned_alloc(count * each + 16, &out) != B200SHA3_OK) {
    throw sha3::b200::DeviceError(B200SHA3_ERR_CUDA, std::string("pinned allocation: ") + b200sha3_last_cuda_error());
  }
  const MessageStream stream(o.seed, total, o.message_size);
  for_each_range(count, [&](std::uint64_t first, std::uint64_t last) {
    for (std::uint64_t i = first; i < last; ++i) stream.write(i, static_cast<std::uint8_t*>(in) + i * o.message_size);
  });
  Row row{count * o.message_size, o.message_size, count};
  int failed = B200SHA3_OK;
  measure(o.repeats, [&] {
    double ms = 0;
    b200sha3_config cfg{};
    cfg.struct_size = sizeof cfg;
    cfg.device = -1;
    cfg.fma_preset = -1;
    cfg.device_ms = &ms;
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = b200sha3_hash_fixed(o.algorithm, static_cast<const std::uint8_t*>(in), o.message_size, count,
                                       o.xof_bits, static_cast<std::uint8_t*>(out), &cfg);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (rc != B200SHA3_OK) failed = rc;
    return Pass{failed ? 1.0 : wall, ms * 1e-3};  // a failing call ends the sampling at once
  }, row);
  b200sha3_pinned_free(in);
  b200sha3_pinned_free(out);
  if (failed) {
    throw sha3::b200::DeviceError(failed, std::string(b200sha3_strerror(failed)) + ": " + b200sha3_last_cuda_error());
  }
  return row;
}

int run_bench(BenchOptions o) {
  if (o.repeats < 3) throw UsageError{"--repeats must be at least 3 (a reported row is a median)"};
  if (o.message_size == 0) throw UsageError{"--message-size must be positive"};
  if (is_xof(o.algorithm) && o.xof_bits == 0) o.xof_bits = o.algorithm == B200SHA3_SHAKE128 ? 256 : 512;
  if (!is_xof(o.algorithm)) o.xof_bits = 0;
  for (const std::uint64_t total : o.totals) {
    if (total < o.message_size) throw UsageError{"a --sizes entry is smaller than one message"};
  }
  const char* backend = o.packed ? "cuda-packed" : "cuda";
  std::vector<Row> rows;
  for (const std::uint64_t total : o.totals) rows.push_back(o.packed ? bench_packed(o, total) : bench_vectors(o, total));

  std::printf("%14s %9s %12s %-12s %12s %16s %7s %12s\n", "total_bytes", "msg_size", "msg_count", "backend", "time_s",
              "throughput_Bps", "repeats", "kernels_s");
  for (const Row& r : rows) {
    std::printf("%14" PRIu64 " %9zu %12" PRIu64 " %-12s %12.6f %16.2f %7u %12.6f\n", r.hashed_bytes, r.message_size,
                r.messages, backend, r.seconds, static_cast<double>(r.hashed_bytes) / r.seconds, r.passes, r.kernels);
  }
  if (o.csv.empty()) return kOk;
  std::FILE* f = std::fopen(o.csv.c_str(), "wb");
  if (!f) {
    std::cerr << "b200sha3cli: cannot write " << o.csv << "\n";
    return kIo;
  }
  // column contract: proj/tools/sha3cli/report.cpp:15-16
  std::fputs("total_bytes,message_size,message_count,backend,time_seconds,throughput_bps,repeats\n", f);
  for (const Row& r : rows) {
    std::fprintf(f, "%" PRIu64 ",%zu,%" PRIu64 ",%s,%.9g,%.9g,%u\n", r.hashed_bytes, r.message_size, r.messages,
                 backend, r.seconds, static_cast<double>(r.hashed_bytes) / r.seconds, r.passes);
  }
  const bool bad = std::ferror(f) != 0;
  return (std::fclose(f) != 0 || bad) ? kIo : kOk;
}

// ---------------------------------------------------------------------------------------
// hash

int run_hash(const std::string& algo_name, std::uint64_t bits, const std::string& path) {
  const int algorithm = algorithm_id(algo_name);
  if (algorithm < 0) throw UsageError{"unknown algorithm '" + algo_name + "'"};
  if (bits && !is_xof(algorithm)) throw UsageError{"--bits applies to XOF variants only"};
  if (is_xof(algorithm) && bits == 0) bits = algorithm == B200SHA3_SHAKE128 ? 256 : 512;
  if (bits % 8) throw UsageError{"--bits must be a multiple of 8"};
  std::ifstream file;
  std::istream* in = &std::cin;
  if (!path.empty() && path != "-") {
    file.open(path, std::ios::binary);
    if (!file) {
      std::cerr << "b200sha3cli: cannot open " << path << "\n";
      return kIo;
    }
    in = &file;
  }
  sha3::b200::BatchHasher hasher(static_cast<sha3::Algorithm>(algorithm), 1);
  std::vector<std::uint8_t> chunk(4u << 20);
  for (;;) {
    in->read(reinterpret_cast<char*>(chunk.data()), static_cast<std::streamsize>(chunk.size()));
    const std::uint64_t got = static_cast<std::uint64_t>(in->gcount());
    if (got) hasher.update_fixed(chunk.data(), got);
    if (!*in) break;
  }
  if (in->bad()) {
    std::cerr << "b200sha3cli: read error\n";
    return kIo;
  }
  std::vector<std::vector<std::uint8_t>> out;
  if (is_xof(algorithm)) {
    hasher.finish();
    out = hasher.read(bits / 8);
  } else {
    out = hasher.digest();
  }
  std::cout << rsp::hex(out[0].data(), out[0].size()) << "\n";
  return kOk;
}

// ---------------------------------------------------------------------------------------

constexpr const char* kUsageText =
    "usage: b200sha3cli vectors --file F.rsp [--algo A]\n"
    "       b200sha3cli bench [--algo A] [--message-size N] [--sizes a,b,c] [--bits B] [--repeats R]\n"
    "                         [--seed S] [--workers W] [--layout vectors|packed] [--csv FILE]\n"
    "       b200sha3cli hash [--algo A] [--bits B] [FILE|-]\n"
    "algorithms: sha3-224 sha3-256 sha3-384 sha3-512 shake128 shake256\n";

struct Options {
  std::map<std::string, std::string> named;
  std::vector<std::string> positional;
  std::string get(const std::string& key, const std::string& fallback) const {
    const auto it = named.find(key);
    return it == named.end() ? fallback : it->second;
  }
  std::uint64_t number(const std::string& key, std::uint64_t fallback) const {
    const auto it = named.find(key);
    if (it == named.end()) return fallback;
    std::size_t used = 0;
    std::uint64_t v = 0;
    try {
      v = std::stoull(it->second, &used);
    } catch (const std::exception&) {
      used = 0;
    }
    if (used == 0 || used != it->second.size()) throw UsageError{"--" + key + " needs a number, got '" + it->second + "'"};
    return v;
  }
};

Options parse_options(int argc, char** argv, const std::vector<std::string>& allowed) {
  Options o;
  for (int i = 2; i < argc; ++i) {
    const std::string arg = argv[i];
    if (arg.size() > 2 && arg.compare(0, 2, "--") == 0) {
      const std::string key = arg.substr(2);
      if (std::find(allowed.begin(), allowed.end(), key) == allowed.end()) throw UsageError{"unknown option " + arg};
      if (i + 1 >= argc) throw UsageError{arg + " needs a value"};
      o.named[key] = argv[++i];
    } else {
      o.positional.push_back(arg);
    }
  }
  return o;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const std::string command = argc > 1 ? argv[1] : "";
    if (command == "vectors") {
      const Options o = parse_options(argc, argv, {"file", "algo"});
      if (!o.named.count("file") || !o.positional.empty()) throw UsageError{"vectors needs --file"};
      return run_vectors(o.get("file", ""), o.get("algo", ""));
    }
    if (command == "bench") {
      const Options o = parse_options(argc, argv, {"algo", "message-size", "sizes", "bits", "repeats", "seed",
                                                   "workers", "layout", "csv", "backend", "chunk"});
      if (!o.positional.empty()) throw UsageError{"unexpected argument " + o.positional[0]};
      BenchOptions b;
      b.algorithm = algorithm_id(o.get("algo", "sha3-256"));
      if (b.algorithm < 0) throw UsageError{"unknown algorithm '" + o.get("algo", "") + "'"};
      b.xof_bits = o.number("bits", 0);
      b.message_size = o.number("message-size", b.message_size);
      b.seed = o.number("seed", b.seed);
      b.repeats = static_cast<unsigned>(o.number("repeats", b.repeats));
      b.workers = static_cast<unsigned>(o.number("workers", 0));
      b.csv = o.get("csv", "");
      const std::string layout = o.get("layout", "vectors");
      if (layout != "vectors" && layout != "packed") throw UsageError{"--layout must be vectors or packed"};
      b.packed = layout == "packed";
      if (o.named.count("sizes")) {
        b.totals.clear();
        const std::string list = o.get("sizes", "");
        for (std::size_t at = 0; at <= list.size();) {
          const std::size_t comma = std::min(list.find(',', at), list.size());
          Options one;
          one.named["sizes"] = list.substr(at, comma - at);
          b.totals.push_back(one.number("sizes", 0));
          at = comma + 1;
        }
      }
      return run_bench(b);
    }
    if (command == "hash") {
      const Options o = parse_options(argc, argv, {"algo", "bits"});
      if (o.positional.size() > 1) throw UsageError{"hash takes at most one FILE"};
      return run_hash(o.get("algo", "sha3-256"), o.number("bits", 0), o.positional.empty() ? "-" : o.positional[0]);
    }
    throw UsageError{command.empty() ? "a sub-command is required" : "unknown sub-command '" + command + "'"};
  } catch (const UsageError& e) {
    std::cerr << "b200sha3cli: " << e.text << "\n" << kUsageText;
    return kUsage;
  } catch (const std::invalid_argument& e) {
    std::cerr << "b200sha3cli: " << e.what() << "\n";
    return kUsage;
  } catch (const std::exception& e) {
    std::cerr << "b200sha3cli: " << e.what() << "\n";
    return kIo;
  }
}
