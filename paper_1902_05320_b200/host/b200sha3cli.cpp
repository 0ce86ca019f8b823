// b200sha3cli.cpp -- the two callers either side of the hot path, on the GPU
// backend:
//
//   b200sha3cli bench   --algo A --message-size N --sizes a,b,c [--bits B] [--repeats R]
//                       [--seed S] [--csv FILE] [--workers W]
//       the `sha3cli bench` sweep (proj/tools/sha3cli/main.cpp:85-124) with backend
//       "cuda": same workload stream (workload.cpp:16-47), same methodology
//       (runner.cpp:30-76: one warm-up, >= R (>= 3) timed runs until >= 1 ms
//       aggregate, median of BatchResult::elapsed), same console table and the same
//       CSV columns (report.cpp:15-16) so rows can be concatenated with the
//       reference's own output.
//   b200sha3cli vectors --file F.rsp [--algo A]
//       the `sha3cli vectors` verifier (main.cpp:126-160, vectors.cpp:42-179): the
//       whole response file goes through the GPU as ONE batch.
//
// Exit codes follow main.cpp:21-24: 0 ok, 1 verification failed, 2 usage, 3 I/O.
#include <algorithm>
#include <cctype>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "b200sha3/batch.hpp"

namespace {

constexpr int kExitOk = 0, kExitVerifyFailed = 1, kExitUsage = 2, kExitIo = 3;

const char* const kNames[6] = {"sha3-224", "sha3-256", "sha3-384", "sha3-512", "shake128", "shake256"};

std::string lowered(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

// parse_algorithm (proj/core/src/sha3.cpp:39-49)
std::optional<sha3::Algorithm> parse_algorithm(const std::string& name) {
  const std::string n = lowered(name);
  for (int i = 0; i < 6; ++i) {
    if (n == kNames[i]) return static_cast<sha3::Algorithm>(i);
  }
  if (n == "shake-128") return sha3::Algorithm::shake128;
  if (n == "shake-256") return sha3::Algorithm::shake256;
  return std::nullopt;
}

bool is_xof(sha3::Algorithm a) { return a == sha3::Algorithm::shake128 || a == sha3::Algorithm::shake256; }

// ---- workload (proj/tools/sha3cli/workload.cpp:9-47) -------------------------------
struct SplitMix64 {
  std::uint64_t state;
  std::uint64_t next() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
};

sha3::HashBatch generate_workload(sha3::Algorithm algorithm, std::uint64_t xof_bits,
                                  std::size_t message_size, std::uint64_t seed,
                                  std::uint64_t total_bytes) {
  sha3::HashBatch batch;
  batch.algorithm = algorithm;
  if (is_xof(algorithm)) {
    batch.xof_output_bits = xof_bits ? xof_bits : (algorithm == sha3::Algorithm::shake128 ? 256 : 512);
  }
  SplitMix64 rng{seed ^ (total_bytes * 0x9e3779b97f4a7c15ull)};
  batch.messages.resize(total_bytes / message_size);
  for (auto& msg : batch.messages) {
    msg.resize(message_size);
    for (std::size_t i = 0; i < message_size;) {
      const std::uint64_t word = rng.next();
      for (int k = 0; k < 8 && i < message_size; ++k, ++i) msg[i] = static_cast<std::uint8_t>(word >> (8 * k));
    }
  }
  return batch;
}

// ---- bench (runner.cpp:30-76, report.cpp:52-143) -----------------------------------
struct Record {
  std::uint64_t total_bytes;
  std::size_t message_size, message_count;
  double time_seconds, throughput_bps;
  unsigned repeats;
  double wall_seconds;  // whole hash_batch call (pack + copies + kernels + unpack); console only
};

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  const std::size_t n = v.size();
  return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

int cmd_bench(sha3::Algorithm algorithm, std::uint64_t bits, std::size_t message_size,
              const std::vector<std::uint64_t>& sizes, std::uint64_t seed, unsigned repeats,
              unsigned workers, const std::string& csv_path) {
  if (repeats < 3) {
    std::cerr << "b200sha3cli: reported rows need at least 3 repeats\n";
    return kExitUsage;
  }
  if (message_size == 0) {
    std::cerr << "b200sha3cli: message size must be positive\n";
    return kExitUsage;
  }
  sha3::EngineConfig config;
  config.workers = workers;
  std::vector<Record> records;
  for (const std::uint64_t total : sizes) {
    if (total < message_size) {
      std::cerr << "b200sha3cli: total size smaller than one message\n";
      return kExitUsage;
    }
    const sha3::HashBatch batch = generate_workload(algorithm, bits, message_size, seed, total);
    const std::uint64_t hashed = static_cast<std::uint64_t>(batch.messages.size()) * message_size;
    sha3::b200::hash_batch(batch, config);  // warm-up, not recorded
    std::vector<double> samples, walls;
    double aggregate = 0;
    while (samples.size() < repeats || aggregate < 1e-3) {
      const auto t0 = std::chrono::steady_clock::now();
      const sha3::BatchResult result = sha3::b200::hash_batch(batch, config);
      walls.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      samples.push_back(result.elapsed.count());  // `result` dies after the clock was read
      aggregate += samples.back();
      if (samples.size() >= 1u << 20) break;
    }
    double time = median(samples);
    if (time <= 0) time = aggregate / static_cast<double>(samples.size());
    records.push_back({hashed, message_size, batch.messages.size(), time,
                       static_cast<double>(hashed) / time, static_cast<unsigned>(samples.size()),
                       median(walls)});
  }
  // the reference's table (report.cpp:113-143) plus one column: the wall time of the call
  std::printf("%12s %9s %10s %-10s %14s %16s %8s %8s %12s\n", "total_bytes", "msg_size", "msg_count",
              "backend", "time_s", "throughput_Bps", "repeats", "speedup", "call_wall_s");
  for (const Record& r : records) {
    std::printf("%12" PRIu64 " %9zu %10zu %-10s %14.6f %16.2f %8u %8s %12.6f\n", r.total_bytes,
                r.message_size, r.message_count, "cuda", r.time_seconds, r.throughput_bps, r.repeats, "",
                r.wall_seconds);
  }
  if (!csv_path.empty()) {
    std::ofstream out(csv_path, std::ios::binary);
    if (!out) {
      std::cerr << "b200sha3cli: cannot write " << csv_path << "\n";
      return kExitIo;
    }
    out << "total_bytes,message_size,message_count,backend,time_seconds,throughput_bps,repeats\n";
    char buf[256];
    for (const Record& r : records) {
      std::snprintf(buf, sizeof buf, "%" PRIu64 ",%zu,%zu,cuda,%.9g,%.9g,%u\n", r.total_bytes,
                    r.message_size, r.message_count, r.time_seconds, r.throughput_bps, r.repeats);
      out << buf;
    }
    if (!out) return kExitIo;
  }
  return kExitOk;
}

// ---- vectors (vectors.cpp:42-179) ---------------------------------------------------
struct Entry {
  std::size_t line = 0;
  std::uint64_t msg_bits = 0;
  std::vector<std::uint8_t> message, expected;
};

std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r\n");
  if (b == std::string::npos) return "";
  return s.substr(b, s.find_last_not_of(" \t\r\n") - b + 1);
}

bool key_value(const std::string& line, std::string& key, std::string& value) {
  const auto eq = line.find('=');
  if (eq == std::string::npos) return false;
  key = trim(line.substr(0, eq));
  value = trim(line.substr(eq + 1));
  return !key.empty();
}

std::optional<std::vector<std::uint8_t>> from_hex(const std::string& s) {
  if (s.size() % 2) return std::nullopt;
  std::vector<std::uint8_t> out(s.size() / 2);
  auto nib = [](char c) -> int {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    return -1;
  };
  for (std::size_t i = 0; i < out.size(); ++i) {
    const int hi = nib(s[2 * i]), lo = nib(s[2 * i + 1]);
    if (hi < 0 || lo < 0) return std::nullopt;
    out[i] = static_cast<std::uint8_t>(hi * 16 + lo);
  }
  return out;
}

std::string to_hex(const std::vector<std::uint8_t>& v) {
  static const char* d = "0123456789abcdef";
  std::string s;
  for (std::uint8_t b : v) {
    s.push_back(d[b >> 4]);
    s.push_back(d[b & 15]);
  }
  return s;
}

struct ParseError {
  std::string what;
};

void parse_file(std::istream& in, std::uint64_t& output_bits, std::vector<Entry>& entries) {
  std::string line;
  std::size_t line_no = 0;
  std::optional<Entry> pending;
  bool have_msg = false;
  auto fail = [&](const std::string& what) {
    throw ParseError{"vector file line " + std::to_string(line_no) + ": " + what};
  };
  while (std::getline(in, line)) {
    ++line_no;
    const std::string text = trim(line);
    if (text.empty() || text[0] == '#') continue;
    std::string key, value;
    if (text.front() == '[' && text.back() == ']') {
      if (key_value(text.substr(1, text.size() - 2), key, value) && key == "Outputlen") {
        try {
          output_bits = std::stoull(value);
        } catch (const std::exception&) {
          fail("bad Outputlen value '" + value + "'");
        }
      }
      continue;
    }
    if (!key_value(text, key, value)) fail("expected 'Key = value', got '" + text + "'");
    if (key == "Len") {
      if (pending) fail("new Len before the previous vector was completed");
      Entry e;
      e.line = line_no;
      try {
        e.msg_bits = std::stoull(value);
      } catch (const std::exception&) {
        fail("bad Len value '" + value + "'");
      }
      if (e.msg_bits % 8) fail("only byte-aligned lengths are supported (Len = " + value + ")");
      pending = std::move(e);
      have_msg = false;
    } else if (key == "Msg") {
      if (!pending) fail("Msg without a preceding Len");
      auto bytes = from_hex(value);
      if (!bytes) fail("Msg is not valid hex");
      if (pending->msg_bits > 0) {
        if (bytes->size() < pending->msg_bits / 8) fail("Msg shorter than Len");
        bytes->resize(pending->msg_bits / 8);
        pending->message = std::move(*bytes);
      }
      have_msg = true;
    } else if (key == "MD" || key == "Output") {
      if (!pending || !have_msg) fail(key + " without a preceding Len/Msg pair");
      const auto bytes = from_hex(value);
      if (!bytes || bytes->empty()) fail(key + " is not valid hex");
      pending->expected = *bytes;
      entries.push_back(std::move(*pending));
      pending.reset();
    } else {
      fail("unknown key '" + key + "'");
    }
  }
  if (pending) fail("file ended in the middle of a vector");
}

std::optional<sha3::Algorithm> algorithm_from_filename(const std::string& path) {
  std::string name = path.substr(path.find_last_of('/') == std::string::npos ? 0 : path.find_last_of('/') + 1);
  name = lowered(name);
  for (const char* sep : {"_", "-", ""}) {
    const std::pair<std::string, int> tags[] = {
        {std::string("sha3") + sep + "224", 0}, {std::string("sha3") + sep + "256", 1},
        {std::string("sha3") + sep + "384", 2}, {std::string("sha3") + sep + "512", 3},
        {std::string("shake") + sep + "128", 4}, {std::string("shake") + sep + "256", 5}};
    for (const auto& [tag, id] : tags) {
      if (name.find(tag) != std::string::npos) return static_cast<sha3::Algorithm>(id);
    }
  }
  return std::nullopt;
}

int cmd_vectors(const std::string& path, const std::string& algo_name) {
  std::optional<sha3::Algorithm> algorithm;
  if (!algo_name.empty()) {
    algorithm = parse_algorithm(algo_name);
    if (!algorithm) {
      std::cerr << "b200sha3cli: unknown algorithm '" << algo_name << "'\n";
      return kExitUsage;
    }
  } else {
    algorithm = algorithm_from_filename(path);
    if (!algorithm) {
      std::cerr << "b200sha3cli: cannot infer the algorithm from '" << path << "'; pass --algo\n";
      return kExitUsage;
    }
  }
  std::uint64_t output_bits = 0;
  std::vector<Entry> entries;
  {
    std::ifstream in(path);
    if (!in) {
      std::cerr << "b200sha3cli: cannot open vector file: " << path << "\n";
      return kExitIo;
    }
    try {
      parse_file(in, output_bits, entries);
    } catch (const ParseError& e) {
      std::cerr << "b200sha3cli: " << e.what << "\n";
      return kExitIo;
    }
  }
  // One GPU batch per distinct output length (one batch in practice: hash variants
  // have a fixed length and XOF files carry one [Outputlen]).
  std::map<std::uint64_t, std::vector<std::size_t>> groups;
  for (std::size_t i = 0; i < entries.size(); ++i) {
    const std::uint64_t bits = is_xof(*algorithm) ? (output_bits ? output_bits : entries[i].expected.size() * 8) : 0;
    groups[bits].push_back(i);
  }
  std::size_t passed = 0;
  try {
    for (const auto& [bits, idx] : groups) {
      sha3::HashBatch batch;
      batch.algorithm = *algorithm;
      batch.xof_output_bits = bits;
      for (std::size_t i : idx) batch.messages.push_back(entries[i].message);
      const sha3::BatchResult res = sha3::b200::hash_batch(batch);
      for (std::size_t k = 0; k < idx.size(); ++k) {
        const Entry& e = entries[idx[k]];
        if (res.digests[k] == e.expected) {
          ++passed;
        } else {
          std::cout << "FAIL line " << e.line << " (Len = " << e.msg_bits << ")\n"
                    << "  expected " << to_hex(e.expected) << "\n"
                    << "  actual   " << to_hex(res.digests[k]) << "\n";
        }
      }
    }
  } catch (const std::exception& e) {
    std::cerr << "b200sha3cli: " << e.what() << "\n";
    return kExitIo;
  }
  std::cout << passed << "/" << entries.size() << " vectors passed ("
            << kNames[static_cast<int>(*algorithm)] << ", cuda)\n";
  return passed == entries.size() ? kExitOk : kExitVerifyFailed;
}

int usage() {
  std::cerr << "usage: b200sha3cli bench --algo A --message-size N --sizes a,b,c [--bits B] [--repeats R]"
               " [--seed S] [--workers W] [--csv FILE]\n"
               "       b200sha3cli vectors --file F.rsp [--algo A]\n";
  return kExitUsage;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  const std::string cmd = argv[1];
  std::map<std::string, std::string> opt;
  for (int i = 2; i < argc; ++i) {
    const std::string key = argv[i];
    if (key.rfind("--", 0) != 0 || i + 1 >= argc) return usage();
    opt[key.substr(2)] = argv[++i];
  }
  auto get = [&](const std::string& k, const std::string& dflt) {
    const auto it = opt.find(k);
    return it == opt.end() ? dflt : it->second;
  };
  try {
    if (cmd == "vectors") {
      if (!opt.count("file")) return usage();
      return cmd_vectors(opt["file"], get("algo", ""));
    }
    if (cmd == "bench") {
      const auto algorithm = parse_algorithm(get("algo", "sha3-256"));
      if (!algorithm) {
        std::cerr << "b200sha3cli: unknown algorithm '" << get("algo", "") << "'\n";
        return kExitUsage;
      }
      // defaults of WorkloadSpec (workload.hpp:15-20): the paper's Table 3 sweep
      std::vector<std::uint64_t> sizes;
      std::stringstream ss(get("sizes", "1202,4652,9302,18602,37202,74402,148802,297602,595202,1190402"));
      for (std::string tok; std::getline(ss, tok, ',');) sizes.push_back(std::stoull(tok));
      return cmd_bench(*algorithm, std::stoull(get("bits", "0")), std::stoull(get("message-size", "10")),
                       sizes, std::stoull(get("seed", "1")),
                       static_cast<unsigned>(std::stoul(get("repeats", "3"))),
                       static_cast<unsigned>(std::stoul(get("workers", "0"))), get("csv", ""));
    }
  } catch (const std::invalid_argument& e) {
    std::cerr << "b200sha3cli: " << e.what() << "\n";
    return kExitUsage;
  } catch (const std::exception& e) {
    std::cerr << "b200sha3cli: " << e.what() << "\n";
    return kExitIo;
  }
  return usage();
}
