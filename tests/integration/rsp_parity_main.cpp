// tests/integration/rsp_parity_main.cpp -- parser parity for SURVEY.md 8(f) row f-2:
// our packed response-file reader (paper_1902_05320_b200/host/rsp_reader.cpp) against the
// reference's parse_vector_file (proj/tools/sha3cli/vectors.cpp, compiled unmodified from
// /root/reference by oracle/Makefile).  CPU only.  One line per file:
//   <file> same <n>          both parsed it into the same n vectors
//   <file> reject <line>     both rejected it, naming the same line
//   <file> DIFFER <detail>   anything else (exit code 1)
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <regex>
#include <string>

#include "rsp_reader.hpp"
#include "vectors.hpp"

namespace {

long line_in(const std::string& what) {  // "vector file line N: ..."
  std::smatch m;
  return std::regex_search(what, m, std::regex("line ([0-9]+)")) ? std::stol(m[1]) : -1;
}

}  // namespace

int main(int argc, char** argv) {
  int status = 0;
  for (int i = 1; i < argc; ++i) {
    std::ifstream in(argv[i], std::ios::binary);
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    long ref_line = 0, our_line = 0;
    sha3::bench::VectorFile ref;
    b200sha3::rsp::PackedVectors ours;
    try {
      std::ifstream again(argv[i]);
      ref = sha3::bench::parse_vector_file(again);
    } catch (const std::exception& e) {
      ref_line = line_in(e.what());
    }
    try {
      ours = b200sha3::rsp::parse(text);
    } catch (const b200sha3::rsp::SyntaxError& e) {
      our_line = static_cast<long>(e.line());
    }
    if (ref_line || our_line) {
      if (ref_line == our_line) {
        std::printf("%s reject %ld\n", argv[i], our_line);
      } else {
        std::printf("%s DIFFER reference line %ld, ours line %ld\n", argv[i], ref_line, our_line);
        status = 1;
      }
      continue;
    }
    std::string detail;
    if (ref.entries.size() != ours.size()) detail = "vector counts";
    if (ref.output_bits != ours.output_bits) detail = "Outputlen";
    for (std::size_t k = 0; detail.empty() && k < ours.size(); ++k) {
      const auto& e = ref.entries[k];
      const bool same = e.line == ours.source_line[k] && e.msg_bits == ours.message_bits[k] &&
                        e.message.size() == ours.lengths[k] && e.expected.size() == ours.expected_lengths[k] &&
                        ours.offsets[k] % 8 == 0 &&
                        std::memcmp(e.message.data(), ours.messages.data() + ours.offsets[k], e.message.size()) == 0 &&
                        std::memcmp(e.expected.data(), ours.expected.data() + ours.expected_offsets[k],
                                    e.expected.size()) == 0;
      if (!same) detail = "vector " + std::to_string(k);
    }
    if (detail.empty()) {
      std::printf("%s same %zu\n", argv[i], ours.size());
    } else {
      std::printf("%s DIFFER %s\n", argv[i], detail.c_str());
      status = 1;
    }
  }
  return status;
}
