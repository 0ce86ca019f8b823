// rsp_reader.hpp -- NIST-style response files (`Len = / Msg = / MD =` triples) read
// straight into the packed batch layout of the C ABI (include/b200sha3.h): one byte
// arena for all messages plus offsets[] / lengths[], one arena for the expected
// digests.  A whole file is then ONE b200sha3_hash_batch call; there is no
// per-vector container to convert from.
//
// File convention (the format contract of proj/tools/sha3cli/vectors.hpp:42-45):
//   * `Len = <bits>`, `Msg = <hex>`, `MD = <hex>` (or `Output = <hex>`), in that order;
//   * Msg carries a placeholder when Len = 0 and is ignored then; a Msg longer than
//     Len / 8 bytes is cut to Len / 8;
//   * blank lines and `#` comments are skipped; `[...]` header lines are skipped except
//     `[Outputlen = N]`, the XOF output length of the file;
//   * only whole-byte message lengths are accepted.
// Malformed input raises rsp::SyntaxError carrying the 1-based line number.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace b200sha3::rsp {

class SyntaxError : public std::runtime_error {
 public:
  SyntaxError(std::size_t line, const std::string& what)
      : std::runtime_error("line " + std::to_string(line) + ": " + what), line_(line) {}
  std::size_t line() const { return line_; }

 private:
  std::size_t line_;
};

// All vectors of one file, packed.  Vector i: message bytes
// messages[offsets[i] .. offsets[i] + lengths[i]), expected digest
// expected[expected_offsets[i] .. + expected_lengths[i]).
struct PackedVectors {
  std::vector<std::uint8_t> messages;
  std::vector<std::uint64_t> offsets, lengths;
  std::vector<std::uint8_t> expected;
  std::vector<std::uint64_t> expected_offsets, expected_lengths;
  std::vector<std::uint64_t> message_bits;  // the Len field as written
  std::vector<std::size_t> source_line;     // line of the Len field
  std::uint64_t output_bits = 0;            // [Outputlen = N]; 0 when the file has none

  std::size_t size() const { return lengths.size(); }
  // XOF output length of vector i: the file's [Outputlen], else the length of its digest.
  std::uint64_t xof_bits(std::size_t i) const {
    return output_bits ? output_bits : 8 * expected_lengths[i];
  }
};

// Parses the text of a response file.  Message starts are padded to `align` bytes
// (8 lets the device use aligned 64-bit loads; 1 packs back to back).
PackedVectors parse(std::string_view text, std::size_t align = 8);

// Reads and parses a file; std::runtime_error("cannot open ...") when unreadable.
PackedVectors load(const std::string& path, std::size_t align = 8);

// Algorithm id (0..5, the C ABI's order) named in a file name such as
// SHA3_256ShortMsg.rsp, shake-128.rsp or sha3512long.rsp; -1 when there is none.
int algorithm_in_filename(std::string_view path);

std::string hex(const std::uint8_t* bytes, std::size_t n);

}  // namespace b200sha3::rsp
