// rsp_reader.cpp -- see rsp_reader.hpp.  A line classifier plus a three-state record
// builder that appends decoded bytes directly to the packed arenas.
#include "rsp_reader.hpp"

#include <array>
#include <cctype>
#include <charconv>
#include <fstream>
#include <iterator>

namespace b200sha3::rsp {

namespace {

constexpr std::string_view kSpace = " \t\r\n\v\f";

std::string_view strip(std::string_view s) {
  const std::size_t first = s.find_first_not_of(kSpace);
  if (first == std::string_view::npos) return {};
  return s.substr(first, s.find_last_not_of(kSpace) - first + 1);
}

constexpr std::array<std::int8_t, 256> make_nibbles() {
  std::array<std::int8_t, 256> t{};
  for (auto& v : t) v = -1;
  for (int d = 0; d < 10; ++d) t['0' + d] = static_cast<std::int8_t>(d);
  for (int d = 0; d < 6; ++d) {
    t['a' + d] = static_cast<std::int8_t>(10 + d);
    t['A' + d] = static_cast<std::int8_t>(10 + d);
  }
  return t;
}
constexpr std::array<std::int8_t, 256> kNibble = make_nibbles();

// Appends the bytes spelled by `digits` to `arena`; false (arena restored) unless `digits`
// is an even number of hex characters.  At most `limit` bytes are kept.
bool append_hex(std::string_view digits, std::vector<std::uint8_t>& arena,
                std::size_t limit = static_cast<std::size_t>(-1)) {
  if (digits.size() % 2) return false;
  const std::size_t mark = arena.size();
  for (std::size_t i = 0; i < digits.size(); i += 2) {
    const int hi = kNibble[static_cast<unsigned char>(digits[i])];
    const int lo = kNibble[static_cast<unsigned char>(digits[i + 1])];
    if ((hi | lo) < 0) {
      arena.resize(mark);
      return false;
    }
    if (i / 2 < limit) arena.push_back(static_cast<std::uint8_t>(hi << 4 | lo));
  }
  return true;
}

bool to_u64(std::string_view s, std::uint64_t& out) {
  if (s.empty()) return false;
  const auto [end, ec] = std::from_chars(s.data(), s.data() + s.size(), out, 10);
  return ec == std::errc() && end == s.data() + s.size();
}

struct Field {
  std::string_view key, value;
};

// "key = value" -> Field; no '=' or nothing before it -> false.
bool split_field(std::string_view text, Field& f) {
  const std::size_t eq = text.find('=');
  if (eq == std::string_view::npos) return false;
  f.key = strip(text.substr(0, eq));
  f.value = strip(text.substr(eq + 1));
  return !f.key.empty();
}

// Assembles records from the fields of a file; every record goes Len -> Msg -> digest.
class RecordBuilder {
 public:
  RecordBuilder(PackedVectors& out, std::size_t align) : out_(out), align_(align ? align : 1) {}

  void field(std::size_t line, const Field& f) {
    if (f.key == "Len") {
      begin(line, f.value);
    } else if (f.key == "Msg") {
      message(line, f.value);
    } else if (f.key == "MD" || f.key == "Output") {
      digest(line, f);
    } else {
      throw SyntaxError(line, "'" + std::string(f.key) + "' is not a response-file key (Len, Msg, MD, Output)");
    }
  }

  void end_of_file(std::size_t last_line) const {
    if (stage_ != Stage::idle) throw SyntaxError(last_line, "the last vector is incomplete (no MD / Output line)");
  }

 private:
  enum class Stage { idle, have_len, have_msg };

  void begin(std::size_t line, std::string_view value) {
    if (stage_ != Stage::idle) {
      throw SyntaxError(line, "Len starts a new vector but the one from line " + std::to_string(len_line_) +
                                  " has no MD / Output yet");
    }
    if (!to_u64(value, bits_)) throw SyntaxError(line, "Len must be a decimal bit count, not '" + std::string(value) + "'");
    if (bits_ % 8) {
      throw SyntaxError(line, "Len = " + std::string(value) + " is not byte-aligned; bit-granular messages are not supported");
    }
    len_line_ = line;
    stage_ = Stage::have_len;
  }

  void message(std::size_t line, std::string_view value) {
    if (stage_ == Stage::idle) throw SyntaxError(line, "Msg needs a Len line first");
    const std::size_t want = static_cast<std::size_t>(bits_ / 8);
    if (stage_ == Stage::have_len) {  // first Msg of the record: open its slot in the arena
      out_.messages.resize((out_.messages.size() + align_ - 1) / align_ * align_, 0);
      start_ = out_.messages.size();
    } else {                          // a second Msg line replaces the first
      out_.messages.resize(start_);
    }
    // Len = 0 files carry a placeholder byte ("00"): checked for syntax, not kept.
    if (!append_hex(value, out_.messages, want)) throw SyntaxError(line, "Msg is not an even run of hex digits");
    if (out_.messages.size() - start_ < want) {
      throw SyntaxError(line, "Msg has " + std::to_string(out_.messages.size() - start_) + " bytes, Len asks for " +
                                  std::to_string(want));
    }
    stage_ = Stage::have_msg;
  }

  void digest(std::size_t line, const Field& f) {
    if (stage_ != Stage::have_msg) throw SyntaxError(line, std::string(f.key) + " needs a Len and a Msg line first");
    const std::size_t mark = out_.expected.size();
    if (!append_hex(f.value, out_.expected) || out_.expected.size() == mark) {
      throw SyntaxError(line, std::string(f.key) + " is not a non-empty even run of hex digits");
    }
    out_.offsets.push_back(start_);
    out_.lengths.push_back(bits_ / 8);
    out_.expected_offsets.push_back(mark);
    out_.expected_lengths.push_back(out_.expected.size() - mark);
    out_.message_bits.push_back(bits_);
    out_.source_line.push_back(len_line_);
    stage_ = Stage::idle;
  }

  PackedVectors& out_;
  const std::size_t align_;
  Stage stage_ = Stage::idle;
  std::uint64_t bits_ = 0;
  std::size_t len_line_ = 0, start_ = 0;
};

}  // namespace

PackedVectors parse(std::string_view text, std::size_t align) {
  PackedVectors out;
  out.messages.reserve(text.size() / 2);
  RecordBuilder builder(out, align);
  std::size_t line_no = 0;
  for (std::size_t pos = 0; pos < text.size();) {
    const std::size_t nl = text.find('\n', pos);
    const std::string_view line = strip(text.substr(pos, nl == std::string_view::npos ? nl : nl - pos));
    pos = nl == std::string_view::npos ? text.size() : nl + 1;
    ++line_no;
    if (line.empty() || line.front() == '#') continue;
    Field f;
    if (line.front() == '[' && line.back() == ']') {  // section header
      if (split_field(line.substr(1, line.size() - 2), f) && f.key == "Outputlen" && !to_u64(f.value, out.output_bits)) {
        throw SyntaxError(line_no, "Outputlen must be a decimal bit count, not '" + std::string(f.value) + "'");
      }
      continue;
    }
    if (!split_field(line, f)) throw SyntaxError(line_no, "not a 'Key = value' line: '" + std::string(line) + "'");
    builder.field(line_no, f);
  }
  builder.end_of_file(line_no);
  out.messages.resize(out.messages.size() + 8, 0);  // slack so the arena is never empty
  return out;
}

PackedVectors load(const std::string& path, std::size_t align) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  if (in.bad()) throw std::runtime_error("read error on " + path);
  return parse(text, align);
}

int algorithm_in_filename(std::string_view path) {
  const std::size_t slash = path.find_last_of('/');
  if (slash != std::string_view::npos) path.remove_prefix(slash + 1);
  // family and strength may be joined by '_', '-' or nothing: compare on the name with
  // those two separators dropped
  std::string name;
  for (const char c : path) {
    if (c != '_' && c != '-') name.push_back(static_cast<char>(std::tolower(static_cast<unsigned char>(c))));
  }
  static constexpr std::string_view kTags[6] = {"sha3224", "sha3256", "sha3384", "sha3512", "shake128", "shake256"};
  for (int id = 0; id < 6; ++id) {
    if (name.find(kTags[id]) != std::string::npos) return id;
  }
  return -1;
}

std::string hex(const std::uint8_t* bytes, std::size_t n) {
  std::string s(2 * n, '0');
  for (std::size_t i = 0; i < n; ++i) {
    s[2 * i] = "0123456789abcdef"[bytes[i] >> 4];
    s[2 * i + 1] = "0123456789abcdef"[bytes[i] & 15];
  }
  return s;
}

}  // namespace b200sha3::rsp
