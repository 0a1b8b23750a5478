// io.cpp — on-disk exchange formats of the reference (proj/src/io.cpp,
// io.hpp:12-36), host side, behind the C ABI (include/sige_b200.h):
//  * SIGT tensors: "SIGT", u32 version 1, u32 dims n/c/h/w, n*c*h*w float32
//    bit patterns, all little-endian, no trailing bytes (io.cpp:34-85);
//  * plain PBM (P1) masks: "P1\n<w> <h>\n", rows of '0'/'1' separated by
//    spaces; on read, comments and whitespace-free packing are accepted
//    (io.cpp:102-160);
//  * sige_blocks_v1 block stacks: the (count, C, bh, bh) payload as SIGT plus a
//    json sidecar with the geometry and origin indices (io.cpp:405-457). The
//    sidecar is written byte-identically to the reference's dump(2) with the
//    nlohmann build in this image (3.11.3 as bundled with cudnn_frontend: keys
//    sorted, 2-space indent, arrays of numbers on one line) and read with a
//    small json reader for that schema.
// Error messages are the reference's ConfigError texts.
#include <cctype>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "common.hpp"

namespace sige_b200 {

namespace {

void put_u32(std::ostream& os, uint32_t v) {
  const char b[4] = {static_cast<char>(v & 0xff), static_cast<char>((v >> 8) & 0xff),
                     static_cast<char>((v >> 16) & 0xff), static_cast<char>((v >> 24) & 0xff)};
  os.write(b, 4);
}

uint32_t get_u32(std::istream& is, const std::string& path) {
  unsigned char b[4];
  if (!is.read(reinterpret_cast<char*>(b), 4)) throw ConfigError(path + ": truncated tensor file");
  return static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) | (static_cast<uint32_t>(b[2]) << 16) |
         (static_cast<uint32_t>(b[3]) << 24);
}

}  // namespace

void io_write_sigt(const std::string& path, const uint32_t d[4], const float* data) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw ConfigError(path + ": cannot open for writing");
  os.write("SIGT", 4);
  put_u32(os, 1);
  for (int i = 0; i < 4; ++i) put_u32(os, d[i]);
  const size_t count = static_cast<size_t>(d[0]) * d[1] * d[2] * d[3];
  std::vector<char> buf(count * 4);
  for (size_t i = 0; i < count; ++i) {
    uint32_t bits;
    std::memcpy(&bits, data + i, 4);
    for (int k = 0; k < 4; ++k) buf[4 * i + k] = static_cast<char>((bits >> (8 * k)) & 0xff);
  }
  os.write(buf.data(), static_cast<std::streamsize>(buf.size()));
  if (!os) throw ConfigError(path + ": write failed");
}

// Header only (dims), or header + payload into `out` (capacity in floats).
void io_read_sigt(const std::string& path, uint32_t d[4], float* out, size_t cap) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw ConfigError(path + ": cannot open");
  char magic[4];
  if (!is.read(magic, 4) || std::memcmp(magic, "SIGT", 4) != 0)
    throw ConfigError(path + ": not a SIGT tensor file (bad magic)");
  const uint32_t version = get_u32(is, path);
  if (version != 1) throw ConfigError(path + ": unsupported SIGT version " + std::to_string(version));
  for (int i = 0; i < 4; ++i) d[i] = get_u32(is, path);
  const size_t count = static_cast<size_t>(d[0]) * d[1] * d[2] * d[3];
  if (count > (1ull << 31)) throw ConfigError(path + ": unreasonable tensor size");
  if (!out) return;
  if (cap < count) throw ConfigError(path + ": output buffer too small");
  std::vector<unsigned char> buf(count * 4);
  if (count && !is.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size())))
    throw ConfigError(path + ": truncated tensor file");
  for (size_t i = 0; i < count; ++i) {
    const uint32_t bits = static_cast<uint32_t>(buf[4 * i]) | (static_cast<uint32_t>(buf[4 * i + 1]) << 8) |
                          (static_cast<uint32_t>(buf[4 * i + 2]) << 16) | (static_cast<uint32_t>(buf[4 * i + 3]) << 24);
    std::memcpy(out + i, &bits, 4);
  }
  char extra;
  if (is.read(&extra, 1)) throw ConfigError(path + ": trailing bytes");
}

void io_save_mask_pbm(const std::string& path, const uint8_t* m, int h, int w) {
  std::ofstream os(path);
  if (!os) throw ConfigError(path + ": cannot open for writing");
  std::string s = "P1\n" + std::to_string(w) + " " + std::to_string(h) + "\n";
  s.reserve(s.size() + static_cast<size_t>(h) * w * 2);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      s.push_back(m[static_cast<size_t>(y) * w + x] ? '1' : '0');
      s.push_back(x + 1 == w ? '\n' : ' ');
    }
  os << s;
  if (!os) throw ConfigError(path + ": write failed");
}

namespace {

// The file is read whole and scanned by position (the reference streams it,
// io.cpp:118-160; the accepted grammar and the error texts are the same).
// Header fields are runs of non-space bytes; a field opening with '#' comments
// out the rest of its line. Payload bits may be packed without separators.
class PbmScanner {
 public:
  PbmScanner(std::string text, const std::string& path) : s_(std::move(text)), path_(path) {}

  std::string field() {
    for (;;) {
      while (pos_ < s_.size() && is_space(s_[pos_])) ++pos_;
      if (pos_ == s_.size()) throw ConfigError(path_ + ": truncated PBM file");
      const size_t from = pos_;
      while (pos_ < s_.size() && !is_space(s_[pos_])) ++pos_;
      if (s_[from] != '#') return s_.substr(from, pos_ - from);
      skip_line();
    }
  }

  // Fills up to n bits; returns how many were present.
  size_t bits(uint8_t* out, size_t n) {
    size_t got = 0;
    while (got < n && pos_ < s_.size()) {
      const char c = s_[pos_++];
      if (c == '0' || c == '1') {
        out[got++] = static_cast<uint8_t>(c - '0');
      } else if (c == '#') {
        skip_line();
      } else if (!is_space(c)) {
        throw ConfigError(path_ + ": unexpected character in PBM payload");
      }
    }
    return got;
  }

 private:
  static bool is_space(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }
  void skip_line() {
    const size_t nl = s_.find('\n', pos_);
    pos_ = nl == std::string::npos ? s_.size() : nl + 1;
  }
  std::string s_;
  const std::string& path_;
  size_t pos_ = 0;
};

}  // namespace

// dims only when out == nullptr
void io_load_mask_pbm(const std::string& path, int* h, int* w, uint8_t* out, size_t cap) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw ConfigError(path + ": cannot open");
  PbmScanner sc(std::string(std::istreambuf_iterator<char>(is), std::istreambuf_iterator<char>()), path);
  const std::string magic = sc.field();
  if (magic != "P1") throw ConfigError(path + ": expected plain PBM (P1), got '" + magic + "'");
  const int ww = std::stoi(sc.field());
  const int hh = std::stoi(sc.field());
  if (ww < 1 || hh < 1) throw ConfigError(path + ": bad PBM dimensions");
  *h = hh;
  *w = ww;
  if (!out) return;
  const size_t n = static_cast<size_t>(hh) * ww;
  if (cap < n) throw ConfigError(path + ": output buffer too small");
  if (sc.bits(out, n) != n) throw ConfigError(path + ": truncated PBM file");
}

// ------------------------------------------------------------ block stacks

namespace {

// Minimal json value for the sige_blocks_v1 sidecar: objects, arrays,
// integers (and strings for "format"); anything else is a parse error.
struct JVal {
  enum Kind { kNull, kNum, kStr, kArr, kObj } kind = kNull;
  long long num = 0;
  std::string str;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;
};

struct JParser {
  const std::string& s;
  size_t i = 0;
  std::string where;
  [[noreturn]] void fail(const std::string& why) {
    throw ConfigError(where + ": json parse error: " + why + " at offset " + std::to_string(i));
  }
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  JVal value() {
    ws();
    if (i >= s.size()) fail("unexpected end");
    JVal v;
    const char c = s[i];
    if (c == '{') {
      v.kind = JVal::kObj;
      ++i;
      ws();
      if (i < s.size() && s[i] == '}') return ++i, v;
      for (;;) {
        ws();
        JVal k = value();
        if (k.kind != JVal::kStr) fail("object key is not a string");
        ws();
        if (i >= s.size() || s[i] != ':') fail("expected ':'");
        ++i;
        v.obj[k.str] = value();
        ws();
        if (i < s.size() && s[i] == ',') {
          ++i;
          continue;
        }
        if (i < s.size() && s[i] == '}') return ++i, v;
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = JVal::kArr;
      ++i;
      ws();
      if (i < s.size() && s[i] == ']') return ++i, v;
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (i < s.size() && s[i] == ',') {
          ++i;
          continue;
        }
        if (i < s.size() && s[i] == ']') return ++i, v;
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = JVal::kStr;
      ++i;
      while (i < s.size() && s[i] != '"') {
        if (s[i] == '\\') fail("escapes are not used by sige_blocks_v1");
        v.str.push_back(s[i++]);
      }
      if (i >= s.size()) fail("unterminated string");
      ++i;
      return v;
    }
    if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) {
      v.kind = JVal::kNum;
      size_t j = i + (c == '-');
      while (j < s.size() && std::isdigit(static_cast<unsigned char>(s[j]))) ++j;
      if (j < s.size() && (s[j] == '.' || s[j] == 'e' || s[j] == 'E')) fail("non-integer number");
      v.num = std::stoll(s.substr(i, j - i));
      i = j;
      return v;
    }
    fail("unexpected character");
  }
};

const JVal& at(const JVal& o, const char* key, const std::string& where) {
  if (o.kind != JVal::kObj) throw ConfigError(where + ": json parse error: expected an object");
  auto it = o.obj.find(key);
  if (it == o.obj.end()) throw ConfigError(where + ": json parse error: missing key '" + key + "'");
  return it->second;
}

int as_int(const JVal& v, const std::string& where) {
  if (v.kind != JVal::kNum) throw ConfigError(where + ": json parse error: expected a number");
  return static_cast<int>(v.num);
}

}  // namespace

void io_save_block_stack(const std::string& prefix, const float* data, int count, int channels, int block,
                         int overlap, int origin_block, int origin_h, int origin_w, const int32_t* idx) {
  const int bh = block + overlap;
  const uint32_t d[4] = {static_cast<uint32_t>(count), static_cast<uint32_t>(channels), static_cast<uint32_t>(bh),
                         static_cast<uint32_t>(bh)};
  io_write_sigt(prefix + ".sigt", d, data);
  // nlohmann::json::dump(2) of {block, format, indices, origin, overlap} (std::map order)
  std::ostringstream js;
  js << "{\n  \"block\": " << block << ",\n  \"format\": \"sige_blocks_v1\",\n  \"indices\": ";
  if (count == 0) {
    js << "[]";
  } else {
    js << "[\n";
    for (int g = 0; g < count; ++g) {
      js << "    [" << idx[3 * g] << "," << idx[3 * g + 1] << "," << idx[3 * g + 2] << "]"
         << (g + 1 < count ? ",\n" : "\n");
    }
    js << "  ]";
  }
  js << ",\n  \"origin\": {\n    \"block_size\": " << origin_block << ",\n    \"h\": " << origin_h
     << ",\n    \"w\": " << origin_w << "\n  },\n  \"overlap\": " << overlap << "\n}\n";
  std::ofstream os(prefix + ".json");
  if (!os) throw ConfigError(prefix + ".json: cannot open for writing");
  os << js.str();
  if (!os) throw ConfigError(prefix + ".json: write failed");
}

// meta = {count, channels, block, overlap, origin_block, origin_h, origin_w};
// payload / indices only when the output pointers are non-null.
void io_load_block_stack(const std::string& prefix, int meta[7], float* data, size_t cap, int32_t* idx,
                         size_t idx_cap) {
  const std::string jpath = prefix + ".json";
  std::ifstream is(jpath);
  if (!is) throw ConfigError(jpath + ": cannot open");
  std::stringstream ss;
  ss << is.rdbuf();
  const std::string text = ss.str();
  JParser jp{text, 0, jpath};
  const JVal j = jp.value();
  jp.ws();
  if (jp.i != text.size()) jp.fail("trailing characters");
  if (j.kind != JVal::kObj || !j.obj.count("format") || j.obj.at("format").kind != JVal::kStr ||
      j.obj.at("format").str != "sige_blocks_v1")
    throw ConfigError(jpath + ": not a sige_blocks_v1 file");
  const int block = as_int(at(j, "block", jpath), jpath), overlap = as_int(at(j, "overlap", jpath), jpath);
  const JVal& org = at(j, "origin", jpath);
  const JVal& ind = at(j, "indices", jpath);
  if (ind.kind != JVal::kArr) throw ConfigError(jpath + ": json parse error: indices is not an array");
  uint32_t d[4];
  io_read_sigt(prefix + ".sigt", d, nullptr, 0);
  if (d[0] != ind.arr.size()) throw ConfigError(prefix + ": payload/index count mismatch");
  if (static_cast<int>(d[2]) != block + overlap || static_cast<int>(d[3]) != block + overlap)
    throw ConfigError(prefix + ": payload block geometry mismatch");
  meta[0] = static_cast<int>(d[0]);
  meta[1] = static_cast<int>(d[1]);
  meta[2] = block;
  meta[3] = overlap;
  meta[4] = as_int(at(org, "block_size", jpath), jpath);
  meta[5] = as_int(at(org, "h", jpath), jpath);
  meta[6] = as_int(at(org, "w", jpath), jpath);
  if (idx) {
    if (idx_cap < 3 * ind.arr.size()) throw ConfigError(prefix + ": index buffer too small");
    for (size_t g = 0; g < ind.arr.size(); ++g) {
      const JVal& e = ind.arr[g];
      if (e.kind != JVal::kArr || e.arr.size() < 3) throw ConfigError(jpath + ": json parse error: bad index entry");
      for (int k = 0; k < 3; ++k) idx[3 * g + k] = as_int(e.arr[k], jpath);
    }
  }
  if (data) io_read_sigt(prefix + ".sigt", d, data, cap);
}

}  // namespace sige_b200
