// PGM codec of the C ABI (gpf_read_pgm / gpf_decode_pgm / gpf_write_pgm /
// gpf_encode_pgm / gpf_free_bytes; reference ref.h:171-190, capi.cpp:311-349,
// behaviour of proj/src/core/pgm_io.cpp): the data format on either side of the
// GPF path. Host code: parsing and quantisation only.
//
// Accepted: "P5" (binary) or "P2" (ASCII) magic; header tokens separated by
// whitespace, '#' comments to the end of line; width and height in 1..2^20;
// maxval exactly 255; a P5 raster starts after exactly one whitespace byte.
// Failures carry a status (bad magic / dims / maxval / truncated / bad pixel)
// and a message "PGM parse error (<kind>) at byte <offset>: <detail>".
// Encoding writes P5 with samples rounded half away from zero and clamped to
// [0, 255] (NaN and non-positive values -> 0).
#include "pgm.h"

#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

namespace gpfb {
namespace pgm {

namespace {

const char* kind_name(gpf_status s) {
  switch (s) {
    case GPF_ERR_PGM_BAD_MAGIC: return "bad_magic";
    case GPF_ERR_PGM_BAD_DIMS: return "bad_dims";
    case GPF_ERR_PGM_BAD_MAXVAL: return "bad_maxval";
    case GPF_ERR_PGM_TRUNCATED: return "truncated";
    case GPF_ERR_PGM_BAD_PIXEL: return "bad_pixel";
    default: return "unknown";
  }
}

[[noreturn]] void parse_error(gpf_status s, size_t offset, const std::string& detail) {
  throw Error{s, std::string("PGM parse error (") + kind_name(s) + ") at byte " +
                     std::to_string(offset) + ": " + detail};
}

inline bool space(uint8_t c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

class Tokens {
 public:
  Tokens(const uint8_t* b, size_t n, size_t start) : b_(b), n_(n), at_(start) {}

  size_t at() const { return at_; }
  size_t token_start() const { return tok_; }
  bool done() const { return at_ >= n_; }
  uint8_t peek() const { return b_[at_]; }
  void advance() { ++at_; }

  // Next unsigned decimal token, bounded by `limit`; failures report `kind`.
  long long number(gpf_status kind, const char* what, long long limit) {
    skip();
    if (at_ >= n_) parse_error(GPF_ERR_PGM_TRUNCATED, n_, std::string("missing ") + what);
    tok_ = at_;
    long long v = 0;
    size_t digits = 0;
    for (; at_ < n_ && b_[at_] >= '0' && b_[at_] <= '9'; ++at_, ++digits) {
      v = 10 * v + (b_[at_] - '0');
      if (v > limit) parse_error(kind, tok_, std::string(what) + " exceeds " + std::to_string(limit));
    }
    const bool ends = at_ >= n_ || space(b_[at_]) || b_[at_] == '#';
    if (digits == 0 || !ends) parse_error(kind, tok_, std::string("malformed ") + what);
    return v;
  }

 private:
  void skip() {
    while (at_ < n_) {
      if (space(b_[at_])) {
        ++at_;
      } else if (b_[at_] == '#') {
        while (at_ < n_ && b_[at_] != '\n') ++at_;
      } else {
        return;
      }
    }
  }

  const uint8_t* b_;
  size_t n_, at_, tok_ = 0;
};

}  // namespace

Decoded decode(const uint8_t* bytes, size_t size) {
  if (size < 2 || bytes[0] != 'P' || (bytes[1] != '2' && bytes[1] != '5'))
    parse_error(GPF_ERR_PGM_BAD_MAGIC, 0, "expected magic \"P5\" or \"P2\"");
  const bool raw = bytes[1] == '5';
  Tokens t(bytes, size, 2);
  constexpr long long kMaxDim = 1 << 20;
  const long long w = t.number(GPF_ERR_PGM_BAD_DIMS, "width", kMaxDim);
  if (w < 1) parse_error(GPF_ERR_PGM_BAD_DIMS, t.token_start(), "width must be positive");
  const long long h = t.number(GPF_ERR_PGM_BAD_DIMS, "height", kMaxDim);
  if (h < 1) parse_error(GPF_ERR_PGM_BAD_DIMS, t.token_start(), "height must be positive");
  const long long maxval = t.number(GPF_ERR_PGM_BAD_MAXVAL, "maxval", 255);
  if (maxval != 255) parse_error(GPF_ERR_PGM_BAD_MAXVAL, t.token_start(), "only maxval 255 is supported");
  Decoded d;
  d.w = static_cast<int>(w);
  d.h = static_cast<int>(h);
  const size_t count = static_cast<size_t>(w) * static_cast<size_t>(h);
  d.pixels.resize(count);
  if (raw) {
    if (t.done()) parse_error(GPF_ERR_PGM_TRUNCATED, size, "missing raster");
    if (!space(t.peek()))
      parse_error(GPF_ERR_PGM_BAD_MAXVAL, t.at(), "expected a single whitespace byte after maxval");
    t.advance();
    const size_t left = size - t.at();
    if (left < count)
      parse_error(GPF_ERR_PGM_TRUNCATED, size,
                  "raster has " + std::to_string(left) + " of " + std::to_string(count) + " bytes");
    const uint8_t* r = bytes + t.at();
    for (size_t i = 0; i < count; ++i) d.pixels[i] = r[i];
  } else {
    for (size_t i = 0; i < count; ++i)
      d.pixels[i] = static_cast<double>(t.number(GPF_ERR_PGM_BAD_PIXEL, "sample", 255));
  }
  return d;
}

uint8_t quantize(double v) {
  if (!(v > 0.0)) return 0;
  if (v >= 255.0) return 255;
  return static_cast<uint8_t>(std::lround(v));
}

std::vector<uint8_t> encode(const double* px, int w, int h) {
  const std::string head = "P5\n" + std::to_string(w) + " " + std::to_string(h) + "\n255\n";
  std::vector<uint8_t> out(head.begin(), head.end());
  const size_t count = static_cast<size_t>(w) * static_cast<size_t>(h);
  out.reserve(out.size() + count);
  for (size_t i = 0; i < count; ++i) out.push_back(quantize(px[i]));
  return out;
}

std::vector<uint8_t> read_file(const char* path) {
  std::FILE* fp = std::fopen(path, "rb");
  if (!fp) throw Error{GPF_ERR_IO, std::string("cannot open ") + path + " for reading"};
  std::vector<uint8_t> buf;
  uint8_t chunk[1 << 16];
  size_t got;
  while ((got = std::fread(chunk, 1, sizeof(chunk), fp)) > 0) buf.insert(buf.end(), chunk, chunk + got);
  const bool bad = std::ferror(fp) != 0;
  std::fclose(fp);
  if (bad) throw Error{GPF_ERR_IO, std::string("read failure on ") + path};
  return buf;
}

void write_file(const char* path, const std::vector<uint8_t>& bytes) {
  std::FILE* fp = std::fopen(path, "wb");
  if (!fp) throw Error{GPF_ERR_IO, std::string("cannot open ") + path + " for writing"};
  const size_t put = std::fwrite(bytes.data(), 1, bytes.size(), fp);
  const bool bad = put != bytes.size() || std::fclose(fp) != 0;
  if (bad) throw Error{GPF_ERR_IO, std::string("write failure on ") + path};
}

}  // namespace pgm
}  // namespace gpfb
