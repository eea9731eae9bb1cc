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

#include <algorithm>
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

// Header scanner. A token is a maximal run of bytes that are neither
// whitespace nor '#'; separators are whitespace and '#'-to-end-of-line
// comments. next() returns the token's [begin, end) or begin == n at the end
// of the input.
struct Span {
  size_t begin, end;
};

Span next_token(const uint8_t* b, size_t n, size_t& pos) {
  for (;;) {
    while (pos < n && space(b[pos])) ++pos;
    if (pos < n && b[pos] == '#') {
      while (pos < n && b[pos] != '\n') ++pos;
      continue;
    }
    break;
  }
  const size_t begin = pos;
  while (pos < n && !space(b[pos]) && b[pos] != '#') ++pos;
  return {begin, pos};
}

// One header / ASCII-raster field: an unsigned decimal no larger than
// `limit`. The value is checked digit by digit (a too-long number is reported
// as exceeding the limit even if it is followed by garbage); a token that is
// empty or not all digits is malformed. Errors carry the token's offset.
long long field(const uint8_t* b, size_t n, size_t& pos, gpf_status kind, const char* what,
                long long limit, size_t* where = nullptr) {
  const Span t = next_token(b, n, pos);
  if (t.begin == n) parse_error(GPF_ERR_PGM_TRUNCATED, n, std::string("missing ") + what);
  if (where) *where = t.begin;
  long long v = 0;
  size_t k = t.begin;
  while (k < t.end && b[k] >= '0' && b[k] <= '9') {
    v = 10 * v + (b[k++] - '0');
    if (v > limit) parse_error(kind, t.begin, std::string(what) + " exceeds " + std::to_string(limit));
  }
  if (k == t.begin || k != t.end) parse_error(kind, t.begin, std::string("malformed ") + what);
  return v;
}

}  // namespace

Decoded decode(const uint8_t* bytes, size_t size) {
  if (size < 2 || bytes[0] != 'P' || (bytes[1] != '2' && bytes[1] != '5'))
    parse_error(GPF_ERR_PGM_BAD_MAGIC, 0, "expected magic \"P5\" or \"P2\"");
  const bool raw = bytes[1] == '5';
  size_t pos = 2, at = 0;
  constexpr long long kMaxDim = 1 << 20;
  long long dims[2];
  const char* names[2] = {"width", "height"};
  for (int k = 0; k < 2; ++k) {
    dims[k] = field(bytes, size, pos, GPF_ERR_PGM_BAD_DIMS, names[k], kMaxDim, &at);
    if (dims[k] < 1) parse_error(GPF_ERR_PGM_BAD_DIMS, at, std::string(names[k]) + " must be positive");
  }
  if (field(bytes, size, pos, GPF_ERR_PGM_BAD_MAXVAL, "maxval", 255, &at) != 255)
    parse_error(GPF_ERR_PGM_BAD_MAXVAL, at, "only maxval 255 is supported");
  Decoded d;
  d.w = static_cast<int>(dims[0]);
  d.h = static_cast<int>(dims[1]);
  const size_t count = static_cast<size_t>(dims[0]) * static_cast<size_t>(dims[1]);
  d.pixels.resize(count);
  if (!raw) {  // P2: every sample is a field of its own
    for (double& v : d.pixels) v = static_cast<double>(field(bytes, size, pos, GPF_ERR_PGM_BAD_PIXEL, "sample", 255));
    return d;
  }
  // P5: the maxval token is followed by exactly one whitespace byte, then the raster
  if (pos == size) parse_error(GPF_ERR_PGM_TRUNCATED, size, "missing raster");
  if (!space(bytes[pos]))
    parse_error(GPF_ERR_PGM_BAD_MAXVAL, pos, "expected a single whitespace byte after maxval");
  const uint8_t* raster = bytes + pos + 1;
  const size_t avail = size - pos - 1;
  if (avail < count)
    parse_error(GPF_ERR_PGM_TRUNCATED, size,
                "raster has " + std::to_string(avail) + " of " + std::to_string(count) + " bytes");
  std::copy(raster, raster + count, d.pixels.begin());
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
