// PGM codec (host side of the C ABI's PGM entries; see pgm.cpp).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "gpf_internal.h"
#include "gpfilter/gpfilter.h"

namespace gpfb {
namespace pgm {

struct Decoded {
  int w = 0, h = 0;
  std::vector<double> pixels;
};

Decoded decode(const uint8_t* bytes, size_t size);             // throws Error (GPF_ERR_PGM_*)
std::vector<uint8_t> encode(const double* px, int w, int h);   // P5
uint8_t quantize(double v);
std::vector<uint8_t> read_file(const char* path);             // throws Error (GPF_ERR_IO)
void write_file(const char* path, const std::vector<uint8_t>& bytes);

}  // namespace pgm
}  // namespace gpfb
