// gpfilter.hpp -- C++ entry point of the B200 GPF path.
//
// The reference's C++ API for the Gauss-polynomial filter is
//   gpfilter::gpf(const Image&, const SpatialParams&, const RangeParams&,
//                 SpatialBackend, const GpfOptions& = {}) -> FilterResult
// (/root/reference/proj/src/core/bilateral.hpp:73-75, "ref" below), the only
// way to reach midpoint centering (ref bilateral.hpp:15-21). This header
// declares the same names, members, defaults and exceptions in namespace
// gpfilter, so C++ callers of that path recompile against libgpfilter_b200.so
// unchanged:
//   Image                ref image.hpp:14-41 (row-major doubles, w, h >= 1)
//   IntensityRange       ref image.hpp:44-47
//   Boundary, SpatialParams, SigmaTooSmallError, default_window_radius
//                        ref spatial.hpp:13-34
//   RangeParams          ref range_kernel.hpp:13-18
//   SpatialBackend, CenteringMode, GpfOptions, FilterResult, GpfState, gpf, kQMin
//                        ref bilateral.hpp:13-28, 38-68, 73-85
// Errors are thrown as in the reference: std::invalid_argument for invalid
// parameters (same messages), SigmaTooSmallError for sigma_s < 0.5 on the
// recursive backend; GPU failures as std::runtime_error. The filter runs on the
// current CUDA device through the drop-in engine of gpf_filter_gpf (plan cache,
// AUTO precision: fp32 planes inside their validated envelope, the
// reference-exact fp64 mode outside it; gpfilter_b200.h).
#ifndef GPFILTER_B200_GPFILTER_HPP
#define GPFILTER_B200_GPFILTER_HPP

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace gpfilter {

class Image {
 public:
  Image() = default;
  Image(int width, int height, double fill = 0.0);  // throws std::invalid_argument if w or h < 1

  int width() const { return width_; }
  int height() const { return height_; }
  std::size_t pixels() const { return samples_.size(); }

  double* data() { return samples_.data(); }
  const double* data() const { return samples_.data(); }

  double& at(int row, int col) { return samples_[static_cast<std::size_t>(row) * width_ + col]; }
  double at(int row, int col) const { return samples_[static_cast<std::size_t>(row) * width_ + col]; }

  bool same_size(const Image& o) const { return width_ == o.width_ && height_ == o.height_; }

 private:
  int width_ = 0;
  int height_ = 0;
  std::vector<double> samples_;
};

struct IntensityRange {
  double low = 0.0;
  double high = 255.0;
};

enum class Boundary { replicate, reflect, zero };

struct SigmaTooSmallError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

struct SpatialParams {
  double sigma_s = 2.0;
  int window_radius = 6;
  Boundary boundary = Boundary::replicate;
  double kernel_scale = 1.0;

  static SpatialParams make(double sigma_s);  // window_radius = ceil(3 sigma_s)
  void validate() const;                      // throws std::invalid_argument
};

int default_window_radius(double sigma_s);

struct RangeParams {
  double sigma_r = 30.0;
  int degree = 20;

  void validate() const;  // throws std::invalid_argument
};

enum class SpatialBackend { direct, recursive };

enum class CenteringMode { mean, midpoint };

struct GpfOptions {
  bool centering = true;
  CenteringMode mode = CenteringMode::mean;
  IntensityRange range;  // midpoint mode: t_c = (low + high) / 2
};

struct FilterResult {
  Image image;
  long long fallback_count = 0;
};

// Gauss-polynomial bilateral filter on the GPU: constant time per pixel with
// SpatialBackend::recursive (the hot path), O(window_radius) with
// SpatialBackend::direct (windowed passes, fp64 mode); degree <= 62.
FilterResult gpf(const Image& img, const SpatialParams& sp, const RangeParams& rp,
                 SpatialBackend backend, const GpfOptions& opts = {});

inline constexpr double kQMin = 1e-8;

// The other entry points of the reference core, same signatures and exceptions,
// each running on the GPU through the C ABI entry of the same name (gpfilter.h):
//   exact_bilateral, taylor_bilateral            ref bilateral.hpp:30-36, 76-80
//   direct_gaussian, recursive_gaussian, kernel_mass_1d
//                                                ref spatial.hpp:46-64
//   mean_intensity, shift, max_abs_diff          ref image.hpp:49-57
//   ErrorReport, compare, mse_db, kMseDbFloor    ref metrics.hpp:11-33
//   gaussian_range, gauss_polynomial, taylor_polynomial, RangeApprox, sup_error
//                                                ref range_kernel.hpp:20-43 (host scalar)
Image exact_bilateral(const Image& img, const SpatialParams& sp, const RangeParams& rp);
FilterResult taylor_bilateral(const Image& img, const SpatialParams& sp, const RangeParams& rp,
                              SpatialBackend backend);
Image direct_gaussian(const Image& img, const SpatialParams& p);
Image recursive_gaussian(const Image& img, double sigma_s, double kernel_scale = 1.0);
double kernel_mass_1d(double sigma_s, int window_radius);
// index i mapped onto [0, n) by the boundary rule, -1 where zero padding drops the sample
// (ref spatial.hpp:38-40); unnormalised 2-D weight exp(-(jr^2 + jc^2) / 2 sigma_s^2) (42-43)
int boundary_index(int i, int n, Boundary boundary);
double spatial_weight(int j_row, int j_col, double sigma_s);
// ref parallel.hpp:20-22: recorded, not used -- the device work is deterministic and does not
// depend on a host thread count
void set_num_threads(int n);
int num_threads();

double mean_intensity(const Image& img);         // deterministic double-double mean on the GPU
Image shift(const Image& img, double c);         // every sample decreased by c
double max_abs_diff(const Image& a, const Image& b);  // throws std::invalid_argument on size mismatch

struct ErrorReport {
  double mse = 0.0;
  double mse_db = 0.0;  // 10 log10(mse), kMseDbFloor when mse == 0
  double max_abs = 0.0;
  long long pixels = 0;
};
inline constexpr double kMseDbFloor = -400.0;
double mse_db(double mse);
ErrorReport compare(const Image& ref, const Image& test, int exclude_border = 0);

double gaussian_range(double t, double tau, const RangeParams& p);
double gauss_polynomial(double t, double tau, const RangeParams& p);
double taylor_polynomial(double t, double tau, const RangeParams& p);
enum class RangeApprox { gauss_polynomial, taylor };
double sup_error(const RangeParams& p, double tau, const IntensityRange& range, double step,
                 RangeApprox which);

// PGM codec (ref pgm_io.hpp:17-54; host code, the C ABI's gpf_decode_pgm / gpf_encode_pgm /
// gpf_read_pgm / gpf_write_pgm are the same routines): P5 and P2 decode with comments, canonical
// P5 encode, clamp-and-round-half-away quantisation; parse failures carry their kind and the byte
// offset, file failures are std::runtime_error.
enum class PgmErrorKind { bad_magic, bad_dims, bad_maxval, truncated, bad_pixel };
const char* pgm_error_kind_name(PgmErrorKind kind);
class PgmParseError : public std::runtime_error {
 public:
  PgmParseError(PgmErrorKind kind, std::size_t offset, const std::string& detail);
  PgmErrorKind kind() const { return kind_; }
  std::size_t offset() const { return offset_; }

 private:
  PgmErrorKind kind_;
  std::size_t offset_;
};
Image decode_pgm(const std::uint8_t* bytes, std::size_t size);
std::vector<std::uint8_t> encode_pgm(const Image& img);
std::uint8_t quantize_sample(double v);
Image read_pgm(const std::string& path);
void write_pgm(const Image& img, const std::string& path);

// Step-wise form of gpf (ref bilateral.hpp:38-68): init, then degree + 1 calls
// of step(), then finalize(); after n steps c = 1/n!, G = H^n, F = H^n F_0.
// The state images are public host images, as in the reference; every phase
// runs on the GPU in the reference-exact fp64 arithmetic (the reference's
// operation order; F_0's exp() is correctly rounded, one ulp from glibc's on ~0.1 % of arguments) on the images as they
// stand, so a caller may inspect or edit them between steps. It is the
// inspection tool, not the fast path: each step round-trips its images over
// PCIe (gpf() keeps the planes on the device).
struct GpfState {
  Image G;     // running power image H^n
  Image F;     // Gaussian-weighted moment image
  Image Fbar;  // spatially filtered F
  Image P;     // numerator accumulator
  Image Q;     // denominator accumulator
  Image H;     // h / sigma_r
  double c = 1.0;
  int n = 0;  // completed steps
  double t_c = 0.0;

  static GpfState init(const Image& img, const SpatialParams& sp, const RangeParams& rp,
                       SpatialBackend backend, const GpfOptions& opts);
  void step();
  FilterResult finalize(const Image& input) const;  // sigma_r (P / Q) + t_c, fallback rule

 private:
  SpatialParams sp_;
  RangeParams rp_;
  SpatialBackend backend_ = SpatialBackend::recursive;
};

}  // namespace gpfilter

#endif  // GPFILTER_B200_GPFILTER_HPP
