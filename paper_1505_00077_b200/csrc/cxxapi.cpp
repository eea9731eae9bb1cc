// C++ entry point (include/gpfilter/gpfilter.hpp): gpfilter::gpf over the
// drop-in engine (dropin.cpp), with the reference's validation order and
// exceptions (proj/src/core/bilateral.cpp:64-106, 150-158; spatial.cpp:25-35,
// 220-230; range_kernel.cpp:22-29; image.cpp:11-18).
#include <cmath>
#include <string>

#include "gpf_internal.h"
#include "gpfilter/gpfilter.hpp"

namespace gpfilter {

Image::Image(int width, int height, double fill) {
  if (width < 1 || height < 1) throw std::invalid_argument("Image dimensions must be >= 1");
  width_ = width;
  height_ = height;
  samples_.assign(static_cast<std::size_t>(width) * height, fill);
}

int default_window_radius(double sigma_s) { return static_cast<int>(std::ceil(3.0 * sigma_s)); }

SpatialParams SpatialParams::make(double sigma_s) {
  SpatialParams p;
  p.sigma_s = sigma_s;
  p.window_radius = default_window_radius(sigma_s);
  return p;
}

void SpatialParams::validate() const {
  if (!(sigma_s > 0.0)) throw std::invalid_argument("SpatialParams: sigma_s must be > 0");
  if (window_radius < 1) throw std::invalid_argument("SpatialParams: window_radius must be >= 1");
  if (!(kernel_scale > 0.0)) throw std::invalid_argument("SpatialParams: kernel_scale must be > 0");
}

void RangeParams::validate() const {
  if (!(sigma_r > 0.0)) throw std::invalid_argument("RangeParams: sigma_r must be > 0");
  if (degree < 0) throw std::invalid_argument("RangeParams: degree must be >= 0");
}

FilterResult gpf(const Image& img, const SpatialParams& sp, const RangeParams& rp,
                 SpatialBackend backend, const GpfOptions& opts) {
  // GpfState::init (bilateral.cpp:67-72): parameters, then the range option
  sp.validate();
  rp.validate();
  if (!(opts.range.low < opts.range.high))
    throw std::invalid_argument("GpfOptions: range.low must be < range.high");
  if (img.pixels() == 0) throw std::invalid_argument("Image dimensions must be >= 1");
  // apply_spatial (bilateral.cpp:58-62): direct_gaussian (spatial.cpp:112-129)
  // or recursive_gaussian (spatial.cpp:222-230)
  if (backend == SpatialBackend::recursive) {
    if (!(sp.sigma_s > 0.0) || !(sp.kernel_scale > 0.0))
      throw std::invalid_argument("recursive_gaussian: sigma_s and kernel_scale must be > 0");
    if (sp.sigma_s < 0.5)
      throw SigmaTooSmallError(
          "recursive_gaussian: sigma_s < 0.5 is not supported; use the direct backend");
  }
  if (rp.degree > gpfb::kMaxDegreeF64)
    throw std::invalid_argument("RangeParams: degree must be <= " +
                                std::to_string(gpfb::kMaxDegreeF64) + " in the B200 library");
  gpfb::Params p;
  p.width = img.width();
  p.height = img.height();
  p.sigma_s = sp.sigma_s;
  p.kernel_scale = sp.kernel_scale;
  p.sigma_r = rp.sigma_r;
  p.degree = rp.degree;
  p.backend = backend == SpatialBackend::direct ? 0 : 1;
  p.window_radius = sp.window_radius;
  p.boundary = static_cast<int>(sp.boundary);
  // t_c (bilateral.cpp:77-82): mean, midpoint (low + high) / 2, or 0
  p.centering = !opts.centering ? 0 : (opts.mode == CenteringMode::mean ? 1 : 2);
  p.tc_fixed = (opts.range.low + opts.range.high) / 2.0;
  FilterResult res;
  res.image = Image(img.width(), img.height());
  try {
    res.fallback_count = gpfb::dropin_gpf(img.data(), res.image.data(), p);
  } catch (const gpfb::Error& e) {
    if (e.status == 1) throw std::invalid_argument(e.msg);
    if (e.status == 3) throw SigmaTooSmallError(e.msg);
    throw std::runtime_error(e.msg);
  }
  return res;
}

}  // namespace gpfilter
