// C++ entry point (include/gpfilter/gpfilter.hpp): gpfilter::gpf over the
// drop-in engine (dropin.cpp), with the reference's validation order and
// exceptions (proj/src/core/bilateral.cpp:64-106, 150-158; spatial.cpp:25-35,
// 220-230; range_kernel.cpp:22-29; image.cpp:11-18).
#include <cmath>
#include <string>
#include <utility>

#include <cuda_runtime.h>

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

// ------------------------------------------------------------------ GpfState
namespace {

[[noreturn]] void rethrow(const gpfb::Error& e) {
  if (e.status == 1) throw std::invalid_argument(e.msg);
  if (e.status == 3) throw SigmaTooSmallError(e.msg);
  throw std::runtime_error(e.msg);
}

void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw gpfb::Error{9, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

// n doubles on the device, optionally filled from a host image
struct Dev {
  double* p = nullptr;
  size_t n = 0;
  explicit Dev(size_t count, const double* host = nullptr) : n(count) {
    cu(cudaMalloc(&p, sizeof(double) * count), "cudaMalloc");
    if (host) up(host);
  }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  void up(const double* host) { cu(cudaMemcpy(p, host, sizeof(double) * n, cudaMemcpyHostToDevice), "H2D"); }
  void down(double* host) const { cu(cudaMemcpy(host, p, sizeof(double) * n, cudaMemcpyDeviceToHost), "D2H"); }
};

gpfb::Params state_params(int w, int h, const SpatialParams& sp, const RangeParams& rp,
                          SpatialBackend backend) {
  gpfb::Params p;
  p.width = w;
  p.height = h;
  p.sigma_s = sp.sigma_s;
  p.kernel_scale = sp.kernel_scale;
  p.sigma_r = rp.sigma_r;
  p.degree = rp.degree;
  p.backend = backend == SpatialBackend::direct ? 0 : 1;
  p.window_radius = sp.window_radius;
  p.boundary = static_cast<int>(sp.boundary);
  return p;
}

void require_device() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw std::runtime_error("no CUDA device available (the B200 library has no CPU path)");
  }
}

}  // namespace

GpfState GpfState::init(const Image& img, const SpatialParams& sp, const RangeParams& rp,
                        SpatialBackend backend, const GpfOptions& opts) {
  // bilateral.cpp:67-72, then the first apply_spatial's checks (spatial.cpp:222-230)
  sp.validate();
  rp.validate();
  if (!(opts.range.low < opts.range.high))
    throw std::invalid_argument("GpfOptions: range.low must be < range.high");
  if (img.pixels() == 0) throw std::invalid_argument("Image dimensions must be >= 1");
  if (backend == SpatialBackend::recursive && sp.sigma_s < 0.5)
    throw SigmaTooSmallError(
        "recursive_gaussian: sigma_s < 0.5 is not supported; use the direct backend");
  require_device();
  GpfState s;
  s.sp_ = sp;
  s.rp_ = rp;
  s.backend_ = backend;
  const int w = img.width(), h = img.height();
  const size_t n = img.pixels();
  s.G = Image(w, h, 1.0);
  s.P = Image(w, h, 0.0);
  s.Q = Image(w, h, 0.0);
  s.H = Image(w, h);
  s.F = Image(w, h);
  s.Fbar = Image(w, h);
  gpfb::Params p = state_params(w, h, sp, rp, backend);
  // t_c (bilateral.cpp:77-82): mean, midpoint (low + high) / 2, or 0
  p.centering = !opts.centering ? 0 : (opts.mode == CenteringMode::mean ? 1 : 2);
  p.tc_fixed = (opts.range.low + opts.range.high) / 2.0;
  try {
    Dev in(n, img.data()), dH(n), dF(n), dFbar(n), tmp(n), scal(2 + 4 * (size_t)gpfb::kF64MeanBlocks);
    gpfb::state_init_f64(in.p, dH.p, dF.p, scal.p, scal.p + 2, p, nullptr);
    gpfb::state_spatial_f64(dF.p, dFbar.p, tmp.p, p, nullptr);
    cu(cudaMemcpy(&s.t_c, scal.p, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    dH.down(s.H.data());
    dF.down(s.F.data());
    dFbar.down(s.Fbar.data());
  } catch (const gpfb::Error& e) {
    rethrow(e);
  }
  s.c = 1.0;
  s.n = 0;
  return s;
}

void GpfState::step() {
  require_device();
  const size_t count = F.pixels();
  const gpfb::Params p = state_params(F.width(), F.height(), sp_, rp_, backend_);
  try {
    Dev dG(count, G.data()), dF(count, F.data()), dFbar(count, Fbar.data()), dP(count, P.data()),
        dQ(count, Q.data()), dH(count, H.data()), tmp(count);
    gpfb::state_step_a_f64(dQ.p, dF.p, dG.p, dFbar.p, dH.p, c, (long long)count, nullptr);
    gpfb::state_spatial_f64(dF.p, dFbar.p, tmp.p, p, nullptr);
    gpfb::state_step_b_f64(dP.p, dG.p, dFbar.p, dH.p, c, (long long)count, nullptr);
    dQ.down(Q.data());
    dF.down(F.data());
    dFbar.down(Fbar.data());
    dP.down(P.data());
    dG.down(G.data());
  } catch (const gpfb::Error& e) {
    rethrow(e);
  }
  c = c / (n + 1);
  ++n;
}

FilterResult GpfState::finalize(const Image& input) const {
  if (!input.same_size(P) || !input.same_size(Q))
    throw std::invalid_argument("GpfState::finalize: input and state images differ in size");
  require_device();
  FilterResult res;
  res.image = Image(input.width(), input.height());
  const size_t count = input.pixels();
  try {
    Dev in(count, input.data()), dP(count, P.data()), dQ(count, Q.data()), out(count), fb(1);
    gpfb::state_finalize_f64(in.p, dP.p, dQ.p, out.p, (long long)count, rp_.sigma_r, t_c,
                             reinterpret_cast<unsigned long long*>(fb.p), nullptr);
    out.down(res.image.data());
    unsigned long long f = 0;
    cu(cudaMemcpy(&f, fb.p, sizeof(f), cudaMemcpyDeviceToHost), "D2H");
    res.fallback_count = static_cast<long long>(f);
  } catch (const gpfb::Error& e) {
    rethrow(e);
  }
  return res;
}

}  // namespace gpfilter
