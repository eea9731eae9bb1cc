// C++ entry point (include/gpfilter/gpfilter.hpp): gpfilter::gpf over the
// drop-in engine (dropin.cpp), with the reference's validation order and
// exceptions (proj/src/core/bilateral.cpp:64-106, 150-158; spatial.cpp:25-35,
// 220-230; range_kernel.cpp:22-29; image.cpp:11-18).
#include <algorithm>
#include <cmath>
#include <string>
#include <utility>

#include <cuda_runtime.h>

#include "gpf_internal.h"
#include "gpfilter/gpfilter.h"
#include "gpfilter/gpfilter.hpp"
#include "pgm.h"

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

// ------------------------------------- the other entry points, over the C ABI
namespace {

// a gpf_image handle holding a copy of `img` (or an output of the C ABI)
struct Handle {
  gpf_image* h = nullptr;
  Handle() = default;
  explicit Handle(const Image& img) {
    if (img.pixels() == 0) throw std::invalid_argument("Image dimensions must be >= 1");
    if (gpf_image_create(img.width(), img.height(), &h) != GPF_OK) throw std::runtime_error(gpf_last_error());
    std::copy(img.data(), img.data() + img.pixels(), gpf_image_data(h));
  }
  ~Handle() { gpf_image_destroy(h); }
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  Image take() const {
    Image out(gpf_image_width(h), gpf_image_height(h));
    std::copy(gpf_image_cdata(h), gpf_image_cdata(h) + out.pixels(), out.data());
    return out;
  }
};

// status -> the exception the reference core throws for it
void raise(gpf_status st) {
  if (st == GPF_OK) return;
  const std::string msg = gpf_last_error();
  if (st == GPF_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (st == GPF_ERR_SIGMA_TOO_SMALL) throw SigmaTooSmallError(msg);
  throw std::runtime_error(msg);
}

gpf_spatial_params c_spatial(const SpatialParams& sp) {
  sp.validate();  // window_radius >= 1 here: the C struct's "<= 0 selects the default" never applies
  gpf_spatial_params c;
  c.sigma_s = sp.sigma_s;
  c.window_radius = sp.window_radius;
  c.boundary = static_cast<gpf_boundary>(static_cast<int>(sp.boundary));
  c.kernel_scale = sp.kernel_scale;
  return c;
}

gpf_range_params c_range(const RangeParams& rp) {
  rp.validate();
  return gpf_range_params{rp.sigma_r, rp.degree};
}

}  // namespace

Image exact_bilateral(const Image& img, const SpatialParams& sp, const RangeParams& rp) {
  const gpf_spatial_params csp = c_spatial(sp);
  const gpf_range_params crp = c_range(rp);
  Handle in(img), out;
  raise(gpf_filter_exact(in.h, &csp, &crp, &out.h));
  return out.take();
}

FilterResult taylor_bilateral(const Image& img, const SpatialParams& sp, const RangeParams& rp,
                              SpatialBackend backend) {
  const gpf_spatial_params csp = c_spatial(sp);
  const gpf_range_params crp = c_range(rp);
  Handle in(img), out;
  FilterResult res;
  raise(gpf_filter_taylor(in.h, &csp, &crp,
                          backend == SpatialBackend::direct ? GPF_BACKEND_DIRECT : GPF_BACKEND_RECURSIVE,
                          &res.fallback_count, &out.h));
  res.image = out.take();
  return res;
}

Image direct_gaussian(const Image& img, const SpatialParams& p) {
  const gpf_spatial_params csp = c_spatial(p);
  Handle in(img), out;
  raise(gpf_gaussian_direct(in.h, &csp, &out.h));
  return out.take();
}

Image recursive_gaussian(const Image& img, double sigma_s, double kernel_scale) {
  if (!(sigma_s > 0.0) || !(kernel_scale > 0.0))
    throw std::invalid_argument("recursive_gaussian: sigma_s and kernel_scale must be > 0");
  if (sigma_s < 0.5)
    throw SigmaTooSmallError(
        "recursive_gaussian: sigma_s < 0.5 is not supported; use the direct backend");
  Handle in(img), out;
  raise(gpf_gaussian_recursive(in.h, sigma_s, kernel_scale, &out.h));
  return out.take();
}

double kernel_mass_1d(double sigma_s, int window_radius) { return gpfb::kernel_mass_1d(sigma_s, window_radius); }

int boundary_index(int i, int n, Boundary boundary) {
  if (i >= 0 && i < n) return i;
  if (boundary == Boundary::replicate) return i < 0 ? 0 : n - 1;
  if (boundary == Boundary::zero) return -1;
  const long long period = 2LL * n;  // half-sample symmetric: -1 -> 0, n -> n - 1
  long long m = i % period;
  if (m < 0) m += period;
  return static_cast<int>(m < n ? m : period - 1 - m);
}

double spatial_weight(int j_row, int j_col, double sigma_s) {
  const double r2 = static_cast<double>(j_row) * j_row + static_cast<double>(j_col) * j_col;
  return std::exp(-r2 / (2.0 * sigma_s * sigma_s));
}

void set_num_threads(int n) { gpf_set_num_threads(std::max(1, n)); }
int num_threads() { return gpf_get_num_threads(); }

Image shift(const Image& img, double c) {
  Image out = img;
  for (std::size_t i = 0; i < out.pixels(); ++i) out.data()[i] -= c;
  return out;
}

double max_abs_diff(const Image& a, const Image& b) {
  if (!a.same_size(b)) throw std::invalid_argument("max_abs_diff: image dimensions differ");
  double worst = 0.0;
  for (std::size_t i = 0; i < a.pixels(); ++i) worst = std::fmax(worst, std::fabs(a.data()[i] - b.data()[i]));
  return worst;
}

double mse_db(double mse) {
  if (mse < 0.0) throw std::invalid_argument("mse_db: mse must be non-negative");
  return mse == 0.0 ? kMseDbFloor : std::fmax(10.0 * std::log10(mse), kMseDbFloor);
}

ErrorReport compare(const Image& ref, const Image& test, int exclude_border) {
  if (!ref.same_size(test)) throw std::invalid_argument("compare: images differ in size");
  Handle a(ref), b(test);
  gpf_error_report r;
  raise(gpf_compare(a.h, b.h, exclude_border, &r));
  return ErrorReport{r.mse, r.mse_db, r.max_abs, r.pixels};
}

namespace {
template <class F>
double scalar(F&& f) {
  try {
    return f();
  } catch (const gpfb::Error& e) {
    throw std::invalid_argument(e.msg);
  }
}
}  // namespace

double gaussian_range(double t, double tau, const RangeParams& p) {
  p.validate();
  return scalar([&] { return gpfb::kernel_gauss(t, tau, p.sigma_r); });
}
double gauss_polynomial(double t, double tau, const RangeParams& p) {
  return scalar([&] { return gpfb::kernel_gauss_poly(t, tau, p.sigma_r, p.degree); });
}
double taylor_polynomial(double t, double tau, const RangeParams& p) {
  return scalar([&] { return gpfb::kernel_taylor(t, tau, p.sigma_r, p.degree); });
}
double sup_error(const RangeParams& p, double tau, const IntensityRange& range, double step,
                 RangeApprox which) {
  return scalar([&] {
    return gpfb::kernel_sup_error(p.sigma_r, p.degree, tau, range.low, range.high, step,
                                  which == RangeApprox::taylor);
  });
}

// ----------------------------------------------------------------- PGM codec
const char* pgm_error_kind_name(PgmErrorKind kind) {
  static const char* const names[] = {"bad_magic", "bad_dims", "bad_maxval", "truncated", "bad_pixel"};
  const int k = static_cast<int>(kind);
  return k >= 0 && k < 5 ? names[k] : "unknown";
}

PgmParseError::PgmParseError(PgmErrorKind kind, std::size_t offset, const std::string& detail)
    : std::runtime_error(std::string("PGM parse error (") + pgm_error_kind_name(kind) + ") at byte " +
                         std::to_string(offset) + ": " + detail),
      kind_(kind),
      offset_(offset) {}

namespace {
// the codec (pgm.cpp) reports "PGM parse error (<kind>) at byte <offset>: <detail>" with a
// GPF_ERR_PGM_* status: back to the typed exception
[[noreturn]] void rethrow_pgm(const gpfb::Error& e) {
  if (e.status >= GPF_ERR_PGM_BAD_MAGIC && e.status <= GPF_ERR_PGM_BAD_PIXEL) {
    const std::string key = ") at byte ";
    const std::size_t at = e.msg.find(key);
    std::size_t offset = 0;
    std::string detail = e.msg;
    if (at != std::string::npos) {
      const std::size_t colon = e.msg.find(": ", at);
      offset = static_cast<std::size_t>(std::stoull(e.msg.substr(at + key.size())));
      detail = colon == std::string::npos ? "" : e.msg.substr(colon + 2);
    }
    throw PgmParseError(static_cast<PgmErrorKind>(e.status - GPF_ERR_PGM_BAD_MAGIC), offset, detail);
  }
  throw std::runtime_error(e.msg);
}
}  // namespace

Image decode_pgm(const std::uint8_t* bytes, std::size_t size) {
  try {
    gpfb::pgm::Decoded d = gpfb::pgm::decode(bytes, size);
    Image img(d.w, d.h);
    std::copy(d.pixels.begin(), d.pixels.end(), img.data());
    return img;
  } catch (const gpfb::Error& e) {
    rethrow_pgm(e);
  }
}

std::vector<std::uint8_t> encode_pgm(const Image& img) {
  return gpfb::pgm::encode(img.data(), img.width(), img.height());
}

std::uint8_t quantize_sample(double v) { return gpfb::pgm::quantize(v); }

Image read_pgm(const std::string& path) {
  try {
    const std::vector<std::uint8_t> bytes = gpfb::pgm::read_file(path.c_str());
    return decode_pgm(bytes.data(), bytes.size());
  } catch (const gpfb::Error& e) {
    rethrow_pgm(e);
  }
}

void write_pgm(const Image& img, const std::string& path) {
  try {
    gpfb::pgm::write_file(path.c_str(), encode_pgm(img));
  } catch (const gpfb::Error& e) {
    rethrow_pgm(e);
  }
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
  // the state images are public: a caller may have replaced one
  for (const Image* im : {&G, &Fbar, &P, &Q, &H})
    if (!im->same_size(F) || F.pixels() == 0)
      throw std::invalid_argument("GpfState::step: state images differ in size");
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

// mean_intensity (image.cpp:20-37): the deterministic double-double mean of the
// GPF path (K0), equal to the reference's compensated sum whenever that is
// correctly rounded
double mean_intensity(const Image& img) {
  if (img.pixels() == 0) throw std::invalid_argument("Image dimensions must be >= 1");
  require_device();
  double t_c = 0.0;
  try {
    Dev in(img.pixels(), img.data()), scal(2 + 4 * (size_t)gpfb::kF64MeanBlocks);
    gpfb::launch_mean_f64(in.p, (long long)img.pixels(), 1, 0.0, 1.0, scal.p + 2, gpfb::kF64MeanBlocks,
                          scal.p, nullptr);
    cu(cudaMemcpy(&t_c, scal.p, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  } catch (const gpfb::Error& e) {
    rethrow(e);
  }
  return t_c;
}

}  // namespace gpfilter
