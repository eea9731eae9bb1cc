// C ABI of libgpfilter_b200 (include/gpfilter/gpfilter.h, gpfilter_b200.h).
//
// Mirrors the reference's proj/src/capi.cpp for the GPF path: same validation
// order and messages (to_spatial 65-80, to_backend 82-88, SpatialParams /
// RangeParams validate, spatial.cpp:25-35 / range_kernel.cpp:22-29,
// recursive_gaussian's SigmaTooSmallError, spatial.cpp:222-230), thread-local
// last error (capi.cpp:28-33), *out = NULL before work, fallback_count written
// only on success. There is no CPU compute path: every filter call runs the
// sm_100a kernels, and a missing device is an error.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <atomic>
#include <map>
#include <memory>
#include <list>
#include <cstdlib>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "gpf_internal.h"
#include "gpfilter/gpfilter.h"
#include "pgm.h"
#include "gpfilter/gpfilter_b200.h"

// Image storage. Frames of 4 MiB and more live in page-locked host memory
// (cudaMallocHost, recycled through a small pool) so that the drop-in entry's
// copies run at full PCIe speed instead of through the driver's pageable
// staging; smaller ones (and any image on a machine without a CUDA device) use
// ordinary heap memory. The layout the caller sees is the reference's:
// row-major doubles (proj/src/core/image.hpp:14-41).
namespace {
constexpr size_t kPinnedMinBytes = size_t(4) << 20;
constexpr size_t kPinnedPoolBytes = size_t(8) << 30;

struct HostPool {
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks;  // bytes -> block
  size_t pooled = 0;
};
HostPool& host_pool() {
  static HostPool* p = new HostPool();  // never destroyed: blocks may outlive static teardown
  return *p;
}

double* host_alloc(size_t n, bool& pinned) {
  const size_t bytes = std::max<size_t>(n, 1) * sizeof(double);
  pinned = false;
  if (bytes >= kPinnedMinBytes) {
    HostPool& hp = host_pool();
    {
      std::lock_guard<std::mutex> lock(hp.mu);
      auto it = hp.free_blocks.lower_bound(bytes);
      if (it != hp.free_blocks.end() && it->first <= 2 * bytes) {
        void* b = it->second;
        hp.pooled -= it->first;
        hp.free_blocks.erase(it);
        pinned = true;
        // remember the block's real size in front of the data
        return static_cast<double*>(b) + 1;
      }
    }
    void* b = nullptr;
    if (cudaMallocHost(&b, bytes + sizeof(double)) == cudaSuccess) {
      *static_cast<size_t*>(b) = bytes;
      pinned = true;
      return static_cast<double*>(b) + 1;
    }
    cudaGetLastError();  // no device / pinned memory exhausted: pageable storage
  }
  auto* d = static_cast<double*>(std::malloc(bytes));
  if (!d) throw std::bad_alloc();
  return d;
}

void host_free(double* d, bool pinned) {
  if (!d) return;
  if (!pinned) {
    std::free(d);
    return;
  }
  void* b = d - 1;
  const size_t bytes = *static_cast<size_t*>(b);
  HostPool& hp = host_pool();
  {
    std::lock_guard<std::mutex> lock(hp.mu);
    if (hp.pooled + bytes <= kPinnedPoolBytes) {
      hp.free_blocks.emplace(bytes, b);
      hp.pooled += bytes;
      return;
    }
  }
  cudaFreeHost(b);
}
}  // namespace

struct gpf_image {
  int w = 0, h = 0;
  double* px = nullptr;
  bool pinned = false;
  gpf_image(int w_, int h_) : w(w_), h(h_) { px = host_alloc((size_t)w * h, pinned); }
  ~gpf_image() { host_free(px, pinned); }
  gpf_image(const gpf_image&) = delete;
  gpf_image& operator=(const gpf_image&) = delete;
  size_t n() const { return (size_t)w * h; }
};

struct gpf_b200_plan {
  gpfb::Plan plan;
  unsigned long long* d_fb = nullptr;  // per-frame counters (grown on demand)
  int d_fb_cap = 0;
  // Host-entry pipeline: two staging slots; compute on the plan's stream (or
  // the caller's), H2D / D2H on the device's shared copy streams, so frame f+1
  // uploads while f computes and f-1 downloads.
  float* d_stage_in[2] = {nullptr, nullptr};
  float* d_stage_out[2] = {nullptr, nullptr};
  cudaStream_t s_comp = nullptr;
  cudaEvent_t in_ready[2] = {}, computed[2] = {}, out_free[2] = {};
  unsigned long long* h_fb = nullptr;  // pinned readback of the counters
  int h_fb_cap = 0;
};

namespace {

thread_local std::string g_last_error;
void batch_release();  // cached plans of gpf_b200_filter_batch (defined with it)
std::atomic<int> g_threads{1};

gpf_status fail(gpf_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear a non-sticky error (e.g. a failed allocation) for the caller
    throw gpfb::Error{GPF_ERR_UNKNOWN, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

template <typename Fn>
gpf_status guarded(Fn&& fn) {
  try {
    fn();
    return GPF_OK;
  } catch (const gpfb::Error& e) {
    return fail(static_cast<gpf_status>(e.status), e.msg);
  } catch (const std::bad_alloc&) {
    return fail(GPF_ERR_UNKNOWN, "std::bad_alloc");
  } catch (const std::exception& e) {
    return fail(GPF_ERR_UNKNOWN, e.what());
  }
}

[[noreturn]] void invalid(const std::string& m) { throw gpfb::Error{GPF_ERR_INVALID_ARGUMENT, m}; }

// Validation of the GPF path, in the reference's order.
gpfb::Params validate(int w, int h, const gpf_spatial_params& sp, const gpf_range_params& rp,
                      gpf_backend backend, int centering, int max_degree) {
  // to_spatial (capi.cpp:65-80): boundary enum checked even though unused.
  if (sp.boundary != GPF_BOUNDARY_REPLICATE && sp.boundary != GPF_BOUNDARY_REFLECT &&
      sp.boundary != GPF_BOUNDARY_ZERO)
    invalid("boundary must be replicate, reflect, or zero");
  // to_backend (capi.cpp:82-88)
  if (backend != GPF_BACKEND_DIRECT && backend != GPF_BACKEND_RECURSIVE)
    invalid("backend must be direct or recursive");
  // SpatialParams::validate (spatial.cpp:25-35)
  const int radius = sp.window_radius > 0 ? sp.window_radius : gpfb::default_window_radius(sp.sigma_s);
  if (!(sp.sigma_s > 0.0)) invalid("SpatialParams: sigma_s must be > 0");
  if (radius < 1) invalid("SpatialParams: window_radius must be >= 1");
  if (!(sp.kernel_scale > 0.0)) invalid("SpatialParams: kernel_scale must be > 0");
  // RangeParams::validate (range_kernel.cpp:22-29)
  if (!(rp.sigma_r > 0.0)) invalid("RangeParams: sigma_r must be > 0");
  if (rp.degree < 0) invalid("RangeParams: degree must be >= 0");
  // recursive_gaussian (spatial.cpp:222-230); the direct backend takes any sigma_s > 0
  if (backend == GPF_BACKEND_RECURSIVE && sp.sigma_s < 0.5)
    throw gpfb::Error{GPF_ERR_SIGMA_TOO_SMALL,
                      "recursive_gaussian: sigma_s < 0.5 is not supported; use the direct backend"};
  if (rp.degree > max_degree)
    invalid("RangeParams: degree must be <= " + std::to_string(max_degree) +
            (max_degree == gpfb::kMaxDegreeF64 ? " in the B200 library"
                                               : " for the fp32 plan entries of the B200 library"));
  if (w < 1 || h < 1) invalid("Image dimensions must be >= 1");
  gpfb::Params p;
  p.width = w;
  p.height = h;
  p.sigma_s = sp.sigma_s;
  p.kernel_scale = sp.kernel_scale;
  p.sigma_r = rp.sigma_r;
  p.degree = rp.degree;
  p.centering = centering != 0 ? 1 : 0;
  p.backend = backend == GPF_BACKEND_DIRECT ? 0 : 1;
  p.window_radius = radius;
  p.boundary = static_cast<int>(sp.boundary);
  return p;
}

// Validation of the exact filter (to_spatial / to_range, SpatialParams and
// RangeParams::validate): returns the window radius.
int validate_exact(const gpf_spatial_params& sp, const gpf_range_params& rp) {
  if (sp.boundary != GPF_BOUNDARY_REPLICATE && sp.boundary != GPF_BOUNDARY_REFLECT &&
      sp.boundary != GPF_BOUNDARY_ZERO)
    invalid("boundary must be replicate, reflect, or zero");
  const int radius = sp.window_radius > 0 ? sp.window_radius : gpfb::default_window_radius(sp.sigma_s);
  if (!(sp.sigma_s > 0.0)) invalid("SpatialParams: sigma_s must be > 0");
  if (radius < 1) invalid("SpatialParams: window_radius must be >= 1");
  if (!(sp.kernel_scale > 0.0)) invalid("SpatialParams: kernel_scale must be > 0");
  if (!(rp.sigma_r > 0.0)) invalid("RangeParams: sigma_r must be > 0");
  if (rp.degree < 0) invalid("RangeParams: degree must be >= 0");
  return radius;
}

void fill_report(const gpfb::ErrorStats& st, gpf_error_report* out) {
  out->mse = st.mse;
  out->mse_db = st.mse == 0.0 ? -400.0 : std::max(10.0 * std::log10(st.mse), -400.0);  // metrics.cpp:12-18
  out->max_abs = st.max_abs;
  out->pixels = st.pixels;
}

void check_compare_dims(int w, int h, int border) {  // metrics.cpp:20-33
  if (border < 0) invalid("compare: exclude_border must be >= 0");
  if (2 * border >= w || 2 * border >= h) invalid("compare: exclude_border leaves no interior pixels");
}

int current_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw gpfb::Error{GPF_ERR_UNKNOWN, "no CUDA device available (the B200 library has no CPU path)"};
  }
  int d = 0;
  cuda_check(cudaGetDevice(&d), "cudaGetDevice");
  return d;
}

// RAII device buffer
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t n) { cuda_check(cudaMalloc(&p, n), "cudaMalloc"); }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

struct PlanGuard {
  gpfb::Plan plan;
  bool live = false;
  ~PlanGuard() {
    if (live) gpfb::plan_free(plan);
  }
};

// Host<->device copy streams shared by every plan on a device. One FIFO per
// direction means concurrent host-entry calls (several plans, several host
// threads) upload one frame at a time at full link speed instead of sharing
// the link and then all computing / downloading at once; the calls then
// stagger and the frames' copies overlap each other's compute. Never freed
// (they live as long as the process's CUDA context).
struct CopyStreams {
  cudaStream_t h2d = nullptr, d2h = nullptr;
};

CopyStreams copy_streams(int device) {
  static std::mutex mu;
  static std::vector<CopyStreams> per_dev;
  std::lock_guard<std::mutex> lock(mu);
  if ((int)per_dev.size() <= device) per_dev.resize(device + 1);
  CopyStreams& cs = per_dev[device];
  if (!cs.h2d) {
    cuda_check(cudaStreamCreateWithFlags(&cs.h2d, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaStreamCreateWithFlags(&cs.d2h, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  return cs;
}

}  // namespace

extern "C" {

const char* gpf_status_name(gpf_status status) {
  switch (status) {
    case GPF_OK: return "GPF_OK";
    case GPF_ERR_INVALID_ARGUMENT: return "GPF_ERR_INVALID_ARGUMENT";
    case GPF_ERR_IO: return "GPF_ERR_IO";
    case GPF_ERR_SIGMA_TOO_SMALL: return "GPF_ERR_SIGMA_TOO_SMALL";
    case GPF_ERR_PGM_BAD_MAGIC: return "GPF_ERR_PGM_BAD_MAGIC";
    case GPF_ERR_PGM_BAD_DIMS: return "GPF_ERR_PGM_BAD_DIMS";
    case GPF_ERR_PGM_BAD_MAXVAL: return "GPF_ERR_PGM_BAD_MAXVAL";
    case GPF_ERR_PGM_TRUNCATED: return "GPF_ERR_PGM_TRUNCATED";
    case GPF_ERR_PGM_BAD_PIXEL: return "GPF_ERR_PGM_BAD_PIXEL";
    case GPF_ERR_UNKNOWN: return "GPF_ERR_UNKNOWN";
  }
  return "GPF_ERR_UNKNOWN";
}

const char* gpf_last_error(void) { return g_last_error.c_str(); }

// the ABI version implemented (the reference pins "1.0.0", proj/tests/test_capi.cpp:37)
const char* gpf_version(void) { return "1.0.0"; }

gpf_status gpf_image_create(int width, int height, gpf_image** out) {
  if (out == nullptr) return fail(GPF_ERR_INVALID_ARGUMENT, "out is null");
  *out = nullptr;
  if (width < 1 || height < 1) return fail(GPF_ERR_INVALID_ARGUMENT, "Image dimensions must be >= 1");
  return guarded([&] {
    auto* img = new gpf_image(width, height);
    std::memset(img->px, 0, img->n() * sizeof(double));
    *out = img;
  });
}

void gpf_image_destroy(gpf_image* img) { delete img; }
int gpf_image_width(const gpf_image* img) { return img ? img->w : 0; }
int gpf_image_height(const gpf_image* img) { return img ? img->h : 0; }
double* gpf_image_data(gpf_image* img) { return img ? img->px : nullptr; }
const double* gpf_image_cdata(const gpf_image* img) { return img ? img->px : nullptr; }

void gpf_spatial_params_init(gpf_spatial_params* sp) {
  if (!sp) return;
  sp->sigma_s = 2.0;
  sp->window_radius = 0;
  sp->boundary = GPF_BOUNDARY_REPLICATE;
  sp->kernel_scale = 1.0;
}

void gpf_range_params_init(gpf_range_params* rp) {
  if (!rp) return;
  rp->sigma_r = 30.0;
  rp->degree = 20;
}

gpf_status gpf_filter_gpf(const gpf_image* in, const gpf_spatial_params* sp,
                          const gpf_range_params* rp, gpf_backend backend, int centering,
                          long long* fallback_count, gpf_image** out) {
  if (in == nullptr || sp == nullptr || rp == nullptr || out == nullptr)
    return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    const gpfb::Params p = validate(in->w, in->h, *sp, *rp, backend, centering, gpfb::kMaxDegreeF64);
    auto* res = new gpf_image(p.width, p.height);
    std::unique_ptr<gpf_image> hold(res);
    const long long fb = gpfb::dropin_gpf(in->px, res->px, p);
    if (fallback_count != nullptr) *fallback_count = fb;
    *out = hold.release();
  });
}
gpf_status gpf_gaussian_direct(const gpf_image* in, const gpf_spatial_params* sp, gpf_image** out) {
  if (in == nullptr || sp == nullptr || out == nullptr)
    return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    // to_spatial (capi.cpp:65-80), SpatialParams::validate (spatial.cpp:25-35)
    if (sp->boundary != GPF_BOUNDARY_REPLICATE && sp->boundary != GPF_BOUNDARY_REFLECT &&
        sp->boundary != GPF_BOUNDARY_ZERO)
      invalid("boundary must be replicate, reflect, or zero");
    const int radius =
        sp->window_radius > 0 ? sp->window_radius : gpfb::default_window_radius(sp->sigma_s);
    if (!(sp->sigma_s > 0.0)) invalid("SpatialParams: sigma_s must be > 0");
    if (radius < 1) invalid("SpatialParams: window_radius must be >= 1");
    if (!(sp->kernel_scale > 0.0)) invalid("SpatialParams: kernel_scale must be > 0");
    current_device();
    const size_t n = (size_t)in->w * in->h;
    DevBuf din(n * sizeof(double)), dtmp(n * sizeof(double));
    cuda_check(cudaMemcpy(din.p, in->px, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    gpfb::run_direct_gaussian_f64(static_cast<const double*>(din.p), static_cast<double*>(din.p),
                                  static_cast<double*>(dtmp.p), in->w, in->h, 1, sp->sigma_s,
                                  sp->kernel_scale, radius, static_cast<int>(sp->boundary), nullptr);
    auto* res = new gpf_image(in->w, in->h);
    std::unique_ptr<gpf_image> hold(res);
    cuda_check(cudaMemcpy(res->px, din.p, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    *out = hold.release();
  });
}

gpf_status gpf_gaussian_recursive(const gpf_image* in, double sigma_s, double kernel_scale,
                                  gpf_image** out) {
  if (in == nullptr || out == nullptr) return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    // spatial.cpp:222-230
    if (!(sigma_s > 0.0) || !(kernel_scale > 0.0))
      invalid("recursive_gaussian: sigma_s and kernel_scale must be > 0");
    if (sigma_s < 0.5)
      throw gpfb::Error{GPF_ERR_SIGMA_TOO_SMALL,
                        "recursive_gaussian: sigma_s < 0.5 is not supported; use the direct backend"};
    current_device();
    const size_t n = (size_t)in->w * in->h;
    DevBuf din(n * sizeof(double)), dout(n * sizeof(double)), dtmp(n * sizeof(double));
    cuda_check(cudaMemcpy(din.p, in->px, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    const double mass = gpfb::kernel_mass_1d(sigma_s, gpfb::default_window_radius(sigma_s));
    gpfb::run_gaussian_f64(static_cast<const double*>(din.p), static_cast<double*>(dout.p),
                           static_cast<double*>(dtmp.p), in->w, in->h, sigma_s,
                           mass * mass * kernel_scale, nullptr);
    auto* res = new gpf_image(in->w, in->h);
    std::unique_ptr<gpf_image> hold(res);
    cuda_check(cudaMemcpy(res->px, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    *out = hold.release();
  });
}

gpf_status gpf_filter_taylor(const gpf_image* in, const gpf_spatial_params* sp,
                             const gpf_range_params* rp, gpf_backend backend,
                             long long* fallback_count, gpf_image** out) {
  if (in == nullptr || sp == nullptr || rp == nullptr || out == nullptr)
    return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    const gpfb::Params p = validate(in->w, in->h, *sp, *rp, backend, 0, 1 << 20);
    current_device();
    const size_t n = (size_t)in->w * in->h;
    DevBuf din(n * sizeof(double)), dout(n * sizeof(double)), dfb(sizeof(unsigned long long));
    cuda_check(cudaMemcpy(din.p, in->px, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    gpfb::run_taylor_f64(static_cast<const double*>(din.p), static_cast<double*>(dout.p), p,
                         static_cast<unsigned long long*>(dfb.p), nullptr);
    auto* res = new gpf_image(in->w, in->h);
    std::unique_ptr<gpf_image> hold(res);
    unsigned long long fb = 0;
    cuda_check(cudaMemcpy(res->px, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(&fb, dfb.p, sizeof(fb), cudaMemcpyDeviceToHost), "D2H");
    if (fallback_count) *fallback_count = static_cast<long long>(fb);
    *out = hold.release();
  });
}

gpf_status gpf_filter_exact(const gpf_image* in, const gpf_spatial_params* sp,
                            const gpf_range_params* rp, gpf_image** out) {
  if (in == nullptr || sp == nullptr || rp == nullptr || out == nullptr)
    return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    const int W = validate_exact(*sp, *rp);
    current_device();
    const size_t n = (size_t)in->w * in->h;
    DevBuf din(n * sizeof(double)), dout(n * sizeof(double));
    cuda_check(cudaMemcpy(din.p, in->px, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    gpfb::run_exact_f64(static_cast<const double*>(din.p), static_cast<double*>(dout.p), in->w, in->h,
                        1, W, static_cast<int>(sp->boundary), sp->sigma_s, rp->sigma_r,
                        sp->kernel_scale, nullptr);
    auto* res = new gpf_image(in->w, in->h);
    std::unique_ptr<gpf_image> hold(res);
    cuda_check(cudaMemcpy(res->px, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    *out = hold.release();
  });
}

// y[i] = the fp64 mode's correctly rounded exp(x[i]) evaluated on the device (host
// buffers); exists so that the device instantiation can be compared with the host one
gpf_status gpf_b200_exp_cr(const double* x, double* y, long long n) {
  if (x == nullptr || y == nullptr || n < 0) return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    current_device();
    if (n == 0) return;
    DevBuf dx(n * sizeof(double)), dy(n * sizeof(double));
    cuda_check(cudaMemcpy(dx.p, x, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    gpfb::run_exp_cr_f64(static_cast<const double*>(dx.p), static_cast<double*>(dy.p), n, nullptr);
    cuda_check(cudaMemcpy(y, dy.p, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  });
}

// ------------------------------------------------- range-kernel evaluators
gpf_status gpf_kernel_gauss(double t, double tau, double sigma_r, double* out) {
  if (out == nullptr) return fail(GPF_ERR_INVALID_ARGUMENT, "out is null");
  return guarded([&] { *out = gpfb::kernel_gauss(t, tau, sigma_r); });
}

gpf_status gpf_kernel_gauss_poly(double t, double tau, double sigma_r, int degree, double* out) {
  if (out == nullptr) return fail(GPF_ERR_INVALID_ARGUMENT, "out is null");
  return guarded([&] { *out = gpfb::kernel_gauss_poly(t, tau, sigma_r, degree); });
}

gpf_status gpf_kernel_taylor(double t, double tau, double sigma_r, int degree, double* out) {
  if (out == nullptr) return fail(GPF_ERR_INVALID_ARGUMENT, "out is null");
  return guarded([&] { *out = gpfb::kernel_taylor(t, tau, sigma_r, degree); });
}

gpf_status gpf_kernel_sup_error(double sigma_r, int degree, double tau, double low, double high,
                                double step, gpf_range_approx which, double* out) {
  if (out == nullptr) return fail(GPF_ERR_INVALID_ARGUMENT, "out is null");
  return guarded([&] {
    if (which != GPF_RANGE_APPROX_GAUSS_POLY && which != GPF_RANGE_APPROX_TAYLOR)
      invalid("which must be gauss_poly or taylor");
    *out = gpfb::kernel_sup_error(sigma_r, degree, tau, low, high, step,
                                  which == GPF_RANGE_APPROX_TAYLOR);
  });
}

gpf_status gpf_compare(const gpf_image* ref, const gpf_image* test, int exclude_border,
                       gpf_error_report* out) {
  if (ref == nullptr || test == nullptr || out == nullptr)
    return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    if (ref->w != test->w || ref->h != test->h) invalid("compare: images differ in size");
    check_compare_dims(ref->w, ref->h, exclude_border);
    current_device();
    const size_t n = (size_t)ref->w * ref->h;
    DevBuf da(n * sizeof(double)), db(n * sizeof(double));
    cuda_check(cudaMemcpy(da.p, ref->px, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(db.p, test->px, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    fill_report(gpfb::compare_f64(static_cast<const double*>(da.p), static_cast<const double*>(db.p),
                                  ref->w, ref->h, exclude_border, nullptr),
                out);
  });
}

// ----------------------------------------------------------------- PGM I/O
namespace {
void deliver_pgm(gpfb::pgm::Decoded&& d, gpf_image** out) {
  auto* img = new gpf_image(d.w, d.h);
  std::memcpy(img->px, d.pixels.data(), img->n() * sizeof(double));
  *out = img;
}
}  // namespace

gpf_status gpf_read_pgm(const char* path, gpf_image** out) {
  if (path == nullptr || out == nullptr) return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    const std::vector<uint8_t> bytes = gpfb::pgm::read_file(path);
    deliver_pgm(gpfb::pgm::decode(bytes.data(), bytes.size()), out);
  });
}

gpf_status gpf_decode_pgm(const uint8_t* bytes, size_t size, gpf_image** out) {
  if (bytes == nullptr || out == nullptr) return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] { deliver_pgm(gpfb::pgm::decode(bytes, size), out); });
}

gpf_status gpf_write_pgm(const gpf_image* img, const char* path) {
  if (img == nullptr || path == nullptr) return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] { gpfb::pgm::write_file(path, gpfb::pgm::encode(img->px, img->w, img->h)); });
}

gpf_status gpf_encode_pgm(const gpf_image* img, uint8_t** bytes, size_t* size) {
  if (img == nullptr || bytes == nullptr || size == nullptr)
    return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  *bytes = nullptr;
  *size = 0;
  return guarded([&] {
    const std::vector<uint8_t> buf = gpfb::pgm::encode(img->px, img->w, img->h);
    auto* mem = new uint8_t[buf.size()];
    std::memcpy(mem, buf.data(), buf.size());
    *bytes = mem;
    *size = buf.size();
  });
}

void gpf_free_bytes(uint8_t* bytes) { delete[] bytes; }

gpf_status gpf_b200_set_precision(int mode) {
  if (mode != GPF_B200_PRECISION_AUTO && mode != GPF_B200_PRECISION_FP32 &&
      mode != GPF_B200_PRECISION_FP64)
    return fail(GPF_ERR_INVALID_ARGUMENT, "precision must be AUTO, FP32 or FP64");
  gpfb::set_precision(mode);
  return GPF_OK;
}

int gpf_b200_get_precision(void) { return gpfb::get_precision(); }
int gpf_b200_last_precision(void) { return gpfb::last_precision(); }
double gpf_b200_last_max_abs_h(void) { return gpfb::last_max_abs_h(); }
float gpf_b200_last_device_ms(void) { return gpfb::last_device_ms(); }
double gpf_b200_fp32_h_limit(void) { return gpfb::kH32Limit; }
double gpf_b200_fp32_h_limit_degree(int degree) { return gpfb::fp32_h_limit(degree); }
void gpf_b200_dropin_release(void) {
  batch_release();
  gpfb::dropin_release();
}

gpf_status gpf_set_num_threads(int n) {
  if (n < 1) return fail(GPF_ERR_INVALID_ARGUMENT, "thread count must be >= 1");
  g_threads.store(n);
  return GPF_OK;
}

int gpf_get_num_threads(void) { return g_threads.load(); }

// ---------------------------------------------------------------- B200 plans
gpf_status gpf_b200_plan_create(int width, int height, const gpf_spatial_params* sp,
                                const gpf_range_params* rp, int centering, int device,
                                gpf_b200_plan** out) {
  if (sp == nullptr || rp == nullptr || out == nullptr)
    return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded([&] {
    const gpfb::Params p =
        validate(width, height, *sp, *rp, GPF_BACKEND_RECURSIVE, centering, gpfb::kMaxDegreeF32);
    const int prev = current_device();
    const int dev = device >= 0 ? device : prev;
    struct Restore {  // the caller's current device is left as it was
      int d;
      ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    auto* pl = new gpf_b200_plan();
    std::unique_ptr<gpf_b200_plan> hold(pl);
    gpfb::plan_init(pl->plan, p, dev);
    *out = hold.release();
  });
}

void gpf_b200_plan_destroy(gpf_b200_plan* plan) {
  if (!plan) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(plan->plan.device);
  gpfb::stage_reset(plan->plan);
  gpfb::plan_free(plan->plan);
  cudaFree(plan->d_fb);
  for (int s = 0; s < 2; ++s) {
    cudaFree(plan->d_stage_in[s]);
    cudaFree(plan->d_stage_out[s]);
    if (plan->in_ready[s]) cudaEventDestroy(plan->in_ready[s]);
    if (plan->computed[s]) cudaEventDestroy(plan->computed[s]);
    if (plan->out_free[s]) cudaEventDestroy(plan->out_free[s]);
  }
  if (plan->s_comp) cudaStreamDestroy(plan->s_comp);
  cudaFreeHost(plan->h_fb);
  cudaSetDevice(prev);
  delete plan;
}

gpf_status gpf_b200_plan_set_batch(gpf_b200_plan* plan, int frames) {
  if (plan == nullptr) return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  if (frames < 1) return fail(GPF_ERR_INVALID_ARGUMENT, "frames must be >= 1");
  return guarded([&] {
    int prev = 0;
    cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
    struct Restore {
      int d;
      ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    cuda_check(cudaSetDevice(plan->plan.device), "cudaSetDevice");
    cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    // Build the new workspace first; the plan keeps its old one (and stays
    // usable) if that fails, e.g. when the batch does not fit in HBM.
    gpfb::Plan fresh;
    gpfb::plan_init(fresh, plan->plan.p, plan->plan.device, frames);
    fresh.profile = plan->plan.profile;
    fresh.timer = plan->plan.timer;
    plan->plan.timer = nullptr;
    gpfb::plan_free(plan->plan);
    plan->plan = fresh;
  });
}

gpf_status gpf_b200_plan_set_profiling(gpf_b200_plan* plan, int enable) {
  if (plan == nullptr) return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    gpfb::stage_reset(plan->plan);
    plan->plan.profile = enable != 0;
  });
}

int gpf_b200_plan_stage_times(gpf_b200_plan* plan, float* ms, int max_stages) {
  if (plan == nullptr || ms == nullptr || max_stages <= 0) return 0;
  try {
    return gpfb::stage_times(plan->plan, ms, max_stages);
  } catch (const gpfb::Error& e) {
    fail(static_cast<gpf_status>(e.status), e.msg);
    return 0;
  }
}

int gpf_b200_plan_stage_marks(gpf_b200_plan* plan, void* ref_event, float* t_ms, int* stage,
                              int max_marks) {
  if (plan == nullptr || ref_event == nullptr || t_ms == nullptr || stage == nullptr || max_marks <= 0)
    return 0;
  try {
    return gpfb::stage_marks(plan->plan, static_cast<cudaEvent_t>(ref_event), t_ms, stage, max_marks);
  } catch (const gpfb::Error& e) {
    fail(static_cast<gpf_status>(e.status), e.msg);
    return 0;
  }
}

size_t gpf_b200_plan_workspace_bytes(const gpf_b200_plan* plan) { return plan ? plan->plan.bytes : 0; }

int gpf_b200_plan_launches_per_frame(const gpf_b200_plan* plan) {
  return plan ? plan->plan.launches_per_frame : 0;
}

}  // extern "C"

namespace {
gpf_status filter_f32_impl(gpf_b200_plan* plan, const float* d_in, float* d_out, int count,
                           long long* d_fallbacks, int* d_ill, void* stream, void* front_done) {
  if (plan == nullptr || d_in == nullptr || d_out == nullptr)
    return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  if (count < 0) return fail(GPF_ERR_INVALID_ARGUMENT, "count must be >= 0");
  return guarded([&] {
    cuda_check(cudaSetDevice(plan->plan.device), "cudaSetDevice");
    auto st = static_cast<cudaStream_t>(stream);
    const size_t npx = (size_t)plan->plan.p.width * plan->plan.p.height;
    auto* fb = reinterpret_cast<unsigned long long*>(d_fallbacks);
    const int B = plan->plan.batch;
    if (fb) cuda_check(cudaMemsetAsync(fb, 0, sizeof(long long) * count, st), "cudaMemsetAsync");
    else if (plan->d_fb_cap < B) {
      cudaFree(plan->d_fb);
      plan->d_fb = nullptr;
      plan->d_fb_cap = 0;
      cuda_check(cudaMalloc(&plan->d_fb, sizeof(unsigned long long) * B), "cudaMalloc");
      plan->d_fb_cap = B;
    }
    struct Reset {  // the event and the flag array belong to this call only
      gpfb::Plan& p;
      ~Reset() {
        p.front_done = nullptr;
        p.ill_out = nullptr;
      }
    } reset{plan->plan};
    for (int f = 0; f < count; f += B) {
      const int n = std::min(B, count - f);
      plan->plan.front_done = f + n >= count ? static_cast<cudaEvent_t>(front_done) : nullptr;
      plan->plan.ill_out = d_ill ? d_ill + f : nullptr;
      gpfb::run_frames_f32(plan->plan, d_in + f * npx, d_out + f * npx, n, fb ? fb + f : plan->d_fb, st);
    }
  });
}

// One-shot batched entry: plans cached per device and parameter set, most
// recently used first. A plan's workspace serves one call at a time, so a call
// makes its stream wait for the plan's previous user (`last`).
struct BatchEntry {
  int device, count;
  gpfb::Params p;
  gpf_b200_plan* plan;
  cudaEvent_t last;
};
std::mutex g_batch_mu;
std::list<BatchEntry> g_batch;
constexpr int kBatchPlans = 4;
constexpr size_t kBatchWorkspace = (size_t)16 << 30;  // bound on one plan's batch workspace

bool batch_same(const BatchEntry& e, int device, int count, const gpfb::Params& p) {
  return e.device == device && e.count == count && e.p.width == p.width && e.p.height == p.height &&
         e.p.sigma_s == p.sigma_s && e.p.kernel_scale == p.kernel_scale && e.p.sigma_r == p.sigma_r &&
         e.p.degree == p.degree && e.p.centering == p.centering;
}

void batch_drop(BatchEntry& e) {  // the plan's queued work finishes first
  cudaEventSynchronize(e.last);
  cudaEventDestroy(e.last);
  gpf_b200_plan_destroy(e.plan);
}

void batch_release() {
  std::lock_guard<std::mutex> lock(g_batch_mu);
  for (auto& e : g_batch) batch_drop(e);
  g_batch.clear();
}
}  // namespace

extern "C" {

gpf_status gpf_b200_filter_f32_ev(gpf_b200_plan* plan, const float* d_in, float* d_out, int count,
                                  long long* d_fallbacks, void* stream, void* front_done) {
  return filter_f32_impl(plan, d_in, d_out, count, d_fallbacks, nullptr, stream, front_done);
}

gpf_status gpf_b200_filter_f32(gpf_b200_plan* plan, const float* d_in, float* d_out, int count,
                               long long* d_fallbacks, void* stream) {
  return filter_f32_impl(plan, d_in, d_out, count, d_fallbacks, nullptr, stream, nullptr);
}

gpf_status gpf_b200_filter_f32_checked(gpf_b200_plan* plan, const float* d_in, float* d_out, int count,
                                       long long* d_fallbacks, int* d_ill, void* stream) {
  return filter_f32_impl(plan, d_in, d_out, count, d_fallbacks, d_ill, stream, nullptr);
}

gpf_status gpf_b200_filter_batch(const float* d_in, float* d_out, int width, int height, int count,
                                 const gpf_spatial_params* sp, const gpf_range_params* rp, int centering,
                                 long long* d_fallbacks, void* stream) {
  if (d_in == nullptr || d_out == nullptr || sp == nullptr || rp == nullptr)
    return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  if (count < 0) return fail(GPF_ERR_INVALID_ARGUMENT, "count must be >= 0");
  gpf_status inner = GPF_OK;
  const gpf_status st = guarded([&] {
    const gpfb::Params p =
        validate(width, height, *sp, *rp, GPF_BACKEND_RECURSIVE, centering, gpfb::kMaxDegreeF32);
    if (count == 0) return;
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(g_batch_mu);
    auto it = g_batch.begin();
    while (it != g_batch.end() && !batch_same(*it, dev, count, p)) ++it;
    if (it != g_batch.end()) {
      g_batch.splice(g_batch.begin(), g_batch, it);
    } else {
      while ((int)g_batch.size() >= kBatchPlans) {
        batch_drop(g_batch.back());
        g_batch.pop_back();
      }
      BatchEntry e{dev, count, p, nullptr, nullptr};
      inner = gpf_b200_plan_create(width, height, sp, rp, centering, dev, &e.plan);
      if (inner != GPF_OK) return;
      // frames filtered per launch: the whole batch when its workspace fits the bound
      const size_t per = std::max<size_t>(e.plan->plan.bytes, 1);
      const int frames = (int)std::max<size_t>(1, std::min<size_t>((size_t)count, kBatchWorkspace / per));
      if (frames > 1) inner = gpf_b200_plan_set_batch(e.plan, frames);
      if (inner == GPF_OK && cudaEventCreateWithFlags(&e.last, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        inner = fail(GPF_ERR_UNKNOWN, "cudaEventCreate failed");
      }
      if (inner != GPF_OK) {
        gpf_b200_plan_destroy(e.plan);
        return;
      }
      cuda_check(cudaEventRecord(e.last, static_cast<cudaStream_t>(stream)), "cudaEventRecord");
      g_batch.push_front(e);
    }
    BatchEntry& e = g_batch.front();
    auto cs = static_cast<cudaStream_t>(stream);
    cuda_check(cudaStreamWaitEvent(cs, e.last, 0), "cudaStreamWaitEvent");
    inner = gpf_b200_filter_f32(e.plan, d_in, d_out, count, d_fallbacks, stream);
    cuda_check(cudaEventRecord(e.last, cs), "cudaEventRecord");
  });
  return st != GPF_OK ? st : inner;
}

gpf_status gpf_b200_exact_f32(const float* d_in, float* d_out, int width, int height, int count,
                              const gpf_spatial_params* sp, const gpf_range_params* rp,
                              void* stream) {
  if (d_in == nullptr || d_out == nullptr || sp == nullptr || rp == nullptr)
    return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  if (width < 1 || height < 1) return fail(GPF_ERR_INVALID_ARGUMENT, "Image dimensions must be >= 1");
  if (count < 0) return fail(GPF_ERR_INVALID_ARGUMENT, "count must be >= 0");
  return guarded([&] {
    const int W = validate_exact(*sp, *rp);
    current_device();
    gpfb::run_exact_f32(d_in, d_out, width, height, count, W, static_cast<int>(sp->boundary),
                        sp->sigma_s, rp->sigma_r, static_cast<cudaStream_t>(stream));
  });
}

gpf_status gpf_b200_compare_f32(const float* d_ref, const float* d_test, int width, int height,
                                int exclude_border, gpf_error_report* out, void* stream) {
  if (d_ref == nullptr || d_test == nullptr || out == nullptr)
    return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    check_compare_dims(width, height, exclude_border);
    current_device();
    fill_report(gpfb::compare_f32(d_ref, d_test, width, height, exclude_border,
                                  static_cast<cudaStream_t>(stream)),
                out);
  });
}

gpf_status gpf_b200_filter_f32_host(gpf_b200_plan* plan, const float* h_in, float* h_out, int count,
                                    long long* h_fallbacks, void* stream) {
  if (plan == nullptr || h_in == nullptr || h_out == nullptr)
    return fail(GPF_ERR_INVALID_ARGUMENT, "null argument");
  if (count < 0) return fail(GPF_ERR_INVALID_ARGUMENT, "count must be >= 0");
  return guarded([&] {
    cuda_check(cudaSetDevice(plan->plan.device), "cudaSetDevice");
    if (!plan->s_comp) {
      const unsigned fl = cudaStreamNonBlocking;
      cuda_check(cudaStreamCreateWithFlags(&plan->s_comp, fl), "cudaStreamCreate");
      for (int s = 0; s < 2; ++s) {
        cuda_check(cudaEventCreateWithFlags(&plan->in_ready[s], cudaEventDisableTiming), "event");
        cuda_check(cudaEventCreateWithFlags(&plan->computed[s], cudaEventDisableTiming), "event");
        cuda_check(cudaEventCreateWithFlags(&plan->out_free[s], cudaEventDisableTiming), "event");
      }
    }
    // Null stream -> the plan's own non-blocking stream, so that host threads
    // driving different plans overlap instead of serialising on stream 0.
    auto st = stream ? static_cast<cudaStream_t>(stream) : plan->s_comp;
    const CopyStreams cs = copy_streams(plan->plan.device);
    const size_t npx = (size_t)plan->plan.p.width * plan->plan.p.height;
    const int slots = count > 1 ? 2 : 1;
    for (int s = 0; s < slots; ++s)
      if (!plan->d_stage_in[s]) {
        cuda_check(cudaMalloc(&plan->d_stage_in[s], npx * sizeof(float)), "cudaMalloc");
        cuda_check(cudaMalloc(&plan->d_stage_out[s], npx * sizeof(float)), "cudaMalloc");
      }
    if (plan->d_fb_cap < count) {
      cudaFree(plan->d_fb);
      cuda_check(cudaMalloc(&plan->d_fb, sizeof(unsigned long long) * std::max(count, 1)), "cudaMalloc");
      plan->d_fb_cap = std::max(count, 1);
    }
    if (plan->h_fb_cap < count) {
      cudaFreeHost(plan->h_fb);
      plan->h_fb = nullptr;
      plan->h_fb_cap = 0;
      cuda_check(cudaMallocHost(&plan->h_fb, sizeof(unsigned long long) * count), "cudaMallocHost");
      plan->h_fb_cap = count;
    }
    cuda_check(cudaMemsetAsync(plan->d_fb, 0, sizeof(unsigned long long) * count, st), "memset");
    // The staging slots belong to this plan and its previous host-entry call has
    // completed, so the first uploads need no wait (a wait here would also hold
    // up other plans' uploads queued behind this one on the shared stream).
    for (int f = 0; f < count; ++f) {
      const int s = f % slots;
      // slot s is reused by frame f: its input is free once frame f-2 computed,
      // its output once frame f-2 downloaded.
      if (f >= slots) cuda_check(cudaStreamWaitEvent(cs.h2d, plan->computed[s], 0), "wait");
      cuda_check(cudaMemcpyAsync(plan->d_stage_in[s], h_in + f * npx, npx * sizeof(float),
                                 cudaMemcpyHostToDevice, cs.h2d), "H2D");
      cuda_check(cudaEventRecord(plan->in_ready[s], cs.h2d), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(st, plan->in_ready[s], 0), "wait");
      if (f >= slots) cuda_check(cudaStreamWaitEvent(st, plan->out_free[s], 0), "wait");
      gpfb::run_frames_f32(plan->plan, plan->d_stage_in[s], plan->d_stage_out[s], 1, plan->d_fb + f, st);
      cuda_check(cudaEventRecord(plan->computed[s], st), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(cs.d2h, plan->computed[s], 0), "wait");
      cuda_check(cudaMemcpyAsync(h_out + f * npx, plan->d_stage_out[s], npx * sizeof(float),
                                 cudaMemcpyDeviceToHost, cs.d2h), "D2H");
      cuda_check(cudaEventRecord(plan->out_free[s], cs.d2h), "cudaEventRecord");
    }
    if (count > 0)
      cuda_check(cudaMemcpyAsync(plan->h_fb, plan->d_fb, sizeof(unsigned long long) * count,
                                 cudaMemcpyDeviceToHost, st), "D2H");
    // this call's last download is the last event on out_free[(count-1)%slots]
    if (count > 0) cuda_check(cudaEventSynchronize(plan->out_free[(count - 1) % slots]), "sync");
    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    if (h_fallbacks)
      for (int f = 0; f < count; ++f) h_fallbacks[f] = static_cast<long long>(plan->h_fb[f]);
  });
}

}  // extern "C"
