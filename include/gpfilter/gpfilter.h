/* gpfilter.h -- B200 drop-in for the Gauss-polynomial bilateral filter path.
 *
 * This header declares the C ABI that libgpfilter_b200.so exports. Every
 * entry point keeps the name, argument meaning, status codes and error
 * behaviour of the reference library's public header, so a caller written
 * against the reference binds to this library unchanged for the GPF path.
 * Each declaration cites the reference interface it replaces
 * (/root/reference/proj/include/gpfilter/gpfilter.h, "ref.h" below).
 *
 * Provided: every function of the reference header -- the GPF hot path
 * (gpf_filter_gpf, recursive backend) and the handles, params, status/error
 * plumbing it needs; beside it the exact filter, the Taylor baseline, the
 * single-plane Gaussians, the direct (windowed) backend (fp64 on the GPU,
 * bitwise the reference's), gpf_compare, PGM I/O and the scalar
 * range-kernel evaluators (host). The C++ entry point gpfilter::gpf is in
 * gpfilter/gpfilter.hpp; device-resident batches and the precision modes in
 * gpfilter/gpfilter_b200.h.
 */
#ifndef GPFILTER_B200_GPFILTER_H
#define GPFILTER_B200_GPFILTER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: same numeric values as ref.h:18-29. */
typedef enum gpf_status {
  GPF_OK = 0,
  GPF_ERR_INVALID_ARGUMENT = 1,
  GPF_ERR_IO = 2,
  GPF_ERR_SIGMA_TOO_SMALL = 3,
  GPF_ERR_PGM_BAD_MAGIC = 4,
  GPF_ERR_PGM_BAD_DIMS = 5,
  GPF_ERR_PGM_BAD_MAXVAL = 6,
  GPF_ERR_PGM_TRUNCATED = 7,
  GPF_ERR_PGM_BAD_PIXEL = 8,
  GPF_ERR_UNKNOWN = 9 /* also: CUDA runtime failures (detail in gpf_last_error) */
} gpf_status;

/* ref.h:31-39 */
const char* gpf_status_name(gpf_status status);
const char* gpf_last_error(void); /* thread-local detail of the last failure */
const char* gpf_version(void);

/* Opaque row-major width*height grid of doubles (ref.h:45-58). */
typedef struct gpf_image gpf_image;
gpf_status gpf_image_create(int width, int height, gpf_image** out); /* zero-filled, w,h >= 1 */
void gpf_image_destroy(gpf_image* img);                               /* NULL is a no-op */
int gpf_image_width(const gpf_image* img);                            /* 0 for NULL */
int gpf_image_height(const gpf_image* img);
double* gpf_image_data(gpf_image* img);                               /* NULL for NULL */
const double* gpf_image_cdata(const gpf_image* img);

/* Parameters (ref.h:64-90); identical layout and defaults. */
typedef enum gpf_boundary {
  GPF_BOUNDARY_REPLICATE = 0,
  GPF_BOUNDARY_REFLECT = 1,
  GPF_BOUNDARY_ZERO = 2
} gpf_boundary;

typedef enum gpf_backend {
  GPF_BACKEND_DIRECT = 0,   /* windowed Gaussian, O(window_radius) per pixel; fp64 mode only */
  GPF_BACKEND_RECURSIVE = 1 /* the O(1) Deriche path, sigma_s >= 0.5 */
} gpf_backend;

typedef struct gpf_spatial_params {
  double sigma_s;     /* > 0 */
  int window_radius;  /* <= 0 selects ceil(3 sigma_s); unused by the recursive path */
  gpf_boundary boundary; /* direct backend and exact filter; the recursive path
                            always uses the replicate steady state, as the
                            reference does */
  double kernel_scale;   /* > 0 */
} gpf_spatial_params;

typedef struct gpf_range_params {
  double sigma_r; /* > 0 */
  int degree;     /* polynomial degree N >= 0 (N+2 filtered planes) */
} gpf_range_params;

void gpf_spatial_params_init(gpf_spatial_params* sp); /* 2 / auto / replicate / 1.0 */
void gpf_range_params_init(gpf_range_params* rp);     /* 30 / 20 */

/* The hot path (replaces ref.h:100-107, proj/src/capi.cpp:176-192).
 * Runs on the current CUDA device; precision per gpf_b200_set_precision
 * (default AUTO: the fp32 plane kernels inside their validated envelope, the
 * reference-exact fp64 mode outside it -- gpfilter_b200.h). Degree <= 62.
 * Plans and buffers are cached per device between calls; concurrent calls on
 * one device are serialised. Host images of 4 MiB and more are page-locked.
 * Validation and status mapping follow the reference: NULL in/sp/rp/out ->
 * INVALID_ARGUMENT; *out is set to NULL before work starts; bad backend or
 * boundary enum, sigma_s <= 0, kernel_scale <= 0, sigma_r <= 0, degree < 0 ->
 * INVALID_ARGUMENT (detail names the field); sigma_s < 0.5 with the recursive
 * backend -> GPF_ERR_SIGMA_TOO_SMALL with "direct" in the detail.
 * GPF_BACKEND_DIRECT (apply_spatial -> direct_gaussian,
 * proj/src/core/bilateral.cpp:58-62) filters the planes with the windowed
 * passes of gpf_gaussian_direct, any sigma_s > 0, in the fp64 mode (the fp32
 * mode forced by gpf_b200_set_precision rejects it). fallback_count may be
 * NULL and is written only on success. Pixels with |Q| <= 1e-8 (reference
 * units, proj/src/core/bilateral.hpp:85) keep their input value. */
gpf_status gpf_filter_gpf(const gpf_image* in, const gpf_spatial_params* sp,
                          const gpf_range_params* rp, gpf_backend backend,
                          int centering, long long* fallback_count,
                          gpf_image** out);

/* Spatial windowed Gaussian alone (ref.h:116-117, proj/src/capi.cpp:209-217 ->
 * direct_gaussian, proj/src/core/spatial.cpp:112-129): 2W+1 taps per axis
 * (W = sp->window_radius, or ceil(3 sigma_s) when <= 0), rows then columns,
 * kernel_scale on the row taps, the boundary mode of sp; unnormalised, like
 * the reference. fp64 on the GPU in the reference's accumulation order:
 * bitwise equal to the reference. */
gpf_status gpf_gaussian_direct(const gpf_image* in, const gpf_spatial_params* sp,
                               gpf_image** out);

/* Spatial recursive Gaussian alone (ref.h:118-119, proj/src/capi.cpp:219-228):
 * same Deriche filter, output scaled by kernel_mass_1d(sigma_s)^2*kernel_scale. */
gpf_status gpf_gaussian_recursive(const gpf_image* in, double sigma_s,
                                  double kernel_scale, gpf_image** out);

/* Taylor-polynomial baseline of degree rp->degree, truncation order
 * K = degree / 2 (ref.h:109-113, proj/src/capi.cpp:194-207 -> taylor_bilateral,
 * proj/src/core/bilateral.cpp:160-220): the 2K+2 moment images f^m smoothed by
 * the recursive Gaussian and recombined per pixel; fp64 on the GPU, bitwise
 * equal to the reference, with either backend. Same NULL / validation /
 * status behaviour and fallback rule as gpf_filter_gpf. */
gpf_status gpf_filter_taylor(const gpf_image* in, const gpf_spatial_params* sp,
                             const gpf_range_params* rp, gpf_backend backend,
                             long long* fallback_count, gpf_image** out);

/* Exact brute-force bilateral filter, Eq. (1) over the (2W+1)^2 window with
 * the boundary mode of sp (ref.h:97-98, proj/src/capi.cpp:164-174 ->
 * exact_bilateral, proj/src/core/bilateral.cpp:14-56). The MSE yardstick of
 * the GPF path; runs on the GPU in fp64 with the reference's operation order
 * and weight table (only exp() differs by <= 1 ulp): passes the reference's
 * own pins (impulse within 3e-14, shift invariance within 1e-9). The fp32
 * device entry gpf_b200_exact_f32 is the fast form. Same NULL / validation /
 * status behaviour. */
gpf_status gpf_filter_exact(const gpf_image* in, const gpf_spatial_params* sp,
                            const gpf_range_params* rp, gpf_image** out);

/* Range-kernel evaluation (ref.h:123-143, proj/src/capi.cpp:230-286 ->
 * proj/src/core/range_kernel.cpp): scalar, on the host. NULL out, sigma_r <= 0,
 * degree < 0, low >= high, step <= 0 or a bad `which` -> INVALID_ARGUMENT. */
typedef enum gpf_range_approx {
  GPF_RANGE_APPROX_GAUSS_POLY = 0,
  GPF_RANGE_APPROX_TAYLOR = 1
} gpf_range_approx;
/* exp(-(t - tau)^2 / (2 sigma_r^2)) */
gpf_status gpf_kernel_gauss(double t, double tau, double sigma_r, double* out);
/* its degree-N Gauss-polynomial (Eq. (4)) and Taylor approximations */
gpf_status gpf_kernel_gauss_poly(double t, double tau, double sigma_r, int degree, double* out);
gpf_status gpf_kernel_taylor(double t, double tau, double sigma_r, int degree, double* out);
/* sup over t in [low, high] (stepped by `step`, endpoint included) of the
 * absolute error of the chosen approximation against the exact kernel */
gpf_status gpf_kernel_sup_error(double sigma_r, int degree, double tau, double low, double high,
                                double step, gpf_range_approx which, double* out);

/* Error statistics between equally sized images (ref.h:149-159,
 * proj/src/capi.cpp:288-301 -> metrics::compare, proj/src/core/metrics.cpp). */
typedef struct gpf_error_report {
  double mse;
  double mse_db; /* 10*log10(mse); -400 when mse == 0 */
  double max_abs;
  long long pixels; /* samples compared */
} gpf_error_report;

gpf_status gpf_compare(const gpf_image* ref, const gpf_image* test,
                       int exclude_border, gpf_error_report* out);

/* Thread-count plumbing (ref.h:165-168). Kept for ABI compatibility; the
 * value is recorded but device work is always deterministic and identical
 * for every count. */
gpf_status gpf_set_num_threads(int n);
int gpf_get_num_threads(void);

/* PGM I/O (ref.h:171-186, proj/src/capi.cpp:311-349):
 * binary (P5) or ASCII (P2), maxval 255. Parse failures return one of the
 * GPF_ERR_PGM_* codes and gpf_last_error() names the byte offset; file errors
 * return GPF_ERR_IO. Writing produces "P5\n<w> <h>\n255\n" with samples
 * clamped to [0, 255] and rounded half away from zero. */
gpf_status gpf_read_pgm(const char* path, gpf_image** out);
gpf_status gpf_decode_pgm(const uint8_t* bytes, size_t size, gpf_image** out);
gpf_status gpf_write_pgm(const gpf_image* img, const char* path);
gpf_status gpf_encode_pgm(const gpf_image* img, uint8_t** bytes, size_t* size);

/* Releases a buffer returned by gpf_encode_pgm. */
void gpf_free_bytes(uint8_t* bytes);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* GPFILTER_B200_GPFILTER_H */
