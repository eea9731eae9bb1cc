/* gpfilter_b200.h -- device-resident batched entry points (B200 extension).
 *
 * The reference ABI (gpfilter.h) moves one double image through host memory
 * per call. Throughput users keep fp32 frames resident in HBM and filter a
 * batch per call; these entries expose exactly that, with the same parameter
 * structs, validation and status codes as gpf_filter_gpf.
 *
 * A plan binds (width, height, sigma_s, kernel_scale, sigma_r, degree,
 * centering) to one CUDA device and owns the device workspace (the N+2
 * intermediate planes, carries and per-frame scalars). Plans are not shared
 * between concurrent callers; create one per thread/stream.
 */
#ifndef GPFILTER_B200_EXT_H
#define GPFILTER_B200_EXT_H

#include "gpfilter/gpfilter.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gpf_b200_plan gpf_b200_plan;

/* Validates like gpf_filter_gpf (backend is implied recursive; degree <= 48,
 * the fp32 kernels' limit) and allocates the workspace on `device` (-1 =
 * current device); the caller's current device is left unchanged. The plan
 * entries always run the fp32 plane kernels (see the precision notes below
 * and gpf_b200_filter_f32_checked). */
gpf_status gpf_b200_plan_create(int width, int height, const gpf_spatial_params* sp,
                                const gpf_range_params* rp, int centering, int device,
                                gpf_b200_plan** out);
void gpf_b200_plan_destroy(gpf_b200_plan* plan);

/* Re-sizes the workspace to hold `frames` frames, so that gpf_b200_filter_f32
 * filters up to that many frames per kernel launch (default 1). Frame-level
 * batching is what fills the 148 SMs for small frames (e.g. 3840x2160). The
 * new workspace is built before the old one is released: on failure (e.g. the
 * batch does not fit in HBM) the plan keeps its previous workspace and stays
 * usable. */
gpf_status gpf_b200_plan_set_batch(gpf_b200_plan* plan, int frames);

/* Per-stage timing for benchmarks: when enabled, every launch group records
 * CUDA events between its kernels on the launching stream. stage_times
 * synchronises those events and returns, per stage (0 mean, 1 column
 * carries, 2 column pass, 3 row-carry scan, 4 row pass + contraction), the
 * milliseconds accumulated since profiling was (re)enabled. */
gpf_status gpf_b200_plan_set_profiling(gpf_b200_plan* plan, int enable);
int gpf_b200_plan_stage_times(gpf_b200_plan* plan, float* ms, int max_stages);
/* Timeline of the recorded stage events (profiling enabled): for each mark
 * since the last stage_times / stage_marks call, its stage id (0-4, or -1 for
 * the end of a launch group) and its time in ms after `ref_event` (a
 * cudaEvent_t recorded by the caller on the same device). Synchronises the
 * events and consumes them; returns the number of marks written. */
int gpf_b200_plan_stage_marks(gpf_b200_plan* plan, void* ref_event, float* t_ms, int* stage,
                              int max_marks);

/* Bytes of device workspace held by the plan. */
size_t gpf_b200_plan_workspace_bytes(const gpf_b200_plan* plan);

/* Kernel launches enqueued per frame (for launch accounting in benchmarks). */
int gpf_b200_plan_launches_per_frame(const gpf_b200_plan* plan);

/* Filters `count` contiguous fp32 frames (each width*height, row-major) that
 * live in device memory. d_out may not alias d_in. d_fallbacks (device
 * memory, `count` long longs, may be NULL) receives per-frame fallback
 * counts. Work is enqueued on `stream` (a cudaStream_t, NULL = legacy
 * default stream); the call returns without synchronising. */
gpf_status gpf_b200_filter_f32(gpf_b200_plan* plan, const float* d_in, float* d_out,
                               int count, long long* d_fallbacks, void* stream);

/* Same as gpf_b200_filter_f32, and records `front_done` (a cudaEvent_t) on
 * `stream` once the column half of the last frame (mean, seeds, column
 * carries, column pass) has been enqueued: waiting on it lets the caller start
 * another frame's column half while this frame's row half (row carries, row
 * pass) runs, so HBM-heavy and FMA-heavy kernels of different frames overlap. */
gpf_status gpf_b200_filter_f32_ev(gpf_b200_plan* plan, const float* d_in, float* d_out,
                                  int count, long long* d_fallbacks, void* stream,
                                  void* front_done);

/* Same as gpf_b200_filter_f32, and writes d_ill[f] (device memory, `count`
 * ints) = 1 when frame f lies outside the envelope in which the fp32 kernels
 * are held to the reference within 1e-3 (max|H| = max(f_max - t_c, t_c -
 * f_min) / sigma_r > gpf_b200_fp32_h_limit_degree(degree), measured on the device from the
 * frame itself), else 0. Such a frame's fp32 output is still the fp32
 * evaluation, but the reference's own degree-N series is ill-conditioned there
 * (it may leave the input range); filter it through gpf_filter_gpf (AUTO runs
 * the reference-exact fp64 mode for it). */
gpf_status gpf_b200_filter_f32_checked(gpf_b200_plan* plan, const float* d_in, float* d_out,
                                       int count, long long* d_fallbacks, int* d_ill, void* stream);

/* One-shot batched device entry: gpf_b200_filter_f32 without a
 * plan handle. Filters `count` contiguous fp32 frames (each width*height,
 * row-major) in device memory on the current device with the parameters of
 * gpf_filter_gpf (recursive backend; `centering` as there). The library
 * creates a plan for (device, size, parameters, count) on first use and keeps
 * the four most recently used, so a repeated call allocates nothing; calls
 * that share a cached plan run one after the other on the device (their
 * streams are chained by an event). d_fallbacks: device memory, `count` long
 * longs, may be NULL. Enqueued on `stream`, no synchronisation.
 * gpf_b200_dropin_release() frees the cached plans. */
gpf_status gpf_b200_filter_batch(const float* d_in, float* d_out, int width, int height, int count,
                                 const gpf_spatial_params* sp, const gpf_range_params* rp,
                                 int centering, long long* d_fallbacks, void* stream);

/* Exact (direct O(sigma_s^2)) bilateral filter of `count` contiguous fp32
 * frames in device memory (the gpf_filter_exact definition), on `stream`. */
gpf_status gpf_b200_exact_f32(const float* d_in, float* d_out, int width, int height, int count,
                              const gpf_spatial_params* sp, const gpf_range_params* rp,
                              void* stream);

/* gpf_compare on fp32 device images (deterministic reduction); synchronises
 * `stream`. */
gpf_status gpf_b200_compare_f32(const float* d_ref, const float* d_test, int width, int height,
                                int exclude_border, gpf_error_report* out, void* stream);

/* Same, from host memory to host memory: copies each frame in, filters,
 * copies the result and the fallback counts back, and synchronises `stream`
 * before returning. h_fallbacks (host, `count` entries) may be NULL. */
gpf_status gpf_b200_filter_f32_host(gpf_b200_plan* plan, const float* h_in, float* h_out,
                                    int count, long long* h_fallbacks, void* stream);

/* ------------------------------------------------------------------------
 * Precision of the fp64 drop-in entry gpf_filter_gpf.
 *
 *   FP32  the fp32 plane kernels (the throughput path of gpf_b200_filter_f32),
 *         fp64 input/output and prologue. Held to max |out - reference| <= 1e-3
 *         on [0,255] while max|H| = max(f_max - t_c, t_c - f_min) / sigma_r <=
 *         gpf_b200_fp32_h_limit_degree(degree) (7.0 at the default N = 20;
 *         1.5-10 for other degrees: the truncated series cancels sooner at low
 *         and odd N) and degree <= 48.
 *   FP64  the reference's own fp64 arithmetic replayed on the GPU operation for
 *         operation (exp() is a correctly rounded double-double evaluation,
 *         equal to glibc's on ~99.9 % of arguments): follows the
 *         reference also where its degree-N series is ill-conditioned and its
 *         output leaves the input range (BASELINE C2/C5). Degree <= 62; about
 *         (degree + 2) x 18 B of extra device memory per pixel. Each axis runs
 *         in chunks of 32 samples restarted from recorded recurrence states,
 *         bitwise equal to the line-by-line order of the reference
 *         (environment GPF_B200_F64_SEQUENTIAL=1 selects the literal
 *         sequential replay, the cross-check of the tests).
 *   AUTO  (default; environment GPF_B200_PRECISION=auto|fp32|fp64 sets the
 *         initial mode) measures t_c, f_min and f_max on the device and runs
 *         FP64 outside the FP32 envelope, FP32 inside it.
 * The mode is process-global; gpf_b200_last_precision() reports (per calling
 * thread) which one the last gpf_filter_gpf call ran, and
 * gpf_b200_last_max_abs_h() the max|H| it measured (AUTO only, else 0).
 * ---------------------------------------------------------------------- */
typedef enum gpf_b200_precision {
  GPF_B200_PRECISION_AUTO = 0,
  GPF_B200_PRECISION_FP32 = 1,
  GPF_B200_PRECISION_FP64 = 2
} gpf_b200_precision;

gpf_status gpf_b200_set_precision(int mode);
int gpf_b200_get_precision(void);
int gpf_b200_last_precision(void);
double gpf_b200_last_max_abs_h(void);
double gpf_b200_fp32_h_limit(void);             /* the envelope at the default degree (20) */
double gpf_b200_fp32_h_limit_degree(int degree); /* the envelope at `degree` (0 outside 0..48) */
/* Device time (CUDA events on the drop-in stream) of the filter kernels of this
 * thread's last gpf_filter_gpf call, copies excluded. */
float gpf_b200_last_device_ms(void);

/* gpf_filter_gpf keeps, per device, up to four fp32 plans (keyed by every
 * filter parameter), the fp64 workspace and its device buffers between calls,
 * so repeated calls allocate nothing. This frees all of it. */
void gpf_b200_dropin_release(void);

/* y[i] = exp(x[i]) as the reference-exact fp64 mode evaluates it on the device
 * (csrc/exp_cr.h: double-double, correctly rounded; equals glibc's exp on ~99.9 %
 * of arguments, one ulp apart where glibc itself misrounds). x, y: host arrays of
 * n doubles. A verification hook (tests/test_exp_cr.py), not a fast path. */
gpf_status gpf_b200_exp_cr(const double* x, double* y, long long n);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* GPFILTER_B200_EXT_H */
