// Internal interfaces of libgpfilter_b200: filter constants, plan and launchers.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

#include <cuda.h>
#include <cuda_runtime.h>

namespace gpfb {

constexpr int kMaxPlanes = 64;  // N+2 <= 64  (degree <= 62)
constexpr int kMaxDegreeF32 = 48;  // fp32 plane kernels (shared memory per CTA)
constexpr int kMaxDegreeF64 = 62;  // reference-exact fp64 mode
constexpr int kTile = 32;       // rows per column-pass chunk == columns per row-pass chunk

// Per-call constants of the filter, computed on the host in fp64 from the
// reference's own Deriche coefficients (proj/src/core/spatial.cpp:140-181) and
// passed by value to every kernel.
//
// The 4th-order causal/anticausal recurrences of deriche_line
// (proj/src/core/spatial.cpp:186-216) are realised as two complex first-order
// sections each (partial-fraction expansion over the conjugate pole pairs):
//   causal      w_k[i]   = x[i]   + p_k w_k[i-1],   y+[i] = sum_k Re(A_k w_k[i])
//   anticausal  v_k[i]   = x[i+1] + p_k v_k[i+1],   y-[i] = sum_k Re(B_k v_k[i])
// (A_k, B_k already carry the factor 2 of the conjugate pair.) Same transfer
// function, far better conditioned in fp32 than the direct form. The replicate
// steady-state warm start of the reference is w_k[-1] = x[0]/(1-p_k) and
// v_k[n-1] = x[n-1]/(1-p_k).
// Every coefficient is stored duplicated as (c, c) so that it feeds packed
// fp32x2 instructions directly (the two halves are the two planes of a pair).
struct FilterConsts {
  float2 pr2[2];                   // Re p_k (poles in the upper half plane)
  float2 gr2[2], gi2[2];           // 1/(1-p_k): warm-start gain (standard basis, carry chains)
  float2 ips2[2];                  // 1 / Im(p_k)
  float2 gs2[2];                   // Im(1/(1-p_k)) / Im(p_k): warm start of u2
  // Sweep basis, per direction D (causal c with residues A_k, anticausal a
  // with B_k): u1 = Re w - tau Im w, u2 = Im w / Im p, with tau = Im R / Re R
  // (R = A_k or B_k), so that the section's output Re(R w) = Re R * u1 and the
  // emit costs one FMA per section. The advance stays three FMAs:
  //   u2' = m22 u2 + u1,   u1' = m11 u1 + m12 u2 + x
  //   m11 = Re p - tau Im p,  m22 = Re p + tau Im p,  m12 = -(Im p)^2 (1 + tau^2)
  // (tau = 0 is the plain rescaled basis u2 = Im w / Im p). Only B_1 gets close
  // to a zero real part (sigma_s in [0.96, 1.17]); there tau is clamped to
  // |tau Im p| <= 1 and its emit keeps a u2 term (aev).
  float2 cm11[2], cm12[2], cm22[2];  // causal advance
  float2 am11[2], am12[2], am22[2];  // anticausal advance
  float2 ce[2];                      // causal emit weights Re A_k
  float2 ae[2];                      // anticausal emit weights Re B_k
  float2 aev;                        // anticausal section-1 u2 weight (0 unless tau clamped)
  float2 ntau_a[2];                  // -tau of the anticausal sections (carry -> u1)
  float2 cgu1[2];                    // causal warm start of u1: Re g - tau Im g
  // Emit normalisation: every emit weight is divided by S = Re A_0, so the
  // causal section-0 weight is 1 (its emit needs no multiply). The column
  // pass's input carries S^2 (plane seeds, RangeConsts::e_log2 += seed_log2)
  // and its output S, so the row pass's input carries S and its output none.
  double seed_log2;                  // log2(S^2), host side
};

// Tile constants for exact anticausal carries between chunks of kTile
// samples: the carry entering a chunk from the far side is
//   C = sum_{j < L} p^j x[j]  +  p^L C_next        (L = chunk length)
struct TileConsts {
  float4 w4[kTile];                     // (Re p_0^j, Im p_0^j, Re p_1^j, Im p_1^j), j < kTile
  float2 pTr2[2], pTi2[2];              // p_k^kTile
  float2 pYr2[2], pYi2[2];              // p_k^(rows in the last row chunk)
  float2 pXr2[2], pXi2[2];              // p_k^(columns in the last column strip)
  // G-scaled planes (GPF_GSCALE, pairs <= kGsPairs): the column pass stores
  // plane n as G_n = F_n 2^{s0-64} / n! (every 1/n! folded into the plane, so the
  // row pass contracts with a joint Horner pass for Q and Q' = P and no
  // per-plane weights). With w_n = 2^k/(n+1) (RangeConsts::w_step):
  float2 gstep[16];                     // pair step: (w_2g w_2g+1, w_2g+1 w_2g+2) times m^2
  float gpre[16];                       // prod_{i<2g} w_i: first plane of pair g from es m^{2g}
  float gw[16];                         // w_2g: second plane of pair g from its first (times m)
  float2 gcar[16];                      // (prod_{i<2g} w_i, prod_{i<2g+1} w_i): carry-walk states -> G units
};
constexpr int kGsPairs = 12;            // G-scaled contraction: the k_rowpass2 path (N <= 22)

// Range / plane constants. Plane n holds F_n * 2^{s_n}, s_n = s0 - k*n, so
// that every significant plane value stays in the fp32 normal range (the
// exp(-h^2/2 sr^2) factor alone underflows fp32 for |h| > 13.2 sr).
struct RangeConsts {
  double inv_sr;      // 1/sigma_r
  double inv2s2;      // 1/(2 sigma_r^2)  (same expression as bilateral.cpp:92)
  double sigma_r;
  double e_scale;     // 2^s0
  double e_log2;      // s0
  double exp2_k;      // log2(e) / (2 sigma_r^2)
  float h_step;       // 2^-k      (chain multiplier factor)
  float c0;           // 2^-s0     (weight of plane 0)
  float p_scale;      // 2^k       (P uses planes n+1)
  float w_step[kMaxPlanes];  // 2^k/(n+1): c_{n+1} = c_n * H * w_step[n]
  float k_coef[kMaxPlanes];  // 2^-s0 2^{kn} / n!: c_n = H^n k_coef[n] (Horner contraction)
  float q_thresh;     // kQMin / (mass^2 * kernel_scale)  (bilateral.hpp:85)
  float q_thresh_g;   // the same threshold in G units (q_thresh 2^{s0-64}; GPF_GSCALE)
  int planes;         // N + 2
  int pairs;          // ceil(planes / 2)
  int degree;         // N
  // fp32 prologue (pixel_terms_f32): e_log2 = e_int + e_frac_hi + e_frac_lo,
  // exp2_k = k_hi + k_lo, inv_sr_f = (float)inv_sr (finalize_range_consts)
  int e_int;
  float e_frac_hi, e_frac_lo, k_hi, k_lo, inv_sr_f;
  int centering;      // 0 none / 1 mean / 2 fixed t_c (midpoint)
  double tc_fixed;    // t_c for centering 2
};

struct Params {
  int width = 0, height = 0;
  double sigma_s = 2.0, kernel_scale = 1.0, sigma_r = 30.0;
  int degree = 20, centering = 1;  // centering: 0 none, 1 mean, 2 fixed t_c = tc_fixed
  double tc_fixed = 0.0;           // CenteringMode::midpoint: (range.low + range.high) / 2
  // apply_spatial (bilateral.cpp:58-62): 1 recursive (the hot path), 0 direct
  // (windowed, fp64 mode only: window_radius taps per side, boundary 0
  // replicate / 1 reflect / 2 zero)
  int backend = 1, window_radius = 0, boundary = 0;
};

// Host-side constant builders (coeffs.cpp).
FilterConsts make_filter_consts(double sigma_s);
TileConsts make_tile_consts(double sigma_s, int width, int height);
void fill_gscale_consts(TileConsts& tc, RangeConsts& rc);  // G-scaled plane constants
RangeConsts make_range_consts(const Params& p);
void finalize_range_consts(RangeConsts& rc);  // after e_log2 is final: the fp32 prologue split
double kernel_mass_1d(double sigma_s, int radius);
int default_window_radius(double sigma_s);
// The reference's normalised Deriche coefficients (spatial.cpp:140-181), fp64.
void deriche_coeffs_f64(double sigma, double nc[4], double na[4], double d[4]);

// Device workspace + launch plan for one (w, h, params) on one device.
struct Plan {
  Params p;
  FilterConsts fc;
  TileConsts tc;
  RangeConsts rc;
  int device = 0;
  int batch = 0;       // frames per launch the workspace holds
  int ny = 0, nx = 0;  // row chunks / column strips of kTile
  // workspace (per frame slot)
  float2* V = nullptr;      // [batch][pairs][w][h]   column-pass output, transposed
  float4* CA = nullptr;     // [batch][ny][pairs][w][2] column anticausal carries
  float4* AH = nullptr;     // [batch][nx][pairs][h][2] row aggregates per strip
  float4* CH = nullptr;     // [batch][nx][pairs][h][2] row anticausal carries
  float2* EM = nullptr;     // [batch][h][w_pad] per-pixel plane seeds (E 2^s0, H 2^-k) from K1
  int w_pad = 0;            // EM row pitch in pixels (even: TMA strides are 16-B multiples)
  alignas(64) CUtensorMap vmap;    // TMA map of V: fp32 [batch][pairs][w][2*h_pad] (row-pass loads)
  alignas(64) CUtensorMap vmap8;   // same, 8-row x 33-column boxes (8-row-band row pass)
  alignas(64) CUtensorMap vstore;  // TMA map of V for the column pass's staged chunk stores
  alignas(64) CUtensorMap emmap;   // TMA map of EM: 32x32-pixel tiles for the column pass
  alignas(64) CUtensorMap emcmap;  // TMA map of EM: 64-column x 32-row tiles for the carry walk
  double* scalars = nullptr;   // [batch][2]  t_c, max|H|
  double* partials = nullptr;  // [batch][mean_blocks][4]
  size_t bytes = 0;
  int mean_blocks = 0;
  int launches_per_frame = 0;  // kernels per launch group (independent of batch)
  // optional event recorded after the column pass (set per call by the C ABI)
  cudaEvent_t front_done = nullptr;
  // optional per-frame ill-conditioned flags of this launch group (device, set per call)
  int* ill_out = nullptr;
  // optional row ranges of the row pass for single-frame calls (drop-in D2H overlap):
  // the bands are split into row_ranges launches, range_done[i] recorded after each;
  // the launch reports how many it used and the rows per band
  static constexpr int kMaxRanges = 8;
  int row_ranges = 1;
  cudaEvent_t range_done[kMaxRanges] = {};
  int ranges_launched = 1, range_rows = 16;
  // optional per-stage timing: events recorded on the launching stream
  bool profile = false;
  struct StageTimer* timer = nullptr;
};

// Stage ids for the profiling hook.
enum Stage { kStageMean = 0, kStageColCarry, kStageColPass, kStageRowScan, kStageRowPass, kNumStages };
void stage_mark(Plan& plan, int stage, cudaStream_t st);  // records "stage begins"
void stage_end(Plan& plan, cudaStream_t st);              // records "last stage ends"
int stage_times(Plan& plan, float* ms, int max_stages);   // accumulated ms per stage; syncs
int stage_marks(Plan& plan, cudaEvent_t ref, float* t_ms, int* stage, int max_marks);  // timeline; syncs
void stage_reset(Plan& plan);

// Status-carrying error used inside the library.
struct Error {
  int status;  // gpf_status value
  std::string msg;
};

void plan_init(Plan& plan, const Params& p, int device, int batch = 1);  // throws Error
void plan_free(Plan& plan);
// Enqueue `count` contiguous frames (count <= plan.batch): in -> out; per-frame
// fallback counters d_fb[count] are incremented (caller zeroes them).
void run_frames_f32(Plan& plan, const float* d_in, float* d_out, int count,
                    unsigned long long* d_fb, cudaStream_t st);
void run_frames_f64(Plan& plan, const double* d_in, double* d_out, int count,
                    unsigned long long* d_fb, cudaStream_t st);
// Direct O(sigma_s^2) bilateral (exact_bilateral, bilateral.cpp:14-56) on
// `count` frames; boundary 0 replicate, 1 reflect, 2 zero (exact.cu).
void run_exact_f32(const float* d_in, float* d_out, int w, int h, int count, int W, int boundary,
                   double sigma_s, double sigma_r, cudaStream_t st);
// fp64 form: the reference's per-pixel operation sequence (fp64 taps).
void run_exact_f64(const double* d_in, double* d_out, int w, int h, int count, int W, int boundary,
                   double sigma_s, double sigma_r, double kernel_scale, cudaStream_t st);
// metrics::compare (metrics.cpp:20-56) on device images; synchronises st.
struct ErrorStats {
  double mse = 0.0, max_abs = 0.0;
  long long pixels = 0;
};
ErrorStats compare_f32(const float* d_ref, const float* d_test, int w, int h, int border,
                       cudaStream_t st);
ErrorStats compare_f64(const double* d_ref, const double* d_test, int w, int h, int border,
                       cudaStream_t st);
// Taylor-polynomial baseline (taylor_bilateral, bilateral.cpp:160-220), fp64,
// bitwise equal to the reference; *d_fb receives the fallback count (taylor.cu).
void run_taylor_f64(const double* d_in, double* d_out, const Params& p, unsigned long long* d_fb,
                    cudaStream_t st);
// t_c of one fp64 frame (K0 double-double mean; 0 / tc_fixed per centering) into
// scalars[0];
// scalars[1] = max|H| = max(f_max - t_c, t_c - f_min) / sigma_r; partials
// holds 4*blocks doubles.
void launch_mean_f64(const double* d_in, long long n, int centering, double tc_fixed, double sigma_r,
                     double* partials, int blocks, double* scalars, cudaStream_t st);

// Reference-exact fp64 GPF (gpf_f64.cu): the reference's own fp64 operation
// sequence replayed on the GPU, for inputs whose degree-N series is too
// ill-conditioned for fp32 planes. Workspace grown on demand and reused.
constexpr int kF64MeanBlocks = 592;
struct F64Work {
  double* base = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes);  // throws Error
  void release();
};
size_t f64_workspace_bytes(int w, int h, int degree);
// ranges > 1: the final combine runs in that many pixel ranges, range_done[i]
// recorded after range i (pixels [n i/ranges, n (i+1)/ranges)).
void run_gpf_f64_exact(const double* d_in, double* d_out, const Params& p, F64Work& ws,
                       unsigned long long* d_fb, cudaStream_t st, int ranges = 1,
                       cudaEvent_t* range_done = nullptr);

// GpfState stepping on device buffers (gpf_f64.cu; bilateral.cpp:64-148), fp64,
// the reference's operation order: init (t_c into scalars[0], H, F_0),
// apply_spatial with either backend, the two loops of step(), finalize.
void state_init_f64(const double* d_in, double* H, double* F, double* scalars, double* partials,
                    const Params& p, cudaStream_t st);
void state_spatial_f64(const double* src, double* dst, double* tmp, const Params& p, cudaStream_t st);
void state_step_a_f64(double* Q, double* F, const double* G, const double* Fbar, const double* H,
                      double c, long long n, cudaStream_t st);
void state_step_b_f64(double* P, double* G, const double* Fbar, const double* H, double c, long long n,
                      cudaStream_t st);
void state_finalize_f64(const double* in, const double* P, const double* Q, double* out, long long n,
                        double sigma_r, double t_c, unsigned long long* d_fb, cudaStream_t st);

void run_exp_cr_f64(const double* d_x, double* d_y, long long n, cudaStream_t st);

// Drop-in fp64 host entry (dropin.cpp): gpf_filter_gpf and gpfilter::gpf.
// Per device: an LRU of fp32 plans, the fp64 workspace, device in/out
// buffers and a stream, reused across calls (a repeated call allocates
// nothing). Precision: kPrecFp32 = the fp32 plane kernels, kPrecFp64 = the
// reference-exact fp64 replay, kPrecAuto = fp64 exactly when the frame lies
// outside the envelope where the fp32 kernels are validated against the
// reference (max |H| = max(f_max - t_c, t_c - f_min) / sigma_r > kH32Limit),
// or when the degree exceeds the fp32 kernels' limit.
enum Precision { kPrecAuto = 0, kPrecFp32 = 1, kPrecFp64 = 2 };
extern const double kH32Limit;          // the envelope at the default degree N = 20
double fp32_h_limit(int degree);        // the envelope at degree N (dropin.cpp)
void set_precision(int mode);
int get_precision();
int last_precision();       // mode this thread's last drop-in call ran (1 or 2; 0 = none)
double last_max_abs_h();    // max |H| this thread's last drop-in call measured (auto mode)
float last_device_ms();     // device time of its filter kernels (CUDA events; copies excluded)
long long dropin_gpf(const double* h_in, double* h_out, const Params& p);  // throws Error
void dropin_release();

// Single-plane recursive Gaussian (gpf_gaussian_recursive), fp64 in/out.
void run_gaussian_f64(const double* d_in, double* d_out, double* d_tmp, int w, int h,
                      double sigma_s, double scale, cudaStream_t st);

// The direct (windowed) backend in fp64 (direct.cu): `planes` images of w x h
// (plane stride w h) d_src -> d_dst through d_tmp (d_dst may alias d_src),
// bitwise the reference's direct_gaussian (spatial.cpp:112-129).
void run_direct_gaussian_f64(const double* d_src, double* d_dst, double* d_tmp, int w, int h,
                             int planes, double sigma_s, double kernel_scale, int window_radius,
                             int boundary, cudaStream_t st);
// Scalar range-kernel evaluators (range_kernel.cpp; host fp64, throw Error{1, ...})
double kernel_gauss(double t, double tau, double sigma_r);
double kernel_gauss_poly(double t, double tau, double sigma_r, int degree);
double kernel_taylor(double t, double tau, double sigma_r, int degree);
double kernel_sup_error(double sigma_r, int degree, double tau, double low, double high, double step,
                        int taylor);
// F[p] = H^p F0, p < planes, by step()'s multiply chain (bilateral.cpp:108-129)
void direct_gen_planes_f64(const double* H, const double* F0, double* F, long long n, int planes,
                           cudaStream_t st);

}  // namespace gpfb
