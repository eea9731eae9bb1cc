/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the GPF hot path.
 *
 * A plain-C, fp64 restatement of the reference algorithm on the path
 * gpf_filter_gpf(..., GPF_BACKEND_RECURSIVE, ...) of arXiv 1505.00077's
 * `gpfilter` library. Every function cites the reference file:line it
 * follows (paths relative to /root/reference/proj). Operation order is kept
 * identical so that, compiled with plain -O2 on x86-64 (no FMA contraction),
 * the results are bitwise equal to the reference library; tests pin this
 * against oracle/_ref/libgpfilter_ref.so and tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load this library, and only as the checker. The product path never does.
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- src/core/image.cpp:20-37  mean_intensity (Neumaier summation) ---- */
double oracle_mean(const double* p, long long n) {
  double sum = 0.0, comp = 0.0;
  for (long long i = 0; i < n; ++i) {
    const double t = sum + p[i];
    if (fabs(sum) >= fabs(p[i])) comp += (sum - t) + p[i];
    else comp += (p[i] - t) + sum;
    sum = t;
  }
  return (sum + comp) / (double)n;
}

/* ---- src/core/spatial.cpp:14-16 default_window_radius ---- */
int oracle_default_window_radius(double sigma_s) {
  return (int)ceil(3.0 * sigma_s);
}

/* ---- src/core/spatial.cpp:43-50 kernel_mass_1d ---- */
double oracle_kernel_mass_1d(double sigma_s, int radius) {
  double mass = 0.0;
  for (int k = -radius; k <= radius; ++k)
    mass += exp(-((double)k * k) / (2.0 * sigma_s * sigma_s));
  return mass;
}

/* ---- src/core/spatial.cpp:134-181 DericheCoeffs / deriche_coeffs ---- */
typedef struct { double nc[4], na[4], d[4]; } deriche_t;

void oracle_deriche_coeffs(double sigma, double nc[4], double na[4], double d[4]) {
  const double A1 = 1.6800, C1 = 3.7350, L1 = 1.7830, W1 = 0.6318;
  const double A2 = -0.6803, C2 = -0.2598, L2 = 1.7230, W2 = 1.9970;
  const double e1 = exp(-L1 / sigma), e2 = exp(-L2 / sigma);
  const double cw1 = cos(W1 / sigma), sw1 = sin(W1 / sigma);
  const double cw2 = cos(W2 / sigma), sw2 = sin(W2 / sigma);
  nc[0] = A1 + A2;
  nc[1] = e2 * (C2 * sw2 - (A2 + 2.0 * A1) * cw2) + e1 * (C1 * sw1 - (2.0 * A2 + A1) * cw1);
  nc[2] = 2.0 * e1 * e2 * ((A1 + A2) * cw2 * cw1 - C1 * cw2 * sw1 - C2 * cw1 * sw2) +
          A2 * e1 * e1 + A1 * e2 * e2;
  nc[3] = e2 * e1 * e1 * (C2 * sw2 - A2 * cw2) + e1 * e2 * e2 * (C1 * sw1 - A1 * cw1);
  d[0] = -2.0 * e2 * cw2 - 2.0 * e1 * cw1;
  d[1] = 4.0 * cw2 * cw1 * e1 * e2 + e1 * e1 + e2 * e2;
  d[2] = -2.0 * cw1 * e1 * e2 * e2 - 2.0 * cw2 * e2 * e1 * e1;
  d[3] = e1 * e1 * e2 * e2;
  for (int i = 0; i < 3; ++i) na[i] = nc[i + 1] - d[i] * nc[0];
  na[3] = -d[3] * nc[0];
  double num = 0.0, den = 1.0;
  for (int i = 0; i < 4; ++i) { num += nc[i] + na[i]; den += d[i]; }
  const double dc = num / den;
  for (int i = 0; i < 4; ++i) { nc[i] /= dc; na[i] /= dc; }
}

/* ---- src/core/spatial.cpp:186-216 deriche_line (replicate steady state) ---- */
static void deriche_line(const double* src, double* dst, int n, long long stride,
                         const deriche_t* k) {
  const double den_sum = 1.0 + k->d[0] + k->d[1] + k->d[2] + k->d[3];
  const double x0 = src[0];
  double ss = x0 * (k->nc[0] + k->nc[1] + k->nc[2] + k->nc[3]) / den_sum;
  double xm1 = x0, xm2 = x0, xm3 = x0;
  double ym1 = ss, ym2 = ss, ym3 = ss, ym4 = ss;
  for (int i = 0; i < n; ++i) {
    const double xi = src[i * stride];
    const double yi = k->nc[0] * xi + k->nc[1] * xm1 + k->nc[2] * xm2 + k->nc[3] * xm3 -
                      k->d[0] * ym1 - k->d[1] * ym2 - k->d[2] * ym3 - k->d[3] * ym4;
    dst[i * stride] = yi;
    xm3 = xm2; xm2 = xm1; xm1 = xi;
    ym4 = ym3; ym3 = ym2; ym2 = ym1; ym1 = yi;
  }
  const double xl = src[(long long)(n - 1) * stride];
  ss = xl * (k->na[0] + k->na[1] + k->na[2] + k->na[3]) / den_sum;
  double xp1 = xl, xp2 = xl, xp3 = xl, xp4 = xl;
  double yp1 = ss, yp2 = ss, yp3 = ss, yp4 = ss;
  for (int i = n - 1; i >= 0; --i) {
    const double yi = k->na[0] * xp1 + k->na[1] * xp2 + k->na[2] * xp3 + k->na[3] * xp4 -
                      k->d[0] * yp1 - k->d[1] * yp2 - k->d[2] * yp3 - k->d[3] * yp4;
    dst[i * stride] += yi;
    xp4 = xp3; xp3 = xp2; xp2 = xp1; xp1 = src[i * stride];
    yp4 = yp3; yp3 = yp2; yp2 = yp1; yp1 = yi;
  }
}

/* Worker pool over lines (the reference's parallel_for, src/core/parallel.hpp:27-47:
 * static contiguous chunks, disjoint writes => bitwise identical for any count). */
typedef struct {
  const double* src; double* dst; int n_lines, len; long long line_step, stride;
  const deriche_t* k; int lo, hi;
} lines_job;

static void* lines_worker(void* arg) {
  lines_job* j = (lines_job*)arg;
  for (int l = j->lo; l < j->hi; ++l)
    deriche_line(j->src + (long long)l * j->line_step, j->dst + (long long)l * j->line_step,
                 j->len, j->stride, j->k);
  return NULL;
}

static void run_lines(const double* src, double* dst, int n_lines, int len, long long line_step,
                      long long stride, const deriche_t* k, int threads) {
  if (threads < 1) threads = 1;
  if (threads > n_lines) threads = n_lines;
  pthread_t tid[256];
  lines_job jobs[256];
  if (threads > 256) threads = 256;
  const int chunk = (n_lines + threads - 1) / threads;
  int launched = 0;
  for (int w = 0; w < threads; ++w) {
    const int lo = w * chunk, hi = lo + chunk < n_lines ? lo + chunk : n_lines;
    if (lo >= hi) break;
    jobs[w] = (lines_job){src, dst, n_lines, len, line_step, stride, k, lo, hi};
    if (w == 0) continue;
    pthread_create(&tid[w], NULL, lines_worker, &jobs[w]);
    launched = w;
  }
  if (n_lines > 0) lines_worker(&jobs[0]);
  for (int w = 1; w <= launched; ++w) pthread_join(tid[w], NULL);
}

/* ---- src/core/spatial.cpp:220-251 recursive_gaussian (rows, then columns,
 *      then x mass(sigma, ceil(3 sigma))^2 * kernel_scale) ----
 * Returns 0, or -1 (sigma/scale <= 0), or -3 (sigma < 0.5). */
int oracle_recursive_gaussian(const double* img, int w, int h, double sigma_s,
                              double kernel_scale, double* out, int threads) {
  if (!(sigma_s > 0.0) || !(kernel_scale > 0.0)) return -1;
  if (sigma_s < 0.5) return -3;
  deriche_t k;
  oracle_deriche_coeffs(sigma_s, k.nc, k.na, k.d);
  const size_t n = (size_t)w * h;
  double* tmp = (double*)calloc(n, sizeof(double));
  run_lines(img, tmp, h, w, w, 1, &k, threads);   /* rows: stride 1 */
  memset(out, 0, n * sizeof(double));
  run_lines(tmp, out, w, h, 1, w, &k, threads);   /* columns: stride w */
  free(tmp);
  const double mass = oracle_kernel_mass_1d(sigma_s, oracle_default_window_radius(sigma_s));
  const double scale = mass * mass * kernel_scale;
  for (size_t i = 0; i < n; ++i) out[i] *= scale;
  return 0;
}

/* ---- src/core/bilateral.cpp:64-158 GpfState::init/step/finalize + gpf ----
 * Recursive backend only. kQMin = 1e-8 (src/core/bilateral.hpp:85).
 * centering: 0 off, 1 mean (image.cpp:20-37), 2 midpoint (low+high)/2.
 * Returns 0 ok, -1 invalid argument, -3 sigma too small. */
int oracle_gpf(const double* img, int w, int h, double sigma_s, double kernel_scale,
               double sigma_r, int degree, int centering, double mid_low, double mid_high,
               double* out, long long* fallbacks, double* t_c_out, int threads) {
  if (!(sigma_s > 0.0) || !(kernel_scale > 0.0)) return -1;
  if (!(sigma_r > 0.0) || degree < 0) return -1;
  if (w < 1 || h < 1) return -1;
  if (sigma_s < 0.5) return -3;
  const size_t n = (size_t)w * h;
  double t_c = 0.0;
  if (centering == 1) t_c = oracle_mean(img, (long long)n);
  else if (centering == 2) t_c = (mid_low + mid_high) / 2.0;
  if (t_c_out) *t_c_out = t_c;
  double* G = (double*)malloc(n * sizeof(double));
  double* P = (double*)calloc(n, sizeof(double));
  double* Q = (double*)calloc(n, sizeof(double));
  double* H = (double*)malloc(n * sizeof(double));
  double* F = (double*)malloc(n * sizeof(double));
  double* Fb = (double*)malloc(n * sizeof(double));
  const double inv2s2 = 1.0 / (2.0 * sigma_r * sigma_r);
  for (size_t i = 0; i < n; ++i) {
    G[i] = 1.0;
    const double hv = img[i] - t_c;
    H[i] = hv / sigma_r;
    F[i] = exp(-(hv * hv) * inv2s2);
  }
  oracle_recursive_gaussian(F, w, h, sigma_s, kernel_scale, Fb, threads);
  double c = 1.0;
  for (int s = 0; s <= degree; ++s) {
    for (size_t i = 0; i < n; ++i) {
      Q[i] += c * G[i] * Fb[i];
      F[i] = H[i] * F[i];
    }
    oracle_recursive_gaussian(F, w, h, sigma_s, kernel_scale, Fb, threads);
    for (size_t i = 0; i < n; ++i) {
      P[i] += c * G[i] * Fb[i];
      G[i] = H[i] * G[i];
    }
    c = c / (s + 1);
  }
  long long fb = 0;
  for (size_t i = 0; i < n; ++i) {
    if (fabs(Q[i]) <= 1e-8) { out[i] = img[i]; ++fb; }
    else out[i] = sigma_r * (P[i] / Q[i]) + t_c;
  }
  if (fallbacks) *fallbacks = fb;
  free(G); free(P); free(Q); free(H); free(F); free(Fb);
  return 0;
}


/* Diagnostic twin of oracle_gpf (same arithmetic, src/core/bilateral.cpp:64-158).
 * Also returns, per pixel, the cancellation factor of the truncated series
 *   kappa = sum_n |c G| R(|F_{n+1}|) / |P|  +  sum_n |c G| R(|F_n|) / |Q|
 * where R(|F|) filters the absolute plane: how much a relative rounding of the
 * plane samples (before the spatial sum) is amplified in the output ratio.
 * kappa ~ 1 for well-posed pixels; it explodes where the reference's own
 * degree-N series diverges (hard part 8). Used by the
 * parity tests to scale the tolerance honestly. */
int oracle_gpf_kappa(const double* img, int w, int h, double sigma_s, double kernel_scale,
                     double sigma_r, int degree, double* out, double* kappa, int threads) {
  if (!(sigma_s > 0.0) || !(kernel_scale > 0.0) || !(sigma_r > 0.0) || degree < 0) return -1;
  if (sigma_s < 0.5) return -3;
  const size_t n = (size_t)w * h;
  const double t_c = oracle_mean(img, (long long)n);
  double* G = (double*)malloc(n * sizeof(double));
  double* P = (double*)calloc(n, sizeof(double));
  double* Q = (double*)calloc(n, sizeof(double));
  double* aP = (double*)calloc(n, sizeof(double));
  double* aQ = (double*)calloc(n, sizeof(double));
  double* H = (double*)malloc(n * sizeof(double));
  double* F = (double*)malloc(n * sizeof(double));
  double* A = (double*)malloc(n * sizeof(double));
  double* Fb = (double*)malloc(n * sizeof(double));
  double* Ab = (double*)malloc(n * sizeof(double));
  const double inv2s2 = 1.0 / (2.0 * sigma_r * sigma_r);
  for (size_t i = 0; i < n; ++i) {
    G[i] = 1.0;
    const double hv = img[i] - t_c;
    H[i] = hv / sigma_r;
    F[i] = exp(-(hv * hv) * inv2s2);
    A[i] = fabs(F[i]);
  }
  oracle_recursive_gaussian(F, w, h, sigma_s, kernel_scale, Fb, threads);
  oracle_recursive_gaussian(A, w, h, sigma_s, kernel_scale, Ab, threads);
  double c = 1.0;
  for (int s = 0; s <= degree; ++s) {
    for (size_t i = 0; i < n; ++i) {
      Q[i] += c * G[i] * Fb[i];
      aQ[i] += fabs(c * G[i]) * fabs(Ab[i]);
      F[i] = H[i] * F[i];
      A[i] = fabs(F[i]);
    }
    oracle_recursive_gaussian(F, w, h, sigma_s, kernel_scale, Fb, threads);
    oracle_recursive_gaussian(A, w, h, sigma_s, kernel_scale, Ab, threads);
    for (size_t i = 0; i < n; ++i) {
      P[i] += c * G[i] * Fb[i];
      aP[i] += fabs(c * G[i]) * fabs(Ab[i]);
      G[i] = H[i] * G[i];
    }
    c = c / (s + 1);
  }
  for (size_t i = 0; i < n; ++i) {
    if (fabs(Q[i]) <= 1e-8) { out[i] = img[i]; kappa[i] = 0.0; }
    else {
      out[i] = sigma_r * (P[i] / Q[i]) + t_c;
      kappa[i] = (P[i] != 0.0 ? aP[i] / fabs(P[i]) : 0.0) + aQ[i] / fabs(Q[i]);
    }
  }
  free(G); free(P); free(Q); free(aP); free(aQ); free(H); free(F); free(A); free(Fb); free(Ab);
  return 0;
}

/* ---- src/core/spatial.cpp:37-41, 52-68: spatial_weight, boundary_index ---- */
static int boundary_index(int i, int n, int boundary) {
  if (i >= 0 && i < n) return i;
  if (boundary == 0) return i < 0 ? 0 : n - 1;
  if (boundary == 1) {
    const int period = 2 * n;
    int m = i % period;
    if (m < 0) m += period;
    return m < n ? m : period - 1 - m;
  }
  return -1;
}

/* ---- src/core/bilateral.cpp:14-56 exact_bilateral, evaluated at selected
 *      pixels (offset form; used for the MSE-vs-exact report on samples) ---- */
void oracle_exact_bilateral_at(const double* img, int w, int h, double sigma_s, int radius,
                               int boundary, double kernel_scale, double sigma_r,
                               const long long* idx, long long count, double* out) {
  const int W = radius, span = 2 * W + 1;
  double* ws = (double*)malloc(sizeof(double) * span * span);
  for (int a = -W; a <= W; ++a)
    for (int b = -W; b <= W; ++b) {
      const double r2 = (double)a * a + (double)b * b;
      ws[(a + W) * span + (b + W)] = kernel_scale * exp(-r2 / (2.0 * sigma_s * sigma_s));
    }
  const double inv2s2 = 1.0 / (2.0 * sigma_r * sigma_r);
  for (long long q = 0; q < count; ++q) {
    const int r = (int)(idx[q] / w), x = (int)(idx[q] % w);
    const double fc = img[(size_t)r * w + x];
    double num = 0.0, den = 0.0;
    for (int a = -W; a <= W; ++a) {
      const int rr = boundary_index(r + a, h, boundary);
      if (rr < 0) continue;
      for (int b = -W; b <= W; ++b) {
        const int cc = boundary_index(x + b, w, boundary);
        if (cc < 0) continue;
        const double d = img[(size_t)rr * w + cc] - fc;
        const double wgt = ws[(a + W) * span + (b + W)] * exp(-(d * d) * inv2s2);
        num += wgt * d;
        den += wgt;
      }
    }
    out[q] = fc + num / den;
  }
  free(ws);
}
