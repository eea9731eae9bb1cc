// gpf_b200: command-line front end of libgpfilter_b200 with the reference CLI's
// `filter`, `compare`, `kernel-error` and `bench` subcommands
// (proj/tools/gpf_cli.cpp:53-110, 112-137, 145-199, 200-285; SURVEY.md 8(f)
// row 4): same flags, same CSV protocol
//   method,backend,sigma_s,sigma_r,degree,pixels,repeats,median_seconds
// (only the filter call inside the clock; warm-up runs discarded; median of
// the timed runs), same "error: <flag>: <detail>" diagnostics;
// `kernel-error` writes "tau,approx,sup_error" rows.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "gpfilter/gpfilter.h"

namespace {

// Numbers in the reference's CSV style: integral values as "%.1f", otherwise
// the shortest "%g" rendering that reads back exactly.
std::string num(double v) {
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  char buf[64];
  if (v == std::floor(v) && std::fabs(v) <= 1e9) {
    std::snprintf(buf, sizeof buf, "%.1f", v);
    return buf;
  }
  for (int digits = 6; digits <= 17; ++digits) {
    std::snprintf(buf, sizeof buf, "%.*g", digits, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  return buf;
}

int fail(const char* flag, const std::string& detail) {
  std::fprintf(stderr, "error: %s: %s\n", flag, detail.c_str());
  return 1;
}

struct Img {
  gpf_image* p = nullptr;
  ~Img() { gpf_image_destroy(p); }
};

// --flag value pairs and bare --flags after the subcommand
struct Args {
  std::map<std::string, std::string> kv;
  std::set<std::string> flags;
  std::string bad;

  bool has(const char* k) const { return kv.count(k) != 0; }
  std::string str(const char* k, const std::string& dflt = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? dflt : it->second;
  }
};

Args parse(int argc, char** argv, int from, const std::set<std::string>& bare) {
  Args a;
  for (int i = from; i < argc; ++i) {
    const std::string k = argv[i];
    if (k.rfind("--", 0) != 0) {
      a.bad = k;
      return a;
    }
    const size_t eq = k.find('=');
    if (eq != std::string::npos) {
      a.kv[k.substr(0, eq)] = k.substr(eq + 1);
    } else if (bare.count(k)) {
      a.flags.insert(k);
    } else if (i + 1 < argc) {
      a.kv[k] = argv[++i];
    } else {
      a.bad = k;
      return a;
    }
  }
  return a;
}

bool to_double(const std::string& s, double* v) {
  char* end = nullptr;
  *v = std::strtod(s.c_str(), &end);
  return !s.empty() && end && *end == '\0';
}

bool to_int(const std::string& s, int* v) {
  char* end = nullptr;
  const long x = std::strtol(s.c_str(), &end, 10);
  *v = static_cast<int>(x);
  return !s.empty() && end && *end == '\0';
}

std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  size_t at = 0;
  while (true) {
    const size_t c = s.find(',', at);
    out.push_back(s.substr(at, c == std::string::npos ? std::string::npos : c - at));
    if (c == std::string::npos) break;
    at = c + 1;
  }
  return out;
}

gpf_backend backend_of(const std::string& s) {
  return s == "direct" ? GPF_BACKEND_DIRECT : GPF_BACKEND_RECURSIVE;
}

gpf_boundary boundary_of(const std::string& s) {
  if (s == "reflect") return GPF_BOUNDARY_REFLECT;
  if (s == "zero") return GPF_BOUNDARY_ZERO;
  return GPF_BOUNDARY_REPLICATE;
}

// One filter call of `method` (exact / gpf / taylor).
gpf_status run_method(const std::string& method, const gpf_image* in, const gpf_spatial_params& sp,
                      const gpf_range_params& rp, gpf_backend be, int centering,
                      long long* fallback, gpf_image** out) {
  if (method == "exact") return gpf_filter_exact(in, &sp, &rp, out);
  if (method == "gpf") return gpf_filter_gpf(in, &sp, &rp, be, centering, fallback, out);
  return gpf_filter_taylor(in, &sp, &rp, be, fallback, out);
}

bool is_method(const std::string& m) { return m == "exact" || m == "gpf" || m == "taylor"; }

int cmd_filter(const Args& a) {
  for (const char* k : {"--input", "--output", "--method", "--sigma-s", "--sigma-r"})
    if (!a.has(k)) return fail(k, "is required");
  const std::string method = a.str("--method");
  if (!is_method(method)) return fail("--method", "must be one of exact, gpf, taylor");
  gpf_spatial_params sp;
  gpf_range_params rp;
  gpf_spatial_params_init(&sp);
  gpf_range_params_init(&rp);
  if (!to_double(a.str("--sigma-s"), &sp.sigma_s) || !(sp.sigma_s > 0))
    return fail("--sigma-s", "must be a positive number");
  if (!to_double(a.str("--sigma-r"), &rp.sigma_r) || !(rp.sigma_r > 0))
    return fail("--sigma-r", "must be a positive number");
  rp.degree = 20;
  if (a.has("--degree") && (!to_int(a.str("--degree"), &rp.degree) || rp.degree < 0))
    return fail("--degree", "must be a non-negative integer");
  const std::string be = a.str("--backend", "recursive");
  if (be != "recursive" && be != "direct") return fail("--backend", "must be direct or recursive");
  if (a.has("--window") && (!to_int(a.str("--window"), &sp.window_radius) || sp.window_radius < 1))
    return fail("--window", "must be a positive integer");
  const std::string bd = a.str("--boundary", "replicate");
  if (bd != "replicate" && bd != "reflect" && bd != "zero")
    return fail("--boundary", "must be replicate, reflect or zero");
  sp.boundary = boundary_of(bd);
  int threads = 1;
  if (a.has("--threads") && (!to_int(a.str("--threads"), &threads) || threads < 1))
    return fail("--threads", "must be a positive integer");
  if (gpf_set_num_threads(threads) != GPF_OK) return fail("--threads", gpf_last_error());
  Img in, out;
  if (gpf_read_pgm(a.str("--input").c_str(), &in.p) != GPF_OK) return fail("--input", gpf_last_error());
  long long fallback = 0;
  const gpf_status st = run_method(method, in.p, sp, rp, backend_of(be),
                                   a.flags.count("--no-centering") ? 0 : 1, &fallback, &out.p);
  if (st == GPF_ERR_SIGMA_TOO_SMALL) return fail("--sigma-s", gpf_last_error());
  if (st != GPF_OK) return fail("--method", gpf_last_error());
  if (gpf_write_pgm(out.p, a.str("--output").c_str()) != GPF_OK) return fail("--output", gpf_last_error());
  if (fallback > 0) std::fprintf(stderr, "fallback pixels: %lld\n", fallback);
  return 0;
}

int cmd_compare(const Args& a) {
  for (const char* k : {"--ref", "--test"})
    if (!a.has(k)) return fail(k, "is required");
  int border = 0;
  if (a.has("--exclude-border") && (!to_int(a.str("--exclude-border"), &border) || border < 0))
    return fail("--exclude-border", "must be a non-negative integer");
  Img ref, test;
  if (gpf_read_pgm(a.str("--ref").c_str(), &ref.p) != GPF_OK) return fail("--ref", gpf_last_error());
  if (gpf_read_pgm(a.str("--test").c_str(), &test.p) != GPF_OK) return fail("--test", gpf_last_error());
  gpf_error_report rep;
  if (gpf_compare(ref.p, test.p, border, &rep) != GPF_OK) return fail("--test", gpf_last_error());
  std::printf("mse=%s mse_db=%s max_abs=%s pixels=%lld\n", num(rep.mse).c_str(), num(rep.mse_db).c_str(),
              num(rep.max_abs).c_str(), rep.pixels);
  return 0;
}

// kernel-error: sup |exact - approximation| of the range kernel per tau
// (reference gpf kernel-error, proj/tools/gpf_cli.cpp:145-199): CSV
// "tau,approx,sup_error", approx in {gp, taylor}, rows in tau order, gp first.
int cmd_kernel_error(const Args& a) {
  for (const char* k : {"--sigma-r", "--degree", "--tau-list", "--range", "--step", "--which", "--csv"})
    if (!a.has(k)) return fail(k, "is required");
  double sigma_r, step, lo, hi;
  int degree;
  if (!to_double(a.str("--sigma-r"), &sigma_r) || !(sigma_r > 0)) return fail("--sigma-r", "must be a positive number");
  if (!to_int(a.str("--degree"), &degree) || degree < 0) return fail("--degree", "must be a non-negative integer");
  if (!to_double(a.str("--step"), &step) || !(step > 0)) return fail("--step", "must be a positive number");
  const std::string which = a.str("--which");
  if (which != "gp" && which != "taylor" && which != "both") return fail("--which", "must be one of gp, taylor, both");
  std::vector<double> taus;
  for (const auto& t : split(a.str("--tau-list"))) {
    double v;
    if (!to_double(t, &v)) return fail("--tau-list", "must be numbers");
    taus.push_back(v);
  }
  const std::string range = a.str("--range");
  const size_t colon = range.find(':');
  if (colon == std::string::npos || !to_double(range.substr(0, colon), &lo) ||
      !to_double(range.substr(colon + 1), &hi) || !(lo < hi))
    return fail("--range", "expected LO:HI with LO < HI");
  FILE* csv = std::fopen(a.str("--csv").c_str(), "w");
  if (!csv) return fail("--csv", "cannot open for writing");
  std::fprintf(csv, "tau,approx,sup_error\n");
  for (const double tau : taus) {
    for (const gpf_range_approx ap : {GPF_RANGE_APPROX_GAUSS_POLY, GPF_RANGE_APPROX_TAYLOR}) {
      if (which != "both" && (which == "gp") != (ap == GPF_RANGE_APPROX_GAUSS_POLY)) continue;
      double sup = 0.0;
      if (gpf_kernel_sup_error(sigma_r, degree, tau, lo, hi, step, ap, &sup) != GPF_OK) {
        std::fclose(csv);
        return fail("--range", gpf_last_error());
      }
      std::fprintf(csv, "%s,%s,%s\n", num(tau).c_str(), ap == GPF_RANGE_APPROX_GAUSS_POLY ? "gp" : "taylor",
                   num(sup).c_str());
    }
  }
  if (std::fclose(csv) != 0) return fail("--csv", "write failure");
  return 0;
}

int cmd_bench(const Args& a) {
  for (const char* k : {"--input", "--method", "--sigma-s-list", "--sigma-r", "--degree", "--backend", "--csv"})
    if (!a.has(k)) return fail(k, "is required");
  const std::vector<std::string> methods = split(a.str("--method"));
  for (const auto& m : methods)
    if (!is_method(m)) return fail("--method", "must be one of exact, gpf, taylor");
  std::vector<double> sigmas;
  for (const auto& t : split(a.str("--sigma-s-list"))) {
    double v;
    if (!to_double(t, &v) || !(v > 0)) return fail("--sigma-s-list", "must be positive numbers");
    sigmas.push_back(v);
  }
  gpf_range_params rp;
  gpf_range_params_init(&rp);
  if (!to_double(a.str("--sigma-r"), &rp.sigma_r) || !(rp.sigma_r > 0))
    return fail("--sigma-r", "must be a positive number");
  if (!to_int(a.str("--degree"), &rp.degree) || rp.degree < 0)
    return fail("--degree", "must be a non-negative integer");
  const std::string be = a.str("--backend");
  if (be != "recursive" && be != "direct") return fail("--backend", "must be direct or recursive");
  int repeats = 5, warmup = 1, threads = 1;
  if (a.has("--repeats") && (!to_int(a.str("--repeats"), &repeats) || repeats < 1))
    return fail("--repeats", "must be a positive integer");
  if (a.has("--warmup") && (!to_int(a.str("--warmup"), &warmup) || warmup < 0))
    return fail("--warmup", "must be a non-negative integer");
  if (a.has("--threads") && (!to_int(a.str("--threads"), &threads) || threads < 1))
    return fail("--threads", "must be a positive integer");
  if (gpf_set_num_threads(threads) != GPF_OK) return fail("--threads", gpf_last_error());
  Img in;
  if (gpf_read_pgm(a.str("--input").c_str(), &in.p) != GPF_OK) return fail("--input", gpf_last_error());
  const long long pixels = static_cast<long long>(gpf_image_width(in.p)) * gpf_image_height(in.p);
  std::FILE* csv = std::fopen(a.str("--csv").c_str(), "w");
  if (!csv) return fail("--csv", "cannot open for writing");
  std::fprintf(csv, "method,backend,sigma_s,sigma_r,degree,pixels,repeats,median_seconds\n");
  for (const auto& method : methods) {
    for (const double ss : sigmas) {
      gpf_spatial_params sp;
      gpf_spatial_params_init(&sp);
      sp.sigma_s = ss;
      std::vector<double> secs;
      for (int i = 0; i < warmup + repeats; ++i) {
        Img out;
        const auto t0 = std::chrono::steady_clock::now();
        const gpf_status st = run_method(method, in.p, sp, rp, backend_of(be), 1, nullptr, &out.p);
        const auto t1 = std::chrono::steady_clock::now();
        if (st == GPF_ERR_SIGMA_TOO_SMALL) {
          std::fclose(csv);
          return fail("--sigma-s-list", gpf_last_error());
        }
        if (st != GPF_OK) {
          std::fclose(csv);
          return fail("--method", gpf_last_error());
        }
        if (i >= warmup) secs.push_back(std::chrono::duration<double>(t1 - t0).count());
      }
      std::sort(secs.begin(), secs.end());
      const size_t n = secs.size();
      const double median = n % 2 ? secs[n / 2] : 0.5 * (secs[n / 2 - 1] + secs[n / 2]);
      std::fprintf(csv, "%s,%s,%s,%s,%d,%lld,%d,%s\n", method.c_str(), be.c_str(), num(ss).c_str(),
                   num(rp.sigma_r).c_str(), rp.degree, pixels, repeats, num(median).c_str());
    }
  }
  if (std::fclose(csv) != 0) return fail("--csv", "write failure");
  return 0;
}

void usage() {
  std::fprintf(stderr,
               "usage: gpf_b200 {filter|compare|kernel-error|bench} --flag value ...\n"
               "  filter  --input P --output P --method exact|gpf|taylor --sigma-s S --sigma-r R\n"
               "          [--degree N] [--backend recursive|direct] [--window W] [--boundary B]\n"
               "          [--no-centering] [--threads T]\n"
               "  compare --ref P --test P [--exclude-border B]\n"
               "  kernel-error --sigma-r R --degree N --tau-list T[,T..] --range LO:HI --step S\n"
               "          --which gp|taylor|both --csv P\n"
               "  bench   --input P --method M[,M..] --sigma-s-list S[,S..] --sigma-r R --degree N\n"
               "          --backend recursive|direct --csv P [--repeats K] [--warmup W] [--threads T]\n");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 2 && (!std::strcmp(argv[1], "--version"))) {
    std::printf("%s-b200\n", gpf_version());
    return 0;
  }
  if (argc < 2) {
    usage();
    return 1;
  }
  const std::string cmd = argv[1];
  const Args a = parse(argc, argv, 2, {"--no-centering"});
  if (!a.bad.empty()) return fail(a.bad.c_str(), "unexpected or incomplete argument");
  if (cmd == "filter") return cmd_filter(a);
  if (cmd == "compare") return cmd_compare(a);
  if (cmd == "bench") return cmd_bench(a);
  if (cmd == "kernel-error") return cmd_kernel_error(a);
  usage();
  return 1;
}
