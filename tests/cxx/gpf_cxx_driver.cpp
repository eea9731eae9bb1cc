// TEST INFRASTRUCTURE: one program, compiled twice -- against the reference's
// C++ core (proj/src/core/bilateral.hpp, linked with oracle/_ref's library;
// oracle/Makefile) and against the B200 library's C++ entry point
// (include/gpfilter/gpfilter.hpp; paper_1505_00077_b200/Makefile) -- so that
// tests/test_cxx_api.py runs the same gpfilter::gpf call through both.
//
//   driver IN.raw W H OUT.raw SIGMA_S SIGMA_R DEGREE CENTERING MODE LOW HIGH BACKEND
//          KERNEL_SCALE WINDOW_RADIUS [state:K]
// IN/OUT: W*H little-endian doubles; MODE mean|midpoint; BACKEND direct|recursive.
// Prints "ok <fallback_count>" or "error <exception type> <message>".
// With state:K the run goes through GpfState (init, K steps, finalize) and OUT
// holds the doubles t_c, c, n, then the images G, F, Fbar, P, Q, H, then the
// finalize image. With fn:NAME (exact|taylor|direct|recursive|misc) the named
// core function runs instead of gpf (misc: OUT = mean_intensity, kernel_mass_1d,
// compare(img, shift(img, 1.5), 1).{mse, mse_db, max_abs, pixels}, max_abs_diff,
// gaussian_range / gauss_polynomial / taylor_polynomial / sup_error x 2 at fixed
// arguments).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#ifdef GPF_B200
#include "gpfilter/gpfilter.hpp"
#else
#include "core/bilateral.hpp"
#include "core/metrics.hpp"
#endif

using namespace gpfilter;

int main(int argc, char** argv) {
  if (argc != 15 && argc != 16) {
    std::fprintf(stderr, "usage: see source\n");
    return 2;
  }
  const int w = std::atoi(argv[2]), h = std::atoi(argv[3]);
  SpatialParams sp;
  sp.sigma_s = std::atof(argv[5]);
  sp.kernel_scale = std::atof(argv[13]);
  sp.window_radius = std::atoi(argv[14]);
  RangeParams rp;
  rp.sigma_r = std::atof(argv[6]);
  rp.degree = std::atoi(argv[7]);
  GpfOptions opts;
  opts.centering = std::atoi(argv[8]) != 0;
  opts.mode = std::strcmp(argv[9], "midpoint") == 0 ? CenteringMode::midpoint : CenteringMode::mean;
  opts.range.low = std::atof(argv[10]);
  opts.range.high = std::atof(argv[11]);
  const SpatialBackend be =
      std::strcmp(argv[12], "direct") == 0 ? SpatialBackend::direct : SpatialBackend::recursive;
  try {
    Image img;
    if (w > 0 && h > 0) {
      img = Image(w, h);
      FILE* f = std::fopen(argv[1], "rb");
      if (!f || std::fread(img.data(), sizeof(double), img.pixels(), f) != img.pixels()) return 3;
      std::fclose(f);
    }
    if (argc == 16 && std::strncmp(argv[15], "fn:", 3) == 0) {
      const std::string fn = argv[15] + 3;
      FILE* o = std::fopen(argv[4], "wb");
      long long fb = 0;
      if (fn == "misc") {
        const ErrorReport rep = compare(img, shift(img, 1.5), 1);
        const IntensityRange rg{opts.range.low, opts.range.high};
        const double v[12] = {mean_intensity(img), kernel_mass_1d(sp.sigma_s, sp.window_radius), rep.mse,
                              rep.mse_db, rep.max_abs, static_cast<double>(rep.pixels),
                              max_abs_diff(img, shift(img, -2.25)), gaussian_range(100.0, 40.0, rp),
                              gauss_polynomial(100.0, 40.0, rp), taylor_polynomial(100.0, 40.0, rp),
                              sup_error(rp, 40.0, rg, 0.5, RangeApprox::gauss_polynomial),
                              sup_error(rp, 40.0, rg, 0.5, RangeApprox::taylor)};
        std::fwrite(v, sizeof(double), 12, o);
      } else {
        Image out;
        if (fn == "exact") out = exact_bilateral(img, sp, rp);
        else if (fn == "direct") out = direct_gaussian(img, sp);
        else if (fn == "recursive") out = recursive_gaussian(img, sp.sigma_s, sp.kernel_scale);
        else {
          FilterResult r = taylor_bilateral(img, sp, rp, be);
          out = r.image;
          fb = r.fallback_count;
        }
        std::fwrite(out.data(), sizeof(double), out.pixels(), o);
      }
      std::fclose(o);
      std::printf("ok %lld\n", fb);
      return 0;
    }
    if (argc == 16) {
      const int steps = std::atoi(argv[15] + 6);
      GpfState st = GpfState::init(img, sp, rp, be, opts);
      for (int k = 0; k < steps; ++k) st.step();
      const FilterResult r = st.finalize(img);
      FILE* o = std::fopen(argv[4], "wb");
      const double head[3] = {st.t_c, st.c, static_cast<double>(st.n)};
      std::fwrite(head, sizeof(double), 3, o);
      const Image* dump[7] = {&st.G, &st.F, &st.Fbar, &st.P, &st.Q, &st.H, &r.image};
      for (const Image* im : dump)
        std::fwrite(im->data(), sizeof(double), im->pixels(), o);
      std::fclose(o);
      std::printf("ok %lld\n", r.fallback_count);
      return 0;
    }
    const FilterResult r = gpf(img, sp, rp, be, opts);
    FILE* o = std::fopen(argv[4], "wb");
    std::fwrite(r.image.data(), sizeof(double), r.image.pixels(), o);
    std::fclose(o);
    std::printf("ok %lld\n", r.fallback_count);
  } catch (const SigmaTooSmallError& e) {
    std::printf("error SigmaTooSmallError %s\n", e.what());
  } catch (const std::invalid_argument& e) {
    std::printf("error invalid_argument %s\n", e.what());
  } catch (const std::exception& e) {
    std::printf("error runtime_error %s\n", e.what());
  }
  return 0;
}
