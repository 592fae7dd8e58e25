// Reference-shaped calls on the C++ shim: pcg_jacobi / CsrMatrix::multiply on
// a caller matrix (proj/tests/test_sparse.cpp's 2x2 system) and the observers
// (total_temperature, boundary_flux_profile + integrated_abs_flux) after a few
// steps of a config; with a second (non-separable) config, its assembled
// reduced operator through the shim (a GPU product checked against a host one
// summed in CSR order) and the geometry tooling. Prints one line per check;
// exit code 0 when all pass.
#include <cmath>
#include <cstdio>

#include "thermiga_b200.hpp"

namespace tb = thermiga_b200;

int main(int argc, char** argv) {
  try {
    tb::CsrMatrix A;
    A.rows = A.cols = 2;
    A.row_ptr = {0, 2, 4};
    A.col_idx = {0, 1, 0, 1};
    A.vals = {4.0, 1.0, 1.0, 3.0};
    std::vector<double> b{1.0, 2.0}, x{0.0, 0.0};
    const auto r = tb::pcg_jacobi(A, b, x);
    const bool ok1 = std::abs(x[0] - 1.0 / 11.0) <= 1e-10 && std::abs(x[1] - 7.0 / 11.0) <= 1e-10;
    std::vector<double> y;
    A.multiply(x, y);
    std::printf("pcg 2x2: x = %.15g %.15g its %d  Ax = %.15g %.15g  %s\n", x[0], x[1],
                r.iterations, y[0], y[1], ok1 ? "ok" : "FAIL");
    bool ok2 = false;
    try {
      std::vector<double> x2{0.0, 0.0};
      tb::pcg_jacobi(A, b, x2, {1e-14, 1});
    } catch (const tb::numeric_error& e) {
      // the reference's numeric_error prefixes "numeric error: " (core.hpp:78-80)
      ok2 = std::string(e.what()) ==
            "numeric error: pcg: no convergence in 1 iterations, relative residual 1";
      if (!ok2) std::printf("  numeric_error: %s\n", e.what());
    } catch (const std::exception& e) {
      std::printf("  other exception: %s\n", e.what());
    }
    std::printf("cap raises numeric_error: %s\n", ok2 ? "ok" : "FAIL");
    bool ok3 = true;
    if (argc > 1) {
      tb::Simulation sim(argv[1]);
      int steps = 0;
      tb::State last;
      sim.run_time_loop([&](const tb::State& s) {
        last = s;
        ++steps;
      });
      const auto T = sim.total_temperature({{0.5, 0.5, 1.0}, {0.25, 0.5, 0.5}});
      const auto prof = sim.boundary_flux_profile(2, 21);
      const auto m = tb::integrated_abs_flux(prof);
      ok3 = T.size() == 2 && std::isfinite(T[0]) && prof.samples.size() == 21 &&
            m.integral_analytic >= 0.0;
      std::printf("observers after %d states: T = %.10g %.10g, |q| integral %.6g  %s\n", steps,
                  T[0], T[1], m.integral_net, ok3 ? "ok" : "FAIL");
    }
    bool ok4 = true;
    if (argc > 2) {
      tb::Simulation sim(argv[2]);
      const tb::CsrMatrix Aff = sim.reduced_operator();
      std::vector<double> v(Aff.cols), gpu;
      for (int i = 0; i < Aff.cols; ++i) v[i] = std::sin(0.37 * i);
      Aff.multiply(v, gpu);
      int bad = 0;
      for (int r2 = 0; r2 < Aff.rows; ++r2) {
        double acc = 0.0;
        for (int k = Aff.row_ptr[r2]; k < Aff.row_ptr[r2 + 1]; ++k)
          acc += Aff.vals[k] * v[Aff.col_idx[k]];
        bad += acc != gpu[r2];
      }
      const std::string geo = std::string(argc > 3 ? argv[3] : "/tmp") + "/qc3.geo";
      const std::string src = std::string(argc > 3 ? argv[3] : "/tmp") + "/qc.geo";
      if (FILE* f = std::fopen(src.c_str(), "w")) {
        std::fputs("[geometry]\ncase = quarter_cylinder\n", f);
        std::fclose(f);
      }
      const int up[3] = {1, 2, 2};
      tb::elevate_geometry(src, geo, up);
      FILE* g = std::fopen(geo.c_str(), "r");
      char line[128] = {0};
      bool deg3 = false;
      while (g && std::fgets(line, sizeof(line), g))
        if (std::string(line) == "degrees = 3 3 3\n") deg3 = true;
      if (g) std::fclose(g);
      ok4 = bad == 0 && deg3;
      std::printf("reduced operator %d rows, GPU rows == host CSR-order rows: %d mismatches; "
                  "elevated geometry degree 3: %s  %s\n",
                  Aff.rows, bad, deg3 ? "yes" : "no", ok4 ? "ok" : "FAIL");
    }
    return ok1 && ok2 && ok3 && ok4 ? 0 : 1;
  } catch (const tb::config_error& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
