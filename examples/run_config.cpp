// Example host program: the reference's `thermiga simulate` hot loop through
// the C++ shim (include/thermiga_b200.hpp). Build:
//   g++ -std=c++17 -O2 -Iinclude examples/run_config.cpp \
//       -Lpaper_2511_20432_b200/_lib -lthermiga_b200 -Wl,-rpath,$PWD/paper_2511_20432_b200/_lib
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "thermiga_b200.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s config.cfg\n", argv[0]);
    return 1;
  }
  try {
    thermiga_b200::Simulation sim(argv[1]);
    double peak = 0.0;
    std::vector<double> last;
    long iters = 0;
    if (argc > 2 && std::string(argv[2]) == "free") {
      // the reference's own loop (driver.cpp:126-145) over the free-function
      // shim: assemble_flux_load, dirichlet_values, theta_step
      namespace tb = thermiga_b200;
      const auto boundary = tb::boundary_sets(sim);
      const auto system = tb::dirichlet_system(sim);
      const auto sources = sim.sources();
      const auto mat = sim.material();
      const auto opts = sim.superpose_options();
      std::vector<double> load_n, load_np1;
      tb::assemble_flux_load(boundary, sources, mat, 0.0, -1.0, load_n, opts);
      tb::State state{std::vector<double>(sim.n_free, 0.0),
                      tb::dirichlet_values(boundary, sources, mat, 0.0, opts), 0, 0.0};
      const tb::PcgOptions po{sim.tol, sim.max_iter};
      for (int s = 1; s <= sim.n_steps; ++s) {
        const double t1 = s * sim.dt_solver;
        tb::assemble_flux_load(boundary, sources, mat, t1, -1.0, load_np1, opts);
        const auto g1 = tb::dirichlet_values(boundary, sources, mat, t1, opts);
        tb::PcgResult r{};
        state = tb::theta_step(system, state, load_n, load_np1, g1, po, &r);
        iters += r.iterations;
        std::swap(load_n, load_np1);
        for (double v : state.free_coeffs) peak = v > peak ? v : peak;
      }
      last = state.free_coeffs;
    } else {
      iters = sim.run_time_loop([&](const thermiga_b200::State& s) {
        for (double v : s.free_coeffs) peak = v > peak ? v : peak;
        last = s.free_coeffs;
      });
    }
    double amax = 0.0, l2 = 0.0;
    for (double v : last) {
      amax = std::fmax(amax, std::fabs(v));
      l2 += v * v;
    }
    std::printf("steps %d  cg iterations %ld  max correction coefficient %.6e\n", sim.n_steps,
                iters, peak);
    std::printf("final free coefficients: max|x| %.17g  |x|_2 %.17g\n", amax, std::sqrt(l2));
  } catch (const thermiga_b200::config_error& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  } catch (const thermiga_b200::io_error& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 4;
  } catch (const thermiga_b200::numeric_error& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
