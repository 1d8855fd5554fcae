// Drives libtomo_b200 through the reference-shaped C++ wrapper (include/tomo_b200.hpp):
// geometry -> make_direct_backend / make_fused_backend -> apply_normal / split_bregman_tv, exactly as a caller of
// the reference library (proj/include/tomo/normal_ops.hpp, solver.hpp) would. Writes the
// results as raw doubles for tests/test_cpp_wrapper.py to compare with the oracle.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <vector>

#include "tomo_b200.hpp"

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  using namespace tomo_b200;
  Geometry g = Geometry::preset(32, 25, 6);
  NormalBackend op = make_direct_backend(g);
  std::vector<Complex> u(32 * 32);
  for (size_t i = 0; i < u.size(); ++i) u[i] = Complex(std::sin(0.37 * i), std::cos(0.11 * i));
  std::vector<Complex> nu = apply_normal(op, u);
  std::vector<Complex> f = forward(op, u);
  SolverConfig cfg;
  cfg.alpha = 10.0;
  cfg.lambda = 1.0;
  cfg.max_bregman_iters = 4;
  cfg.cg_steps_per_update = 5;
  cfg.update_tol_rel = 0.0;
  auto [mu, trace] = split_bregman_tv(op, f, cfg);
  std::ofstream os(argv[1], std::ios::binary);
  os.write(reinterpret_cast<const char*>(nu.data()), sizeof(Complex) * nu.size());
  os.write(reinterpret_cast<const char*>(mu.data()), sizeof(double) * mu.size());
  NormalBackend fused = make_fused_backend(g);
  std::vector<Complex> nf = apply_normal(fused, u);
  os.write(reinterpret_cast<const char*>(nf.data()), sizeof(Complex) * nf.size());
  bool threw = false;
  try {
    Geometry bad = Geometry::preset(30, 4, 6);  // m = 60: not a power of two
    NormalBackend b2 = make_direct_backend(bad);
  } catch (const ConfigError&) {
    threw = true;
  }
  std::printf("iterations %d leak %.3e config_error %d\n", trace.iterations, trace.imag_leakage, threw ? 1 : 0);
  return threw ? 0 : 1;
}
