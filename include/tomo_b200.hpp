// tomo_b200.hpp — header-only C++ wrapper that re-exposes the reference's operator/solver API
// (proj/include/tomo/{normal_ops,solver,errors}.hpp) over the C ABI of libtomo_b200.so.
//
// Status codes become the reference's exception classes (errors.hpp:9-30); host vectors in,
// host vectors out (the library stages them through HBM), or raw device pointers for callers
// that keep data resident. Link with -ltomo_b200 (paper_1705_07497_b200/libtomo_b200.so).
#pragma once

#include <complex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tomo_b200.h"

namespace tomo_b200 {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
class NumericalError : public Error {
 public:
  using Error::Error;
};
class IoError : public Error {
 public:
  using Error::Error;
};
class CudaError : public Error {
 public:
  using Error::Error;
};

inline void check(int rc) {
  if (rc == TOMO_OK) return;
  const std::string msg = tomo_last_error();
  switch (rc) {
    case TOMO_ERR_CONFIG: throw ConfigError(msg);
    case TOMO_ERR_NUMERICAL: throw NumericalError(msg);
    case TOMO_ERR_IO: throw IoError(msg);
    case TOMO_ERR_CUDA: throw CudaError(msg);
    default: throw Error(msg);
  }
}

using Complex = std::complex<double>;

// SliceGrid + NufftParams; defaults are the reference's (n_b = n, R = 2, [-m_sp, m_sp],
// tau = m_sp / n^2, theta_a = a*pi/A).
struct Geometry {
  int n = 0, n_angles = 0, n_b = 0, oversample = 2, win_lo = -6, win_hi = 6;
  double tau = 0.0;
  std::vector<double> angles;  // optional

  static Geometry preset(int n, int n_angles, int m_sp) {
    Geometry g;
    g.n = n;
    g.n_angles = n_angles;
    g.win_lo = -m_sp;
    g.win_hi = m_sp;
    return g;
  }
  tomo_geom_desc desc() const {
    tomo_geom_desc d{};
    d.n = n;
    d.n_angles = n_angles;
    d.n_b = n_b;
    d.oversample = oversample;
    d.win_lo = win_lo;
    d.win_hi = win_hi;
    const int m_sp = win_hi > -win_lo ? win_hi : -win_lo;
    d.tau = tau > 0.0 ? tau : static_cast<double>(m_sp) / (static_cast<double>(n) * n);
    d.angles = angles.empty() ? nullptr : angles.data();
    return d;
  }
};

// tomo::SolverConfig (solver.hpp:51-65)
struct SolverConfig {
  double alpha = 1.0, lambda = 1.0;
  int max_bregman_iters = 6000, cg_steps_per_update = 5;
  double update_tol_rel = 1e-8;
  bool warm_start = true;
  bool data_feedback = false;  // solver.hpp:58-61
};

// tomo::SolveTrace subset (solver.hpp:67-80)
struct SolveTrace {
  std::vector<double> update_l1;
  int iterations = 0;
  std::string stopping_reason;
  double first_update_l1 = 0.0, stabilization_shift = 0.0, min_ritz = 0.0, imag_leakage = 0.0;
};

// tomo::NormalBackend (normal_ops.hpp:23-31): an fp64 device operator (the reference computes
// in fp64), W/W^T ("direct") or surrogate stencil.
class NormalBackend {
 public:
  NormalBackend(const Geometry& g, int backend, int surrogate_r = 1, int device = 0, int max_batch = 1,
                int64_t mem_cap_bytes = 0)
      : geom_(g) {
    tomo_geom_desc gd = g.desc();
    tomo_op_desc od{};
    od.backend = backend;
    od.surrogate_r = surrogate_r;
    od.device = device;
    od.max_batch = max_batch;
    od.precision = TOMO_F64;
    od.mem_cap_bytes = mem_cap_bytes;
    tomo_op* op = nullptr;
    check(tomo_op_create(&gd, &od, &op));
    op_.reset(op);
  }
  tomo_op* handle() const { return op_.get(); }
  const Geometry& geometry() const { return geom_; }
  int64_t points() const {
    tomo_op_info info{};
    check(tomo_op_get_info(op_.get(), &info));
    return info.P;
  }

 private:
  struct Del {
    void operator()(tomo_op* p) const { tomo_op_destroy(p); }
  };
  Geometry geom_;
  std::unique_ptr<tomo_op, Del> op_;
};

// make_direct_backend / make_fused_backend / make_surrogate_backend (normal_ops.hpp:35-39)
inline NormalBackend make_direct_backend(const Geometry& g, int device = 0) {
  return NormalBackend(g, TOMO_BACKEND_DIRECT, 1, device);
}
inline NormalBackend make_fused_backend(const Geometry& g, int64_t mem_cap_bytes = int64_t(8) << 30,
                                        int device = 0) {
  return NormalBackend(g, TOMO_BACKEND_FUSED, 1, device, 1, mem_cap_bytes);
}
inline NormalBackend make_surrogate_backend(const Geometry& g, int radius_r = 1, int device = 0) {
  return NormalBackend(g, TOMO_BACKEND_SURROGATE, radius_r, device);
}

// apply_normal (normal_ops.hpp:65)
inline std::vector<Complex> apply_normal(const NormalBackend& b, const std::vector<Complex>& image) {
  std::vector<Complex> out(image.size());
  check(tomo_apply_normal(b.handle(), image.data(), out.data(), 1, nullptr));
  return out;
}

// apply_normal_real (normal_ops.hpp:69)
inline std::vector<double> apply_normal_real(const NormalBackend& b, const std::vector<double>& u) {
  std::vector<double> out(u.size());
  check(tomo_apply_normal_real(b.handle(), u.data(), out.data(), 1, nullptr));
  return out;
}

// SliceTransform::forward / adjoint (fourier_slice.hpp:43,46)
inline std::vector<Complex> forward(const NormalBackend& b, const std::vector<Complex>& image) {
  std::vector<Complex> out(static_cast<size_t>(b.points()));
  check(tomo_forward(b.handle(), image.data(), out.data(), 1, nullptr));
  return out;
}
inline std::vector<Complex> adjoint(const NormalBackend& b, const std::vector<Complex>& samples) {
  const int n = b.geometry().n;
  std::vector<Complex> out(static_cast<size_t>(n) * n);
  check(tomo_adjoint(b.handle(), samples.data(), out.data(), 1, nullptr));
  return out;
}

// split_bregman_tv (solver.hpp:83-85)
inline std::pair<std::vector<double>, SolveTrace> split_bregman_tv(const NormalBackend& b,
                                                                   const std::vector<Complex>& slice_data,
                                                                   const SolverConfig& c) {
  const int n = b.geometry().n;
  tomo_sb_config cfg{c.alpha, c.lambda, c.max_bregman_iters, c.cg_steps_per_update, c.update_tol_rel,
                     c.warm_start ? 1 : 0, -1.0, c.data_feedback ? 1 : 0};
  std::vector<double> mu(static_cast<size_t>(n) * n), upd(c.max_bregman_iters);
  tomo_sb_trace tr{};
  check(tomo_split_bregman(b.handle(), &cfg, slice_data.data(), mu.data(), 1, upd.data(), &tr, nullptr));
  SolveTrace t;
  t.update_l1.assign(upd.begin(), upd.begin() + tr.iterations);
  t.iterations = tr.iterations;
  t.stopping_reason = tr.stopped_on_tolerance ? "tolerance" : "max_iterations";
  t.first_update_l1 = tr.first_update_l1;
  t.stabilization_shift = tr.sigma;
  t.min_ritz = tr.min_ritz;
  t.imag_leakage = tr.imag_leakage;
  return {std::move(mu), std::move(t)};
}

// tikhonov_solve with K = identity (solver.hpp:91-92) at a fixed step count / tolerance
inline std::vector<double> tikhonov_solve(const NormalBackend& b, const std::vector<Complex>& slice_data,
                                          double alpha, int steps = 5000, double rel_tol = 1e-8) {
  const int n = b.geometry().n;
  std::vector<double> mu(static_cast<size_t>(n) * n);
  check(tomo_tikhonov(b.handle(), alpha, slice_data.data(), mu.data(), steps, rel_tol, 1, nullptr));
  return mu;
}

}  // namespace tomo_b200
