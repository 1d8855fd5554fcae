// ref_driver.cpp — C entry points into the REFERENCE library itself (TEST INFRASTRUCTURE).
//
// Compiled together with the reference's unmodified sources from /root/reference/proj/src
// (image, fft, nufft, fourier_slice, sparse, normal_ops, solver) against the Eigen-API
// shim in oracle/eigen_shim, into oracle/_ref/libtomo_ref.so (recipe: oracle/Makefile,
// target `ref`). Every function below only calls the reference's public tomo:: API
// (proj/include/tomo/*.hpp); it exists so Python tests can pin the oracle restatement and
// generate golden vectors, and so bench.py --impl reference can time the reference.
//
// Geometry is the reference's own: n_b = n, R = 2, window [-m_sp, m_sp]; the angle set
// theta_a = a*pi/A is built through the public AngleSet struct (fourier_slice.hpp:12-17),
// which is what make_angle_set produces for count A (fourier_slice.cpp:18).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <memory>
#include <vector>
#include <string>

#include "tomo/fourier_slice.hpp"
#include "tomo/image.hpp"
#include "tomo/normal_ops.hpp"
#include "tomo/nufft.hpp"
#include "tomo/solver.hpp"
#include "tomo/sparse.hpp"

using namespace tomo;

namespace {
thread_local std::string g_err;

struct RefSetup {
  SliceGrid grid;
  NufftParams params;
  std::shared_ptr<const SliceTransform> transform;
};

thread_local int g_nb = 0;  // radial samples per angle for the next setup (0 -> n)
thread_local int g_feedback = 0;  // SolverConfig::data_feedback for the next ref_split_bregman

RefSetup make_setup(int n, int n_angles, int m_sp, double tau) {
  AngleSet set;
  set.subsample_d = 1;
  set.angles.resize(n_angles);
  for (int a = 0; a < n_angles; ++a) set.angles[a] = a * M_PI / n_angles;
  RefSetup s;
  s.params = tau > 0 ? make_params(m_sp, tau, n) : make_params(m_sp, static_cast<double>(m_sp) / (double(n) * n), n);
  const int nb = g_nb > 0 ? g_nb : n;
  if (nb == n) {
    s.grid = slice_points(set, n);
  } else {
    // Extension D1 (n_b != n radial samples): the same angle-major lattice as slice_points
    // (fourier_slice.cpp:22-41) with spacing 2*pi/n_b, fed through the reference's own
    // FrequencyPointSet::make and SliceTransform.
    Eigen::MatrixXd coords(static_cast<Eigen::Index>(n_angles) * nb, 2);
    Eigen::Index row = 0;
    for (int a = 0; a < n_angles; ++a) {
      const double c = std::cos(set.angles[a]), sn = std::sin(set.angles[a]);
      for (int t = 0; t < nb; ++t, ++row) {
        const double k_r = (2.0 * M_PI / nb) * (t - nb / 2);
        coords(row, 0) = k_r * c;
        coords(row, 1) = k_r * sn;
      }
    }
    s.grid.angle_set = set;
    s.grid.n = n;
    s.grid.points = FrequencyPointSet::make(2, std::move(coords));
  }
  s.transform = std::make_shared<const SliceTransform>(s.grid, s.params);
  return s;
}

ComplexVector cvec(const double* p, Eigen::Index len) {
  ComplexVector v(len);
  for (Eigen::Index i = 0; i < len; ++i) v[i] = Complex(p[2 * i], p[2 * i + 1]);
  return v;
}
void put(const ComplexVector& v, double* p) {
  for (Eigen::Index i = 0; i < v.size(); ++i) {
    p[2 * i] = v[i].real();
    p[2 * i + 1] = v[i].imag();
  }
}

int code_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  if (dynamic_cast<const NumericalError*>(&e)) return 3;
  if (dynamic_cast<const IoError*>(&e)) return 4;
  return 2;
}
}  // namespace

#define REF_TRY try {
#define REF_CATCH \
  return 0;       \
  }               \
  catch (const std::exception& e) { return code_of(e); }

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Radial samples per angle for subsequent calls on this thread (0 -> n, the reference).
void ref_set_nb(int nb) { g_nb = nb; }
// SolverConfig::data_feedback (solver.hpp:58-61) for subsequent ref_split_bregman calls.
void ref_set_feedback(int on) { g_feedback = on; }

int ref_points(int n, int A, int m_sp, double tau, double* coords) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  const auto& c = s.grid.points.coords;
  for (Eigen::Index j = 0; j < c.rows(); ++j) {
    coords[2 * j] = c(j, 0);
    coords[2 * j + 1] = c(j, 1);
  }
  REF_CATCH
}

int ref_plan(int n, int A, int m_sp, double tau, int* nearest, double* e1, double* e2, double* e3) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  const auto& p = s.transform->plan();
  for (Eigen::Index j = 0; j < p.points.count(); ++j)
    for (int d = 0; d < 2; ++d) {
      nearest[2 * j + d] = p.nearest_index(j, d);
      e1[2 * j + d] = p.e1(j, d);
      e2[2 * j + d] = p.e2(j, d);
    }
  for (int l = 0; l < 2 * m_sp + 1; ++l) e3[l] = p.e3[l];
  REF_CATCH
}

int ref_type2(int n, int A, int m_sp, double tau, const double* coeffs, double* samples) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  put(s.transform->forward(ComplexImage(n, cvec(coeffs, Eigen::Index(n) * n))), samples);
  REF_CATCH
}

int ref_type1(int n, int A, int m_sp, double tau, const double* samples, double* coeffs) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  put(s.transform->adjoint(cvec(samples, s.grid.points.count())).data, coeffs);
  REF_CATCH
}

int ref_direct_ndft(int n, int A, int m_sp, double tau, const double* in, double* out, int to_type1) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  const Eigen::Index len = to_type1 ? s.grid.points.count() : Eigen::Index(n) * n;
  put(direct_ndft(s.grid.points, n, cvec(in, len), to_type1 ? NdftDirection::type1 : NdftDirection::type2), out);
  REF_CATCH
}

// backend: 0 direct, 1 fused
int ref_apply_normal(int n, int A, int m_sp, double tau, int backend, const double* in, double* out) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  NormalBackend b = backend == 1 ? make_fused_backend(s.transform) : make_direct_backend(s.transform);
  put(apply_normal(b, ComplexImage(n, cvec(in, Eigen::Index(n) * n))).data, out);
  REF_CATCH
}

int ref_apply_normal_real(int n, int A, int m_sp, double tau, int backend, const double* in, double* out) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  NormalBackend b = backend == 1 ? make_fused_backend(s.transform) : make_direct_backend(s.transform);
  Vector u(Eigen::Index(n) * n);
  for (Eigen::Index i = 0; i < u.size(); ++i) u[i] = in[i];
  Vector o = apply_normal_real(b, u);
  for (Eigen::Index i = 0; i < o.size(); ++i) out[i] = o[i];
  REF_CATCH
}

int64_t ref_btb_nnz(int n, int A, int m_sp, double tau) {
  try {
    auto s = make_setup(n, A, m_sp, tau);
    return build_btb(s.transform->plan()).nnz();
  } catch (const std::exception& e) {
    return -code_of(e);
  }
}

// Surrogate stencil = centre row of T (normal_ops.cpp:232-283); returns (2r+1)^2 values.
int ref_surrogate_stencil(int n, int A, int m_sp, double tau, int r, double* stencil) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  NormalBackend fused = make_direct_backend(s.transform);
  fused.kind = BackendKind::fused;  // build_surrogate only reads the transform
  SurrogateConfig cfg;
  cfg.radius_r = r;
  SparseOperator t = build_surrogate(fused, cfg);
  const std::int64_t row = std::int64_t(n / 2) * n + n / 2;
  const int side = 2 * r + 1;
  for (std::int64_t k = t.row_offsets[row]; k < t.row_offsets[row + 1]; ++k) {
    const int col = t.col_indices[k];
    const int di = col / n - n / 2, dj = col % n - n / 2;
    stencil[(di + r) * side + (dj + r)] = t.values[k];
  }
  REF_CATCH
}

int ref_apply_surrogate_real(int n, int A, int m_sp, double tau, int r, const double* in, double* out) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  NormalBackend fused = make_direct_backend(s.transform);
  fused.kind = BackendKind::fused;
  SurrogateConfig cfg;
  cfg.radius_r = r;
  NormalBackend sur;
  sur.kind = BackendKind::surrogate;
  sur.params = s.params;
  sur.transform = s.transform;
  sur.t = std::make_shared<SparseOperator>(build_surrogate(fused, cfg));
  Vector u(Eigen::Index(n) * n);
  for (Eigen::Index i = 0; i < u.size(); ++i) u[i] = in[i];
  Vector o = apply_normal_real(sur, u);
  for (Eigen::Index i = 0; i < o.size(); ++i) out[i] = o[i];
  REF_CATCH
}

// CG on the split-Bregman system alpha*Re(N) + lambda*K'K (solver.cpp:171-173), direct
// backend, through the reference's cg_solve.
int ref_cg_sb_system(int n, int A, int m_sp, double tau, double alpha, double lambda, const double* rhs,
                     const double* x0, int steps, double* x, double* min_ritz) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  NormalBackend b = make_direct_backend(s.transform);
  LinOp op = [&](const Vector& u, Vector& o) {
    o = alpha * apply_normal_real(b, u) + lambda * grad_adjoint(grad(u, n));
  };
  const Eigen::Index L = Eigen::Index(n) * n;
  Vector bb(L), xx(L);
  for (Eigen::Index i = 0; i < L; ++i) {
    bb[i] = rhs[i];
    xx[i] = x0 ? x0[i] : 0.0;
  }
  CgOptions opts;
  opts.steps = steps;
  CgStats st;
  Vector r = cg_solve(op, bb, xx, opts, &st);
  for (Eigen::Index i = 0; i < L; ++i) x[i] = r[i];
  if (min_ritz) *min_ritz = st.min_ritz;
  REF_CATCH
}

// backend: 0 direct, 1 fused, 2 surrogate (radius r, built from the fused backend).
int ref_split_bregman(int n, int A, int m_sp, double tau, int backend, int r, double alpha, double lambda,
                      int iters, int cg_steps, const double* slice_data, double* mu, double* update_l1,
                      double* sigma, double* leak) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  NormalBackend b;
  if (backend == 2) {
    NormalBackend fused = make_direct_backend(s.transform);
    fused.kind = BackendKind::fused;
    SurrogateConfig cfg;
    cfg.radius_r = r;
    b.kind = BackendKind::surrogate;
    b.params = s.params;
    b.transform = s.transform;
    b.t = std::make_shared<SparseOperator>(build_surrogate(fused, cfg));
    b.sample_weights = radial_density_weights(s.grid);
    b.surrogate_r = r;
  } else if (backend == 1) {
    b = make_fused_backend(s.transform);
  } else {
    b = make_direct_backend(s.transform);
  }
  SolverConfig cfg;
  cfg.alpha = alpha;
  cfg.lambda = lambda;
  cfg.max_bregman_iters = iters;
  cfg.cg_steps_per_update = cg_steps;
  cfg.update_tol_rel = 0.0;
  cfg.data_feedback = g_feedback != 0;
  auto res = split_bregman_tv(b, cvec(slice_data, s.grid.points.count()), cfg);
  for (Eigen::Index i = 0; i < res.first.data.size(); ++i) mu[i] = res.first.data[i];
  if (update_l1)
    for (size_t i = 0; i < res.second.update_l1.size(); ++i) update_l1[i] = res.second.update_l1[i];
  if (sigma) *sigma = res.second.stabilization_shift;
  if (leak) *leak = res.second.imag_leakage;
  REF_CATCH
}

// Config-1 KKT/Tikhonov shape: cg_solve on alpha*Re(N) + I with rhs alpha*Re(F_NU f), x0 = 0,
// fixed steps (solver.cpp:309-337 builds the same system; D11 fixes the step count).
int ref_tikhonov_identity(int n, int A, int m_sp, double tau, double alpha, const double* slice_data,
                          int steps, double* mu) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  NormalBackend b = make_direct_backend(s.transform);
  LinOp op = [&](const Vector& u, Vector& o) { o = alpha * apply_normal_real(b, u) + u; };
  Vector rhs = alpha * s.transform->adjoint(cvec(slice_data, s.grid.points.count())).data.real();
  CgOptions opts;
  opts.steps = steps;
  Vector x = cg_solve(op, rhs, Vector::Zero(rhs.size()), opts, nullptr);
  for (Eigen::Index i = 0; i < x.size(); ++i) mu[i] = x[i];
  REF_CATCH
}

int ref_shepp_logan(int n, double* img) {
  REF_TRY
  Image im = generate_shepp_logan(n);
  std::memcpy(img, im.data.data(), sizeof(double) * im.data.size());
  REF_CATCH
}

int ref_synthesize(int n, int A, int m_sp, double tau, const double* phantom, double sigma, uint64_t seed,
                   double* samples) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  Vector v(Eigen::Index(n) * n);
  for (Eigen::Index i = 0; i < v.size(); ++i) v[i] = phantom[i];
  put(synthesize_data(Image(n, v), s.grid, s.params, sigma, seed), samples);
  REF_CATCH
}

// The reference's own on-disk operators (TOMOSPM1, sparse.cpp:68-106): the Gram of
// make_fused_backend and the surrogate T of build_surrogate, written by save_sparse.
int ref_save_btb(int n, int A, int m_sp, double tau, const char* path) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  NormalBackend b = make_fused_backend(s.transform);
  save_sparse(*b.btb, path);
  REF_CATCH
}

int ref_save_surrogate(int n, int A, int m_sp, double tau, int r, int euclidean, const char* path) {
  REF_TRY
  auto s = make_setup(n, A, m_sp, tau);
  NormalBackend fused = make_direct_backend(s.transform);
  fused.kind = BackendKind::fused;
  SurrogateConfig cfg;
  cfg.radius_r = r;
  cfg.euclidean = euclidean != 0;
  save_sparse(build_surrogate(fused, cfg), path);
  REF_CATCH
}

// ---- persistent handles for timing (bench.py --impl reference) ---------------------------
// One geometry + backend built once (operator construction is not timed), then
// timed calls through the reference's public API: apply_normal with time_apply's semantics
// (proj/src/bench.cpp:245-257) and split_bregman_tv (proj/src/solver.cpp:219-307).
struct RefHandle {
  RefSetup s;
  NormalBackend b;
};

// backend: 0 direct, 1 fused, 2 surrogate (radius r). nb: radial samples (0 -> n).
void* ref_backend_new(int n, int A, int m_sp, double tau, int nb, int backend, int r) {
  try {
    g_nb = nb;
    auto* h = new RefHandle;
    h->s = make_setup(n, A, m_sp, tau);
    g_nb = 0;
    if (backend == 2) {
      NormalBackend fused = make_direct_backend(h->s.transform);
      fused.kind = BackendKind::fused;
      SurrogateConfig cfg;
      cfg.radius_r = r;
      h->b.kind = BackendKind::surrogate;
      h->b.params = h->s.params;
      h->b.transform = h->s.transform;
      h->b.t = std::make_shared<SparseOperator>(build_surrogate(fused, cfg));
      h->b.sample_weights = radial_density_weights(h->s.grid);
      h->b.surrogate_r = r;
    } else if (backend == 1) {
      h->b = make_fused_backend(h->s.transform);
    } else {
      h->b = make_direct_backend(h->s.transform);
    }
    return h;
  } catch (const std::exception& e) {
    g_nb = 0;
    code_of(e);
    return nullptr;
  }
}

void ref_backend_free(void* h) { delete static_cast<RefHandle*>(h); }

// time_apply (bench.cpp:245-257): one untimed warm-up apply_normal, then `reps` timed ones;
// returns the median seconds in *median_s and the last output in `out` (complex n^2).
int ref_backend_time_apply(void* hp, const double* in, int reps, double* out, double* median_s) {
  REF_TRY
  auto* h = static_cast<RefHandle*>(hp);
  const int n = h->b.params.n;
  const ComplexImage probe(n, cvec(in, Eigen::Index(n) * n));
  ComplexImage sink = apply_normal(h->b, probe);
  std::vector<double> times;
  for (int rep = 0; rep < reps; ++rep) {
    const auto t0 = std::chrono::steady_clock::now();
    sink = apply_normal(h->b, probe);
    times.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  std::sort(times.begin(), times.end());
  *median_s = times.empty() ? 0.0 : times[times.size() / 2];
  if (out) put(sink.data, out);
  REF_CATCH
}

// One timed split_bregman_tv call: *t_call_s = the whole call (make_subproblem, leak probe,
// back-projection and the Bregman loop), *t_loop_s = the trace's t_total_s at the last
// iteration (the loop only, solver.cpp:255-296).
int ref_backend_split_bregman(void* hp, double alpha, double lambda, int iters, int cg_steps,
                              const double* slice_data, double* mu, double* t_call_s, double* t_loop_s) {
  REF_TRY
  auto* h = static_cast<RefHandle*>(hp);
  SolverConfig cfg;
  cfg.alpha = alpha;
  cfg.lambda = lambda;
  cfg.max_bregman_iters = iters;
  cfg.cg_steps_per_update = cg_steps;
  cfg.update_tol_rel = 0.0;
  const ComplexVector f = cvec(slice_data, h->s.grid.points.count());
  const auto t0 = std::chrono::steady_clock::now();
  auto res = split_bregman_tv(h->b, f, cfg);
  *t_call_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *t_loop_s = res.second.t_total_s.empty() ? 0.0 : res.second.t_total_s.back();
  if (mu)
    for (Eigen::Index i = 0; i < res.first.data.size(); ++i) mu[i] = res.first.data[i];
  REF_CATCH
}

}  // extern "C"
