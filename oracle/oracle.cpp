// oracle.cpp — fp64 CPU restatement of the reference hot path. TEST INFRASTRUCTURE ONLY:
// the product (libtomo_b200.so) never links this; see tomo_oracle.h for who may call it.
//
// Every function cites the reference file:line it restates (paths relative to
// /root/reference). The restatement is single-threaded and keeps the reference's loop
// and operation order wherever that order is observable; reductions are plain
// sequential sums (Eigen's vectorised reductions differ only at the 1e-16 level).
// Independent work (the rows / columns of fft_2d, the samples of interpolate) is split over
// host threads (parallel_for, ORC_THREADS or hardware_concurrency); every output element is
// still computed by the same sequence of operations, so results are bit-identical to a
// single-threaded run (spread's scatter and every reduction stay sequential).
#include "tomo_oracle.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

using cd = std::complex<double>;
using CVec = std::vector<cd>;
using RVec = std::vector<double>;

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

thread_local std::string g_last_error;

// Static-chunked parallel loop over [0, count): chunk c of T covers a contiguous range, so
// which thread computes an element never changes the arithmetic. Small loops run inline.
static int orc_threads() {
  static const int t = [] {
    const char* e = std::getenv("ORC_THREADS");
    int v = e ? std::atoi(e) : static_cast<int>(std::thread::hardware_concurrency());
    return std::max(1, std::min(v, 64));
  }();
  return t;
}

template <class F>
static void parallel_for(int64_t count, int64_t min_parallel, F&& fn) {
  const int nt = orc_threads();
  if (nt <= 1 || count < min_parallel) {
    fn(int64_t(0), count);
    return;
  }
  std::vector<std::thread> pool;
  const int64_t chunk = (count + nt - 1) / nt;
  for (int t = 1; t < nt; ++t) {
    const int64_t b = t * chunk, e = std::min(count, b + chunk);
    if (b < e) pool.emplace_back([&fn, b, e] { fn(b, e); });
  }
  fn(int64_t(0), std::min(count, chunk));
  for (auto& th : pool) th.join();
}

// ---------------------------------------------------------------------------------
// Geometry + spreading plan.
// make_angle_set: proj/src/fourier_slice.cpp:10-20 (theta_a = a*pi/count; explicit count
// is extension D2). slice_points: proj/src/fourier_slice.cpp:22-41 with n_b radial samples
// (extension D1: k_r = t - floor(n_b/2), spacing 2*pi/n_b; n_b = n is the reference).
// FrequencyPointSet::make: proj/src/nufft.cpp:43-54. plan_spreading: nufft.cpp:71-101 with
// the window generalised to [lo, hi] (extension D5) and m = R*n (extension D7).
// ---------------------------------------------------------------------------------
struct Geometry {
  int n = 0, A = 0, nb = 0, R = 2, lo = 0, hi = 0, m = 0, w = 0;
  double tau = 0.0;
  std::vector<double> angles;
  int64_t P = 0;
  std::vector<double> x, y;        // reduced coordinates
  std::vector<int> mjx, mjy;       // nearest_index
  std::vector<double> e1x, e1y, e2x, e2y, e3;
};

static std::unique_ptr<Geometry> make_geometry(const orc_geom* d) {
  if (!d) throw ConfigError("geometry: null descriptor");
  auto g = std::make_unique<Geometry>();
  g->n = d->n;
  g->A = d->n_angles;
  g->nb = d->n_b > 0 ? d->n_b : d->n;
  g->R = d->oversample > 0 ? d->oversample : 2;
  g->lo = d->win_lo;
  g->hi = d->win_hi;
  g->tau = d->tau;
  if (g->n < 4) throw ConfigError("make_params: n must be >= 4");
  if (g->n % 2 != 0) throw ConfigError("slice_points: n must be even");
  if (g->A < 1) throw ConfigError("geometry: need at least one angle");
  if (g->nb < 2) throw ConfigError("geometry: n_b must be >= 2");
  if (g->R < 2) throw ConfigError("geometry: oversampling must be >= 2");
  if (!(g->lo <= 0 && g->hi >= 0)) throw ConfigError("geometry: window must contain 0");
  if (!(g->tau > 0.0)) throw ConfigError("make_params: tau must be positive");
  g->m = g->R * g->n;
  g->w = g->hi - g->lo + 1;
  if (g->w > 64) throw ConfigError("spreading window too wide");
  if (g->w >= g->m) throw ConfigError("geometry: window wider than grid");

  g->angles.resize(g->A);
  for (int a = 0; a < g->A; ++a)
    g->angles[a] = d->angles ? d->angles[a] : a * M_PI / g->A;

  g->P = static_cast<int64_t>(g->A) * g->nb;
  g->x.resize(g->P);
  g->y.resize(g->P);
  constexpr double two_pi = 2.0 * M_PI;
  auto reduce = [](double v) {
    double r = std::fmod(v, two_pi);
    if (r < 0.0) r += two_pi;
    if (r >= two_pi) r = 0.0;  // fmod rounding at the seam (nufft.cpp:49)
    return r;
  };
  int64_t row = 0;
  for (int a = 0; a < g->A; ++a) {
    const double c = std::cos(g->angles[a]);
    const double s = std::sin(g->angles[a]);
    for (int t = 0; t < g->nb; ++t, ++row) {
      const double k_r = (2.0 * M_PI / g->nb) * (t - g->nb / 2);
      g->x[row] = reduce(k_r * c);
      g->y[row] = reduce(k_r * s);
    }
  }

  // plan_spreading (nufft.cpp:71-101)
  const double big_m = g->m / 2.0;
  const double h = M_PI / big_m;
  const double tau = g->tau;
  g->e3.resize(g->w);
  for (int l = g->lo; l <= g->hi; ++l)
    g->e3[l - g->lo] = std::exp(-(M_PI * l / big_m) * (M_PI * l / big_m) / (4.0 * tau));
  g->mjx.resize(g->P);
  g->mjy.resize(g->P);
  g->e1x.resize(g->P);
  g->e1y.resize(g->P);
  g->e2x.resize(g->P);
  g->e2y.resize(g->P);
  for (int64_t j = 0; j < g->P; ++j) {
    for (int dd = 0; dd < 2; ++dd) {
      const double xv = dd == 0 ? g->x[j] : g->y[j];
      int mj = static_cast<int>(std::floor(xv / h));
      if (mj >= g->m) mj = g->m - 1;
      const double xi = xv - h * mj;
      const double f1 = std::exp(-xi * xi / (4.0 * tau));
      const double f2 = std::exp(xi * M_PI / (big_m * 2.0 * tau));
      if (dd == 0) {
        g->mjx[j] = mj; g->e1x[j] = f1; g->e2x[j] = f2;
      } else {
        g->mjy[j] = mj; g->e1y[j] = f1; g->e2y[j] = f2;
      }
    }
  }
  return g;
}

// SpreadingPlan::weights (nufft.cpp:56-69), recurrence outward from l = 0 over [lo, hi].
static void weights(const Geometry& g, int64_t j, int dim, double* w) {
  const double f1 = dim == 0 ? g.e1x[j] : g.e1y[j];
  const double f2 = dim == 0 ? g.e2x[j] : g.e2y[j];
  const double f2inv = 1.0 / f2;
  w[-g.lo] = f1;
  double p = f1, q = f1;
  const int reach = std::max(g.hi, -g.lo);
  for (int l = 1; l <= reach; ++l) {
    p *= f2;
    q *= f2inv;
    if (l <= g.hi) w[l - g.lo] = p * g.e3[l - g.lo];
    if (-l >= g.lo) w[-l - g.lo] = q * g.e3[-l - g.lo];
  }
}

static inline int wrap(int idx, int m) {  // nufft.cpp:105-109
  if (idx < 0) return idx + m;
  if (idx >= m) return idx - m;
  return idx;
}

// ---------------------------------------------------------------------------------
// FFT: the reference calls Eigen::FFT<double> (kissfft) at proj/src/fft.cpp:16-50.
// Conventions restated: forward e^{-i}, unscaled; inverse e^{+i}, scaled 1/m per axis.
// Own implementation: iterative radix-2 for powers of two, direct DFT otherwise.
// ---------------------------------------------------------------------------------
static void fft_1d_inplace(cd* data, int m, bool inverse) {
  if (m <= 1) return;
  const double sign = inverse ? 1.0 : -1.0;
  if ((m & (m - 1)) == 0) {
    for (int i = 1, j = 0; i < m; ++i) {
      int bit = m >> 1;
      for (; j & bit; bit >>= 1) j ^= bit;
      j ^= bit;
      if (i < j) std::swap(data[i], data[j]);
    }
    for (int len = 2; len <= m; len <<= 1) {
      const int half = len / 2;
      for (int k = 0; k < half; ++k) {
        const cd wk = std::polar(1.0, sign * 2.0 * M_PI * k / len);
        for (int i = 0; i < m; i += len) {
          const cd u = data[i + k];
          const cd v = data[i + k + half] * wk;
          data[i + k] = u + v;
          data[i + k + half] = u - v;
        }
      }
    }
  } else {
    CVec out(m);
    for (int k = 0; k < m; ++k) {
      cd acc = 0.0;
      for (int t = 0; t < m; ++t)
        acc += data[t] * std::polar(1.0, sign * 2.0 * M_PI *
                                             static_cast<double>((static_cast<int64_t>(k) * t) % m) / m);
      out[k] = acc;
    }
    std::copy(out.begin(), out.end(), data);
  }
  if (inverse) {
    const double s = 1.0 / m;
    for (int i = 0; i < m; ++i) data[i] *= s;
  }
}

// fft_2d (fft.cpp:26-50): row pass, then column pass via gather/scatter.
static void fft_2d(CVec& grid, int m, bool inverse) {
  if (static_cast<int64_t>(grid.size()) != static_cast<int64_t>(m) * m)
    throw ConfigError("fft_2d: grid size mismatch");
  parallel_for(m, 256, [&](int64_t r0, int64_t r1) {
    for (int64_t r = r0; r < r1; ++r) fft_1d_inplace(grid.data() + r * m, m, inverse);
  });
  parallel_for(m, 256, [&](int64_t c0, int64_t c1) {
    CVec buf(m);
    for (int64_t c = c0; c < c1; ++c) {
      for (int r = 0; r < m; ++r) buf[r] = grid[static_cast<int64_t>(r) * m + c];
      fft_1d_inplace(buf.data(), m, inverse);
      for (int r = 0; r < m; ++r) grid[static_cast<int64_t>(r) * m + c] = buf[r];
    }
  });
}

// ---------------------------------------------------------------------------------
// spread (W^T) nufft.cpp:119-158, interpolate (W) nufft.cpp:160-202.
// ---------------------------------------------------------------------------------
static CVec spread(const Geometry& g, const CVec& samples) {
  if (static_cast<int64_t>(samples.size()) != g.P)
    throw ConfigError("spread: sample count does not match plan");
  const int m = g.m, w = g.w;
  CVec grid(static_cast<size_t>(m) * m, cd(0.0, 0.0));
  double wx[64], wy[64];
  int ix[64], iy[64];
  for (int64_t j = 0; j < g.P; ++j) {
    weights(g, j, 0, wx);
    weights(g, j, 1, wy);
    for (int a = 0; a < w; ++a) ix[a] = wrap(g.mjx[j] + g.lo + a, m);
    for (int b = 0; b < w; ++b) iy[b] = wrap(g.mjy[j] + g.lo + b, m);
    const cd s = samples[j];
    for (int a = 0; a < w; ++a) {
      const cd sa = s * wx[a];
      cd* row = grid.data() + static_cast<int64_t>(ix[a]) * m;
      for (int b = 0; b < w; ++b) row[iy[b]] += sa * wy[b];
    }
  }
  return grid;
}

static CVec interpolate(const Geometry& g, const CVec& grid) {
  const int m = g.m, w = g.w;
  if (static_cast<int64_t>(grid.size()) != static_cast<int64_t>(m) * m)
    throw ConfigError("interpolate: grid size mismatch");
  CVec samples(g.P);
  parallel_for(g.P, 4096, [&](int64_t j0, int64_t j1) {
  for (int64_t j = j0; j < j1; ++j) {
    double wx[64], wy[64];
    int ix[64], iy[64];
    weights(g, j, 0, wx);
    weights(g, j, 1, wy);
    for (int a = 0; a < w; ++a) ix[a] = wrap(g.mjx[j] + g.lo + a, m);
    for (int b = 0; b < w; ++b) iy[b] = wrap(g.mjy[j] + g.lo + b, m);
    cd acc = 0.0;
    for (int a = 0; a < w; ++a) {
      const cd* row = grid.data() + static_cast<int64_t>(ix[a]) * m;
      cd rowacc = 0.0;
      for (int b = 0; b < w; ++b) rowacc += row[iy[b]] * wy[b];
      acc += rowacc * wx[a];
    }
    samples[j] = acc;
  }
  });
  return samples;
}

// deconvolve (nufft.cpp:204-227): a[t] = sqrt(pi/tau) exp(k^2 tau), k = t - n/2.
static RVec deapod_axis(const Geometry& g) {
  RVec axis(g.n);
  const double root = std::sqrt(M_PI / g.tau);
  for (int t = 0; t < g.n; ++t) {
    const double k = t - g.n / 2;
    axis[t] = root * std::exp(k * k * g.tau);
  }
  return axis;
}

static void deconvolve(const Geometry& g, CVec& c) {
  const int n = g.n;
  if (static_cast<int64_t>(c.size()) != static_cast<int64_t>(n) * n)
    throw ConfigError("deconvolve: size mismatch");
  const RVec axis = deapod_axis(g);
  for (int t1 = 0; t1 < n; ++t1)
    for (int t2 = 0; t2 < n; ++t2) c[static_cast<int64_t>(t1) * n + t2] *= axis[t1] * axis[t2];
}

static inline int coeff_bin(int t, int n, int m) { return (t - n / 2 + m) % m; }  // nufft.cpp:232

// nufft_type1 (nufft.cpp:236-259)
static CVec type1(const Geometry& g, const CVec& samples) {
  const int n = g.n, m = g.m;
  CVec grid = spread(g, samples);
  fft_2d(grid, m, false);
  CVec coeffs(static_cast<size_t>(n) * n);
  const double scale = 1.0 / (static_cast<double>(m) * m);
  for (int t1 = 0; t1 < n; ++t1) {
    const int64_t src = static_cast<int64_t>(coeff_bin(t1, n, m)) * m;
    for (int t2 = 0; t2 < n; ++t2)
      coeffs[static_cast<int64_t>(t1) * n + t2] = grid[src + coeff_bin(t2, n, m)] * scale;
  }
  deconvolve(g, coeffs);
  return coeffs;
}

// nufft_type2 (nufft.cpp:261-286)
static CVec type2(const Geometry& g, const CVec& coefficients) {
  const int n = g.n, m = g.m;
  if (static_cast<int64_t>(coefficients.size()) != static_cast<int64_t>(n) * n)
    throw ConfigError("nufft_type2: coefficient size mismatch");
  CVec work = coefficients;
  deconvolve(g, work);
  CVec grid(static_cast<size_t>(m) * m, cd(0.0, 0.0));
  for (int t1 = 0; t1 < n; ++t1) {
    const int64_t dst = static_cast<int64_t>(coeff_bin(t1, n, m)) * m;
    for (int t2 = 0; t2 < n; ++t2) grid[dst + coeff_bin(t2, n, m)] = work[static_cast<int64_t>(t1) * n + t2];
  }
  fft_2d(grid, m, true);
  return interpolate(g, grid);
}

// direct_ndft (nufft.cpp:288-333), 2-D branch.
static CVec direct_ndft(const Geometry& g, const CVec& input, bool to_type1) {
  const int n = g.n;
  const int64_t modes = static_cast<int64_t>(n) * n;
  if (g.P * modes > 100'000'000) throw ConfigError("direct_ndft: refusing more than 1e8 terms");
  if (!to_type1) {
    if (static_cast<int64_t>(input.size()) != modes) throw ConfigError("direct_ndft: coefficient size mismatch");
    CVec out(g.P);
    for (int64_t j = 0; j < g.P; ++j) {
      cd acc = 0.0;
      const double x = g.x[j], y = g.y[j];
      for (int t1 = 0; t1 < n; ++t1)
        for (int t2 = 0; t2 < n; ++t2)
          acc += input[static_cast<int64_t>(t1) * n + t2] *
                 std::polar(1.0, (t1 - n / 2) * x + (t2 - n / 2) * y);
      out[j] = acc;
    }
    return out;
  }
  if (static_cast<int64_t>(input.size()) != g.P) throw ConfigError("direct_ndft: sample size mismatch");
  CVec out(modes, cd(0.0, 0.0));
  for (int64_t j = 0; j < g.P; ++j) {
    const double x = g.x[j], y = g.y[j];
    for (int t1 = 0; t1 < n; ++t1)
      for (int t2 = 0; t2 < n; ++t2)
        out[static_cast<int64_t>(t1) * n + t2] +=
            input[j] * std::polar(1.0, -((t1 - n / 2) * x + (t2 - n / 2) * y));
  }
  return out;
}

// apply_normal_direct (normal_ops.cpp:28-30) = adjoint(forward(u)).
static CVec apply_normal(const Geometry& g, const CVec& u) { return type1(g, type2(g, u)); }

// apply_normal_real (normal_ops.cpp:333-340): real -> complex cast, apply, real part.
// Sensitivity probe (test infrastructure, off by default): with orc_set_perturbation(eps, seed)
// every real apply's input and output are multiplied elementwise by (1 + eps * N(0,1)),
// emulating the rounding of a different but equally exact implementation (errors entering at the
// first FFT stage are amplified by the operator's large eigenvalues), so tests can measure how
// much a solver amplifies per-apply rounding.
static double g_perturb_eps = 0.0;
static std::mt19937_64 g_perturb_rng(1);

static RVec apply_normal_real(const Geometry& g, const RVec& u) {
  CVec c(u.size());
  std::normal_distribution<double> gauss;
  // rounding of the first stage enters before the operator and is amplified by its large
  // eigenvalues: perturb the input, then the output
  for (size_t i = 0; i < u.size(); ++i)
    c[i] = cd(g_perturb_eps > 0.0 ? u[i] * (1.0 + g_perturb_eps * gauss(g_perturb_rng)) : u[i], 0.0);
  CVec o = apply_normal(g, c);
  RVec out(u.size());
  for (size_t i = 0; i < u.size(); ++i) out[i] = o[i].real();
  if (g_perturb_eps > 0.0)
    for (auto& v : out) v *= 1.0 + g_perturb_eps * gauss(g_perturb_rng);
  return out;
}

// ---------------------------------------------------------------------------------
// Fused (Gram) backend: build_btb (normal_ops.cpp:53-173) and apply_normal_fused
// (normal_ops.cpp:175-206). Entry (r, c) = sum_j w(j,r) w(j,c); CSR with sorted columns.
// Dense band accumulator over the whole grid (the reference blocks it by 128 MiB).
// ---------------------------------------------------------------------------------
struct Csr {
  int64_t rows = 0;
  std::vector<int64_t> off;
  std::vector<int32_t> col;
  std::vector<double> val;
};

static Csr build_btb(const Geometry& g) {
  const int m = g.m, w = g.w;
  const int reach = std::max(g.hi, -g.lo);
  const int band = 4 * reach + 1;
  const int64_t G = static_cast<int64_t>(m) * m;
  if (G * band * band * 8 > (int64_t(2) << 30)) throw ConfigError("build_btb: oracle Gram too large");
  std::vector<double> acc(static_cast<size_t>(G) * band * band, 0.0);
  double wx[64], wy[64];
  for (int64_t j = 0; j < g.P; ++j) {
    weights(g, j, 0, wx);
    weights(g, j, 1, wy);
    for (int a = 0; a < w; ++a) {
      const int tx = wrap(g.mjx[j] + g.lo + a, m);
      for (int b = 0; b < w; ++b) {
        const int ty = wrap(g.mjy[j] + g.lo + b, m);
        double* cell = acc.data() + (static_cast<int64_t>(tx) * m + ty) * band * band;
        for (int a2 = 0; a2 < w; ++a2)
          for (int b2 = 0; b2 < w; ++b2)
            cell[(a2 - a + 2 * reach) * band + (b2 - b + 2 * reach)] += wx[a] * wx[a2] * wy[b] * wy[b2];
      }
    }
  }
  Csr op;
  op.rows = G;
  op.off.push_back(0);
  std::vector<std::pair<int32_t, double>> ents;
  for (int tx = 0; tx < m; ++tx)
    for (int ty = 0; ty < m; ++ty) {
      const double* cell = acc.data() + (static_cast<int64_t>(tx) * m + ty) * band * band;
      ents.clear();
      for (int i = 0; i < band; ++i) {
        const int cx = wrap(tx + i - 2 * reach, m);
        for (int k = 0; k < band; ++k) {
          const double v = cell[i * band + k];
          if (v != 0.0) ents.emplace_back(static_cast<int32_t>(static_cast<int64_t>(cx) * m + wrap(ty + k - 2 * reach, m)), v);
        }
      }
      std::sort(ents.begin(), ents.end(), [](auto& l, auto& r) { return l.first < r.first; });
      for (auto& e : ents) {
        op.col.push_back(e.first);
        op.val.push_back(e.second);
      }
      op.off.push_back(static_cast<int64_t>(op.val.size()));
    }
  return op;
}

static CVec apply_normal_fused(const Geometry& g, const Csr& btb, const CVec& u) {
  const int n = g.n, m = g.m;
  CVec work = u;
  deconvolve(g, work);
  CVec grid(static_cast<size_t>(m) * m, cd(0.0, 0.0));
  for (int t1 = 0; t1 < n; ++t1)
    for (int t2 = 0; t2 < n; ++t2)
      grid[static_cast<int64_t>(coeff_bin(t1, n, m)) * m + coeff_bin(t2, n, m)] = work[static_cast<int64_t>(t1) * n + t2];
  fft_2d(grid, m, true);
  CVec y(grid.size());
  for (int64_t i = 0; i < btb.rows; ++i) {  // SparseOperator::apply complex, sparse.cpp:27-42
    double re = 0.0, im = 0.0;
    for (int64_t k = btb.off[i]; k < btb.off[i + 1]; ++k) {
      re += btb.val[k] * grid[btb.col[k]].real();
      im += btb.val[k] * grid[btb.col[k]].imag();
    }
    y[i] = cd(re, im);
  }
  fft_2d(y, m, false);
  CVec out(static_cast<size_t>(n) * n);
  const double scale = 1.0 / (static_cast<double>(m) * m);
  for (int t1 = 0; t1 < n; ++t1)
    for (int t2 = 0; t2 < n; ++t2)
      out[static_cast<int64_t>(t1) * n + t2] = y[static_cast<int64_t>(coeff_bin(t1, n, m)) * m + coeff_bin(t2, n, m)] * scale;
  deconvolve(g, out);
  return out;
}

// ---------------------------------------------------------------------------------
// Surrogate: radial_density_weights (normal_ops.cpp:208-219), apply_weighted_normal_real
// (:221-230), build_surrogate stencil (:232-264) and its translated CSR apply (:266-288).
// ---------------------------------------------------------------------------------
static RVec radial_weights(const Geometry& g) {
  RVec w(g.P);
  int64_t row = 0;
  for (int a = 0; a < g.A; ++a)
    for (int t = 0; t < g.nb; ++t, ++row) {
      const int k_r = t - g.nb / 2;
      w[row] = k_r == 0 ? 0.25 : std::abs(static_cast<double>(k_r));
    }
  return w;
}

static RVec weighted_normal_real(const Geometry& g, const RVec& wts, const RVec& u) {
  CVec c(u.size());
  for (size_t i = 0; i < u.size(); ++i) c[i] = cd(u[i], 0.0);
  CVec s = type2(g, c);
  for (int64_t j = 0; j < g.P; ++j) s[j] *= cd(wts[j], 0.0);
  CVec o = type1(g, s);
  RVec out(u.size());
  for (size_t i = 0; i < u.size(); ++i) out[i] = o[i].real();
  return out;
}

static RVec surrogate_stencil(const Geometry& g, int r) {
  const int n = g.n;
  if (r < 1 || r >= n / 2) throw ConfigError("build_surrogate: radius out of range");
  const RVec wts = radial_weights(g);
  RVec delta(static_cast<size_t>(n) * n, 0.0);
  delta[static_cast<int64_t>(n / 2) * n + n / 2] = 1.0;
  const RVec resp = weighted_normal_real(g, wts, delta);
  const int side = 2 * r + 1;
  RVec st(static_cast<size_t>(side) * side);
  for (int di = -r; di <= r; ++di)
    for (int dj = -r; dj <= r; ++dj) {
      const double fwd = resp[static_cast<int64_t>(n / 2 + di) * n + (n / 2 + dj)];
      const double bwd = resp[static_cast<int64_t>(n / 2 - di) * n + (n / 2 - dj)];
      st[(di + r) * side + (dj + r)] = 0.5 * (fwd + bwd);
    }
  return st;
}

// T u with T the translated stencil, out-of-image entries dropped (normal_ops.cpp:266-281);
// summation in CSR column order (sparse.cpp:10-17).
static void apply_stencil(int n, int r, bool euclid, const double* st, const double* u, double* out) {
  const int side = 2 * r + 1;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int di = -r; di <= r; ++di) {
        const int ii = i + di;
        if (ii < 0 || ii >= n) continue;
        for (int dj = -r; dj <= r; ++dj) {
          const int jj = j + dj;
          if (jj < 0 || jj >= n) continue;
          if (euclid && di * di + dj * dj > r * r) continue;
          acc += st[(di + r) * side + (dj + r)] * u[static_cast<int64_t>(ii) * n + jj];
        }
      }
      out[static_cast<int64_t>(i) * n + j] = acc;
    }
}

// ---------------------------------------------------------------------------------
// Solver pieces: grad / grad_adjoint (solver.cpp:12-43), shrink (:45-54).
// ---------------------------------------------------------------------------------
static void grad(int n, const double* u, double* gx, double* gy) {
  const int64_t L = static_cast<int64_t>(n) * n;
  std::fill(gx, gx + L, 0.0);
  std::fill(gy, gy + L, 0.0);
  for (int i = 0; i < n; ++i) {
    const int64_t row = static_cast<int64_t>(i) * n;
    for (int j = 0; j < n - 1; ++j) gx[row + j] = u[row + j + 1] - u[row + j];
    if (i < n - 1)
      for (int j = 0; j < n; ++j) gy[row + j] = u[row + n + j] - u[row + j];
  }
}

static void grad_adjoint(int n, const double* gx, const double* gy, double* out) {
  const int64_t L = static_cast<int64_t>(n) * n;
  std::fill(out, out + L, 0.0);
  for (int i = 0; i < n; ++i) {
    const int64_t row = static_cast<int64_t>(i) * n;
    for (int j = 0; j < n - 1; ++j) {
      out[row + j + 1] += gx[row + j];
      out[row + j] -= gx[row + j];
    }
    if (i < n - 1)
      for (int j = 0; j < n; ++j) {
        out[row + n + j] += gy[row + j];
        out[row + j] -= gy[row + j];
      }
  }
}

static inline double shrink1(double x, double gamma) {
  const double mm = std::abs(x) - gamma;
  return mm > 0.0 ? (x > 0.0 ? mm : -mm) : 0.0;
}

// Inner products of the CG / Lanczos recurrences with compensated (Neumaier) summation. The
// reference's Eigen dot sums in SIMD packets and a final tree (error ~ N/8 eps); a plain
// sequential sum (error ~ N eps) is measurably worse at 4M-pixel images: in the c5 prox CG
// (kappa ~ 7e5) it moved r.r by 3.7x at step 15, while the compensated oracle agrees with the
// GPU's tree-reduced fp64 dots in both CG forms. g_dot_mode = 0 restores the
// plain sequential sum (probe only).
static int g_dot_mode = 1;
static double dot(const RVec& a, const RVec& b) {
  if (g_dot_mode == 0) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
  }
  double s = 0.0, c = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double x = a[i] * b[i];
    const double t = s + x;
    c += std::abs(s) >= std::abs(x) ? (s - t) + x : (x - t) + s;
    s = t;
  }
  return s + c;
}

// System operators. base_op: solver.cpp:171-173 (alpha*apply_normal_real + lambda*K'K),
// sigma shift: :195-198, identity-K Tikhonov system: :323-327.
struct System {
  const Geometry* g = nullptr;
  int backend = 0;
  int r = 1;
  bool euclid = false;
  double alpha = 1.0, lambda = 1.0, shift = 0.0;
  bool identity_k = false;
  RVec stencil;
  std::shared_ptr<Csr> btb;

  RVec base(const RVec& u) const {
    const int n = g->n;
    RVec nu(u.size());
    if (backend == 2) {
      apply_stencil(n, r, euclid, stencil.data(), u.data(), nu.data());
    } else if (backend == 1) {
      CVec c(u.size());
      for (size_t i = 0; i < u.size(); ++i) c[i] = cd(u[i], 0.0);
      CVec o = apply_normal_fused(*g, *btb, c);
      for (size_t i = 0; i < u.size(); ++i) nu[i] = o[i].real();
    } else {
      nu = apply_normal_real(*g, u);
    }
    return nu;
  }

  void operator()(const RVec& u, RVec& out) const {
    const int n = g->n;
    const RVec nu = base(u);
    out.resize(u.size());
    if (identity_k) {
      for (size_t i = 0; i < u.size(); ++i) out[i] = alpha * nu[i] + u[i] + shift * u[i];
      return;
    }
    RVec gx(u.size()), gy(u.size()), kk(u.size());
    grad(n, u.data(), gx.data(), gy.data());
    grad_adjoint(n, gx.data(), gy.data(), kk.data());
    for (size_t i = 0; i < u.size(); ++i) out[i] = alpha * nu[i] + lambda * kk[i];
    if (shift != 0.0)
      for (size_t i = 0; i < u.size(); ++i) out[i] += shift * u[i];
  }
};

static System make_system(const Geometry& g, const orc_system* s) {
  System sys;
  sys.g = &g;
  sys.backend = s->backend;
  sys.r = s->surrogate_r;
  sys.euclid = s->euclidean != 0;
  sys.alpha = s->alpha;
  sys.lambda = s->lambda;
  sys.shift = s->shift;
  sys.identity_k = s->identity_k != 0;
  if (sys.backend == 2) sys.stencil = surrogate_stencil(g, sys.r);
  if (sys.backend == 1) sys.btb = std::make_shared<Csr>(build_btb(g));
  if (sys.backend < 0 || sys.backend > 2) throw ConfigError("unknown backend");
  return sys;
}

// cg_solve (solver.cpp:56-95).
static RVec cg_solve(const System& op, const RVec& rhs, const RVec& x0, int steps, double tol,
                     orc_cg_stats* stats) {
  if (steps < 1) throw ConfigError("cg_solve: steps must be >= 1");
  RVec x = x0;
  RVec ax;
  op(x, ax);
  RVec r(rhs.size());
  for (size_t i = 0; i < r.size(); ++i) r[i] = rhs[i] - ax[i];
  RVec p = r;
  double rs = dot(r, r);
  const double rhs_norm = std::sqrt(dot(rhs, rhs));
  double min_ritz = std::numeric_limits<double>::infinity();
  RVec ap;
  int step = 0;
  for (; step < steps; ++step) {
    if (rs == 0.0) break;
    op(p, ap);
    const double p_ap = dot(p, ap);
    const double p_p = dot(p, p);
    if (p_p > 0.0) min_ritz = std::min(min_ritz, p_ap / p_p);
    if (p_ap == 0.0) break;
    const double alpha = rs / p_ap;
    bool finite = true;
    for (size_t i = 0; i < x.size(); ++i) {
      x[i] += alpha * p[i];
      finite = finite && std::isfinite(x[i]);
    }
    for (size_t i = 0; i < r.size(); ++i) r[i] -= alpha * ap[i];
    const double rs_next = dot(r, r);
    if (!std::isfinite(rs_next) || !finite) throw NumericalError("cg_solve diverged (non-finite iterate)");
    const double beta = rs_next / rs;
    for (size_t i = 0; i < p.size(); ++i) p[i] = r[i] + beta * p[i];
    rs = rs_next;
    if (tol > 0.0 && rhs_norm > 0.0 && std::sqrt(rs) <= tol * rhs_norm) break;
  }
  if (stats) {
    stats->steps_run = step;
    stats->min_ritz = std::isfinite(min_ritz) ? min_ritz : 0.0;
    stats->final_rs = rs;
  }
  return x;
}

// Extreme eigenvalue of a symmetric tridiagonal matrix by Sturm-sequence bisection
// (stands in for Eigen::SelfAdjointEigenSolver at solver.cpp:121-122).
static double tridiag_extreme(const RVec& a, const RVec& b, bool largest) {
  const int m = static_cast<int>(a.size());
  double lo = std::numeric_limits<double>::infinity(), hi = -lo;
  for (int i = 0; i < m; ++i) {
    double rad = 0.0;
    if (i > 0) rad += std::abs(b[i - 1]);
    if (i + 1 < m) rad += std::abs(b[i]);
    lo = std::min(lo, a[i] - rad);
    hi = std::max(hi, a[i] + rad);
  }
  auto count_below = [&](double x) {  // number of eigenvalues < x
    int cnt = 0;
    double q = 1.0;
    for (int i = 0; i < m; ++i) {
      const double bb = i > 0 ? b[i - 1] * b[i - 1] : 0.0;
      q = a[i] - x - (i > 0 ? bb / q : 0.0);
      if (q == 0.0) q = -1e-300;
      if (q < 0.0) ++cnt;
    }
    return cnt;
  };
  const int target = largest ? m - 1 : 0;  // index of the wanted eigenvalue
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (count_below(mid) > target) hi = mid; else lo = mid;
  }
  return 0.5 * (lo + hi);
}

// lanczos_extreme_ritz (solver.cpp:97-130).
template <typename Op>
static double lanczos(const Op& op, int64_t dim, int iters, uint64_t seed, bool largest) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss;
  RVec v(dim);
  for (int64_t i = 0; i < dim; ++i) v[i] = gauss(rng);
  const double vn = std::sqrt(dot(v, v));
  for (auto& e : v) e /= vn;
  RVec v_prev(dim, 0.0), w;
  RVec alphas, betas;
  double beta = 0.0;
  double extreme = largest ? -std::numeric_limits<double>::infinity() : std::numeric_limits<double>::infinity();
  for (int it = 0; it < iters; ++it) {
    op(v, w);
    const double a = dot(v, w);
    alphas.push_back(a);
    for (int64_t i = 0; i < dim; ++i) w[i] -= a * v[i] + beta * v_prev[i];
    beta = std::sqrt(dot(w, w));
    extreme = tridiag_extreme(alphas, betas, largest);
    if (beta < 1e-12) break;
    betas.push_back(beta);
    v_prev = v;
    for (int64_t i = 0; i < dim; ++i) v[i] = w[i] / beta;
  }
  return extreme;
}

static double surrogate_sigma(const Geometry& g, int r, bool euclid, double alpha, double lambda) {
  orc_system s{2, r, euclid ? 1 : 0, alpha, lambda, 0.0, 0};
  System base = make_system(g, &s);
  const int64_t dim = static_cast<int64_t>(g.n) * g.n;
  return 1.2 * std::max(0.0, -lanczos(base, dim, 40, 7, false));
}

// With data feedback (solver.cpp:176-187): contraction floor from the largest Ritz value of
// alpha F W F* - 2 (alpha T + lambda K'K).
static double surrogate_sigma_feedback(const Geometry& g, int r, bool euclid, double alpha, double lambda) {
  orc_system s{2, r, euclid ? 1 : 0, alpha, lambda, 0.0, 0};
  System base = make_system(g, &s);
  const int64_t dim = static_cast<int64_t>(g.n) * g.n;
  const RVec wts = radial_weights(g);
  auto gap = [&g, &wts, &base, alpha](const RVec& u, RVec& out) {
    RVec tmp;
    base(u, tmp);
    const RVec wn = weighted_normal_real(g, wts, u);
    out.resize(u.size());
    for (size_t i = 0; i < u.size(); ++i) out[i] = alpha * wn[i] - 2.0 * tmp[i];
  };
  return 1.2 * std::max(0.0, 0.5 * lanczos(gap, dim, 40, 7, true));
}

// backproject (solver.cpp:200-213).
static RVec backproject(const Geometry& g, int backend, double alpha, const CVec& f) {
  CVec s = f;
  if (backend == 2) {
    const RVec w = radial_weights(g);
    for (int64_t j = 0; j < g.P; ++j) s[j] *= cd(w[j], 0.0);
  }
  CVec o = type1(g, s);
  RVec out(o.size());
  for (size_t i = 0; i < o.size(); ++i) out[i] = alpha * o[i].real();
  return out;
}

static CVec to_cvec(const double* p, int64_t len) {
  CVec v(len);
  for (int64_t i = 0; i < len; ++i) v[i] = cd(p[2 * i], p[2 * i + 1]);
  return v;
}
static void from_cvec(const CVec& v, double* p) {
  for (size_t i = 0; i < v.size(); ++i) {
    p[2 * i] = v[i].real();
    p[2 * i + 1] = v[i].imag();
  }
}

// split_bregman_tv (solver.cpp:219-307), incl. the optional data feedback.
static RVec split_bregman(const Geometry& g, const orc_sb_config* c, const CVec& f,
                          double* upd_out, orc_sb_trace* tr) {
  if (!(c->alpha > 0.0)) throw ConfigError("SolverConfig: alpha must be positive");
  if (!(c->lambda > 0.0)) throw ConfigError("SolverConfig: lambda must be positive");
  if (c->max_iters < 1) throw ConfigError("SolverConfig: max_bregman_iters >= 1");
  if (c->cg_steps < 1) throw ConfigError("SolverConfig: cg_steps_per_update >= 1");
  if (c->update_tol_rel < 0.0) throw ConfigError("SolverConfig: update_tol_rel >= 0");
  if (static_cast<int64_t>(f.size()) != g.P) throw ConfigError("split_bregman_tv: slice data size mismatch");
  const int n = g.n;
  const int64_t dim = static_cast<int64_t>(n) * n;
  const bool surrogate = c->backend == 2;
  double sigma = 0.0;
  const bool feedback = c->data_feedback != 0;
  if (surrogate)
    sigma = c->sigma_override >= 0.0 ? c->sigma_override
            : feedback ? surrogate_sigma_feedback(g, c->surrogate_r, c->euclidean != 0, c->alpha, c->lambda)
                       : surrogate_sigma(g, c->surrogate_r, c->euclidean != 0, c->alpha, c->lambda);
  orc_system sd{c->backend, c->surrogate_r, c->euclidean, c->alpha, c->lambda, sigma, 0};
  System sys = make_system(g, &sd);

  double leak = 0.0;
  if (!surrogate) {  // conjugation-symmetry probe (solver.cpp:236-247)
    CVec ones(dim, cd(1.0, 0.0));
    CVec nu = c->backend == 1 ? apply_normal_fused(g, *sys.btb, ones) : apply_normal(g, ones);
    double tot = 0.0, im = 0.0;
    for (auto& z : nu) {
      tot += std::norm(z);
      im += z.imag() * z.imag();
    }
    tot = std::sqrt(tot);
    leak = tot > 0.0 ? std::sqrt(im) / tot : 0.0;
    if (leak > 0.1) throw NumericalError("split_bregman_tv: conjugation symmetry broken");
  }

  RVec mu(dim, 0.0), dx(dim, 0.0), dy(dim, 0.0), bx(dim, 0.0), by(dim, 0.0);
  CVec fk = f;  // solver.cpp:252-253
  RVec fid = backproject(g, c->backend, c->alpha, fk);
  const double gamma = 1.0 / c->lambda;
  double min_ritz = std::numeric_limits<double>::infinity();
  double first = 0.0;
  int iters = 0;
  bool tol_stop = false;
  RVec tx(dim), ty(dim), adj(dim), rhs(dim), gx(dim), gy(dim);
  for (int it = 0; it < c->max_iters; ++it) {
    for (int64_t i = 0; i < dim; ++i) {
      tx[i] = dx[i] - bx[i];
      ty[i] = dy[i] - by[i];
    }
    grad_adjoint(n, tx.data(), ty.data(), adj.data());
    for (int64_t i = 0; i < dim; ++i) rhs[i] = fid[i] + c->lambda * adj[i];
    orc_cg_stats st{};
    RVec x0 = c->warm_start ? mu : RVec(dim, 0.0);
    RVec mu_next = cg_solve(sys, rhs, x0, c->cg_steps, 0.0, &st);
    if (st.min_ritz != 0.0) min_ritz = std::min(min_ritz, st.min_ritz);
    grad(n, mu_next.data(), gx.data(), gy.data());
    for (int64_t i = 0; i < dim; ++i) {
      dx[i] = shrink1(gx[i] + bx[i], gamma);
      dy[i] = shrink1(gy[i] + by[i], gamma);
      bx[i] += gx[i] - dx[i];
      by[i] += gy[i] - dy[i];
    }
    if (feedback) {  // fk += f - F_NU^* mu_next; fidelity rhs = backproject(fk) (solver.cpp:283-286)
      CVec cm(dim);
      for (int64_t i = 0; i < dim; ++i) cm[i] = cd(mu_next[i], 0.0);
      const CVec s_mu = type2(g, cm);
      for (int64_t j = 0; j < g.P; ++j) fk[j] += f[j] - s_mu[j];
      fid = backproject(g, c->backend, c->alpha, fk);
    }
    double upd = 0.0;
    bool finite = true;
    for (int64_t i = 0; i < dim; ++i) {
      upd += std::abs(mu_next[i] - mu[i]);
      finite = finite && std::isfinite(mu_next[i]);
    }
    mu = std::move(mu_next);
    if (!finite) throw NumericalError("split_bregman_tv: non-finite iterate");
    if (upd_out) upd_out[it] = upd;
    iters = it + 1;
    if (it == 0) first = upd;
    if (upd <= c->update_tol_rel * first) {
      tol_stop = true;
      break;
    }
  }
  if (tr) {
    tr->iterations = iters;
    tr->first_update_l1 = first;
    tr->sigma = sigma;
    tr->min_ritz = std::isfinite(min_ritz) ? min_ritz : 0.0;
    tr->imag_leakage = leak;
    tr->stopped_on_tolerance = tol_stop ? 1 : 0;
  }
  return mu;
}

// Chambolle-Pock anisotropic TV (extension D10). The primal prox is
// (I + tau_cp*alpha*Re N) u = u_tilde + tau_cp*alpha*Re(F_NU f), 'cg_steps' CG steps warm
// started at the current iterate; the dual prox is the clip to [-lambda, lambda].
static RVec chambolle_pock(const Geometry& g, const orc_cp_config* c, const CVec& f) {
  const int n = g.n;
  const int64_t dim = static_cast<int64_t>(n) * n;
  const RVec bp = backproject(g, 0, c->alpha, f);
  orc_system sd{0, 1, 0, c->tau_cp * c->alpha, 0.0, 0.0, 1};
  System sys = make_system(g, &sd);
  RVec u(dim, 0.0), ubar(dim, 0.0), yx(dim, 0.0), yy(dim, 0.0), gx(dim), gy(dim), div(dim), rhs(dim);
  for (int k = 0; k < c->iters; ++k) {
    grad(n, ubar.data(), gx.data(), gy.data());
    for (int64_t i = 0; i < dim; ++i) {
      yx[i] = std::min(c->lambda, std::max(-c->lambda, yx[i] + c->sigma_cp * gx[i]));
      yy[i] = std::min(c->lambda, std::max(-c->lambda, yy[i] + c->sigma_cp * gy[i]));
    }
    grad_adjoint(n, yx.data(), yy.data(), div.data());
    for (int64_t i = 0; i < dim; ++i) rhs[i] = (u[i] - c->tau_cp * div[i]) + c->tau_cp * bp[i];
    RVec un = cg_solve(sys, rhs, u, c->cg_steps, 0.0, nullptr);
    for (int64_t i = 0; i < dim; ++i) {
      ubar[i] = un[i] + c->theta * (un[i] - u[i]);
      if (!std::isfinite(un[i])) throw NumericalError("chambolle_pock: non-finite iterate");
    }
    u = std::move(un);
  }
  return u;
}

// ---------------------------------------------------------------------------------
// Inputs: Ellipse::contains (image.cpp:22-29), Shepp-Logan (:35-67), random ellipses
// (extension D3), synthesize_data (fourier_slice.cpp:71-83, relative sigma D4).
// ---------------------------------------------------------------------------------
struct Ellipse {
  double intensity, a, b, cx, cy, rot;
  bool contains(double x, double y) const {
    const double c = std::cos(rot), s = std::sin(rot);
    const double dx = x - cx, dy = y - cy;
    const double xr = dx * c + dy * s;
    const double yr = -dx * s + dy * c;
    const double u = xr / a, v = yr / b;
    return u * u + v * v <= 1.0;
  }
};

static void rasterize(int n, const std::vector<Ellipse>& es, double* img) {
  for (int i = 0; i < n; ++i) {
    const double y = -1.0 + (2.0 * i + 1.0) / n;
    for (int j = 0; j < n; ++j) {
      const double x = -1.0 + (2.0 * j + 1.0) / n;
      double v = 0.0;
      for (const auto& e : es)
        if (e.contains(x, y)) v += e.intensity;
      img[static_cast<int64_t>(i) * n + j] = v;
    }
  }
}

// Random-ellipse table: per ellipse six U[0,1) draws u = (rng() >> 11) * 2^-53 from
// mt19937_64(seed), mapped as centre = 1.2u-0.6, semi-axis = 0.05+0.35u,
// rotation = pi(2u-1), intensity = u (documented in DESIGN.md; same mapping in the
// product's tomo_random_ellipses).
static std::vector<Ellipse> random_table(int count, uint64_t seed) {
  std::mt19937_64 rng(seed);
  auto U = [&rng]() { return static_cast<double>(rng() >> 11) * (1.0 / 9007199254740992.0); };
  std::vector<Ellipse> es;
  for (int k = 0; k < count; ++k) {
    Ellipse e{};
    e.cx = 1.2 * U() - 0.6;
    e.cy = 1.2 * U() - 0.6;
    e.a = 0.05 + 0.35 * U();
    e.b = 0.05 + 0.35 * U();
    e.rot = M_PI * (2.0 * U() - 1.0);
    e.intensity = U();
    es.push_back(e);
  }
  return es;
}

static int fail(const std::exception& e, int code) {
  g_last_error = e.what();
  return code;
}

}  // namespace orc

using namespace orc;

#define ORC_TRY try {
#define ORC_CATCH                                            \
  return 0;                                                  \
  }                                                          \
  catch (const orc::ConfigError& e) { return fail(e, 2); }   \
  catch (const orc::NumericalError& e) { return fail(e, 3); } \
  catch (const std::exception& e) { return fail(e, 2); }

extern "C" {

const char* orc_last_error(void) { return g_last_error.c_str(); }

void orc_set_dot_mode(int mode) { g_dot_mode = mode; }

void orc_set_perturbation(double eps, uint64_t seed) {
  g_perturb_eps = eps;
  g_perturb_rng.seed(seed);
}

int64_t orc_num_points(const orc_geom* d) {
  try {
    return make_geometry(d)->P;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return -2;
  }
}

int orc_points(const orc_geom* d, double* coords) {
  ORC_TRY
  auto g = make_geometry(d);
  for (int64_t j = 0; j < g->P; ++j) {
    coords[2 * j] = g->x[j];
    coords[2 * j + 1] = g->y[j];
  }
  ORC_CATCH
}

int orc_plan(const orc_geom* d, int* nearest, double* e1, double* e2, double* e3) {
  ORC_TRY
  auto g = make_geometry(d);
  for (int64_t j = 0; j < g->P; ++j) {
    nearest[2 * j] = g->mjx[j];
    nearest[2 * j + 1] = g->mjy[j];
    e1[2 * j] = g->e1x[j];
    e1[2 * j + 1] = g->e1y[j];
    e2[2 * j] = g->e2x[j];
    e2[2 * j + 1] = g->e2y[j];
  }
  std::copy(g->e3.begin(), g->e3.end(), e3);
  ORC_CATCH
}

int orc_weights(const orc_geom* d, double* wx, double* wy) {
  ORC_TRY
  auto g = make_geometry(d);
  for (int64_t j = 0; j < g->P; ++j) {
    weights(*g, j, 0, wx + j * g->w);
    weights(*g, j, 1, wy + j * g->w);
  }
  ORC_CATCH
}

int orc_deapod(const orc_geom* d, double* a) {
  ORC_TRY
  auto g = make_geometry(d);
  RVec ax = deapod_axis(*g);
  std::copy(ax.begin(), ax.end(), a);
  ORC_CATCH
}

int orc_fft2(int m, double* grid, int inverse) {
  ORC_TRY
  if (m < 1) throw ConfigError("fft2: bad size");
  CVec v = to_cvec(grid, static_cast<int64_t>(m) * m);
  fft_2d(v, m, inverse != 0);
  from_cvec(v, grid);
  ORC_CATCH
}

int orc_interpolate(const orc_geom* d, const double* grid, double* samples) {
  ORC_TRY
  auto g = make_geometry(d);
  from_cvec(interpolate(*g, to_cvec(grid, static_cast<int64_t>(g->m) * g->m)), samples);
  ORC_CATCH
}

int orc_spread(const orc_geom* d, const double* samples, double* grid) {
  ORC_TRY
  auto g = make_geometry(d);
  from_cvec(spread(*g, to_cvec(samples, g->P)), grid);
  ORC_CATCH
}

int orc_type2(const orc_geom* d, const double* coeffs, double* samples) {
  ORC_TRY
  auto g = make_geometry(d);
  from_cvec(type2(*g, to_cvec(coeffs, static_cast<int64_t>(g->n) * g->n)), samples);
  ORC_CATCH
}

int orc_type1(const orc_geom* d, const double* samples, double* coeffs) {
  ORC_TRY
  auto g = make_geometry(d);
  from_cvec(type1(*g, to_cvec(samples, g->P)), coeffs);
  ORC_CATCH
}

int orc_direct_ndft(const orc_geom* d, const double* input, double* output, int to_type1) {
  ORC_TRY
  auto g = make_geometry(d);
  const int64_t len = to_type1 ? g->P : static_cast<int64_t>(g->n) * g->n;
  from_cvec(direct_ndft(*g, to_cvec(input, len), to_type1 != 0), output);
  ORC_CATCH
}

int orc_apply_normal(const orc_geom* d, const double* in, double* out) {
  ORC_TRY
  auto g = make_geometry(d);
  from_cvec(apply_normal(*g, to_cvec(in, static_cast<int64_t>(g->n) * g->n)), out);
  ORC_CATCH
}

int orc_apply_normal_real(const orc_geom* d, const double* in, double* out) {
  ORC_TRY
  auto g = make_geometry(d);
  const int64_t L = static_cast<int64_t>(g->n) * g->n;
  RVec u(in, in + L);
  RVec o = apply_normal_real(*g, u);
  std::copy(o.begin(), o.end(), out);
  ORC_CATCH
}

int64_t orc_btb_nnz(const orc_geom* d) {
  try {
    auto g = make_geometry(d);
    return static_cast<int64_t>(build_btb(*g).val.size());
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return -2;
  }
}

int orc_apply_normal_fused(const orc_geom* d, const double* in, double* out) {
  ORC_TRY
  auto g = make_geometry(d);
  Csr btb = build_btb(*g);
  from_cvec(apply_normal_fused(*g, btb, to_cvec(in, static_cast<int64_t>(g->n) * g->n)), out);
  ORC_CATCH
}

int orc_radial_weights(const orc_geom* d, double* w) {
  ORC_TRY
  auto g = make_geometry(d);
  RVec v = radial_weights(*g);
  std::copy(v.begin(), v.end(), w);
  ORC_CATCH
}

int orc_weighted_normal_real(const orc_geom* d, const double* w, const double* in, double* out) {
  ORC_TRY
  auto g = make_geometry(d);
  const int64_t L = static_cast<int64_t>(g->n) * g->n;
  RVec o = weighted_normal_real(*g, RVec(w, w + g->P), RVec(in, in + L));
  std::copy(o.begin(), o.end(), out);
  ORC_CATCH
}

int orc_surrogate_stencil(const orc_geom* d, int r, double* stencil) {
  ORC_TRY
  auto g = make_geometry(d);
  RVec st = surrogate_stencil(*g, r);
  std::copy(st.begin(), st.end(), stencil);
  ORC_CATCH
}

int orc_apply_stencil(int n, int r, int euclidean, const double* stencil, const double* in, double* out) {
  ORC_TRY
  if (n < 1 || r < 0) throw ConfigError("apply_stencil: bad size");
  apply_stencil(n, r, euclidean != 0, stencil, in, out);
  ORC_CATCH
}

int orc_grad(int n, const double* u, double* gx, double* gy) {
  ORC_TRY
  if (n < 1) throw ConfigError("grad: size mismatch");
  grad(n, u, gx, gy);
  ORC_CATCH
}

int orc_grad_adjoint(int n, const double* gx, const double* gy, double* out) {
  ORC_TRY
  if (n < 1) throw ConfigError("grad_adjoint: size mismatch");
  grad_adjoint(n, gx, gy, out);
  ORC_CATCH
}

int orc_shrink(int64_t len, const double* x, double gamma, double* out) {
  ORC_TRY
  for (int64_t i = 0; i < len; ++i) out[i] = shrink1(x[i], gamma);
  ORC_CATCH
}

int orc_system_apply(const orc_geom* d, const orc_system* s, const double* u, double* out) {
  ORC_TRY
  auto g = make_geometry(d);
  System sys = make_system(*g, s);
  const int64_t L = static_cast<int64_t>(g->n) * g->n;
  RVec o;
  sys(RVec(u, u + L), o);
  std::copy(o.begin(), o.end(), out);
  ORC_CATCH
}

int orc_cg(const orc_geom* d, const orc_system* s, const double* rhs, const double* x0, int steps,
           double rel_tol, double* x, orc_cg_stats* stats) {
  ORC_TRY
  auto g = make_geometry(d);
  System sys = make_system(*g, s);
  const int64_t L = static_cast<int64_t>(g->n) * g->n;
  RVec xx = cg_solve(sys, RVec(rhs, rhs + L), x0 ? RVec(x0, x0 + L) : RVec(L, 0.0), steps, rel_tol, stats);
  std::copy(xx.begin(), xx.end(), x);
  ORC_CATCH
}

int orc_surrogate_sigma(const orc_geom* d, int r, int euclidean, double alpha, double lambda, double* sigma) {
  ORC_TRY
  auto g = make_geometry(d);
  *sigma = surrogate_sigma(*g, r, euclidean != 0, alpha, lambda);
  ORC_CATCH
}

int orc_lanczos_extreme(const orc_geom* d, const orc_system* s, int iters, uint64_t seed, int largest,
                        double* value) {
  ORC_TRY
  auto g = make_geometry(d);
  System sys = make_system(*g, s);
  *value = lanczos(sys, static_cast<int64_t>(g->n) * g->n, iters, seed, largest != 0);
  ORC_CATCH
}

int orc_backproject(const orc_geom* d, int backend, double alpha, const double* slice_data, double* out) {
  ORC_TRY
  auto g = make_geometry(d);
  RVec o = backproject(*g, backend, alpha, to_cvec(slice_data, g->P));
  std::copy(o.begin(), o.end(), out);
  ORC_CATCH
}

int orc_split_bregman(const orc_geom* d, const orc_sb_config* c, const double* slice_data, double* mu,
                      double* update_l1, orc_sb_trace* trace) {
  ORC_TRY
  auto g = make_geometry(d);
  RVec m = split_bregman(*g, c, to_cvec(slice_data, g->P), update_l1, trace);
  std::copy(m.begin(), m.end(), mu);
  ORC_CATCH
}

int orc_tikhonov_identity(const orc_geom* d, double alpha, const double* slice_data, int steps,
                          double rel_tol, double* mu) {
  ORC_TRY
  auto g = make_geometry(d);
  const int64_t L = static_cast<int64_t>(g->n) * g->n;
  RVec rhs = backproject(*g, 0, alpha, to_cvec(slice_data, g->P));
  orc_system sd{0, 1, 0, alpha, 0.0, 0.0, 1};
  System sys = make_system(*g, &sd);
  RVec x = cg_solve(sys, rhs, RVec(L, 0.0), steps, rel_tol, nullptr);
  std::copy(x.begin(), x.end(), mu);
  ORC_CATCH
}

int orc_chambolle_pock(const orc_geom* d, const orc_cp_config* c, const double* slice_data, double* mu) {
  ORC_TRY
  auto g = make_geometry(d);
  RVec u = chambolle_pock(*g, c, to_cvec(slice_data, g->P));
  std::copy(u.begin(), u.end(), mu);
  ORC_CATCH
}

int orc_shepp_logan(int n, double* img) {
  ORC_TRY
  if (n < 4) throw ConfigError("generate_shepp_logan: n must be >= 4");
  constexpr double deg = M_PI / 180.0;
  const std::vector<Ellipse> table = {  // original Shepp-Logan table (image.cpp:37-48)
      {2.00, 0.6900, 0.9200, 0.00, 0.0000, 0.0},     {-0.98, 0.6624, 0.8740, 0.00, -0.0184, 0.0},
      {-0.02, 0.1100, 0.3100, 0.22, 0.0000, -18.0 * deg}, {-0.02, 0.1600, 0.4100, -0.22, 0.0000, 18.0 * deg},
      {0.01, 0.2100, 0.2500, 0.00, 0.3500, 0.0},     {0.01, 0.0460, 0.0460, 0.00, 0.1000, 0.0},
      {0.01, 0.0460, 0.0460, 0.00, -0.1000, 0.0},    {0.01, 0.0460, 0.0230, -0.08, -0.6050, 0.0},
      {0.01, 0.0230, 0.0230, 0.00, -0.6060, 0.0},    {0.01, 0.0230, 0.0460, 0.06, -0.6050, 0.0},
  };
  rasterize(n, table, img);
  ORC_CATCH
}

int orc_random_ellipses(int n, int count, uint64_t seed, double* img) {
  ORC_TRY
  if (n < 4) throw ConfigError("random_ellipses: n must be >= 4");
  rasterize(n, random_table(count, seed), img);
  ORC_CATCH
}

int orc_synthesize(const orc_geom* d, const double* phantom, double noise_frac, uint64_t seed,
                   double* samples, double* sigma_used) {
  ORC_TRY
  auto g = make_geometry(d);
  if (noise_frac < 0.0) throw ConfigError("synthesize_data: negative noise level");
  const int64_t L = static_cast<int64_t>(g->n) * g->n;
  CVec c(L);
  for (int64_t i = 0; i < L; ++i) c[i] = cd(phantom[i], 0.0);
  CVec v = type2(*g, c);
  double mx = 0.0;
  for (auto& z : v) mx = std::max(mx, std::abs(z));
  const double sigma = noise_frac * mx;
  if (sigma > 0.0) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, sigma);
    for (auto& z : v) {
      // The reference writes Complex(gauss(rng), gauss(rng)) (fourier_slice.cpp:80); g++
      // evaluates those arguments right to left, so the imaginary draw comes first.
      const double im = gauss(rng);
      const double re = gauss(rng);
      z += cd(re, im);
    }
  }
  if (sigma_used) *sigma_used = sigma;
  from_cvec(v, samples);
  ORC_CATCH
}

double orc_rel_l1(int64_t len, const double* cand, const double* ref) {
  double num = 0.0, den = 0.0;
  for (int64_t i = 0; i < len; ++i) {
    num += std::abs(cand[i] - ref[i]);
    den += std::abs(ref[i]);
  }
  return den == 0.0 ? -1.0 : num / den;
}

}  // extern "C"
