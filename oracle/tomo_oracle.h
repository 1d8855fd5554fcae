/*
 * tomo_oracle.h — CPU fp64 restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This library is the parity checker for the B200 product library (libtomo_b200.so).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it. The product never links or calls it.
 *
 * It restates, function by function, the reference's single-threaded C++ (Eigen) code
 * under /root/reference/proj (cited per function in oracle.cpp), in plain C++17 with
 * std::complex<double> and its own FFT, plus the documented extensions D1-D5, D7, D10
 * of SURVEY.md §0.1 (n_b radial samples, explicit angle counts, general window
 * [lo,hi], explicit tau, oversampling R, random-ellipse phantom, relative noise,
 * Chambolle-Pock).  With n_b = n, R = 2, window [-m_sp, m_sp], tau = m_sp/n^2 the
 * geometry is the reference's bit for bit.
 *
 * Parity pin: oracle/_ref/libtomo_ref.so is the reference's own sources compiled
 * against an Eigen-API shim (oracle/eigen_shim); tests/test_oracle_pin.py compares the
 * two and tests/golden/ holds vectors generated from the reference build.
 *
 * Complex arrays are interleaved (re, im) doubles. All functions return 0 on success,
 * 2 on a configuration error, 3 on a numerical error (same codes as the reference CLI,
 * proj/tools/tomo_main.cpp:88-97); orc_last_error() gives the message.
 */
#ifndef TOMO_ORACLE_H
#define TOMO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int n;               /* image side, even, >= 4 */
  int n_angles;        /* number of projection angles A */
  int n_b;             /* radial samples per angle (0 -> n, the reference) */
  int oversample;      /* R, grid side m = R*n (0 -> 2, the reference) */
  int win_lo, win_hi;  /* window offsets l in [lo, hi]; reference: [-m_sp, m_sp] */
  double tau;          /* Gaussian parameter; reference: m_sp / n^2 */
  const double* angles;/* optional explicit angles (n_angles); NULL -> theta_a = a*pi/A */
} orc_geom;

const char* orc_last_error(void);

/* Sensitivity probe (tests only; 0 = off, the default): multiply every real normal-operator
 * input and output by (1 + eps * N(0,1)) elementwise, seeded. */
void orc_set_perturbation(double eps, uint64_t seed);
/* Inner-product summation of the CG / Lanczos recurrences: 1 = compensated (default), 0 = plain
 * sequential (probe). */
void orc_set_dot_mode(int mode);

/* ---- geometry / plan (fourier_slice.cpp:10-41, nufft.cpp:43-101) ---- */
int64_t orc_num_points(const orc_geom* g);
int orc_points(const orc_geom* g, double* coords /* P x 2 */);
int orc_plan(const orc_geom* g, int* nearest /* P x 2 */, double* e1 /* P x 2 */,
             double* e2 /* P x 2 */, double* e3 /* w */);
int orc_weights(const orc_geom* g, double* wx /* P x w */, double* wy /* P x w */);
int orc_deapod(const orc_geom* g, double* a /* n */);

/* ---- NUFFT pieces (nufft.cpp:119-286, fft.cpp:26-50) ---- */
int orc_fft2(int m, double* grid /* m*m complex, in place */, int inverse);
int orc_interpolate(const orc_geom* g, const double* grid, double* samples);
int orc_spread(const orc_geom* g, const double* samples, double* grid);
int orc_type2(const orc_geom* g, const double* coeffs, double* samples);
int orc_type1(const orc_geom* g, const double* samples, double* coeffs);
int orc_direct_ndft(const orc_geom* g, const double* input, double* output, int type1);

/* ---- normal operator (normal_ops.cpp:28-30, 175-206, 321-340) ---- */
int orc_apply_normal(const orc_geom* g, const double* in, double* out); /* complex n^2 */
int orc_apply_normal_real(const orc_geom* g, const double* in, double* out); /* real n^2 */
/* Gram (fused) backend: build_btb + apply_normal_fused (normal_ops.cpp:53-206). */
int64_t orc_btb_nnz(const orc_geom* g);
int orc_apply_normal_fused(const orc_geom* g, const double* in, double* out);

/* ---- surrogate (normal_ops.cpp:208-288) ---- */
int orc_radial_weights(const orc_geom* g, double* w /* P */);
int orc_weighted_normal_real(const orc_geom* g, const double* w, const double* in, double* out);
int orc_surrogate_stencil(const orc_geom* g, int r, double* stencil /* (2r+1)^2 */);
int orc_apply_stencil(int n, int r, int euclidean, const double* stencil, const double* in,
                      double* out);

/* ---- solver pieces (solver.cpp:12-54) ---- */
int orc_grad(int n, const double* u, double* gx, double* gy);
int orc_grad_adjoint(int n, const double* gx, const double* gy, double* out);
int orc_shrink(int64_t len, const double* x, double gamma, double* out);

/* System operator  op(u) = alpha*B(u) + lambda*K'K u + shift*u  with
 * B = Re(N) (backend 0, direct W/W^T path) or the surrogate stencil T (backend 2).
 * identity_k != 0 selects the Tikhonov identity-K system alpha*B(u) + u + shift*u
 * (solver.cpp:323-327). */
typedef struct {
  int backend;      /* 0 direct, 1 fused (Gram), 2 surrogate */
  int surrogate_r;  /* radius r */
  int euclidean;    /* surrogate truncation */
  double alpha, lambda, shift;
  int identity_k;
} orc_system;

typedef struct {
  int steps_run;
  double min_ritz;
  double final_rs;
} orc_cg_stats;

int orc_system_apply(const orc_geom* g, const orc_system* s, const double* u, double* out);
int orc_cg(const orc_geom* g, const orc_system* s, const double* rhs, const double* x0,
           int steps, double rel_tol, double* x, orc_cg_stats* stats);
/* sigma of make_subproblem (solver.cpp:175-192), no-feedback branch. */
int orc_surrogate_sigma(const orc_geom* g, int r, int euclidean, double alpha, double lambda,
                        double* sigma);
int orc_lanczos_extreme(const orc_geom* g, const orc_system* s, int iters, uint64_t seed,
                        int largest, double* value);

typedef struct {
  int backend, surrogate_r, euclidean;
  double alpha, lambda;
  int max_iters, cg_steps;
  double update_tol_rel;
  int warm_start;
  double sigma_override; /* < 0 -> compute (Lanczos) */
  int data_feedback;     /* SolverConfig::data_feedback (solver.cpp:176-187, 283-286) */
} orc_sb_config;

typedef struct {
  int iterations;
  double first_update_l1;
  double sigma;
  double min_ritz;
  double imag_leakage;
  int stopped_on_tolerance;
} orc_sb_trace;

int orc_backproject(const orc_geom* g, int backend, double alpha, const double* slice_data,
                    double* out);
int orc_split_bregman(const orc_geom* g, const orc_sb_config* c, const double* slice_data,
                      double* mu, double* update_l1 /* max_iters, may be NULL */,
                      orc_sb_trace* trace);
/* Config-1 KKT solve: cg_solve(alpha N + I, alpha Re(F_NU f), 0, steps, rel_tol). */
int orc_tikhonov_identity(const orc_geom* g, double alpha, const double* slice_data, int steps,
                          double rel_tol, double* mu);

/* Chambolle-Pock anisotropic TV (extension D10). */
typedef struct {
  double alpha, lambda;
  double tau_cp, sigma_cp, theta;
  int iters, cg_steps;
} orc_cp_config;
int orc_chambolle_pock(const orc_geom* g, const orc_cp_config* c, const double* slice_data,
                       double* mu);

/* ---- inputs (image.cpp:22-76, fourier_slice.cpp:71-83) ---- */
int orc_shepp_logan(int n, double* img);
int orc_random_ellipses(int n, int count, uint64_t seed, double* img);
int orc_synthesize(const orc_geom* g, const double* phantom, double noise_frac, uint64_t seed,
                   double* samples, double* sigma_used);
double orc_rel_l1(int64_t len, const double* cand, const double* ref);

#ifdef __cplusplus
}
#endif
#endif
