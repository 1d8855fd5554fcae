/*
 * tomo_b200.h — C ABI of the B200-native (sm_100a) CT normal-operator library
 *               (libtomo_b200.so, built from paper_1705_07497_b200/csrc).
 *
 * Drop-in boundary for the reference's operator/solver API (proj/include/tomo/*.hpp),
 * which has no FFI of its own: build-operator, apply, CG, split-Bregman driver. Each entry
 * point below names the reference interface it replaces. Plain pointers and sizes only; no
 * exceptions cross the ABI (status codes mirror the reference's exception classes and CLI
 * exit codes, proj/include/tomo/errors.hpp:9-30, proj/tools/tomo_main.cpp:88-97).
 *
 * Memory: every array argument may be a DEVICE pointer (cudaMalloc / torch CUDA tensor on
 * the op's device; the call is asynchronous on `stream`) or a HOST pointer (the library
 * stages through device scratch and synchronizes `stream` before returning).
 * Precision: an op is created TOMO_F32 (real arrays float32, complex arrays interleaved
 * complex64) or TOMO_F64 (float64 / complex128); every array passed to that op uses its
 * element type. Images are row-major n x n, slice samples
 * angle-major (row j = a*n_b + t), exactly the reference's layouts
 * (proj/include/tomo/image.hpp:11-13, proj/include/tomo/fourier_slice.hpp:20-27).
 * `batch` independent slices are stored back to back.
 *
 * Threading: an op's tables are immutable after tomo_op_create, and
 * one op may serve several host threads / streams at once. Each call leases a private
 * workspace (device scratch, lanes, captured CUDA graphs) for its stream: concurrent calls on
 * distinct streams run concurrently on distinct workspaces (up to 8 per op); a workspace
 * handed from one stream to another is ordered after the previous stream's work by an event.
 * tomo_op_set_allreduce / tomo_op_attach_nccl must not race with calls on the same op.
 */
#ifndef TOMO_B200_H
#define TOMO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define TOMO_OK 0
#define TOMO_ERR_CONFIG 2    /* tomo::ConfigError    */
#define TOMO_ERR_NUMERICAL 3 /* tomo::NumericalError */
#define TOMO_ERR_IO 4        /* tomo::IoError        */
#define TOMO_ERR_CUDA 5      /* CUDA / NCCL failure (no reference analogue) */

/* precisions (the reference computes in fp64, proj/include/tomo/image.hpp:11-13) */
#define TOMO_F32 0
#define TOMO_F64 1

/* backends — tomo::BackendKind (proj/include/tomo/normal_ops.hpp:10) */
#define TOMO_BACKEND_DIRECT 0    /* W / W^T sparse interpolation pair (the GPU form of "direct") */
#define TOMO_BACKEND_FUSED 1     /* Gram W^T W on the oversampled grid (make_fused_backend) */
#define TOMO_BACKEND_SURROGATE 2 /* truncated translated stencil T */

/* Geometry: SliceGrid + NufftParams (fourier_slice.hpp:24-28, nufft.hpp:16-21) with the
 * documented extensions: n_b radial samples (0 -> n), oversampling R (0 -> 2), window
 * offsets [win_lo, win_hi] (reference: [-m_sp, m_sp]), explicit tau, explicit angles
 * (NULL -> theta_a = a*pi/n_angles, fourier_slice.cpp:18). Same layout as the oracle's. */
typedef struct tomo_geom_desc {
  int n;
  int n_angles;
  int n_b;
  int oversample;
  int win_lo, win_hi;
  double tau;
  const double* angles;
} tomo_geom_desc;

typedef struct tomo_op_desc {
  int backend;      /* TOMO_BACKEND_* */
  int surrogate_r;  /* SurrogateConfig::radius_r (normal_ops.hpp:14), 1..4 */
  int euclidean;    /* SurrogateConfig::euclidean */
  int device;       /* CUDA device ordinal */
  int angle_begin;  /* angle-block row shard [begin, end) of W; 0,0 -> all angles */
  int angle_end;
  int max_batch;    /* slices per call the scratch is sized for (>= 1) */
  int precision;    /* TOMO_F32 | TOMO_F64 */
  int64_t mem_cap_bytes; /* fused backend: refuse Gram builds whose estimate exceeds this
                          * (build_btb, normal_ops.cpp:81-84); 0 -> kDefaultBtbMemCap = 8 GiB */
} tomo_op_desc;

typedef struct tomo_op tomo_op;

typedef struct tomo_op_info {
  int n, m, n_b, n_angles_local, window;
  int64_t P;            /* local slice samples (rows of W) */
  int64_t nnz;          /* W non-zeros (= P * window^2) */
  int64_t wt_rows;      /* touched grid nodes (non-empty W^T rows) */
  int64_t wt_slots;     /* W^T task-SpMV slots incl. padding (32-node blocks, count-sorted rows) */
  int64_t bytes_w;      /* device bytes of the W tables */
  int64_t bytes_wt;     /* device bytes of the W^T tables */
  double stencil[81];   /* surrogate stencil (2r+1)^2, fp64 host copy */
  int surrogate_r;
  int precision;
  int backend;
  int64_t gram_nnz;     /* fused backend: non-zeros of W^T W (= build_btb's CSR nnz) */
  int64_t gram_slots;   /* fused backend: task-SpMV slots incl. padding */
  int64_t bytes_gram;   /* fused backend: device bytes of the Gram tables */
  /* W^T folded onto the Hermitian half grid (rows iy in [0, m/2]) for real-part outputs */
  int64_t herm_nnz;     /* entries (= nnz + the entries of grid rows 0 and m/2, listed twice) */
  int64_t herm_slots;   /* task-SpMV slots incl. padding */
  int64_t herm_touched; /* touched half-grid nodes */
  int herm_tasks;       /* warp tasks (0: not built, real inputs take the full grid) */
  /* Mirror pairs of the parallel-beam samples (bins t and 2 (n_b / 2) - t of one angle lie at
   * mirrored frequencies; with a window [1 - hi, hi] their interpolation windows are mirror images).
   * For real images the normal operator then runs W on one sample per pair and the folded W^T of
   * the pairs' primaries only. With a symmetric window [-m_sp, m_sp] around floor(x / h) (the
   * reference's) the partner's window is the mirror image shifted by one node: W evaluates every
   * sample (sym_P = P) and the pair sums, reading each pair's union window once, and the fold reads
   * the pair sums inside the pairs' common window (63 % of the entries at m_sp = 3). 0 everywhere:
   * no pairs, the full fold runs. */
  int sym_tasks;        /* warp tasks of the primaries' folded W^T (0: not built) */
  int64_t sym_pairs;    /* samples that have a mirror partner (both members counted) */
  int64_t sym_P;        /* samples W evaluates on the real-subspace normal operator */
  int64_t sym_nnz;      /* entries of the primaries' folded W^T */
  int64_t sym_slots;    /* its task-SpMV slots incl. padding */
} tomo_op_info;

const char* tomo_last_error(void);

/* make_direct_backend / make_fused_backend / make_surrogate_backend (normal_ops.hpp:35-39)
 * over a SliceTransform(SliceGrid, NufftParams) (fourier_slice.hpp:39). Builds W (separable
 * per-sample window factors), its row-sorted transpose W^T and the Hermitian fold of W^T
 * (real-part outputs on half the grid rows), deapodisation and FFT tables on `device`; for the
 * fused backend also
 * the Gram W^T W (build_btb, normal_ops.hpp:47); for the surrogate also the stencil
 * (build_surrogate, normal_ops.hpp:60). */
int tomo_op_create(const tomo_geom_desc* geom, const tomo_op_desc* desc, tomo_op** out);
void tomo_op_destroy(tomo_op* op);
int tomo_op_get_info(const tomo_op* op, tomo_op_info* info);

/* ---- the reference's on-disk operators, TOMOSPM1 (save_sparse / load_sparse,
 * proj/src/sparse.cpp:68-141; cache keying bench.cpp:62-114) ---- */
typedef struct tomo_tspm_meta {
  int64_t rows, cols, nnz;
  int symmetric;
  int n, m_sp;          /* provenance trailer (SparseOperator::Meta, sparse.hpp:20-28) */
  double tau;
  int angle_count, d, r; /* r = 0: Gram B*B (fused); r >= 1: surrogate T */
} tomo_tspm_meta;
/* load_sparse + SparseOperator::validate of `path` (no GPU needed). */
int tomo_tspm_info(const char* path, tomo_tspm_meta* info);
/* make_fused_backend / make_surrogate_backend with the sparse operator read from a TOMOSPM1
 * file (bench.cpp:78-114 load_or_build_sparse): desc->backend TOMO_BACKEND_FUSED takes a Gram,
 * TOMO_BACKEND_SURROGATE a surrogate T (radius and truncation from the file). The trailer must
 * match the geometry (meta_matches, bench.cpp:78-84) -> TOMO_ERR_CONFIG otherwise; unreadable
 * or truncated files -> TOMO_ERR_IO. */
int tomo_op_create_tspm(const tomo_geom_desc* geom, const tomo_op_desc* desc, const char* path, tomo_op** out);
/* save_sparse of the op's Gram (fused) or surrogate T in the reference's layout, with the
 * trailer {n, m_sp, tau, angle_count, d = angle_subsample_d, r}. */
int tomo_op_save_tspm(const tomo_op* op, const char* path, int angle_subsample_d);

/* apply_normal (normal_ops.hpp:65): complex n^2 -> complex n^2, batch slices. */
int tomo_apply_normal(tomo_op* op, const void* in, void* out, int batch, void* stream);
/* apply_normal_real (normal_ops.hpp:69): Re(N u) for real u (surrogate: T u). */
int tomo_apply_normal_real(tomo_op* op, const void* in, void* out, int batch, void* stream);
/* SliceTransform::forward (type-2, fourier_slice.hpp:43): complex image n^2 -> samples P. */
int tomo_forward(tomo_op* op, const void* image, void* samples, int batch, void* stream);
/* forward_transform (fourier_slice.cpp:61-64): type-2 of a REAL image n^2 -> complex samples P
 * (the image's Hermitian spectrum: half the grid rows are transformed). */
int tomo_forward_real(tomo_op* op, const void* image, void* samples, int batch, void* stream);
/* SliceTransform::adjoint (type-1, fourier_slice.hpp:46): complex samples P -> image n^2. */
int tomo_adjoint(tomo_op* op, const void* samples, void* image, int batch, void* stream);
/* interpolate (W, nufft.hpp:66) / spread (W^T, nufft.hpp:62) alone, on the op's internal
 * grid layout: node = iy*m + ix (the reference's grid[ix*m + iy] transposed). */
int tomo_spmv_w(tomo_op* op, const void* grid, void* samples, int batch, void* stream);
int tomo_spmv_wt(tomo_op* op, const void* samples, void* grid, int batch, void* stream);
/* Back-projection of make_subproblem (solver.cpp:200-213): alpha*Re(F_NU f); weighted=1
 * multiplies samples by the radial density weights first (surrogate fidelity). */
int tomo_backproject(tomo_op* op, double alpha, int weighted, const void* slice_data, void* out, int batch,
                     void* stream);

/* ---- CG (cg_solve, solver.hpp:43-44) on op(u) = alpha*B(u) + lambda*K'K u + shift*u, with
 * B = Re(N) (direct) or T (surrogate). The reference's systems: split Bregman
 * (alpha, lambda, sigma); Tikhonov identity-K: (alpha, 0, 1 + sigma). */
typedef struct tomo_system {
  double alpha, lambda, shift;
} tomo_system;

typedef struct tomo_cg_stats { /* CgStats (solver.hpp:34-38) */
  int steps_run;
  double min_ritz;
  double final_rs;
} tomo_cg_stats;

/* x0 may be NULL (zero start). stats: host array of `batch` entries or NULL. */
int tomo_cg(tomo_op* op, const tomo_system* sys, const void* rhs, const void* x0, void* x, int steps,
            double rel_tol, int batch, tomo_cg_stats* stats, void* stream);

/* ---- split_bregman_tv (solver.hpp:83-85) */
typedef struct tomo_sb_config { /* SolverConfig (solver.hpp:51-65) */
  double alpha, lambda;
  int max_iters;        /* max_bregman_iters */
  int cg_steps;         /* cg_steps_per_update */
  double update_tol_rel;
  int warm_start;
  double sigma_override; /* < 0: surrogate sigma from Lanczos (solver.cpp:175-192) */
  int data_feedback;     /* outer residual feedback on the data term (solver.hpp:58-61,
                          * solver.cpp:176-187, 283-286); 0 = off (the reference default) */
} tomo_sb_config;

typedef struct tomo_sb_trace { /* SolveTrace (solver.hpp:67-80), per slice */
  int iterations;
  double first_update_l1;
  double sigma;
  double min_ritz;
  double imag_leakage;
  int stopped_on_tolerance;
} tomo_sb_trace;

/* slice_data: batch x P complex; mu: batch x n^2 real. update_l1: host, batch x
 * max_iters (or NULL); trace: host, batch entries (or NULL). Synchronizes `stream`. */
int tomo_split_bregman(tomo_op* op, const tomo_sb_config* cfg, const void* slice_data, void* mu, int batch,
                       double* update_l1, tomo_sb_trace* trace, void* stream);
/* The same solve with the reference's full per-iteration trace (SolveTrace, solver.hpp:67-80;
 * record_reference, solver.cpp:291-294): update_l1 and rel_l1_err (batch x max_iters, host;
 * rel_l1_err needs `reference`, batch x n^2 of the op's element type, else NULL), t_total_s and
 * t_cg_s (max_iters, host; CUDA-event times from the start of the Bregman loop, the CG part
 * accumulated like t_cg). One CG graph and one update graph per iteration. */
int tomo_split_bregman_record(tomo_op* op, const tomo_sb_config* cfg, const void* slice_data, void* mu, int batch,
                              const void* reference, double* update_l1, double* rel_l1_err, double* t_total_s,
                              double* t_cg_s, tomo_sb_trace* trace, void* stream);

/* ---- tikhonov_solve with K = identity (solver.cpp:309-337) at a fixed step count:
 * cg_solve(alpha N + I, alpha Re(F_NU f), 0, steps, rel_tol). */
int tomo_tikhonov(tomo_op* op, double alpha, const void* slice_data, void* mu, int steps, double rel_tol,
                  int batch, void* stream);

/* ---- Chambolle-Pock anisotropic TV (extension): prox of the data term
 * (I + tau_cp*alpha*Re N) u = u~ + tau_cp*alpha*Re(F_NU f) by `cg_steps` CG steps. */
typedef struct tomo_cp_config {
  double alpha, lambda, tau_cp, sigma_cp, theta;
  int iters, cg_steps;
} tomo_cp_config;
int tomo_chambolle_pock(tomo_op* op, const tomo_cp_config* cfg, const void* slice_data, void* mu, int batch,
                        void* stream);

/* ---- angle-row sharding across GPUs: the partial adjoint images of each rank's angle
 * block are summed by this hook (in place, `count` elements of the op's precision, float32
 * or float64 as `precision` says, ordered on `stream`) after every type-1 transform. The hook
 * runs on the host and may synchronize `stream`; an op with a hook (and no NCCL communicator)
 * therefore runs its solver loops without CUDA graphs. tomo_op_attach_nccl installs an NCCL all-reduce over a communicator built from
 * a unique id obtained with tomo_nccl_unique_id on one rank and broadcast by the caller. */
typedef int (*tomo_allreduce_fn)(void* buf, size_t count, int precision, void* stream, void* user);
int tomo_op_set_allreduce(tomo_op* op, tomo_allreduce_fn fn, void* user);
int tomo_nccl_unique_id(char out[128]);
int tomo_op_attach_nccl(tomo_op* op, const char id[128], int nranks, int rank);

/* ---- element pieces (solver.cpp:12-54), device pointers of the given precision */
int tomo_grad(int n, int precision, const void* u, void* gx, void* gy, int batch, void* stream);
int tomo_grad_adjoint(int n, int precision, const void* gx, const void* gy, void* out, int batch, void* stream);
int tomo_shrink(int64_t len, int precision, const void* x, double gamma, void* out, void* stream);

/* ---- synthetic inputs (host): image.cpp:22-67 rasteriser; random-ellipse table (extension,
 * same mapping as the oracle: centre 1.2u-0.6, semi-axes 0.05+0.35u, rotation pi(2u-1),
 * intensity u, u = (mt19937_64() >> 11) * 2^-53). */
int tomo_shepp_logan(int n, float* img);
int tomo_random_ellipses(int n, int count, uint64_t seed, float* img);

/* Test hook: one batch of length-m FFT rows through the in-CTA Stockham kernel. */
int tomo_fft_rows(int m, int rows, int precision, const void* in, void* out, int inverse, void* stream);

/* Stage profiler (measurement, not part of the reference API): runs `reps` solver steps of
 * the op's hot path on internal scratch with CUDA events between kernels on `stream` and
 * returns, per stage, the mean device time (ms) and the algorithmic HBM bytes one launch
 * moves. complex_io = 0: the solvers' real-image path (the
 * Hermitian half grid where available); 1: complex applies (complex in, complex out). Stage ids:
 *   0 t2_rows (P1: p-update + deapod + pad + row iFFT)   1 t2_cols (P2: column iFFT)
 *   2 w (W: separable window SpMV)   3 wt_spread (W^T task SpMV + split-block fix-up)
 *   4 t1_cols (PA: grid-row FFT, pruned)   5 t1_rows (PB: FFT + crop + deapod + CG epilogue)
 *   6 cg_update   7 sb_post   8 stencil (surrogate T + K'K + CG dots)
 * Stages that do not apply to the backend report 0. Returns TOMO_OK. */
#define TOMO_NUM_STAGES 9
int tomo_profile_stages(tomo_op* op, int batch, int reps, int complex_io, double* ms, double* bytes, void* stream);

/* Number of library kernels launched since load (for the bench's gpu_launches claim). */
int64_t tomo_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif
