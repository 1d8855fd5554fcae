// kernels.h — host-side declarations of the sm_100a kernels' launchers and the device
// structures they share. No torch types; plain pointers and sizes. Every launcher is a
// template over the real type R (float or double), explicitly instantiated for both.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace tomo_b200 {

// Launch accounting + error check after every kernel launch (defined in tomo_capi.cu).
void note_launch();
// Error check of a cudaLaunchKernelEx status (throws CudaError).
void check_launch(cudaError_t e);
#define CK_LAUNCH(x) ::tomo_b200::check_launch(x)

// W^T entry: sample index + weight. fp32: 8 B {j, w}; fp64: 16 B {j, pad, w}.
template <typename R>
struct WtEnt;
template <>
struct alignas(8) WtEnt<float> {
  int j;
  float w;
};
template <>
struct alignas(16) WtEnt<double> {
  int j;
  int pad;
  double w;
};

// A sparse operator on the grid's row-sorted 32-node blocks, applied as a balanced list of warp
// tasks (used for W^T, input = samples, and for the Gram W^T W, input = the grid).
template <typename R>
struct TaskSpmv {
  const WtEnt<R>* ent;      // chunk-major: entry (chunk c, lane l) at [c*32 + l]; .j = input index
  const int4* tasks;        // {block, chunk0, nchunks, slot (-1: direct)}
  int n_tasks;
  const uint16_t* perm;     // [blocks*32] sorted position -> ix of the block's grid row
  const int4* heavy;        // {block, slot0, nslots, 0}
  const int* slot_heavy;    // slot -> heavy block index
  unsigned* heavy_cnt;      // B x n_heavy task tickets (zero between launches)
  int n_heavy;
  int n_slots;
  cplx<R>* part;            // B x n_slots x 32 partial sums of split blocks
};

// Operator tables + scratch for one device-resident normal operator (see DESIGN.md
// "HBM layout"). Grid nodes are stored transposed relative to the reference:
// node = iy*m + ix, where the reference has grid[ix*m + iy] (proj/src/nufft.cpp:185-200).
template <typename R>
struct OpDev {
  int n, m, nb, P, Ppad;
  int G32;                         // number of 32-node SELL blocks of W^T (= m*m/32)
  const R* apod;                   // n   : a[t]/m  (deconvolve, nufft.cpp:204-227, with 1/m per axis)
  const cplx<R>* tw;               // m   : e^{-2 pi i k/m}
  const cplx<R>* tw_half;          // m/2 : e^{-2 pi i k/(m/2)} (the split grid-row passes' half transforms)
  // Separable ("rank-1 block") storage of W: row j's w x w block is
  // wx_j[a] * wy_j[b] at nodes ((iy0+b) mod m, (ix0+a) mod m) (nufft.cpp:185-200).
  const int* w_base;               // [Ppad] ix0 | iy0 << 16
  const R* w_x;                    // [w][Ppad]
  const R* w_y;                    // [w][Ppad]
  const int* w_perm;               // [P] table position -> sample index: the separable tables are
                                   // stored in grid-tile order (spatial locality of the gathers).
                                   // With w_perm set, the op's internal sample vectors (W output,
                                   // W^T input, W^T entry indices) use positions; the reference
                                   // order only at the API boundary (forward/adjoint).
  int w_out_pos;                   // W writes sample t at position t (1) or at w_perm[t] (0)
  int w;                           // window width
  // W^T: nodes of each grid row sorted by entry count (SELL-32-sigma, sigma = one grid row);
  // the 32-node blocks are processed as a balanced list of warp tasks of <= kWtMaxChunks
  // chunks; blocks longer than that are split and their partial sums combined by a fix-up.
  const WtEnt<R>* wt_ent;          // chunk-major: entry (chunk c, lane l) at [c*32 + l]
  const int4* wt_tasks;            // {block, chunk0, nchunks, slot (-1: direct)}
  int n_tasks;
  const uint16_t* wt_perm;         // [G32*32] sorted position -> ix of the block's row
  const int4* wt_heavy;            // {block, slot0, nslots, 0}
  const int* wt_slot_heavy;        // slot -> heavy block index
  unsigned* wt_heavy_cnt;          // B x n_heavy task tickets (zero between launches)
  int n_heavy;
  int n_slots;
  cplx<R>* wt_part;                // B x n_slots x 32 partial sums of split blocks
  cplx<R>* Gt;                     // B x m x m  spread grid [iy][ix]; untouched nodes stay 0
  cplx<R>* Gth;                    // B x m x m  the folded spread grid, rows [0, m/2] (herm_out; own buffer)
  cplx<R>* H;                      // B x m x n  (type-2 row pass output, [iy][t1])
  cplx<R>* g;                      // B x m x m  (oversampled spatial grid, [iy][ix])
  cplx<R>* s;                      // B x P      (slice samples)
  cplx<R>* K;                      // B x n x m  (type-1 row pass output, [t1][iy])
  TaskSpmv<R> gram;                // fused backend: W^T W on the grid (n_tasks == 0 if not built)
  // Real-subspace ("Hermitian") pipeline, selected per call: a real input image has a Hermitian
  // spectrum, so type-2 keeps only grid rows iy in [0, m/2] (P1 transforms two real image rows
  // as one complex row, P2 runs m/2 + 1 rows, W reads row -iy as the conjugate of row iy); a
  // real-part output needs only the Hermitian part of the spread grid, so type-1 applies the
  // folded W^T (wth) onto rows [0, m/2], PA runs m/2 + 1 rows and PB transforms two image rows
  // per complex row (Hermitian extension on load).
  TaskSpmv<R> wth;                 // W^T folded onto rows [0, m/2] (entry .j bit 31 = conjugate)
  int herm_in;                     // type-2 of a real image through the half grid
  int herm_out;                    // type-1 real-part output through the folded half grid
  int s_stride;                    // slice stride of the sample vector (P; overlap pairs: 2P = samples | pair sums)

  TaskSpmv<R> wt_view() const {
    return TaskSpmv<R>{wt_ent, wt_tasks, n_tasks, wt_perm, wt_heavy, wt_slot_heavy, wt_heavy_cnt, n_heavy, n_slots,
                       wt_part};
  }
};

constexpr int kWtMaxChunks = 24;
// chunks per W^T / Gram warp task (longer blocks are split): kWtMaxChunks unless
// TOMO_WT_MAXCH overrides it (A/B runs; read once per process)
int wt_max_chunks();

// Per-slice scalar state of the device-resident CG / split-Bregman loops. All reductions
// land here through the last-block-reduces pattern (deterministic order).
struct SliceScalars {
  double rr[2];       // r.r, parity-indexed by CG step
  double pap, pp;     // p.Ap, p.p of the current step
  double bb;          // rhs.rhs (relative-tolerance test)
  double min_ritz;    // min p.Ap/p.p over the current CG call
  double upd;         // ||mu_new - mu_old||_1 of the last Bregman update
  double leak_num, leak_den;
  double first_upd;   // split Bregman: first update (stopping rule, solver.cpp:298-303)
  double sb_tol;      // update_tol_rel
  double dot;         // scratch dot product (Lanczos)
  double cg_alpha, cg_beta, cg_pp;  // Chronopoulos-Gear CG: alpha_k, beta_k, p.p (recurrence)
  double rs_last;     // the last r.r computed (CgStats::final_rs)
  int done;           // CG finished early (rs == 0, pAp == 0, tolerance)
  int nonfinite;      // sticky non-finite flag (-> NumericalError)
  int steps_run;
  int frozen;         // split Bregman stopped on tolerance: later iterations pass through
  int sb_iters;       // split Bregman iterations run
  int logged;         // iterations already appended to the recorded log (k_sb_log)
  unsigned counter[4];
};

// Reduction scratch: partials[slice][MAX_PART_BLOCKS][2].
constexpr int MAX_PART_BLOCKS = 8192;

struct Reduce {
  SliceScalars* sc;   // [B]
  double* part;       // [B][MAX_PART_BLOCKS][2]
};

// CG system: op(u) = alpha*B(u) + lambda*K'K u + shift*u  (solver.cpp:171-198, 323-327)
struct SysParams {
  double alpha, lambda, shift;
  double tol;          // relative residual tolerance (0 = off)
};

// PB_CGCG: Chronopoulos-Gear step (input r_k: w = A r_k, dots r.w and r.r; the last CTA
// derives alpha_k, beta_k and p.Ap by the recurrences, see cgcg_finalize)
enum PbMode { PB_COMPLEX = 0, PB_REAL = 1, PB_CG_STEP = 2, PB_CG_INIT = 3, PB_CGCG = 4 };

template <typename R>
struct PbEpi {
  int mode;
  R scale;                  // multiplies N u (alpha)
  cplx<R>* out_c;           // PB_COMPLEX
  R* out_r;                 // PB_REAL (and the sharded partial)
  // CG modes
  const R* p;               // STEP: p (after update); INIT: x0
  const R* b;               // INIT: rhs
  R* ap;                    // STEP: Ap out; INIT: r out
  R* p_out;                 // INIT: p = r
  R* x_out;                 // INIT: x = x0
  SysParams sys;
  int step;                 // CG step index (parity for rr)
  Reduce red;
};

// CG p-update fused into the first kernel of a step: p = r + beta p, beta = rr[k]/rr[k-1].
template <typename R>
struct PUpd {
  int enabled;              // 0: plain input
  R* r;                     // cgcg: read and written in place
  R* p;                     // read and written in place
  int step;
  Reduce red;
  // Chronopoulos-Gear (cgcg = 1, step k > 0): the vector update of step k-1 fused into the
  // load, p = r + beta p, s = w + beta s, x += alpha p, r -= alpha s; the FFT input is the new r
  int cgcg;
  const R* w;               // A r of step k-1
  R* s;                     // A p (recurrence)
  R* x;
};

// ---- launchers (nufft.cu) ----
template <typename R>
void launch_t2_rows(const OpDev<R>& d, int B, const void* in, bool in_complex, const PUpd<R>& pu, cudaStream_t st);
template <typename R>
void launch_t2_cols(const OpDev<R>& d, int B, const SliceScalars* skip, cudaStream_t st);
template <typename R>
void launch_w(const OpDev<R>& d, int B, const cplx<R>* grid, cplx<R>* samples, const SliceScalars* skip,
              cudaStream_t st);
template <typename R>
void launch_wt_rows(const OpDev<R>& d, int B, const SliceScalars* skip, cudaStream_t st);
// Overlap pairs, W by units (a mirror pair, or an unpaired sample): one thread reads the pair's
// (w + 1) x (w + 1) union window once and writes s_primary, s_partner = conj(sum with the shifted
// factors) and the pair sum. Tables in unit order (the tile order of the primaries / unpaired).
template <typename R>
struct PairW {
  int U, Upad;           // units, padded to 32
  const int* base;       // [Upad] the primary's (unpaired sample's) window base ix0 | iy0 << 16
  const R* fx;           // [w + 1][Upad] taps 0..w-1: the primary's x factors; tap w: the partner's own tap 0
  const R* fy;           // [w + 1][Upad]
  const int* pos;        // [Upad] output position of the primary (unpaired sample)
  const int* ppos;       // [Upad] output position of the partner, -1: unpaired
};
template <typename R>
void launch_w_pair(const OpDev<R>& d, const PairW<R>& pw, int B, const cplx<R>* grid, cplx<R>* samples,
                   const SliceScalars* skip, cudaStream_t st);
// Overlap pairs (opbuild.cu): s[P + t] = s[t] + conj(s[ppos[t]]) for the positions t of pair primaries
template <typename R>
void launch_pair_sigma(cplx<R>* s, int B, int P, int stride, const int* ppos, cudaStream_t st);
// W^T SpMV alone: samples -> spread grid (task kernel + split-block fix-up); `grid` must hold
// zeros at untouched nodes (they are never written).
template <typename R>
void launch_wt_spread(const OpDev<R>& d, int B, const cplx<R>* samples, cplx<R>* grid, const SliceScalars* skip,
                      cudaStream_t st);
template <typename R>
void launch_t1_cols_only(const OpDev<R>& d, int B, const SliceScalars* skip, cudaStream_t st);
// Fused (Gram) backend: grid_out = (W^T W) grid_in on the oversampled grid.
template <typename R>
void launch_gram(const OpDev<R>& d, int B, const cplx<R>* grid_in, cplx<R>* grid_out, const SliceScalars* skip,
                 cudaStream_t st);
template <typename R>
void launch_t1_rows(const OpDev<R>& d, int B, const PbEpi<R>& e, cudaStream_t st);
template <typename R>
void launch_wt_grid(const OpDev<R>& d, int B, const cplx<R>* samples, cplx<R>* grid, cudaStream_t st);
template <typename R>
void launch_weight_samples(cplx<R>* s, int B, int P, int nb, const int* perm, cudaStream_t st);
// out[b][t] = in[b][perm[t]] (reference sample order -> the op's position order)
template <typename R>
void launch_gather_samples(const cplx<R>* in, cplx<R>* out, const int* perm, int B, int P, cudaStream_t st);
// fk += f - s, s = fk (split-Bregman data feedback)
template <typename R>
void launch_feedback_samples(int64_t n, cplx<R>* fk, const cplx<R>* f, cplx<R>* s, cudaStream_t st);
template <typename R>
void launch_fft_rows_test(int m, int rows, const cplx<R>* tw, const cplx<R>* in, cplx<R>* out, bool inverse,
                          cudaStream_t st);

// ---- operator construction on the device (opbuild.cu) ----
struct BuildArgs {
  int m, nb, lo, hi, w;
  int64_t P, Ppad;
  double tau;
};
struct GpuBuildSizes {
  int64_t chunks = 0;   // W^T chunks (slots / 32)
  int n_tasks = 0, n_slots = 0, n_heavy = 0;
  int64_t touched = 0;  // non-empty W^T rows
  int64_t nnz = 0;      // entries
};
struct GpuBuild;
bool wt_row_order(int m);  // W^T warp-task order (opbuild.cu)
// plan + separable W (written to base/wx/wy) + W^T structure; returns the table sizes
template <typename R>
GpuBuild* gpu_build_begin(const BuildArgs& a, const double* h_cs, const double* h_e3, int* base, R* wx, R* wy,
                          cudaStream_t st, GpuBuildSizes* sizes);
// W^T entries / tasks / perm / heavy tables into caller-allocated buffers
template <typename R>
void gpu_build_finish(GpuBuild* b, WtEnt<R>* ent, int4* tasks, uint16_t* perm, int4* heavy, int* slot_heavy,
                      cudaStream_t st);
void gpu_build_free(GpuBuild* b);
// The Gram W^T W of the fused backend from fp64 window factors (P x w each) and window bases
// (ix0 | iy0 << 16); same tables as the host TaskBuilder path. nullptr: too large for this
// builder (the host build runs instead). Finish with gpu_build_finish.
template <typename R>
GpuBuild* gpu_build_gram_begin(int m, int w, int64_t P, const int* h_base, const double* h_wx, const double* h_wy,
                               cudaStream_t st, GpuBuildSizes* sizes, int64_t* nnz_out);
// Re-order the separable W tables (base, wx, wy; [Ppad] / [w][Ppad]) by 16x16 grid tile of the
// window base; perm[t] = sample stored at position t.
// ent / ent2: W^T entry streams whose sample indices are remapped to positions (bit 31, the
// Hermitian fold's conj flag, is kept).
template <typename R>
void gpu_sort_w_tables(int m, int64_t P, int64_t Ppad, int w, int* base, R* wx, R* wy, int* perm, WtEnt<R>* ent,
                       int64_t n_ent, WtEnt<R>* ent2, int64_t n_ent2, cudaStream_t st);
// Hermitian fold of a finished (unfolded) W^T build: nodes of grid rows [0, m/2], each with its own
// entries and the conjugated entries of its mirror node (-iy, -ix). Finish with gpu_build_finish.
template <typename R>
GpuBuild* gpu_build_fold(const GpuBuild* src, cudaStream_t st, GpuBuildSizes* sizes, const int* pair = nullptr,
                         const int* base = nullptr);
// Mirror pairs of the samples (opbuild.cu "mirror pairs"): pair[j] = mirror sample or -1, from the
// separable W tables in sample order; returns the number of paired samples. With `pair`,
// gpu_build_fold drops the secondaries' entries and doubles the primaries' (entry indices stay
// sample indices until gpu_half_w_finish remaps them).
template <typename R>
int64_t gpu_find_pairs(const BuildArgs& a, const int* base, const R* wx, const R* wy, int* pair, cudaStream_t st);
// The half W: the tile-ordered separable tables (after gpu_sort_w_tables; perm = position -> sample)
// compacted to the samples that are not secondaries (Ph of them, order kept); `ent` (the mirror-pair
// W^T's entries, sample indices) is remapped to the compact positions, a secondary to its primary's.
// Overlap pairs (windows [-h, h] around floor(x / h): the mirror sample's window is the mirror image
// shifted by one node): with `base` (sample order) gpu_build_fold keeps every sample's own entries
// outside the overlap, drops the secondaries' overlap entries and points the primaries' at the pair
// sum (index P + j). gpu_pair_sigma_setup then remaps the entries to positions (P + position for
// pair sums) and fills ppos[t] = position of the partner of the primary at position t, else -1.
template <typename R>
void gpu_pair_sigma_setup(int64_t P, const int* perm, const int* pair, WtEnt<R>* ent, int64_t n_ent, int* ppos,
                          cudaStream_t st);
struct HalfWBuild;
HalfWBuild* gpu_half_w_begin(int64_t P, const int* perm, const int* pair, cudaStream_t st, int64_t* Ph);
template <typename R>
void gpu_half_w_finish(HalfWBuild* hb, int64_t Ppad, int64_t Ppad_h, int w, const int* perm, const int* pair,
                       const int* base, const R* wx, const R* wy, int* base_h, R* wx_h, R* wy_h, WtEnt<R>* ent,
                       int64_t n_ent, cudaStream_t st);
void gpu_half_w_free(HalfWBuild* hb);
// Overlap pairs: the unit tables of PairW from the tile-ordered W tables, the kept flags / compact
// indices of gpu_half_w_begin (units = the samples that are not secondaries) and the partner
// positions `ppos` of gpu_pair_sigma_setup.
template <typename R>
void gpu_pair_w_finish(HalfWBuild* hb, int64_t Ppad, int64_t Upad, int w, const int* ppos, const int* base,
                       const R* wx, const R* wy, int* ubase, R* ufx, R* ufy, int* upos, int* uppos, cudaStream_t st);

// ---- launchers (solver.cu) ----
struct StencilCoef {
  double c[81];             // (2r+1)^2 row-major, r <= 4
};
template <typename R>
void launch_cg_update(int n, int B, const R* p, const R* ap, R* x, R* r, const SysParams& sys, int step,
                      const Reduce& red, cudaStream_t st);
template <typename R>
void launch_cgcg_final(int n, int B, const R* w, R* p, R* s, R* x, R* r, const SysParams& sys, int steps,
                       const Reduce& red, cudaStream_t st);
// Surrogate system apply with fused p-update (mode 0: step, 1: init, 2: plain apply out=op(in)).
template <typename R>
void launch_stencil(int n, int B, int rad, const StencilCoef& coef, int mode, const R* in, const R* r_in, R* p_out,
                    R* ap_out, const R* b, R* x_out, const SysParams& sys, int step, const Reduce& red,
                    cudaStream_t st);
// Sharded-operator CG epilogue: ap = red + lambda K'K p + shift p (mode 0) / init (mode 1).
template <typename R>
void launch_cg_epilogue(int n, int B, int mode, const R* nred, const R* p, const R* b, R* ap, R* p_out, R* x_out,
                        const SysParams& sys, int step, const Reduce& red, cudaStream_t st);
template <typename R>
void launch_sb_post(int n, int B, R* mu_new, const R* mu_old, const R* bx_old, const R* by_old, R* bx_new, R* by_new,
                    const R* fid, R* rhs, double lambda, const Reduce& red, cudaStream_t st);
template <typename R>
void launch_cp_dual(int n, int B, const R* u_cur, const R* u_prev, const R* yx_old, const R* yy_old, R* yx_new,
                    R* yy_new, const R* bp, R* rhs, double tau, double sigma, double theta, double lambda,
                    cudaStream_t st);
template <typename R>
void launch_axpby(int64_t len, double a, const R* x, double b, const R* y, R* out, cudaStream_t st);
template <typename R>
void launch_dot(int n, int B, const R* x, const R* y, const Reduce& red, cudaStream_t st);
template <typename R>
void launch_leak(int64_t len, const cplx<R>* v, const Reduce& red, cudaStream_t st);
template <typename R>
void launch_sb_log(int n, int B, const R* mu, const R* ref, double* upd_log, double* rel_log, const Reduce& red,
                   cudaStream_t st);
template <typename R>
void launch_grad(int n, int B, const R* u, R* gx, R* gy, cudaStream_t st);
template <typename R>
void launch_grad_adjoint(int n, int B, const R* gx, const R* gy, R* out, cudaStream_t st);
template <typename R>
void launch_shrink(int64_t len, const R* x, double gamma, R* out, cudaStream_t st);

}  // namespace tomo_b200
