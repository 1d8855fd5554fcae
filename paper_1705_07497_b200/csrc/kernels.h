// kernels.h — host-side declarations of the sm_100a kernels' launchers and the device
// structures they share. No torch types; plain pointers and sizes.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tomo_b200 {

// Launch accounting + error check after every kernel launch (defined in tomo_capi.cu).
void note_launch();

// Operator tables + scratch for one device-resident normal operator (see DESIGN.md
// "HBM layout"). Grid nodes are stored transposed relative to the reference:
// node = iy*m + ix, where the reference's grid[ix*m + iy] (proj/src/nufft.cpp:185-200).
struct OpDev {
  int n, m, nb, P, Ppad, nq;      // nq = padded window entries / 4
  int G32;                         // number of 32-node SELL blocks of W^T (= m*m/32)
  const float* apod;               // n   : a[t]/m  (deconvolve, nufft.cpp:204-227, with 1/m per axis)
  const float2* tw;                // m   : e^{-2 pi i k/m}
  const int4* w_cols;              // SELL-32 ELL of W: [(Ppad/32) * nq * 32] int4
  const float4* w_vals;            //                   [(Ppad/32) * nq * 32] float4
  const uint32_t* wt_chunk;        // G32+1 offsets (units of 32 entries)
  const int2* wt_ent;              // {sample j, float bits of weight}
  float2* H;                       // B x m x n  (type-2 row pass output, [iy][t1])
  float2* g;                       // B x m x m  (oversampled spatial grid, [iy][ix])
  float2* s;                       // B x P      (slice samples)
  float2* K;                       // B x n x m  (type-1 row pass output, [t1][iy])
};

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
  int done;           // CG finished early (rs == 0, pAp == 0, tolerance)
  int nonfinite;      // sticky non-finite flag (-> NumericalError)
  int steps_run;
  int frozen;         // split Bregman stopped on tolerance: later iterations pass through
  int sb_iters;       // split Bregman iterations run
  int pad_;
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
  float alpha, lambda, shift;
  double tol;          // relative residual tolerance (0 = off)
};

enum PbMode { PB_COMPLEX = 0, PB_REAL = 1, PB_CG_STEP = 2, PB_CG_INIT = 3 };

struct PbEpi {
  int mode;
  float scale;              // multiplies N u (alpha)
  float2* out_c;            // PB_COMPLEX
  float* out_r;             // PB_REAL (and the sharded partial)
  // CG modes
  const float* p;           // STEP: p (after update); INIT: x0
  const float* b;           // INIT: rhs
  float* ap;                // STEP: Ap out; INIT: r out
  float* p_out;             // INIT: p = r
  float* x_out;             // INIT: x = x0
  SysParams sys;
  int step;                 // CG step index (parity for rr)
  Reduce red;
};

// CG p-update fused into the first kernel of a step: p = r + beta p, beta = rr[k]/rr[k-1].
struct PUpd {
  int enabled;              // 0: plain input
  const float* r;
  float* p;                 // read and written in place (P1) / written (stencil)
  int step;
  Reduce red;
};

// ---- launchers (nufft.cu) ----
void launch_t2_rows(const OpDev& d, int B, const void* in, bool in_complex, const PUpd& pu, cudaStream_t st);
void launch_t2_cols(const OpDev& d, int B, const SliceScalars* skip, cudaStream_t st);
void launch_w(const OpDev& d, int B, const float2* grid, float2* samples, const SliceScalars* skip,
              cudaStream_t st);
void launch_wt_rows(const OpDev& d, int B, const SliceScalars* skip, cudaStream_t st);
void launch_t1_rows(const OpDev& d, int B, const PbEpi& e, cudaStream_t st);
void launch_wt_grid(const OpDev& d, int B, const float2* samples, float2* grid, cudaStream_t st);
void launch_weight_samples(float2* s, int B, int P, int nb, int angle0, cudaStream_t st);
void launch_fft_rows_test(int m, int rows, const float2* tw, const float2* in, float2* out, bool inverse,
                          cudaStream_t st);

// ---- launchers (solver.cu) ----
struct StencilCoef {
  float c[81];              // (2r+1)^2 row-major, r <= 4
};
void launch_cg_update(int n, int B, const float* p, const float* ap, float* x, float* r, const SysParams& sys,
                      int step, const Reduce& red, cudaStream_t st);
// Surrogate system apply with fused p-update (mode 0: step, 1: init, 2: plain apply out=op(in)).
void launch_stencil(int n, int B, int rad, int euclid, const StencilCoef& coef, int mode, const float* in,
                    const float* r_in, float* p_out, float* ap_out, const float* b, float* x_out,
                    const SysParams& sys, int step, const Reduce& red, cudaStream_t st);
// Sharded-operator CG epilogue: ap = red + lambda K'K p + shift p (mode 0) / init (mode 1).
void launch_cg_epilogue(int n, int B, int mode, const float* nred, const float* p, const float* b, float* ap,
                        float* p_out, float* x_out, const SysParams& sys, int step, const Reduce& red,
                        cudaStream_t st);
void launch_sb_post(int n, int B, float* mu_new, const float* mu_old, const float* bx_old,
                    const float* by_old, float* bx_new, float* by_new, const float* fid, float* rhs,
                    float lambda, const Reduce& red, cudaStream_t st);
void launch_cp_dual(int n, int B, const float* u_cur, const float* u_prev, const float* yx_old,
                    const float* yy_old, float* yx_new, float* yy_new, const float* bp, float* rhs, float tau,
                    float sigma, float theta, float lambda, cudaStream_t st);
void launch_scale_real(int64_t len, const float2* in, float* out, float alpha, cudaStream_t st);
void launch_axpby(int64_t len, float a, const float* x, float b, const float* y, float* out, cudaStream_t st);
void launch_dot(int n, int B, const float* x, const float* y, double* out_host_visible, const Reduce& red,
                cudaStream_t st);
void launch_leak(int64_t len, const float2* v, const Reduce& red, cudaStream_t st);
void launch_grad(int n, int B, const float* u, float* gx, float* gy, cudaStream_t st);
void launch_grad_adjoint(int n, int B, const float* gx, const float* gy, float* out, cudaStream_t st);
void launch_shrink(int64_t len, const float* x, float gamma, float* out, cudaStream_t st);
void launch_reset_scalars(SliceScalars* sc, int B, cudaStream_t st);

}  // namespace tomo_b200
