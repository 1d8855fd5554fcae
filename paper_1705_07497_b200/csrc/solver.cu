// solver.cu — device-resident CG / split-Bregman / Chambolle-Pock vector kernels (sm_100a).
//
// cg_solve (proj/src/solver.cpp:56-95) runs as two kernels per step: the system apply (the
// NUFFT chain of nufft.cu, or the surrogate stencil below) with the p-update of the
// previous step fused into its load and the p.Ap / p.p dots fused into its epilogue, then
// the x/r update with the r.r dot. All scalars (alpha, beta, rs, pAp, min-Ritz, done /
// non-finite flags) stay on the device (SliceScalars); the reference's early exits
// (rs == 0, pAp == 0, relative tolerance; solver.cpp:70,75,86-88) become device predicates.
//
// grad / grad_adjoint / shrink (solver.cpp:12-54) and the Bregman update + next right-hand
// side (solver.cpp:264-282) are one fused pass (k_sb_post); the surrogate T (a translated
// stencil, normal_ops.cpp:266-281) is applied as a shared-memory tiled stencil fused with
// lambda K'K + sigma I and the CG dots. Templated on the real type R; dots in fp64.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace tomo_b200 {

namespace {

constexpr int kVecThreads = 256;

template <typename R>
struct Vec16;
template <>
struct Vec16<float> {
  using T = float4;
};
template <>
struct Vec16<double> {
  using T = double2;
};

int vec_blocks(int64_t L, int B) {
  // ~4 elements per thread, but keep the per-slice block count (and so the cost of the
  // last-block reduction) bounded when a batch of slices already fills the GPU.
  const int64_t per_block = static_cast<int64_t>(kVecThreads) * 4;
  int64_t nb = (L + per_block - 1) / per_block;
  const int64_t cap = std::max<int64_t>(8, 16 * 148 / std::max(B, 1));
  nb = std::min(nb, cap);
  return static_cast<int>(std::min<int64_t>(std::max<int64_t>(nb, 1), MAX_PART_BLOCKS));
}

__device__ __forceinline__ bool slice_live(const SliceScalars& sc, int step) {
  return !sc.done && !sc.frozen && sc.rr[step & 1] != 0.0;
}

__device__ __forceinline__ int64_t gtid() { return static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return static_cast<int64_t>(gridDim.x) * blockDim.x; }

// ------------------------------------------------------------------ CG x/r update
template <typename R>
__global__ void __launch_bounds__(kVecThreads) k_cg_update(int64_t L, const R* __restrict__ p, const R* __restrict__ ap,
                                                           R* __restrict__ x, R* __restrict__ r, SysParams sys,
                                                           int step, Reduce red) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  SliceScalars& sc = red.sc[b];
  if (!slice_live(sc, step)) return;
  const double rs = sc.rr[step & 1];
  const double pap = sc.pap, pp = sc.pp;
  if (blockIdx.x == 0 && threadIdx.x == 0 && pp > 0.0) sc.min_ritz = fmin(sc.min_ritz, pap / pp);
  if (pap == 0.0) {  // solver.cpp:75
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      sc.done = 1;
      sc.steps_run = step;
    }
    return;
  }
  const R alpha = static_cast<R>(rs / pap);
  const size_t off = static_cast<size_t>(b) * L;
  double rr = 0.0;
  bool fin = true;
  // 16-byte vectors (float4 / double2), two per iteration: 8 independent loads in flight
  using V = typename Vec16<R>::T;
  constexpr int VW = 16 / sizeof(R);
  const int64_t nv = L / VW;  // L = n^2 with n even: multiple of 4
  const V* p4 = reinterpret_cast<const V*>(p + off);
  const V* ap4 = reinterpret_cast<const V*>(ap + off);
  V* x4 = reinterpret_cast<V*>(x + off);
  V* r4 = reinterpret_cast<V*>(r + off);
  for (int64_t i = gtid(); i < nv; i += gstride()) {
    V pv = p4[i], av = ap4[i], xv = x4[i], rv = r4[i];
    R* pe = reinterpret_cast<R*>(&pv);
    R* ae = reinterpret_cast<R*>(&av);
    R* xe = reinterpret_cast<R*>(&xv);
    R* re = reinterpret_cast<R*>(&rv);
#pragma unroll
    for (int k = 0; k < VW; ++k) {
      xe[k] += alpha * pe[k];
      re[k] -= alpha * ae[k];
      fin = fin && finite_r(xe[k]);
      rr += static_cast<double>(re[k]) * re[k];
    }
    x4[i] = xv;
    r4[i] = rv;
  }
  if (!fin) sc.nonfinite = 1;
  double t0, t1;
  double* part = red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
  if (reduce2_last(rr, 0.0, part, gridDim.x, blockIdx.x, &sc.counter[1], scratch, t0, t1) && threadIdx.x == 0) {
    sc.rr[(step + 1) & 1] = t0;
    sc.rs_last = t0;
    if (!isfinite(t0)) sc.nonfinite = 1;
    sc.steps_run = step + 1;
    if (sys.tol > 0.0 && sc.bb > 0.0 && sqrt(t0) <= sys.tol * sqrt(sc.bb)) {  // solver.cpp:86-88
      sc.done = 1;
      sc.steps_run = step;
    }
  }
}

// ------------------------------------------------------------------ Chronopoulos-Gear CG: last update
// After the last step's apply (k = steps - 1, scalars from cgcg_finalize): p = r + beta p,
// s = w + beta s, x += alpha p, r -= alpha s, with r.r for the reference's final tolerance test
// (solver.cpp:86-88: a break in the last step reports steps_run = steps - 1). The updates of
// the earlier steps are fused into the next step's first FFT pass (k_t2_rows).
template <typename R>
__global__ void __launch_bounds__(kVecThreads) k_cgcg_final(int64_t L, const R* __restrict__ w, R* __restrict__ p,
                                                            R* __restrict__ s, R* __restrict__ x, R* __restrict__ r,
                                                            SysParams sys, int steps, Reduce red) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  SliceScalars& sc = red.sc[b];
  if (sc.done || sc.frozen) return;
  const R alpha = static_cast<R>(sc.cg_alpha), beta = static_cast<R>(sc.cg_beta);
  const bool first = steps == 1;  // beta_0 = 0: p_0 = r_0, s_0 = w_0
  const size_t off = static_cast<size_t>(b) * L;
  double rr = 0.0;
  bool fin = true;
  for (int64_t i = gtid(); i < L; i += gstride()) {
    const size_t o = off + i;
    R rv = r[o];
    R pv = rv, sv = w[o];
    if (!first) {
      pv += beta * p[o];
      sv += beta * s[o];
    }
    const R xv = x[o] + alpha * pv;
    rv -= alpha * sv;
    x[o] = xv;
    r[o] = rv;
    fin = fin && finite_r(xv);
    rr += static_cast<double>(rv) * rv;
  }
  if (!fin) sc.nonfinite = 1;
  double t0, t1;
  double* part = red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
  if (reduce2_last(rr, 0.0, part, gridDim.x, blockIdx.x, &sc.counter[1], scratch, t0, t1) && threadIdx.x == 0) {
    if (!isfinite(t0)) sc.nonfinite = 1;
    sc.rr[steps & 1] = t0;
    sc.rs_last = t0;
    sc.steps_run = steps;
    if (sys.tol > 0.0 && sc.bb > 0.0 && sqrt(t0) <= sys.tol * sqrt(sc.bb)) sc.steps_run = steps - 1;
  }
}

// ------------------------------------------------------------------ surrogate stencil
// Tile of 32x32 outputs, 256 threads (32 x 8, 4 rows each). Halo H = max(rad, 1).
// 64x64 outputs per CTA (256 threads = 64 columns x 4, 16 rows each): the halo and the
// per-CTA dot reduction are amortised over 4096 pixels.
constexpr int kTile = 64;
constexpr int kTileRows = 4;  // thread rows

// Radius 1 (the surrogate default): 8 resident CTAs per SM for fp32 (32 registers; measured
// c4 stencil 69.0 -> 67.4 us against the unconstrained 84-register build); TOMO_STENCIL_MINB
// overrides for A/B runs.
#ifndef TOMO_STENCIL_MINB
#define TOMO_STENCIL_MINB 0
#endif
template <int RAD, typename R>
constexpr int stencil_minb() {
  return TOMO_STENCIL_MINB > 0 ? TOMO_STENCIL_MINB : RAD == 1 ? (sizeof(R) == 4 ? 8 : 4) : 1;
}

template <int RAD, typename R>
__global__ void __launch_bounds__(256, stencil_minb<RAD, R>()) k_stencil(int n, StencilCoef coef, int mode, const R* __restrict__ in,
                                                 const R* __restrict__ r_in, R* __restrict__ p_out,
                                                 R* __restrict__ ap_out, const R* __restrict__ bvec,
                                                 R* __restrict__ x_out, SysParams sys, int step, Reduce red) {
  constexpr int HALO = RAD > 1 ? RAD : 1;
  constexpr int W = kTile + 2 * HALO;
  constexpr int SIDE = 2 * RAD + 1;
  constexpr int VW = 16 / sizeof(R);
  // smem tile: the interior columns start at PADL (16-byte aligned rows: vector stores), the
  // halo columns sit just left / right of them; logical column lj lives at q[.][CO + lj]
  constexpr int PADL = ((HALO + VW - 1) / VW) * VW;
  constexpr int CO = PADL - HALO;
  constexpr int QS = PADL + kTile + PADL;
  __shared__ __align__(16) R q[W][QS];
  __shared__ R cf[SIDE * SIDE];
  __shared__ double scratch[32];
  const int b = blockIdx.z;
  R beta = 0;
  if (mode != 2 && red.sc[b].frozen) return;
  if (mode == 0) {
    SliceScalars& sc = red.sc[b];
    if (sc.done) return;
    const double rs = sc.rr[step & 1];
    if (rs == 0.0) {
      sc.done = 1;
      return;
    }
    if (step > 0) beta = static_cast<R>(rs / sc.rr[(step + 1) & 1]);
  }
  for (int k = threadIdx.x; k < SIDE * SIDE; k += blockDim.x) cf[k] = static_cast<R>(coef.c[k]);
  const size_t off = static_cast<size_t>(b) * n * n;
  const int i0 = blockIdx.y * kTile - HALO, j0 = blockIdx.x * kTile - HALO;
  const bool upd = mode == 0 && step > 0;  // q = r + beta p (the CG p-update, solver.cpp:84)
  // the halo tile. n % VW == 0: the kTile interior columns of each row with 16-byte vector
  // loads and stores (aligned: they start at a multiple of kTile), the 2*HALO halo columns
  // scalar; otherwise every element scalar.
  if (n % VW == 0) {
    using V = typename Vec16<R>::T;
    constexpr int VPR = kTile / VW;   // vectors per interior row
    constexpr int RPP = 256 / VPR;    // rows per pass of the 256 threads
    const int vq = threadIdx.x % VPR, lr = threadIdx.x / VPR;
    const int gj = j0 + HALO + vq * VW;
#pragma unroll 3
    for (int li = lr; li < W; li += RPP) {
      const int gi = i0 + li;
      V a, rr;
      R* ae = reinterpret_cast<R*>(&a);
      R* re = reinterpret_cast<R*>(&rr);
#pragma unroll
      for (int e = 0; e < VW; ++e) ae[e] = re[e] = R(0);
      if (gi >= 0 && gi < n && gj < n) {
        const size_t o = off + static_cast<size_t>(gi) * n + gj;
        a = *reinterpret_cast<const V*>(in + o);
        if (upd) rr = *reinterpret_cast<const V*>(r_in + o);
      }
      if (upd) {
#pragma unroll
        for (int e = 0; e < VW; ++e) ae[e] = re[e] + beta * ae[e];
      }
      *reinterpret_cast<V*>(&q[li][PADL + vq * VW]) = a;
    }
    for (int idx = threadIdx.x; idx < W * 2 * HALO; idx += 256) {
      const int li = idx / (2 * HALO), h = idx - li * (2 * HALO);
      const int lj = h < HALO ? h : kTile + h;
      const int gi = i0 + li, gj2 = j0 + lj;
      R v = 0, rv = 0;
      if (gi >= 0 && gi < n && gj2 >= 0 && gj2 < n) {
        const size_t o = off + static_cast<size_t>(gi) * n + gj2;
        v = in[o];
        if (upd) rv = r_in[o];
      }
      q[li][CO + lj] = upd ? rv + beta * v : v;
    }
  } else {
#pragma unroll 6
    for (int idx = threadIdx.x; idx < W * W; idx += blockDim.x) {
      const int li = idx / W, lj = idx - li * W;
      const int gi = i0 + li, gj2 = j0 + lj;
      R v = 0, rv = 0;
      if (gi >= 0 && gi < n && gj2 >= 0 && gj2 < n) {
        const size_t o = off + static_cast<size_t>(gi) * n + gj2;
        v = in[o];
        if (upd) rv = r_in[o];
      }
      q[li][CO + lj] = upd ? rv + beta * v : v;
    }
  }
  __syncthreads();
  // each thread: one column, kTile / kTileRows consecutive rows, the (2RAD+1)^2 neighbourhood in
  // a register window that slides down one row per output (2RAD+1 smem reads per output)
  constexpr int RPT = kTile / kTileRows;
  const int tj = threadIdx.x % kTile, ti = threadIdx.x / kTile;
  const R alpha = static_cast<R>(sys.alpha), lam = static_cast<R>(sys.lambda), shift = static_cast<R>(sys.shift);
  double acc0 = 0.0, acc1 = 0.0;
  const int lj = tj + HALO, r0 = ti * RPT + HALO;
  const int gj = j0 + lj;
  R win[SIDE][SIDE];
#pragma unroll
  for (int k = 0; k < SIDE - 1; ++k)
#pragma unroll
    for (int dj = 0; dj < SIDE; ++dj) win[k + 1][dj] = q[r0 - RAD + k][CO + lj - RAD + dj];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int li = r0 + k;
#pragma unroll
    for (int a = 0; a < SIDE - 1; ++a)
#pragma unroll
      for (int dj = 0; dj < SIDE; ++dj) win[a][dj] = win[a + 1][dj];
#pragma unroll
    for (int dj = 0; dj < SIDE; ++dj) win[SIDE - 1][dj] = q[li + RAD][CO + lj - RAD + dj];
    const int gi = i0 + li;
    if (gi >= n || gj >= n) continue;
    const R c = win[RAD][RAD];
    R tq = 0;
#pragma unroll
    for (int di = 0; di < SIDE; ++di)
#pragma unroll
      for (int dj = 0; dj < SIDE; ++dj) tq += cf[di * SIDE + dj] * win[di][dj];
    R kk = 0;
    if (gj >= 1) kk += c - win[RAD][RAD - 1];
    if (gj <= n - 2) kk -= win[RAD][RAD + 1] - c;
    if (gi >= 1) kk += c - win[RAD - 1][RAD];
    if (gi <= n - 2) kk -= win[RAD + 1][RAD] - c;
    const R ax = alpha * tq + lam * kk + shift * c;
    const size_t o = off + static_cast<size_t>(gi) * n + gj;
    if (mode == 0) {
      if (step > 0) p_out[o] = c;
      ap_out[o] = ax;
      acc0 += static_cast<double>(c) * ax;
      acc1 += static_cast<double>(c) * c;
    } else if (mode == 1) {
      const R bv = bvec[o];
      const R rv = bv - ax;
      ap_out[o] = rv;
      p_out[o] = rv;
      x_out[o] = c;
      acc0 += static_cast<double>(rv) * rv;
      acc1 += static_cast<double>(bv) * bv;
    } else {
      ap_out[o] = ax;
    }
  }
  if (mode == 2) return;
  SliceScalars& sc = red.sc[b];
  double t0, t1;
  double* part = red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
  const int nblk = gridDim.x * gridDim.y, blk = blockIdx.y * gridDim.x + blockIdx.x;
  if (reduce2_last(acc0, acc1, part, nblk, blk, &sc.counter[0], scratch, t0, t1) && threadIdx.x == 0) {
    if (mode == 0) {
      sc.pap = t0;
      sc.pp = t1;
    } else {
      sc.rr[0] = t0;
      sc.rs_last = t0;
      sc.bb = t1;
      sc.done = 0;
      sc.steps_run = 0;
      sc.min_ritz = __longlong_as_double(0x7ff0000000000000LL);
    }
  }
}

template <typename R>
__device__ __forceinline__ R ktk_g(const R* __restrict__ p, int n, int i, int j) {
  const size_t o = static_cast<size_t>(i) * n + j;
  const R c = p[o];
  R v = 0;
  if (j >= 1) v += c - p[o - 1];
  if (j <= n - 2) v -= p[o + 1] - c;
  if (i >= 1) v += c - p[o - n];
  if (i <= n - 2) v -= p[o + n] - c;
  return v;
}

// Sharded-operator epilogue: nred = all-reduced alpha*Re(N p) partial sums.
template <typename R>
__global__ void __launch_bounds__(kVecThreads) k_cg_epilogue(int n, int mode, const R* __restrict__ nred,
                                                             const R* __restrict__ p, const R* __restrict__ bvec,
                                                             R* __restrict__ ap, R* __restrict__ p_out,
                                                             R* __restrict__ x_out, SysParams sys, int step,
                                                             Reduce red) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  SliceScalars& sc = red.sc[b];
  if (sc.frozen || (mode == 0 && !slice_live(sc, step))) return;
  const int64_t L = static_cast<int64_t>(n) * n;
  const size_t off = static_cast<size_t>(b) * L;
  const R* pb = p + off;
  const R lam = static_cast<R>(sys.lambda), shift = static_cast<R>(sys.shift);
  double acc0 = 0.0, acc1 = 0.0;
  for (int64_t i = gtid(); i < L; i += gstride()) {
    const int ii = static_cast<int>(i) / n, jj = static_cast<int>(i) - ii * n;
    const R pv = pb[i];
    R ax = nred[off + i];
    if (lam != R(0)) ax += lam * ktk_g(pb, n, ii, jj);
    ax += shift * pv;
    if (mode == 0) {
      ap[off + i] = ax;
      acc0 += static_cast<double>(pv) * ax;
      acc1 += static_cast<double>(pv) * pv;
    } else {
      const R bv = bvec[off + i];
      const R rv = bv - ax;
      ap[off + i] = rv;
      p_out[off + i] = rv;
      x_out[off + i] = pv;
      acc0 += static_cast<double>(rv) * rv;
      acc1 += static_cast<double>(bv) * bv;
    }
  }
  double t0, t1;
  double* part = red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
  if (reduce2_last(acc0, acc1, part, gridDim.x, blockIdx.x, &sc.counter[0], scratch, t0, t1) && threadIdx.x == 0) {
    if (mode == 0) {
      sc.pap = t0;
      sc.pp = t1;
    } else {
      sc.rr[0] = t0;
      sc.rs_last = t0;
      sc.bb = t1;
      sc.done = 0;
      sc.steps_run = 0;
      sc.min_ritz = __longlong_as_double(0x7ff0000000000000LL);
    }
  }
}

// ------------------------------------------------------------------ split-Bregman update
// One pass: g = grad(mu_new), d = shrink(g + b_old, 1/lambda), b_new = b_old + g - d
// (solver.cpp:278-282), next rhs = fid + lambda grad^T(d - b_new) (solver.cpp:264-265),
// and ||mu_new - mu_old||_1 (solver.cpp:288). d is never stored: d - b_new is recomputed at
// the two neighbours grad^T needs.
template <typename R>
__device__ __forceinline__ R shrinkr(R x, R gamma) {
  const R m = fabs(x) - gamma;
  return m > R(0) ? (x > R(0) ? m : -m) : R(0);
}

template <typename R>
__global__ void __launch_bounds__(kVecThreads) k_sb_post(int n, R* __restrict__ mu_new, const R* __restrict__ mu_old,
                                                         const R* __restrict__ bx_old, const R* __restrict__ by_old,
                                                         R* __restrict__ bx_new, R* __restrict__ by_new,
                                                         const R* __restrict__ fid, R* __restrict__ rhs,
                                                         double lambda_d, Reduce red) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const int64_t L = static_cast<int64_t>(n) * n;
  const size_t off = static_cast<size_t>(b) * L;
  SliceScalars& sc = red.sc[b];
  if (sc.frozen) {  // stopped on tolerance: carry the state through unchanged
    for (int64_t i = gtid(); i < L; i += gstride()) {
      mu_new[off + i] = mu_old[off + i];
      bx_new[off + i] = bx_old[off + i];
      by_new[off + i] = by_old[off + i];
    }
    return;
  }
  const R* mu = mu_new + off;
  const R* bxo = bx_old + off;
  const R* byo = by_old + off;
  const R lambda = static_cast<R>(lambda_d);
  const R gamma = static_cast<R>(1.0 / lambda_d);
  double upd = 0.0;
  bool fin = true;
  for (int64_t i = gtid(); i < L; i += gstride()) {
    const int ii = static_cast<int>(i) / n, jj = static_cast<int>(i) - ii * n;  // 32-bit: L < 2^31
    const R c = mu[i];
    fin = fin && finite_r(c);
    upd += fabs(static_cast<double>(c) - static_cast<double>(mu_old[off + i]));
    const R gx = jj < n - 1 ? mu[i + 1] - c : R(0);
    const R gy = ii < n - 1 ? mu[i + n] - c : R(0);
    const R dx = shrinkr(gx + bxo[i], gamma), dy = shrinkr(gy + byo[i], gamma);
    const R bxn = bxo[i] + gx - dx, byn = byo[i] + gy - dy;
    bx_new[off + i] = bxn;
    by_new[off + i] = byn;
    R div = 0;
    if (jj <= n - 2) div -= dx - bxn;
    if (ii <= n - 2) div -= dy - byn;
    if (jj >= 1) {  // tx at (ii, jj-1)
      const R gxl = c - mu[i - 1];
      const R dxl = shrinkr(gxl + bxo[i - 1], gamma);
      div += dxl - (bxo[i - 1] + gxl - dxl);
    }
    if (ii >= 1) {  // ty at (ii-1, jj)
      const R gyu = c - mu[i - n];
      const R dyu = shrinkr(gyu + byo[i - n], gamma);
      div += dyu - (byo[i - n] + gyu - dyu);
    }
    rhs[off + i] = fid[off + i] + lambda * div;
  }
  if (!fin) sc.nonfinite = 1;
  double t0, t1;
  double* part = red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
  if (reduce2_last(upd, 0.0, part, gridDim.x, blockIdx.x, &sc.counter[2], scratch, t0, t1) && threadIdx.x == 0) {
    sc.upd = t0;
    sc.sb_iters += 1;
    if (sc.sb_iters == 1) sc.first_upd = t0;
    if (t0 <= sc.sb_tol * sc.first_upd) sc.frozen = 1;  // solver.cpp:298-303
  }
}

// The same pass four columns at a time (n % 4 == 0): 16-byte vector loads of the row, the rows
// above / below and b, instead of ~11 scalar loads per pixel; per-pixel arithmetic unchanged.
template <typename R>
struct Q4 {
  R v[4];
};
template <typename R>
__device__ __forceinline__ Q4<R> ld4(const R* p) {
  Q4<R> q;
  if constexpr (sizeof(R) == 4) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    q.v[0] = t.x;
    q.v[1] = t.y;
    q.v[2] = t.z;
    q.v[3] = t.w;
  } else {
    const double2 a = *reinterpret_cast<const double2*>(p), c = *reinterpret_cast<const double2*>(p + 2);
    q.v[0] = a.x;
    q.v[1] = a.y;
    q.v[2] = c.x;
    q.v[3] = c.y;
  }
  return q;
}
template <typename R>
__device__ __forceinline__ void st4(R* p, const Q4<R>& q) {
  if constexpr (sizeof(R) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(q.v[0], q.v[1], q.v[2], q.v[3]);
  } else {
    *reinterpret_cast<double2*>(p) = make_double2(q.v[0], q.v[1]);
    *reinterpret_cast<double2*>(p + 2) = make_double2(q.v[2], q.v[3]);
  }
}

template <typename R>
__global__ void __launch_bounds__(kVecThreads) k_sb_post4(int n, R* __restrict__ mu_new, const R* __restrict__ mu_old,
                                                          const R* __restrict__ bx_old, const R* __restrict__ by_old,
                                                          R* __restrict__ bx_new, R* __restrict__ by_new,
                                                          const R* __restrict__ fid, R* __restrict__ rhs,
                                                          double lambda_d, Reduce red) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const int64_t L = static_cast<int64_t>(n) * n;
  const size_t off = static_cast<size_t>(b) * L;
  SliceScalars& sc = red.sc[b];
  const int64_t nq = L / 4;
  if (sc.frozen) {  // stopped on tolerance: carry the state through unchanged
    for (int64_t q = gtid(); q < nq; q += gstride()) {
      st4(mu_new + off + 4 * q, ld4(mu_old + off + 4 * q));
      st4(bx_new + off + 4 * q, ld4(bx_old + off + 4 * q));
      st4(by_new + off + 4 * q, ld4(by_old + off + 4 * q));
    }
    return;
  }
  const R* mu = mu_new + off;
  const R* bxo = bx_old + off;
  const R* byo = by_old + off;
  const R lambda = static_cast<R>(lambda_d);
  const R gamma = static_cast<R>(1.0 / lambda_d);
  double upd = 0.0;
  bool fin = true;
  for (int64_t q = gtid(); q < nq; q += gstride()) {
    const int i = static_cast<int>(4 * q);
    const int ii = i / n, jj = i - ii * n;
    const Q4<R> c = ld4(mu + i), bx = ld4(bxo + i), by = ld4(byo + i);
    const Q4<R> mo = ld4(mu_old + off + i), fd = ld4(fid + off + i);
    Q4<R> dn{}, up{}, byu{};
    if (ii < n - 1) dn = ld4(mu + i + n);
    if (ii >= 1) {
      up = ld4(mu + i - n);
      byu = ld4(byo + i - n);
    }
    const R right = jj + 4 < n ? mu[i + 4] : R(0);
    const R left = jj >= 1 ? mu[i - 1] : R(0), bxl = jj >= 1 ? bxo[i - 1] : R(0);
    Q4<R> obx, oby, orhs;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = jj + k;
      const R cc = c.v[k];
      fin = fin && finite_r(cc);
      upd += fabs(static_cast<double>(cc) - static_cast<double>(mo.v[k]));
      const R gx = j < n - 1 ? (k < 3 ? c.v[k + 1] : right) - cc : R(0);
      const R gy = ii < n - 1 ? dn.v[k] - cc : R(0);
      const R dx = shrinkr(gx + bx.v[k], gamma), dy = shrinkr(gy + by.v[k], gamma);
      const R bxn = bx.v[k] + gx - dx, byn = by.v[k] + gy - dy;
      obx.v[k] = bxn;
      oby.v[k] = byn;
      R div = 0;
      if (j <= n - 2) div -= dx - bxn;
      if (ii <= n - 2) div -= dy - byn;
      if (j >= 1) {  // tx at (ii, j-1)
        const R cl = k > 0 ? c.v[k - 1] : left, bl = k > 0 ? bx.v[k - 1] : bxl;
        const R gxl = cc - cl;
        const R dxl = shrinkr(gxl + bl, gamma);
        div += dxl - (bl + gxl - dxl);
      }
      if (ii >= 1) {  // ty at (ii-1, j)
        const R gyu = cc - up.v[k];
        const R dyu = shrinkr(gyu + byu.v[k], gamma);
        div += dyu - (byu.v[k] + gyu - dyu);
      }
      orhs.v[k] = fd.v[k] + lambda * div;
    }
    st4(bx_new + off + i, obx);
    st4(by_new + off + i, oby);
    st4(rhs + off + i, orhs);
  }
  if (!fin) sc.nonfinite = 1;
  double t0, t1;
  double* part = red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
  if (reduce2_last(upd, 0.0, part, gridDim.x, blockIdx.x, &sc.counter[2], scratch, t0, t1) && threadIdx.x == 0) {
    sc.upd = t0;
    sc.sb_iters += 1;
    if (sc.sb_iters == 1) sc.first_upd = t0;
    if (t0 <= sc.sb_tol * sc.first_upd) sc.frozen = 1;  // solver.cpp:298-303
  }
}

// ------------------------------------------------------------------ Chambolle-Pock dual step
template <typename R>
__global__ void __launch_bounds__(kVecThreads) k_cp_dual(int n, const R* __restrict__ u_cur, const R* __restrict__ u_prev,
                                                         const R* __restrict__ yx_old, const R* __restrict__ yy_old,
                                                         R* __restrict__ yx_new, R* __restrict__ yy_new,
                                                         const R* __restrict__ bp, R* __restrict__ rhs, R tau, R sigma,
                                                         R theta, R lambda) {
  const int b = blockIdx.y;
  const int64_t L = static_cast<int64_t>(n) * n;
  const size_t off = static_cast<size_t>(b) * L;
  const R* uc = u_cur + off;
  const R* up = u_prev + off;
  auto ubar = [&](int64_t k) { return uc[k] + theta * (uc[k] - up[k]); };
  auto clampl = [&](R v) { return fmin(lambda, fmax(-lambda, v)); };
  for (int64_t i = gtid(); i < L; i += gstride()) {
    const int ii = static_cast<int>(i) / n, jj = static_cast<int>(i) - ii * n;
    const R c = ubar(i);
    const R gx = jj < n - 1 ? ubar(i + 1) - c : R(0);
    const R gy = ii < n - 1 ? ubar(i + n) - c : R(0);
    const R yxn = clampl(yx_old[off + i] + sigma * gx);
    const R yyn = clampl(yy_old[off + i] + sigma * gy);
    yx_new[off + i] = yxn;
    yy_new[off + i] = yyn;
    R div = 0;
    if (jj <= n - 2) div -= yxn;
    if (ii <= n - 2) div -= yyn;
    if (jj >= 1) div += clampl(yx_old[off + i - 1] + sigma * (c - ubar(i - 1)));
    if (ii >= 1) div += clampl(yy_old[off + i - n] + sigma * (c - ubar(i - n)));
    rhs[off + i] = (uc[i] - tau * div) + tau * bp[off + i];
  }
}

// ------------------------------------------------------------------ small helpers
template <typename R>
__global__ void k_axpby(int64_t len, R a, const R* __restrict__ x, R b, const R* __restrict__ y, R* __restrict__ out) {
  for (int64_t i = gtid(); i < len; i += gstride()) out[i] = a * x[i] + b * y[i];
}

template <typename R>
__global__ void __launch_bounds__(kVecThreads) k_dot(int64_t L, const R* __restrict__ x, const R* __restrict__ y,
                                                     Reduce red) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const size_t off = static_cast<size_t>(b) * L;
  double acc = 0.0;
  for (int64_t i = gtid(); i < L; i += gstride()) acc += static_cast<double>(x[off + i]) * y[off + i];
  double t0, t1;
  double* part = red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
  if (reduce2_last(acc, 0.0, part, gridDim.x, blockIdx.x, &red.sc[b].counter[3], scratch, t0, t1) &&
      threadIdx.x == 0)
    red.sc[b].dot = t0;
}

// Per-iteration split-Bregman log for the recorded (host-timed) driver: ||mu - ref||_1 and
// ||ref||_1 (relative_l1_error, image.cpp:69-76) reduced in fixed order; the last block appends
// update_l1 / rel_l1 at the slice's iteration count if an iteration ran since the last log.
template <typename R>
__global__ void __launch_bounds__(kVecThreads) k_sb_log(int64_t L, int B, const R* __restrict__ mu,
                                                        const R* __restrict__ ref, double* upd_log, double* rel_log,
                                                        Reduce red) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const size_t off = static_cast<size_t>(b) * L;
  double num = 0.0, den = 0.0;
  if (ref)
    for (int64_t i = gtid(); i < L; i += gstride()) {
      const double r = ref[off + i];
      num += fabs(static_cast<double>(mu[off + i]) - r);
      den += fabs(r);
    }
  double t0, t1;
  double* part = red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
  if (reduce2_last(num, den, part, gridDim.x, blockIdx.x, &red.sc[b].counter[3], scratch, t0, t1) &&
      threadIdx.x == 0) {
    SliceScalars& sc = red.sc[b];
    if (sc.sb_iters > sc.logged) {
      const size_t it = static_cast<size_t>(sc.sb_iters - 1);
      upd_log[it * B + b] = sc.upd;
      if (rel_log) rel_log[it * B + b] = t1 > 0.0 ? t0 / t1 : 0.0;
      sc.logged = sc.sb_iters;
    }
  }
}

template <typename R>
__global__ void __launch_bounds__(kVecThreads) k_leak(int64_t len, const cplx<R>* __restrict__ v, Reduce red) {
  __shared__ double scratch[32];
  double a = 0.0, im = 0.0;
  for (int64_t i = gtid(); i < len; i += gstride()) {
    const cplx<R> z = v[i];
    a += static_cast<double>(z.x) * z.x + static_cast<double>(z.y) * z.y;
    im += static_cast<double>(z.y) * z.y;
  }
  double t0, t1;
  if (reduce2_last(a, im, red.part, gridDim.x, blockIdx.x, &red.sc[0].counter[3], scratch, t0, t1) &&
      threadIdx.x == 0) {
    red.sc[0].leak_den = t0;
    red.sc[0].leak_num = t1;
  }
}

template <typename R>
__global__ void k_grad(int n, const R* __restrict__ u, R* __restrict__ gx, R* __restrict__ gy) {
  const int64_t L = static_cast<int64_t>(n) * n;
  const size_t off = static_cast<size_t>(blockIdx.y) * L;
  for (int64_t i = gtid(); i < L; i += gstride()) {
    const int ii = static_cast<int>(i / n), jj = static_cast<int>(i % n);
    const R c = u[off + i];
    gx[off + i] = jj < n - 1 ? u[off + i + 1] - c : R(0);
    gy[off + i] = ii < n - 1 ? u[off + i + n] - c : R(0);
  }
}

template <typename R>
__global__ void k_grad_adjoint(int n, const R* __restrict__ gx, const R* __restrict__ gy, R* __restrict__ out) {
  const int64_t L = static_cast<int64_t>(n) * n;
  const size_t off = static_cast<size_t>(blockIdx.y) * L;
  for (int64_t i = gtid(); i < L; i += gstride()) {
    const int ii = static_cast<int>(i / n), jj = static_cast<int>(i % n);
    R v = 0;
    if (jj >= 1) v += gx[off + i - 1];
    if (jj <= n - 2) v -= gx[off + i];
    if (ii >= 1) v += gy[off + i - n];
    if (ii <= n - 2) v -= gy[off + i];
    out[off + i] = v;
  }
}

template <typename R>
__global__ void k_shrink(int64_t len, const R* __restrict__ x, R gamma, R* __restrict__ out) {
  for (int64_t i = gtid(); i < len; i += gstride()) out[i] = shrinkr(x[i], gamma);
}

unsigned blocks_for(int64_t len, int threads) {
  return static_cast<unsigned>(std::min<int64_t>((len + threads - 1) / threads, 16 * 148));
}

}  // namespace

template <typename R>
void launch_cg_update(int n, int B, const R* p, const R* ap, R* x, R* r, const SysParams& sys, int step,
                      const Reduce& red, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  CK_LAUNCH(launch_k(k_cg_update<R>, dim3(vec_blocks(L, B), B), kVecThreads, 0, st, L, p, ap, x, r, sys, step, red));
  note_launch();
}

template <typename R>
void launch_cgcg_final(int n, int B, const R* w, R* p, R* s, R* x, R* r, const SysParams& sys, int steps,
                       const Reduce& red, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  CK_LAUNCH(launch_k(k_cgcg_final<R>, dim3(vec_blocks(L, B), B), kVecThreads, 0, st, L, w, p, s, x, r, sys, steps, red));
  note_launch();
}

template <typename R>
void launch_stencil(int n, int B, int rad, const StencilCoef& coef, int mode, const R* in, const R* r_in, R* p_out,
                    R* ap_out, const R* b, R* x_out, const SysParams& sys, int step, const Reduce& red,
                    cudaStream_t st) {
  dim3 grid((n + kTile - 1) / kTile, (n + kTile - 1) / kTile, B);
  switch (rad) {
    case 1: CK_LAUNCH(launch_k(k_stencil<1, R>, grid, 256, 0, st, n, coef, mode, in, r_in, p_out, ap_out, b, x_out, sys, step, red)); break;
    case 2: CK_LAUNCH(launch_k(k_stencil<2, R>, grid, 256, 0, st, n, coef, mode, in, r_in, p_out, ap_out, b, x_out, sys, step, red)); break;
    case 3: CK_LAUNCH(launch_k(k_stencil<3, R>, grid, 256, 0, st, n, coef, mode, in, r_in, p_out, ap_out, b, x_out, sys, step, red)); break;
    default: CK_LAUNCH(launch_k(k_stencil<4, R>, grid, 256, 0, st, n, coef, mode, in, r_in, p_out, ap_out, b, x_out, sys, step, red)); break;
  }
  note_launch();
}

template <typename R>
void launch_cg_epilogue(int n, int B, int mode, const R* nred, const R* p, const R* b, R* ap, R* p_out, R* x_out,
                        const SysParams& sys, int step, const Reduce& red, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  CK_LAUNCH(launch_k(k_cg_epilogue<R>, dim3(vec_blocks(L, B), B), kVecThreads, 0, st, n, mode, nred, p, b, ap, p_out, x_out, sys, step,
                                                                      red));
  note_launch();
}

template <typename R>
void launch_sb_post(int n, int B, R* mu_new, const R* mu_old, const R* bx_old, const R* by_old, R* bx_new, R* by_new,
                    const R* fid, R* rhs, double lambda, const Reduce& red, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  if (n % 4 == 0)  // 16-byte vectors (the slice offsets b*n^2 stay 16-byte aligned)
    CK_LAUNCH(launch_k(k_sb_post4<R>, dim3(vec_blocks(L, B), B), kVecThreads, 0, st, n, mu_new, mu_old, bx_old,
                       by_old, bx_new, by_new, fid, rhs, lambda, red));
  else
    CK_LAUNCH(launch_k(k_sb_post<R>, dim3(vec_blocks(L, B), B), kVecThreads, 0, st, n, mu_new, mu_old, bx_old, by_old,
                       bx_new, by_new, fid, rhs, lambda, red));
  note_launch();
}

template <typename R>
void launch_cp_dual(int n, int B, const R* u_cur, const R* u_prev, const R* yx_old, const R* yy_old, R* yx_new,
                    R* yy_new, const R* bp, R* rhs, double tau, double sigma, double theta, double lambda,
                    cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  CK_LAUNCH(launch_k(k_cp_dual<R>, dim3(vec_blocks(L, B), B), kVecThreads, 0, st, n, u_cur, u_prev, yx_old, yy_old, yx_new, yy_new, bp,
                                                                  rhs, R(tau), R(sigma), R(theta), R(lambda)));
  note_launch();
}

template <typename R>
void launch_axpby(int64_t len, double a, const R* x, double b, const R* y, R* out, cudaStream_t st) {
  CK_LAUNCH(launch_k(k_axpby<R>, blocks_for(len, 256), 256, 0, st, len, R(a), x, R(b), y, out));
  note_launch();
}

template <typename R>
void launch_dot(int n, int B, const R* x, const R* y, const Reduce& red, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  CK_LAUNCH(launch_k(k_dot<R>, dim3(vec_blocks(L, B), B), kVecThreads, 0, st, L, x, y, red));
  note_launch();
}

template <typename R>
void launch_sb_log(int n, int B, const R* mu, const R* ref, double* upd_log, double* rel_log, const Reduce& red,
                   cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  CK_LAUNCH(launch_k(k_sb_log<R>, dim3(vec_blocks(L, B), B), kVecThreads, 0, st, L, B, mu, ref, upd_log, rel_log,
                     red));
  note_launch();
}

template <typename R>
void launch_leak(int64_t len, const cplx<R>* v, const Reduce& red, cudaStream_t st) {
  CK_LAUNCH(launch_k(k_leak<R>, vec_blocks(len, 1), kVecThreads, 0, st, len, v, red));
  note_launch();
}

template <typename R>
void launch_grad(int n, int B, const R* u, R* gx, R* gy, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  CK_LAUNCH(launch_k(k_grad<R>, dim3(vec_blocks(L, B), B), kVecThreads, 0, st, n, u, gx, gy));
  note_launch();
}

template <typename R>
void launch_grad_adjoint(int n, int B, const R* gx, const R* gy, R* out, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  CK_LAUNCH(launch_k(k_grad_adjoint<R>, dim3(vec_blocks(L, B), B), kVecThreads, 0, st, n, gx, gy, out));
  note_launch();
}

template <typename R>
void launch_shrink(int64_t len, const R* x, double gamma, R* out, cudaStream_t st) {
  CK_LAUNCH(launch_k(k_shrink<R>, blocks_for(len, 256), 256, 0, st, len, x, R(gamma), out));
  note_launch();
}

#define TOMO_INST_SOLVER(R)                                                                                        \
  template void launch_sb_log<R>(int, int, const R*, const R*, double*, double*, const Reduce&, cudaStream_t); \
  template void launch_cgcg_final<R>(int, int, const R*, R*, R*, R*, R*, const SysParams&, int, const Reduce&,     \
                                     cudaStream_t);                                                                \
  template void launch_cg_update<R>(int, int, const R*, const R*, R*, R*, const SysParams&, int, const Reduce&,     \
                                    cudaStream_t);                                                                 \
  template void launch_stencil<R>(int, int, int, const StencilCoef&, int, const R*, const R*, R*, R*, const R*, R*, \
                                  const SysParams&, int, const Reduce&, cudaStream_t);                             \
  template void launch_cg_epilogue<R>(int, int, int, const R*, const R*, const R*, R*, R*, R*, const SysParams&, int, \
                                      const Reduce&, cudaStream_t);                                                \
  template void launch_sb_post<R>(int, int, R*, const R*, const R*, const R*, R*, R*, const R*, R*, double,          \
                                  const Reduce&, cudaStream_t);                                                    \
  template void launch_cp_dual<R>(int, int, const R*, const R*, const R*, const R*, R*, R*, const R*, R*, double,    \
                                  double, double, double, cudaStream_t);                                           \
  template void launch_axpby<R>(int64_t, double, const R*, double, const R*, R*, cudaStream_t);                    \
  template void launch_dot<R>(int, int, const R*, const R*, const Reduce&, cudaStream_t);                          \
  template void launch_leak<R>(int64_t, const cplx<R>*, const Reduce&, cudaStream_t);                              \
  template void launch_grad<R>(int, int, const R*, R*, R*, cudaStream_t);                                          \
  template void launch_grad_adjoint<R>(int, int, const R*, const R*, R*, cudaStream_t);                            \
  template void launch_shrink<R>(int64_t, const R*, double, R*, cudaStream_t);

TOMO_INST_SOLVER(float)
TOMO_INST_SOLVER(double)

}  // namespace tomo_b200
