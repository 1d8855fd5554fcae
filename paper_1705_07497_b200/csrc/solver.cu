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
// lambda K'K + sigma I and the CG dots.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace tomo_b200 {

namespace {

constexpr int kVecThreads = 256;

int vec_blocks(int64_t L, int B) {
  // ~2-4 float4 per thread; fewer when the batch already fills the GPU
  int64_t per_block = static_cast<int64_t>(kVecThreads) * 4;
  int64_t nb = (L + per_block - 1) / per_block;
  if (nb * B > 8 * 148) nb = std::max<int64_t>(1, (8 * 148 + B - 1) / B);
  return static_cast<int>(std::min<int64_t>(std::max<int64_t>(nb, 1), MAX_PART_BLOCKS));
}

__device__ __forceinline__ bool slice_live(const SliceScalars& sc, int step) {
  return !sc.done && !sc.frozen && sc.rr[step & 1] != 0.0;
}

// ------------------------------------------------------------------ CG x/r update
__global__ void __launch_bounds__(kVecThreads) k_cg_update(int64_t L, const float* __restrict__ p,
                                                           const float* __restrict__ ap, float* __restrict__ x,
                                                           float* __restrict__ r, SysParams sys, int step,
                                                           Reduce red) {
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
  const float alpha = static_cast<float>(rs / pap);
  const size_t off = static_cast<size_t>(b) * L;
  const float4* p4 = reinterpret_cast<const float4*>(p + off);
  const float4* ap4 = reinterpret_cast<const float4*>(ap + off);
  float4* x4 = reinterpret_cast<float4*>(x + off);
  float4* r4 = reinterpret_cast<float4*>(r + off);
  double rr = 0.0;
  bool fin = true;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L / 4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 pv = p4[i], av = ap4[i];
    float4 xv = x4[i], rv = r4[i];
    xv.x += alpha * pv.x; xv.y += alpha * pv.y; xv.z += alpha * pv.z; xv.w += alpha * pv.w;
    rv.x -= alpha * av.x; rv.y -= alpha * av.y; rv.z -= alpha * av.z; rv.w -= alpha * av.w;
    x4[i] = xv;
    r4[i] = rv;
    fin = fin && finite_f(xv.x) && finite_f(xv.y) && finite_f(xv.z) && finite_f(xv.w);
    rr += static_cast<double>(rv.x) * rv.x + static_cast<double>(rv.y) * rv.y +
          static_cast<double>(rv.z) * rv.z + static_cast<double>(rv.w) * rv.w;
  }
  if (!fin) sc.nonfinite = 1;
  double t0, t1;
  double* part = red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
  if (reduce2_last(rr, 0.0, part, gridDim.x, blockIdx.x, &sc.counter[1], scratch, t0, t1) && threadIdx.x == 0) {
    sc.rr[(step + 1) & 1] = t0;
    if (!isfinite(t0)) sc.nonfinite = 1;
    sc.steps_run = step + 1;
    if (sys.tol > 0.0 && sc.bb > 0.0 && sqrt(t0) <= sys.tol * sqrt(sc.bb)) {  // solver.cpp:86-88
      sc.done = 1;
      sc.steps_run = step;
    }
  }
}

// ------------------------------------------------------------------ surrogate stencil
// Tile of 32x32 outputs, 256 threads (32 x 8, 4 rows each). Halo H = max(rad, 1).
constexpr int kTile = 32;

template <int RAD>
__global__ void __launch_bounds__(256) k_stencil(int n, StencilCoef coef, int mode, const float* __restrict__ in,
                                                 const float* __restrict__ r_in, float* __restrict__ p_out,
                                                 float* __restrict__ ap_out, const float* __restrict__ bvec,
                                                 float* __restrict__ x_out, SysParams sys, int step, Reduce red) {
  constexpr int HALO = RAD > 1 ? RAD : 1;
  constexpr int W = kTile + 2 * HALO;
  constexpr int SIDE = 2 * RAD + 1;
  __shared__ float q[W][W + 1];
  __shared__ double scratch[32];
  const int b = blockIdx.z;
  float beta = 0.f;
  if (mode != 2 && red.sc[b].frozen) return;
  if (mode == 0) {
    SliceScalars& sc = red.sc[b];
    if (sc.done) return;
    const double rs = sc.rr[step & 1];
    if (rs == 0.0) {
      sc.done = 1;
      return;
    }
    if (step > 0) beta = static_cast<float>(rs / sc.rr[(step + 1) & 1]);
  }
  const size_t off = static_cast<size_t>(b) * n * n;
  const int i0 = blockIdx.y * kTile - HALO, j0 = blockIdx.x * kTile - HALO;
  for (int idx = threadIdx.x; idx < W * W; idx += blockDim.x) {
    const int li = idx / W, lj = idx - li * W;
    const int gi = i0 + li, gj = j0 + lj;
    float v = 0.f;
    if (gi >= 0 && gi < n && gj >= 0 && gj < n) {
      const size_t o = off + static_cast<size_t>(gi) * n + gj;
      v = in[o];
      if (mode == 0 && step > 0) v = r_in[o] + beta * v;
    }
    q[li][lj] = v;
  }
  __syncthreads();
  const int tj = threadIdx.x & 31, ti = threadIdx.x >> 5;
  double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int li = ti + 8 * k + HALO, lj = tj + HALO;
    const int gi = i0 + li, gj = j0 + lj;
    if (gi >= n || gj >= n) continue;
    const float c = q[li][lj];
    float tq = 0.f;
#pragma unroll
    for (int di = -RAD; di <= RAD; ++di)
#pragma unroll
      for (int dj = -RAD; dj <= RAD; ++dj) tq += coef.c[(di + RAD) * SIDE + (dj + RAD)] * q[li + di][lj + dj];
    float kk = 0.f;
    if (gj >= 1) kk += c - q[li][lj - 1];
    if (gj <= n - 2) kk -= q[li][lj + 1] - c;
    if (gi >= 1) kk += c - q[li - 1][lj];
    if (gi <= n - 2) kk -= q[li + 1][lj] - c;
    const float ax = sys.alpha * tq + sys.lambda * kk + sys.shift * c;
    const size_t o = off + static_cast<size_t>(gi) * n + gj;
    if (mode == 0) {
      if (step > 0) p_out[o] = c;
      ap_out[o] = ax;
      acc0 += static_cast<double>(c) * ax;
      acc1 += static_cast<double>(c) * c;
    } else if (mode == 1) {
      const float bv = bvec[o];
      const float rv = bv - ax;
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
      sc.bb = t1;
      sc.done = 0;
      sc.steps_run = 0;
      sc.min_ritz = __longlong_as_double(0x7ff0000000000000LL);
    }
  }
}

__device__ __forceinline__ float ktk_g(const float* __restrict__ p, int n, int i, int j) {
  const size_t o = static_cast<size_t>(i) * n + j;
  const float c = p[o];
  float v = 0.f;
  if (j >= 1) v += c - p[o - 1];
  if (j <= n - 2) v -= p[o + 1] - c;
  if (i >= 1) v += c - p[o - n];
  if (i <= n - 2) v -= p[o + n] - c;
  return v;
}

// Sharded-operator epilogue: nred = all-reduced alpha*Re(N p) partial sums.
__global__ void __launch_bounds__(kVecThreads) k_cg_epilogue(int n, int mode, const float* __restrict__ nred,
                                                             const float* __restrict__ p, const float* __restrict__ bvec,
                                                             float* __restrict__ ap, float* __restrict__ p_out,
                                                             float* __restrict__ x_out, SysParams sys, int step,
                                                             Reduce red) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  SliceScalars& sc = red.sc[b];
  if (sc.frozen || (mode == 0 && !slice_live(sc, step))) return;
  const int64_t L = static_cast<int64_t>(n) * n;
  const size_t off = static_cast<size_t>(b) * L;
  const float* pb = p + off;
  double acc0 = 0.0, acc1 = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ii = static_cast<int>(i / n), jj = static_cast<int>(i - static_cast<int64_t>(ii) * n);
    const float pv = pb[i];
    float ax = nred[off + i];
    if (sys.lambda != 0.f) ax += sys.lambda * ktk_g(pb, n, ii, jj);
    ax += sys.shift * pv;
    if (mode == 0) {
      ap[off + i] = ax;
      acc0 += static_cast<double>(pv) * ax;
      acc1 += static_cast<double>(pv) * pv;
    } else {
      const float bv = bvec[off + i];
      const float rv = bv - ax;
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
__device__ __forceinline__ float shrinkf(float x, float gamma) {
  const float m = fabsf(x) - gamma;
  return m > 0.f ? (x > 0.f ? m : -m) : 0.f;
}

__global__ void __launch_bounds__(kVecThreads) k_sb_post(int n, float* __restrict__ mu_new,
                                                         const float* __restrict__ mu_old, const float* __restrict__ bx_old,
                                                         const float* __restrict__ by_old, float* __restrict__ bx_new,
                                                         float* __restrict__ by_new, const float* __restrict__ fid,
                                                         float* __restrict__ rhs, float lambda, Reduce red) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const int64_t L = static_cast<int64_t>(n) * n;
  const size_t off = static_cast<size_t>(b) * L;
  SliceScalars& sc = red.sc[b];
  if (sc.frozen) {  // stopped on tolerance: carry the state through unchanged
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      mu_new[off + i] = mu_old[off + i];
      bx_new[off + i] = bx_old[off + i];
      by_new[off + i] = by_old[off + i];
    }
    return;
  }
  const float* mu = mu_new + off;
  const float* bxo = bx_old + off;
  const float* byo = by_old + off;
  const float gamma = 1.0f / lambda;
  double upd = 0.0;
  bool fin = true;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ii = static_cast<int>(i / n), jj = static_cast<int>(i - static_cast<int64_t>(ii) * n);
    const float c = mu[i];
    fin = fin && finite_f(c);
    upd += fabs(static_cast<double>(c) - static_cast<double>(mu_old[off + i]));
    // own pixel
    const float gx = jj < n - 1 ? mu[i + 1] - c : 0.f;
    const float gy = ii < n - 1 ? mu[i + n] - c : 0.f;
    const float dx = shrinkf(gx + bxo[i], gamma), dy = shrinkf(gy + byo[i], gamma);
    const float bxn = bxo[i] + gx - dx, byn = byo[i] + gy - dy;
    bx_new[off + i] = bxn;
    by_new[off + i] = byn;
    float div = 0.f;
    if (jj <= n - 2) div -= dx - bxn;
    if (ii <= n - 2) div -= dy - byn;
    if (jj >= 1) {  // tx at (ii, jj-1)
      const float gxl = c - mu[i - 1];
      const float dxl = shrinkf(gxl + bxo[i - 1], gamma);
      div += dxl - (bxo[i - 1] + gxl - dxl);
    }
    if (ii >= 1) {  // ty at (ii-1, jj)
      const float gyu = c - mu[i - n];
      const float dyu = shrinkf(gyu + byo[i - n], gamma);
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

// ------------------------------------------------------------------ Chambolle-Pock dual step
__global__ void __launch_bounds__(kVecThreads) k_cp_dual(int n, const float* __restrict__ u_cur,
                                                         const float* __restrict__ u_prev, const float* __restrict__ yx_old,
                                                         const float* __restrict__ yy_old, float* __restrict__ yx_new,
                                                         float* __restrict__ yy_new, const float* __restrict__ bp,
                                                         float* __restrict__ rhs, float tau, float sigma, float theta,
                                                         float lambda) {
  const int b = blockIdx.y;
  const int64_t L = static_cast<int64_t>(n) * n;
  const size_t off = static_cast<size_t>(b) * L;
  const float* uc = u_cur + off;
  const float* up = u_prev + off;
  auto ubar = [&](int64_t k) { return uc[k] + theta * (uc[k] - up[k]); };
  auto clampl = [&](float v) { return fminf(lambda, fmaxf(-lambda, v)); };
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ii = static_cast<int>(i / n), jj = static_cast<int>(i - static_cast<int64_t>(ii) * n);
    const float c = ubar(i);
    const float gx = jj < n - 1 ? ubar(i + 1) - c : 0.f;
    const float gy = ii < n - 1 ? ubar(i + n) - c : 0.f;
    const float yxn = clampl(yx_old[off + i] + sigma * gx);
    const float yyn = clampl(yy_old[off + i] + sigma * gy);
    yx_new[off + i] = yxn;
    yy_new[off + i] = yyn;
    float div = 0.f;
    if (jj <= n - 2) div -= yxn;
    if (ii <= n - 2) div -= yyn;
    if (jj >= 1) div += clampl(yx_old[off + i - 1] + sigma * (c - ubar(i - 1)));
    if (ii >= 1) div += clampl(yy_old[off + i - n] + sigma * (c - ubar(i - n)));
    rhs[off + i] = (uc[i] - tau * div) + tau * bp[off + i];
  }
}

// ------------------------------------------------------------------ small helpers
__global__ void k_scale_real(int64_t len, const float2* __restrict__ in, float* __restrict__ out, float alpha) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < len) out[i] = alpha * in[i].x;
}

__global__ void k_axpby(int64_t len, float a, const float* __restrict__ x, float b, const float* __restrict__ y,
                        float* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < len) out[i] = a * x[i] + b * y[i];
}

__global__ void __launch_bounds__(kVecThreads) k_dot(int64_t L, const float* __restrict__ x, const float* __restrict__ y,
                                                     double* out, Reduce red) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const size_t off = static_cast<size_t>(b) * L;
  double acc = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    acc += static_cast<double>(x[off + i]) * y[off + i];
  double t0, t1;
  double* part = red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
  if (reduce2_last(acc, 0.0, part, gridDim.x, blockIdx.x, &red.sc[b].counter[3], scratch, t0, t1) &&
      threadIdx.x == 0)
    out[b] = t0;
}

__global__ void __launch_bounds__(kVecThreads) k_leak(int64_t len, const float2* __restrict__ v, Reduce red) {
  __shared__ double scratch[32];
  double a = 0.0, im = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < len;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float2 z = v[i];
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

__global__ void k_grad(int n, const float* __restrict__ u, float* __restrict__ gx, float* __restrict__ gy) {
  const int64_t L = static_cast<int64_t>(n) * n;
  const int b = blockIdx.y;
  const size_t off = static_cast<size_t>(b) * L;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ii = static_cast<int>(i / n), jj = static_cast<int>(i % n);
    const float c = u[off + i];
    gx[off + i] = jj < n - 1 ? u[off + i + 1] - c : 0.f;
    gy[off + i] = ii < n - 1 ? u[off + i + n] - c : 0.f;
  }
}

__global__ void k_grad_adjoint(int n, const float* __restrict__ gx, const float* __restrict__ gy, float* __restrict__ out) {
  const int64_t L = static_cast<int64_t>(n) * n;
  const int b = blockIdx.y;
  const size_t off = static_cast<size_t>(b) * L;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ii = static_cast<int>(i / n), jj = static_cast<int>(i % n);
    float v = 0.f;
    if (jj >= 1) v += gx[off + i - 1];
    if (jj <= n - 2) v -= gx[off + i];
    if (ii >= 1) v += gy[off + i - n];
    if (ii <= n - 2) v -= gy[off + i];
    out[off + i] = v;
  }
}

__global__ void k_shrink(int64_t len, const float* __restrict__ x, float gamma, float* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < len) out[i] = shrinkf(x[i], gamma);
}

unsigned blocks_for(int64_t len, int threads) { return static_cast<unsigned>((len + threads - 1) / threads); }

}  // namespace

void launch_cg_update(int n, int B, const float* p, const float* ap, float* x, float* r, const SysParams& sys,
                      int step, const Reduce& red, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  dim3 grid(vec_blocks(L / 4, B) , B);
  k_cg_update<<<grid, kVecThreads, 0, st>>>(L, p, ap, x, r, sys, step, red);
  note_launch();
}

void launch_stencil(int n, int B, int rad, int euclid, const StencilCoef& coef, int mode, const float* in,
                    const float* r_in, float* p_out, float* ap_out, const float* b, float* x_out,
                    const SysParams& sys, int step, const Reduce& red, cudaStream_t st) {
  (void)euclid;  // masked taps carry zero coefficients
  dim3 grid((n + kTile - 1) / kTile, (n + kTile - 1) / kTile, B);
  switch (rad) {
    case 1: k_stencil<1><<<grid, 256, 0, st>>>(n, coef, mode, in, r_in, p_out, ap_out, b, x_out, sys, step, red); break;
    case 2: k_stencil<2><<<grid, 256, 0, st>>>(n, coef, mode, in, r_in, p_out, ap_out, b, x_out, sys, step, red); break;
    case 3: k_stencil<3><<<grid, 256, 0, st>>>(n, coef, mode, in, r_in, p_out, ap_out, b, x_out, sys, step, red); break;
    default: k_stencil<4><<<grid, 256, 0, st>>>(n, coef, mode, in, r_in, p_out, ap_out, b, x_out, sys, step, red); break;
  }
  note_launch();
}

void launch_cg_epilogue(int n, int B, int mode, const float* nred, const float* p, const float* b, float* ap,
                        float* p_out, float* x_out, const SysParams& sys, int step, const Reduce& red,
                        cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  dim3 grid(vec_blocks(L, B), B);
  k_cg_epilogue<<<grid, kVecThreads, 0, st>>>(n, mode, nred, p, b, ap, p_out, x_out, sys, step, red);
  note_launch();
}

void launch_sb_post(int n, int B, float* mu_new, const float* mu_old, const float* bx_old,
                    const float* by_old, float* bx_new, float* by_new, const float* fid, float* rhs,
                    float lambda, const Reduce& red, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  dim3 grid(vec_blocks(L, B), B);
  k_sb_post<<<grid, kVecThreads, 0, st>>>(n, mu_new, mu_old, bx_old, by_old, bx_new, by_new, fid, rhs, lambda, red);
  note_launch();
}

void launch_cp_dual(int n, int B, const float* u_cur, const float* u_prev, const float* yx_old,
                    const float* yy_old, float* yx_new, float* yy_new, const float* bp, float* rhs, float tau,
                    float sigma, float theta, float lambda, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  dim3 grid(vec_blocks(L, B), B);
  k_cp_dual<<<grid, kVecThreads, 0, st>>>(n, u_cur, u_prev, yx_old, yy_old, yx_new, yy_new, bp, rhs, tau, sigma,
                                          theta, lambda);
  note_launch();
}

void launch_scale_real(int64_t len, const float2* in, float* out, float alpha, cudaStream_t st) {
  k_scale_real<<<blocks_for(len, 256), 256, 0, st>>>(len, in, out, alpha);
  note_launch();
}

void launch_axpby(int64_t len, float a, const float* x, float b, const float* y, float* out, cudaStream_t st) {
  k_axpby<<<blocks_for(len, 256), 256, 0, st>>>(len, a, x, b, y, out);
  note_launch();
}

void launch_dot(int n, int B, const float* x, const float* y, double* out, const Reduce& red, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  dim3 grid(vec_blocks(L, B), B);
  k_dot<<<grid, kVecThreads, 0, st>>>(L, x, y, out, red);
  note_launch();
}

void launch_leak(int64_t len, const float2* v, const Reduce& red, cudaStream_t st) {
  k_leak<<<vec_blocks(len, 1), kVecThreads, 0, st>>>(len, v, red);
  note_launch();
}

void launch_grad(int n, int B, const float* u, float* gx, float* gy, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  k_grad<<<dim3(vec_blocks(L, B), B), kVecThreads, 0, st>>>(n, u, gx, gy);
  note_launch();
}

void launch_grad_adjoint(int n, int B, const float* gx, const float* gy, float* out, cudaStream_t st) {
  const int64_t L = static_cast<int64_t>(n) * n;
  k_grad_adjoint<<<dim3(vec_blocks(L, B), B), kVecThreads, 0, st>>>(n, gx, gy, out);
  note_launch();
}

void launch_shrink(int64_t len, const float* x, float gamma, float* out, cudaStream_t st) {
  k_shrink<<<blocks_for(len, 256), 256, 0, st>>>(len, x, gamma, out);
  note_launch();
}

void launch_reset_scalars(SliceScalars* sc, int B, cudaStream_t st) {
  cudaMemsetAsync(sc, 0, sizeof(SliceScalars) * B, st);
}

}  // namespace tomo_b200
