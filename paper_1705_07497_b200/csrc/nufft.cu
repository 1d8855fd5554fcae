// nufft.cu — the FFT passes of the normal-operator hot path on sm_100a (the W / W^T SpMVs are in
// spmv.cu):
//
//   type-2 (F_NU^*, proj/src/nufft.cpp:261-286):  P1 deapod+pad+row iFFT  ->  P2 column iFFT
//                                                  -> W  (separable window SpMV, interpolate :160-202)
//   type-1 (F_NU,   proj/src/nufft.cpp:236-259):  W^T (SpMV over the precomputed, count-sorted
//                                                  transpose, spread :119-158) -> PA grid-row
//                                                  FFT -> PB image-row FFT + crop + deapod
//
// The 2-D transforms (fft.cpp:26-50) are split into a pass over the n non-zero image rows and
// a pass over the m grid rows; zero padding and cropping (coeff_bin, nufft.cpp:232) are
// pruned: only n of m inputs are loaded and only n of m outputs are stored. The spatial grid
// is kept transposed ([iy][ix]) so every pass reads and writes contiguous rows; W's column
// indices are built for that layout. All kernels are templated on the real type R.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.h"

#include <cuda_pipeline.h>
#include <cooperative_groups.h>

namespace tomo_b200 {

namespace {

__device__ __forceinline__ int bin_of(int t, int n, int M) { return (t - n / 2 + M) & (M - 1); }

// FFT-row kernels: at most 512 threads per CTA so ptxas may give each thread up to 128
// registers (a radix-16 fp64 butterfly holds 64 registers of data alone).
constexpr int kFftThreads = 512;
#ifndef TOMO_FFT_MINB_F32
#define TOMO_FFT_MINB_F32 2
#endif
#ifndef TOMO_FFT_MINB_F64
#define TOMO_FFT_MINB_F64 1
#endif
constexpr size_t kMaxSmem = 220 * 1024;  // dynamic smem a persistent FFT CTA may use
// Persistent prefetching FFT-row kernels measured faster only for the longest rows (c5,
// m = 8192); below that the one-shot kernels (more CTAs in flight) win.
constexpr int kPersistMinM = 4096;

// beta for the fused CG p-update (solver.cpp:84): rr[k] / rr[k-1]; returns false when the
// slice's CG is finished (done flag or rs == 0, solver.cpp:70).
__device__ __forceinline__ bool cg_step_live(const Reduce& red, int b, int step, double& beta) {
  SliceScalars& sc = red.sc[b];
  if (sc.done || sc.frozen) return false;
  const double rs = sc.rr[step & 1];
  if (rs == 0.0) {
    sc.done = 1;
    return false;
  }
  beta = step > 0 ? rs / sc.rr[(step + 1) & 1] : 0.0;
  return true;
}

// Transposed store of rpc staged rows: dst[k * ld + q] = sm[q * STRIDE + pad16(k)] for k < K,
// q < ncols (<= rpc). Consecutive threads take consecutive q, then k, so each warp store
// covers whole 32-byte row segments (measured: one thread per k with 16-byte vector stores
// was slower, 2 half-sector stores per lane). rpc is a power of two: shifts, no divisions.
template <int STRIDE, typename C2>
TOMO_DEV void store_transposed(const C2* sm, int rpc, int ncols, int K, C2* __restrict__ dst, size_t ld) {
  const int lg = __ffs(rpc) - 1;
  for (int idx = threadIdx.x; idx < (K << lg); idx += blockDim.x) {
    const int k = idx >> lg, q = idx & (rpc - 1);
    if (q < ncols) dst[static_cast<size_t>(k) * ld + q] = sm[q * STRIDE + pad16(k)];
  }
}
struct NoStore {
  template <typename C2>
  TOMO_DEV void operator()(int, C2) const {}
};

// ---------------------------------------------------------------- P1: image rows (t1)
// deapodise + pad + inverse FFT along t2; the CG p-update (p = r + beta p) is fused into the
// load; output transposed to H[iy][t1] through smem.
// IN: the input mode, a compile-time constant so the per-element load carries no mode branches:
// 0 complex input, 1 real input, 2 standard CG p-update, 3 Chronopoulos-Gear update.
template <int M, int RB, typename R, bool HALF = false, int IN = 0>
__global__ void __launch_bounds__(kFftThreads, sizeof(R) == 4 ? TOMO_FFT_MINB_F32 : TOMO_FFT_MINB_F64) k_t2_rows(OpDev<R> d, const void* __restrict__ in,
                                                  PUpd<R> pu, int rpc) {
  using S = FftShape<M, RB>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  const int b = blockIdx.y;
  double beta = 0.0, alpha = 0.0;
  if constexpr (IN == 3) {
    const SliceScalars& sc = pu.red.sc[b];
    if (sc.done || sc.frozen) return;
    beta = sc.cg_beta;
    alpha = sc.cg_alpha;
  } else if constexpr (IN == 2) {
    if (!cg_step_live(pu.red, b, pu.step, beta)) return;
  } else {
    if (pu.red.sc && pu.red.sc[b].frozen) return;
  }
  const int rr = threadIdx.x / S::T, t = threadIdx.x % S::T;
  const int n = HALF ? M / 2 : d.n /* compile-time at 2x oversampling */;
  const int t10 = blockIdx.x * rpc;
  const int t1 = t10 + rr;
  const bool active = rr < rpc && t1 < n;
  C2* row = sm + rr * S::STRIDE;
  const size_t base = (static_cast<size_t>(b) * n + (active ? t1 : 0)) * n;
  const R a1 = active ? d.apod[t1] : R(0);
  const R bt = static_cast<R>(beta), al = static_cast<R>(alpha);
  auto load = [&](int i) -> C2 {
    const int t2 = (i + n / 2) & (M - 1);
    C2 v = czero<C2>();
    if (t2 < n) {
      const R sc = a1 * __ldg(&d.apod[t2]);
      if constexpr (IN == 0) {
        v = reinterpret_cast<const C2*>(in)[base + t2];
      } else if constexpr (IN == 3) {
        const size_t o = base + t2;
        R rv = pu.r[o];
        if (pu.step > 0) {
          // step k-1's update; at k = 1 (beta_0 = 0) p and s are not read (p_0 = r_0, s_0 = w_0)
          R pv = rv, sv = pu.w[o];
          if (pu.step > 1) {
            pv += bt * pu.p[o];
            sv += bt * pu.s[o];
          }
          const R xv = pu.x[o] + al * pv;
          rv -= al * sv;
          pu.p[o] = pv;
          pu.s[o] = sv;
          pu.x[o] = xv;
          pu.r[o] = rv;
          if (!finite_r(xv)) pu.red.sc[b].nonfinite = 1;
        }
        v.x = rv;
      } else if constexpr (IN == 2) {
        R pv = pu.p[base + t2];
        if (pu.step > 0) {
          pv = pu.r[base + t2] + bt * pv;
          pu.p[base + t2] = pv;
        }
        v.x = pv;
      } else {
        v.x = reinterpret_cast<const R*>(in)[base + t2];
      }
      v = cconj(cscale(v, sc));  // inverse transform: conj in, conj out
    }
    return v;
  };
  auto store = [&](int k, C2 v) { row[pad16(k)] = cconj(v); };
  fft_row<M, RB, true, C2, HALF ? 1 : 0>(row, d.tw, t, active, load, store);
  // transposed store H[b][k][t1]: rpc consecutive t1 per k
  C2* H = d.H + static_cast<size_t>(b) * M * n;
  store_transposed<S::STRIDE>(sm, rpc, min(rpc, n - t10), M, H + t10, static_cast<size_t>(n));
}

// P1 for a real image (real input or the real CG vectors): image rows 2q and 2q+1 are
// transformed together as the one complex row a + ib; their spectra are separated on the
// transposed store, A[k] = (Z[k] + conj Z[-k]) / 2, B[k] = (Z[k] - conj Z[-k]) / 2i, and only
// the rows iy in [0, m/2] of H are written (H[-iy] = conj H[iy]). IN: 1 real input, 2 standard
// CG p-update, 3 Chronopoulos-Gear update (as k_t2_rows; applied to both rows of the pair).
template <int M, int RB, typename R, bool HALF, int IN>
__global__ void __launch_bounds__(kFftThreads, sizeof(R) == 4 ? TOMO_FFT_MINB_F32 : TOMO_FFT_MINB_F64)
k_t2_rows_pk(OpDev<R> d, const void* __restrict__ in, PUpd<R> pu, int rpc) {
  using S = FftShape<M, RB>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  const int b = blockIdx.y;
  double beta = 0.0, alpha = 0.0;
  if constexpr (IN == 3) {
    const SliceScalars& sc = pu.red.sc[b];
    if (sc.done || sc.frozen) return;
    beta = sc.cg_beta;
    alpha = sc.cg_alpha;
  } else if constexpr (IN == 2) {
    if (!cg_step_live(pu.red, b, pu.step, beta)) return;
  } else {
    if (pu.red.sc && pu.red.sc[b].frozen) return;
  }
  const int rr = threadIdx.x / S::T, t = threadIdx.x % S::T;
  const int n = HALF ? M / 2 : d.n /* compile-time at 2x oversampling */, npair = n >> 1;
  const int q0 = blockIdx.x * rpc;
  const int q = q0 + rr;
  const bool active = rr < rpc && q < npair;
  C2* row = sm + rr * S::STRIDE;
  const size_t base = (static_cast<size_t>(b) * n + (active ? 2 * q : 0)) * n;  // row 2q; row 2q+1 at + n
  const R a1a = active ? d.apod[2 * q] : R(0), a1b = active ? d.apod[2 * q + 1] : R(0);
  const R bt = static_cast<R>(beta), al = static_cast<R>(alpha);
  auto value = [&](size_t o) -> R {
    if constexpr (IN == 3) {
      R rv = pu.r[o];
      if (pu.step > 0) {
        R pv = rv, sv = pu.w[o];
        if (pu.step > 1) {
          pv += bt * pu.p[o];
          sv += bt * pu.s[o];
        }
        const R xv = pu.x[o] + al * pv;
        rv -= al * sv;
        pu.p[o] = pv;
        pu.s[o] = sv;
        pu.x[o] = xv;
        pu.r[o] = rv;
        if (!finite_r(xv)) pu.red.sc[b].nonfinite = 1;
      }
      return rv;
    } else if constexpr (IN == 2) {
      R pv = pu.p[o];
      if (pu.step > 0) {
        pv = pu.r[o] + bt * pv;
        pu.p[o] = pv;
      }
      return pv;
    } else {
      return reinterpret_cast<const R*>(in)[o];
    }
  };
  auto load = [&](int i) -> C2 {
    const int t2 = (i + n / 2) & (M - 1);
    C2 v = czero<C2>();
    if (t2 < n) {
      const R ap = __ldg(&d.apod[t2]);
      const R va = value(base + t2) * (a1a * ap);
      const R vb = value(base + n + t2) * (a1b * ap);
      v = mk<C2>(va, -vb);  // inverse transform: conj in, conj out
    }
    return v;
  };
  auto store = [&](int k, C2 v) { row[pad16(k)] = cconj(v); };
  fft_row<M, RB, true, C2, HALF ? 1 : 0>(row, d.tw, t, active, load, store);
  // separate the two spectra; transposed store H[b][k][t1] for k in [0, M/2], 2 rpc consecutive t1
  const int ncols = 2 * max(0, min(rpc, npair - q0));
  const int w2 = 2 * rpc, lg = __ffs(w2) - 1;
  const int c = threadIdx.x & (w2 - 1);  // loop-invariant output column (blockDim.x is a multiple of 2 rpc)
  if (c >= ncols) return;
  C2* H = d.H + static_cast<size_t>(b) * M * n + 2 * q0 + c;
  const C2* rw = sm + (c >> 1) * S::STRIDE;
  const bool odd = c & 1;
  const R h = R(0.5);
  const int step = blockDim.x >> lg;
  for (int k = threadIdx.x >> lg; k <= M / 2; k += step) {
    const C2 z = rw[pad16(k)], zm = rw[pad16((M - k) & (M - 1))];
    H[static_cast<size_t>(k) * n] = odd ? mk<C2>(h * (z.y + zm.y), h * (zm.x - z.x))
                                        : mk<C2>(h * (z.x + zm.x), h * (z.y - zm.y));
  }
}

// ---------------------------------------------------------------- P2: grid rows (iy)
template <int M, int RB, typename R, bool HALF = false>
__global__ void __launch_bounds__(kFftThreads, sizeof(R) == 4 ? TOMO_FFT_MINB_F32 : TOMO_FFT_MINB_F64) k_t2_cols(OpDev<R> d, int rpc, int nrows, const SliceScalars* skip) {
  using S = FftShape<M, RB>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  const int b = blockIdx.y;
  if (skip && (skip[b].done || skip[b].frozen)) return;
  const int rr = threadIdx.x / S::T, t = threadIdx.x % S::T;
  const int n = HALF ? M / 2 : d.n /* compile-time at 2x oversampling */;
  const int iy = blockIdx.x * rpc + rr;
  const bool active = rr < rpc && iy < nrows;  // nrows: m, or m/2 + 1 rows of a Hermitian spectrum
  C2* row = sm + rr * S::STRIDE;
  const C2* H = d.H + (static_cast<size_t>(b) * M + (active ? iy : 0)) * n;
  C2* g = d.g + (static_cast<size_t>(b) * M + (active ? iy : 0)) * M;
  auto load = [&](int i) -> C2 {
    const int t1 = (i + n / 2) & (M - 1);
    return t1 < n ? cconj(H[t1]) : czero<C2>();
  };
  auto store = [&](int k, C2 v) { g[k] = cconj(v); };
  fft_row<M, RB, false, C2, HALF ? 1 : 0>(row, d.tw, t, active, load, store);
}

// ---------------------------------------------------------------- PA: grid rows (iy), type 1
// forward FFT along ix of the spread grid row, pruned to the n bins, transposed to K[t1][iy].
template <int M, int RB, typename R, bool HALF = false>
__global__ void __launch_bounds__(kFftThreads, sizeof(R) == 4 ? TOMO_FFT_MINB_F32 : TOMO_FFT_MINB_F64) k_t1_cols(OpDev<R> d, int rpc, int nrows, const SliceScalars* skip) {
  using S = FftShape<M, RB>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  const int b = blockIdx.y;
  if (skip && (skip[b].done || skip[b].frozen)) return;
  const int n = HALF ? M / 2 : d.n /* compile-time at 2x oversampling */;
  const int iy0 = blockIdx.x * rpc;
  const int rr = threadIdx.x / S::T, t = threadIdx.x % S::T;
  const bool active = rr < rpc && iy0 + rr < nrows;
  C2* row = sm + rr * S::STRIDE;
  const C2* Gr = d.Gt + (static_cast<size_t>(b) * M + iy0 + (active ? rr : 0)) * M;
  auto load = [&](int i) -> C2 { return Gr[i]; };
  auto store = [&](int k, C2 v) {
    const int t1 = (k + n / 2) & (M - 1);  // inverse of bin_of
    if (t1 < n) row[pad16(t1)] = v;
  };
  fft_row<M, RB, true, C2, HALF ? 2 : 0>(row, d.tw, t, active, load, store);
  C2* K = d.K + static_cast<size_t>(b) * n * M;
  store_transposed<S::STRIDE>(sm, rpc, min(rpc, nrows - iy0), n, K + iy0, static_cast<size_t>(M));
}

template <typename R>
__device__ __forceinline__ R ktk_at(const R* __restrict__ p, int n, int i, int j, R c) {
  // (grad^T grad p)(i,j) with the reference's Neumann boundary (solver.cpp:12-43)
  const size_t o = static_cast<size_t>(i) * n + j;
  R v = 0;
  if (j >= 1) v += c - p[o - 1];
  if (j <= n - 2) v -= p[o + 1] - c;
  if (i >= 1) v += c - p[o - n];
  if (i <= n - 2) v -= p[o + n] - c;
  return v;
}

// Chronopoulos-Gear step k from gamma = r_k.r_k and delta = r_k.(A r_k) (one reduction per
// step instead of standard CG's two): beta_k = gamma_k / gamma_{k-1}, p.Ap = delta - beta_k
// gamma_k / alpha_{k-1}, alpha_k = gamma_k / p.Ap, p.p = gamma_k + beta_k^2 p.p_{k-1}. The
// reference's exits (solver.cpp:70-90) in its order: the tolerance test on rs_k (made at the
// end of step k-1, steps_run = k-1), rs == 0 (steps_run = k), p.Ap == 0 (steps_run = k).
__device__ __forceinline__ void cgcg_finalize(SliceScalars& sc, double delta, double gamma, const SysParams& sys,
                                              int k) {
  if (!isfinite(gamma)) sc.nonfinite = 1;
  const double gamma_prev = sc.rr[(k + 1) & 1];
  sc.rr[k & 1] = gamma;
  sc.rs_last = gamma;
  if (k > 0 && sys.tol > 0.0 && sc.bb > 0.0 && sqrt(gamma) <= sys.tol * sqrt(sc.bb)) {
    sc.done = 1;
    sc.steps_run = k - 1;
    return;
  }
  if (gamma == 0.0) {
    sc.done = 1;
    sc.steps_run = k;
    return;
  }
  const double beta = k > 0 ? gamma / gamma_prev : 0.0;
  const double pap = k > 0 ? delta - beta * gamma / sc.cg_alpha : delta;
  const double pp = k > 0 ? gamma + beta * beta * sc.cg_pp : gamma;
  if (pp > 0.0) sc.min_ritz = fmin(sc.min_ritz, pap / pp);
  if (pap == 0.0) {
    sc.done = 1;
    sc.steps_run = k;
    return;
  }
  sc.cg_beta = beta;
  sc.cg_alpha = gamma / pap;
  sc.cg_pp = pp;
  sc.steps_run = k;
}

// ---------------------------------------------------------------- PB: image rows (t1)
// forward FFT along iy, crop to the n bins, deapodise, then the epilogue: complex / real
// output or the CG system apply alpha*Re(N p) + lambda K'K p + shift p with the dots.
// EPI: 0 complex output, 1 real output, 2 the CG modes (compile time: no per-element branches)
template <int M, int RB, typename R, bool HALF = false, int EPI = 2>
__global__ void __launch_bounds__(kFftThreads, sizeof(R) == 4 ? TOMO_FFT_MINB_F32 : TOMO_FFT_MINB_F64) k_t1_rows(OpDev<R> d, PbEpi<R> e, int rpc) {
  using S = FftShape<M, RB>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  __shared__ double red_scratch[32];
  const int b = blockIdx.y;
  if ((e.mode == PB_CG_STEP || e.mode == PB_CGCG) && (e.red.sc[b].done || e.red.sc[b].frozen)) return;
  if (e.mode == PB_CG_INIT && e.red.sc[b].frozen) return;
  const int n = d.n;
  const int rr = threadIdx.x / S::T, t = threadIdx.x % S::T;
  const int t1 = blockIdx.x * rpc + rr;
  const bool active = rr < rpc && t1 < n;
  C2* row = sm + rr * S::STRIDE;
  const C2* Kr = d.K + (static_cast<size_t>(b) * n + (active ? t1 : 0)) * M;
  const R a1 = active ? d.apod[t1] * e.scale : R(0);
  const size_t base = (static_cast<size_t>(b) * n + (active ? t1 : 0)) * n;
  const R lam = static_cast<R>(e.sys.lambda), shift = static_cast<R>(e.sys.shift);
  const R* p = e.p ? e.p + static_cast<size_t>(b) * n * n : nullptr;
  double acc0 = 0.0, acc1 = 0.0;
  auto load = [&](int i) -> C2 { return Kr[i]; };
  auto store = [&](int k, C2 X) {
    const int t2 = (k + n / 2) & (M - 1);
    if (t2 >= n) return;
    const R sc = a1 * __ldg(&d.apod[t2]);
    const size_t o = base + t2;
    if constexpr (EPI == 0) {
      e.out_c[o] = cscale(X, sc);
    } else if constexpr (EPI == 1) {
      e.out_r[o] = X.x * sc;
    } else {
      const R pv = p[static_cast<size_t>(t1) * n + t2];
      R ax = X.x * sc;
      if (lam != R(0)) ax += lam * ktk_at<R>(p, n, t1, t2, pv);
      ax += shift * pv;
      if (e.mode != PB_CG_INIT) {  // STEP: Ap, p.Ap, p.p; CGCG: w = A r, r.w, r.r
        e.ap[o] = ax;
        acc0 += static_cast<double>(pv) * ax;
        acc1 += static_cast<double>(pv) * pv;
      } else {  // PB_CG_INIT: r = b - A x0, p = r, x = x0
        const R bv = e.b[o];
        const R rv = bv - ax;
        e.ap[o] = rv;
        e.p_out[o] = rv;
        e.x_out[o] = pv;
        acc0 += static_cast<double>(rv) * rv;
        acc1 += static_cast<double>(bv) * bv;
      }
    }
  };
  fft_row<M, RB, false, C2, HALF ? 2 : 0>(row, d.tw, t, active, load, store);
  if (EPI == 2) {
    double t0s, t1s;
    SliceScalars& sc = e.red.sc[b];
    double* part = e.red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
    if (reduce2_last(acc0, acc1, part, gridDim.x, blockIdx.x, &sc.counter[0], red_scratch, t0s, t1s) &&
        threadIdx.x == 0) {
      if (e.mode == PB_CGCG) {
        cgcg_finalize(sc, t0s, t1s, e.sys, e.step);
      } else if (e.mode == PB_CG_STEP) {
        sc.pap = t0s;
        sc.pp = t1s;
      } else {
        sc.rr[0] = t0s;
        sc.rs_last = t0s;
        sc.bb = t1s;
        sc.done = 0;
        sc.steps_run = 0;
        sc.min_ritz = __longlong_as_double(0x7ff0000000000000LL);  // +inf
      }
    }
  }
}

// PB for a real-part output from a Hermitian K (rows iy in [0, m/2] stored, K[t1][-iy] =
// conj K[t1][iy]): image rows 2q and 2q+1 as the one complex row Xa + i Xb (Hermitian extension
// on load), whose transform is xa + i xb with both real. The folded W^T computed twice the
// Hermitian part of the spread grid: the 1/2 is folded into the deapodisation. EPI: 1 real
// output, 2 the CG modes (as k_t1_rows, per row of the pair).
template <int M, int RB, typename R, bool HALF, int EPI>
__global__ void __launch_bounds__(kFftThreads, sizeof(R) == 4 ? TOMO_FFT_MINB_F32 : TOMO_FFT_MINB_F64)
k_t1_rows_pk(OpDev<R> d, PbEpi<R> e, int rpc) {
  using S = FftShape<M, RB>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  __shared__ double red_scratch[32];
  const int b = blockIdx.y;
  if ((e.mode == PB_CG_STEP || e.mode == PB_CGCG) && (e.red.sc[b].done || e.red.sc[b].frozen)) return;
  if (e.mode == PB_CG_INIT && e.red.sc[b].frozen) return;
  const int n = d.n, npair = n >> 1;
  const int rr = threadIdx.x / S::T, t = threadIdx.x % S::T;
  const int q = blockIdx.x * rpc + rr;
  const bool active = rr < rpc && q < npair;
  const int ta = active ? 2 * q : 0;
  C2* row = sm + rr * S::STRIDE;
  const C2* Ka = d.K + (static_cast<size_t>(b) * n + ta) * M;
  const C2* Kb = Ka + M;
  const R a1a = active ? d.apod[ta] * e.scale * R(0.5) : R(0);
  const R a1b = active ? d.apod[ta + 1] * e.scale * R(0.5) : R(0);
  const size_t base = (static_cast<size_t>(b) * n + ta) * n;  // row ta; row ta+1 at + n
  const R lam = static_cast<R>(e.sys.lambda), shift = static_cast<R>(e.sys.shift);
  const R* p = e.p ? e.p + static_cast<size_t>(b) * n * n : nullptr;
  double acc0 = 0.0, acc1 = 0.0;
  auto load = [&](int k) -> C2 {
    C2 xa, xb;
    if (k <= M / 2) {
      xa = Ka[k];
      xb = Kb[k];
    } else {
      xa = cconj(Ka[M - k]);
      xb = cconj(Kb[M - k]);
    }
    return mk<C2>(xa.x - xb.y, xa.y + xb.x);  // xa + i xb
  };
  auto epi = [&](int t1, size_t o, int t2, R v) {
    if constexpr (EPI == 1) {
      e.out_r[o] = v;
    } else {
      const R pv = p[static_cast<size_t>(t1) * n + t2];
      R ax = v;
      if (lam != R(0)) ax += lam * ktk_at<R>(p, n, t1, t2, pv);
      ax += shift * pv;
      if (e.mode != PB_CG_INIT) {
        e.ap[o] = ax;
        acc0 += static_cast<double>(pv) * ax;
        acc1 += static_cast<double>(pv) * pv;
      } else {
        const R bv = e.b[o];
        const R rv = bv - ax;
        e.ap[o] = rv;
        e.p_out[o] = rv;
        e.x_out[o] = pv;
        acc0 += static_cast<double>(rv) * rv;
        acc1 += static_cast<double>(bv) * bv;
      }
    }
  };
  auto store = [&](int k, C2 X) {
    const int t2 = (k + n / 2) & (M - 1);
    if (t2 >= n) return;
    const R ap = __ldg(&d.apod[t2]);
    epi(ta, base + t2, t2, X.x * (a1a * ap));
    epi(ta + 1, base + n + t2, t2, X.y * (a1b * ap));
  };
  fft_row<M, RB, false, C2, HALF ? 2 : 0>(row, d.tw, t, active, load, store);
  if (EPI == 2) {
    double t0s, t1s;
    SliceScalars& sc = e.red.sc[b];
    double* part = e.red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
    if (reduce2_last(acc0, acc1, part, gridDim.x, blockIdx.x, &sc.counter[0], red_scratch, t0s, t1s) &&
        threadIdx.x == 0) {
      if (e.mode == PB_CGCG) {
        cgcg_finalize(sc, t0s, t1s, e.sys, e.step);
      } else if (e.mode == PB_CG_STEP) {
        sc.pap = t0s;
        sc.pp = t1s;
      } else {
        sc.rr[0] = t0s;
        sc.rs_last = t0s;
        sc.bb = t1s;
        sc.done = 0;
        sc.steps_run = 0;
        sc.min_ritz = __longlong_as_double(0x7ff0000000000000LL);  // +inf
      }
    }
  }
}

// PB on image-row pairs with the 8192-point fp64 row split over two CTAs (decimation in frequency, as
// k_t1_cols_dif): CTA h transforms y_h from the Hermitian-extended pair row and owns outputs 2k + h.
template <int M, int RB, typename R, int EPI>
__global__ void __launch_bounds__(M / 2 / RB, 2) k_t1_rows_pk_dif(OpDev<R> d, PbEpi<R> e) {
  constexpr int MH = M / 2;
  using S = FftShape<MH, RB>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  __shared__ double red_scratch[32];
  const int b = blockIdx.y;
  if ((e.mode == PB_CG_STEP || e.mode == PB_CGCG) && (e.red.sc[b].done || e.red.sc[b].frozen)) return;
  if (e.mode == PB_CG_INIT && e.red.sc[b].frozen) return;
  const int n = d.n, npair = n >> 1;
  const int t = threadIdx.x, h = blockIdx.x & 1;
  const int q = blockIdx.x >> 1;
  const bool active = q < npair;
  const int ta = active ? 2 * q : 0;
  C2* row = sm;
  const C2* Ka = d.K + (static_cast<size_t>(b) * n + ta) * M;
  const C2* Kb = Ka + M;
  const R a1a = active ? d.apod[ta] * e.scale * R(0.5) : R(0);
  const R a1b = active ? d.apod[ta + 1] * e.scale * R(0.5) : R(0);
  const size_t base = (static_cast<size_t>(b) * n + ta) * n;  // row ta; row ta+1 at + n
  const R lam = static_cast<R>(e.sys.lambda), shift = static_cast<R>(e.sys.shift);
  const R* p = e.p ? e.p + static_cast<size_t>(b) * n * n : nullptr;
  double acc0 = 0.0, acc1 = 0.0;
  auto full = [&](int k) -> C2 {  // the pair row Xa + i Xb at k in [0, M)
    C2 xa, xb;
    if (k <= M / 2) {
      xa = Ka[k];
      xb = Kb[k];
    } else {
      xa = cconj(Ka[M - k]);
      xb = cconj(Kb[M - k]);
    }
    return mk<C2>(xa.x - xb.y, xa.y + xb.x);  // xa + i xb
  };
  auto load = [&](int i) -> C2 {
    const C2 x0 = full(i), x1 = full(i + MH);
    return h == 0 ? cadd(x0, x1) : cmul(csub(x0, x1), __ldg(&d.tw[i]));
  };
  auto epi = [&](int t1, size_t o, int t2, R v) {
    if constexpr (EPI == 1) {
      e.out_r[o] = v;
    } else {
      const R pv = p[static_cast<size_t>(t1) * n + t2];
      R ax = v;
      if (lam != R(0)) ax += lam * ktk_at<R>(p, n, t1, t2, pv);
      ax += shift * pv;
      if (e.mode != PB_CG_INIT) {
        e.ap[o] = ax;
        acc0 += static_cast<double>(pv) * ax;
        acc1 += static_cast<double>(pv) * pv;
      } else {
        const R bv = e.b[o];
        const R rv = bv - ax;
        e.ap[o] = rv;
        e.p_out[o] = rv;
        e.x_out[o] = pv;
        acc0 += static_cast<double>(rv) * rv;
        acc1 += static_cast<double>(bv) * bv;
      }
    }
  };
  auto store = [&](int kh, C2 X) {
    const int t2 = (2 * kh + h + n / 2) & (M - 1);
    if (t2 >= n) return;
    const R ap = __ldg(&d.apod[t2]);
    epi(ta, base + t2, t2, X.x * (a1a * ap));
    epi(ta + 1, base + n + t2, t2, X.y * (a1b * ap));
  };
  fft_row<MH, RB, false, C2, 0>(row, d.tw_half, t, active, load, store);
  if (EPI == 2) {
    double t0s, t1s;
    SliceScalars& sc = e.red.sc[b];
    double* part = e.red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
    if (reduce2_last(acc0, acc1, part, gridDim.x, blockIdx.x, &sc.counter[0], red_scratch, t0s, t1s) &&
        threadIdx.x == 0) {
      if (e.mode == PB_CGCG) {
        cgcg_finalize(sc, t0s, t1s, e.sys, e.step);
      } else if (e.mode == PB_CG_STEP) {
        sc.pap = t0s;
        sc.pp = t1s;
      } else {
        sc.rr[0] = t0s;
        sc.rs_last = t0s;
        sc.bb = t1s;
        sc.done = 0;
        sc.steps_run = 0;
        sc.min_ritz = __longlong_as_double(0x7ff0000000000000LL);  // +inf
      }
    }
  }
}

// ================================================================ persistent FFT-row kernels
// Grid (CTAs per slice, B). Each CTA walks its slice's rows g = blockIdx.x, blockIdx.x +
// gridDim.x, ... (rpc rows per step). The next step's input rows are copied global -> smem
// with cp.async (LDGSTS) right after the current step's first pass has consumed the staging
// buffer, so the copy overlaps the remaining FFT passes and the stores (one staging buffer,
// no extra registers).

template <typename C2>
TOMO_DEV void async_copy(C2* dst_smem, const C2* src) {
  __pipeline_memcpy_async(dst_smem, src, sizeof(C2));
}

// P2: inverse FFT along ix of H rows (t1 at the n bins), natural store g[iy][ix].
template <int M, int RB, typename R>
__global__ void __launch_bounds__(kFftThreads, sizeof(R) == 4 ? TOMO_FFT_MINB_F32 : TOMO_FFT_MINB_F64)
k_t2_cols_p(OpDev<R> d, int nrows, const SliceScalars* skip) {
  using S = FftShape<M, RB>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* row = reinterpret_cast<C2*>(smraw);
  C2* stage = row + S::STRIDE;  // n entries (compact t1)
  const int b = blockIdx.y;
  if (skip && (skip[b].done || skip[b].frozen)) return;  // CTA-uniform
  const int n = d.n, t = threadIdx.x;
  const C2* Hb = d.H + static_cast<size_t>(b) * M * n;
  C2* gb = d.g + static_cast<size_t>(b) * M * M;
  auto issue = [&](int iy) {
    const C2* H = Hb + static_cast<size_t>(iy) * n;
    for (int k = t; k < n; k += S::T) async_copy(&stage[k], &H[k]);
  };
  int iy = blockIdx.x;
  if (iy < nrows) issue(iy);
  __pipeline_commit();
  for (; iy < nrows; iy += gridDim.x) {
    __pipeline_wait_prior(0);
    __syncthreads();
    C2 pre[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int t1 = (t + r * S::T + n / 2) & (M - 1);
      pre[r] = t1 < n ? cconj(stage[t1]) : czero<C2>();
    }
    __syncthreads();  // staging consumed by every thread
    if (iy + static_cast<int>(gridDim.x) < nrows) issue(iy + gridDim.x);
    __pipeline_commit();
    C2* gout = gb + static_cast<size_t>(iy) * M;
    fft_row_pre<M, RB, false, C2>(row, d.tw, t, true, pre, [&](int k, C2 v) { gout[k] = cconj(v); });
  }
  __pipeline_wait_prior(0);
}

// PA: forward FFT of rpc spread-grid rows, pruned to the n bins, transposed store K[t1][iy].
template <int M, int RB, typename R>
__global__ void __launch_bounds__(kFftThreads, sizeof(R) == 4 ? TOMO_FFT_MINB_F32 : TOMO_FFT_MINB_F64)
k_t1_cols_p(OpDev<R> d, int rpc, int nrows, const SliceScalars* skip) {
  using S = FftShape<M, RB>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  C2* stage = sm + static_cast<size_t>(rpc) * S::STRIDE;  // rpc x M
  const int b = blockIdx.y;
  if (skip && (skip[b].done || skip[b].frozen)) return;
  const int n = d.n;
  const int rr = threadIdx.x / S::T, t = threadIdx.x % S::T;
  C2* row = sm + rr * S::STRIDE;
  const int steps = (nrows + rpc - 1) / rpc;  // the last step's staging may cover rows >= nrows (not stored)
  const C2* Gb = d.Gt + static_cast<size_t>(b) * M * M;
  C2* K = d.K + static_cast<size_t>(b) * n * M;
  auto issue = [&](int st) {
    const C2* Gr = Gb + static_cast<size_t>(st) * rpc * M;  // rpc consecutive rows
    for (int k = threadIdx.x; k < rpc * M; k += blockDim.x) async_copy(&stage[k], &Gr[k]);
  };
  int st = blockIdx.x;
  if (st < steps) issue(st);
  __pipeline_commit();
  for (; st < steps; st += gridDim.x) {
    __pipeline_wait_prior(0);
    __syncthreads();
    C2 pre[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) pre[r] = stage[rr * M + t + r * S::T];
    __syncthreads();
    if (st + static_cast<int>(gridDim.x) < steps) issue(st + gridDim.x);
    __pipeline_commit();
    const int iy0 = st * rpc;
    fft_row_pre<M, RB, true, C2>(row, d.tw, t, true, pre, [&](int k, C2 v) {
      const int t1 = (k + n / 2) & (M - 1);  // inverse of bin_of
      if (t1 < n) row[pad16(t1)] = v;
    });
    store_transposed<S::STRIDE>(sm, rpc, min(rpc, nrows - iy0), n, K + iy0, static_cast<size_t>(M));
  }
  __pipeline_wait_prior(0);
}

// PB: forward FFT along iy of K rows, crop + deapodise + epilogue (as k_t1_rows); the CG dots
// are accumulated over all rows of the CTA and reduced once per CTA.
template <int M, int RB, typename R>
__global__ void __launch_bounds__(kFftThreads, sizeof(R) == 4 ? TOMO_FFT_MINB_F32 : TOMO_FFT_MINB_F64)
k_t1_rows_p(OpDev<R> d, PbEpi<R> e) {
  using S = FftShape<M, RB>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* row = reinterpret_cast<C2*>(smraw);
  C2* stage = row + S::STRIDE;  // M entries
  __shared__ double red_scratch[32];
  const int b = blockIdx.y;
  if ((e.mode == PB_CG_STEP || e.mode == PB_CGCG) && (e.red.sc[b].done || e.red.sc[b].frozen)) return;
  if (e.mode == PB_CG_INIT && e.red.sc[b].frozen) return;
  const int n = d.n, t = threadIdx.x;
  const C2* Kb = d.K + static_cast<size_t>(b) * n * M;
  auto issue = [&](int t1) {
    const C2* Kr = Kb + static_cast<size_t>(t1) * M;
    for (int k = t; k < M; k += S::T) async_copy(&stage[k], &Kr[k]);
  };
  const R lam = static_cast<R>(e.sys.lambda), shift = static_cast<R>(e.sys.shift);
  const R* p = e.p ? e.p + static_cast<size_t>(b) * n * n : nullptr;
  double acc0 = 0.0, acc1 = 0.0;
  int t1 = blockIdx.x;
  if (t1 < n) issue(t1);
  __pipeline_commit();
  for (; t1 < n; t1 += gridDim.x) {
    __pipeline_wait_prior(0);
    __syncthreads();
    C2 pre[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) pre[r] = stage[t + r * S::T];
    __syncthreads();
    if (t1 + static_cast<int>(gridDim.x) < n) issue(t1 + gridDim.x);
    __pipeline_commit();
    const R a1 = d.apod[t1] * e.scale;
    const size_t base = (static_cast<size_t>(b) * n + t1) * n;
    fft_row_pre<M, RB, false, C2>(row, d.tw, t, true, pre, [&](int k, C2 X) {
      const int t2 = (k + n / 2) & (M - 1);
      if (t2 >= n) return;
      const R sc = a1 * __ldg(&d.apod[t2]);
      const size_t o = base + t2;
      if (e.mode == PB_COMPLEX) {
        e.out_c[o] = cscale(X, sc);
      } else if (e.mode == PB_REAL) {
        e.out_r[o] = X.x * sc;
      } else {
        const R pv = p[static_cast<size_t>(t1) * n + t2];
        R ax = X.x * sc;
        if (lam != R(0)) ax += lam * ktk_at<R>(p, n, t1, t2, pv);
        ax += shift * pv;
        if (e.mode != PB_CG_INIT) {  // STEP: Ap, p.Ap, p.p; CGCG: w = A r, r.w, r.r
          e.ap[o] = ax;
          acc0 += static_cast<double>(pv) * ax;
          acc1 += static_cast<double>(pv) * pv;
        } else {  // PB_CG_INIT: r = b - A x0, p = r, x = x0
          const R bv = e.b[o];
          const R rv = bv - ax;
          e.ap[o] = rv;
          e.p_out[o] = rv;
          e.x_out[o] = pv;
          acc0 += static_cast<double>(rv) * rv;
          acc1 += static_cast<double>(bv) * bv;
        }
      }
    });
  }
  __pipeline_wait_prior(0);
  if (e.mode < PB_CG_STEP) return;
  double t0s, t1s;
  SliceScalars& sc = e.red.sc[b];
  double* part = e.red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
  if (reduce2_last(acc0, acc1, part, gridDim.x, blockIdx.x, &sc.counter[0], red_scratch, t0s, t1s) &&
      threadIdx.x == 0) {
    if (e.mode == PB_CGCG) {
      cgcg_finalize(sc, t0s, t1s, e.sys, e.step);
    } else if (e.mode == PB_CG_STEP) {
      sc.pap = t0s;
      sc.pp = t1s;
    } else {
      sc.rr[0] = t0s;
      sc.rs_last = t0s;
      sc.bb = t1s;
      sc.done = 0;
      sc.steps_run = 0;
      sc.min_ritz = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    }
  }
}

// ================================================================ split grid rows (fp64, m = 8192)
// A grid row of 8192 fp64 points (128 KB + padding) admits one 512-thread CTA per SM, which then
// serialises its row load, FFT and stores. One decimation-in-frequency step splits the row over two
// CTAs: X[2k+h] = FFT_{M/2}(y_h)[k], y_0[i] = x[i] + x[i+M/2], y_1[i] = (x[i] - x[i+M/2]) W_M^i; each
// CTA (h = blockIdx.x & 1) loads the whole row, combines its halves on load and transforms M/2 points
// in 70 KB of shared memory (two CTAs per SM, one loading while the other computes).

// P1 on image-row pairs at fp64 m = 8192, split over a cluster of two CTAs (decimation in frequency).
// The fused CG update must write each image element once, so CTA 0 updates (and deapodises, packs)
// the pair's t2 in [n/2, n) and CTA 1 the t2 in [0, n/2) into its shared memory; after a cluster
// barrier each CTA's first pass reads both halves, one of them from the peer CTA's shared memory
// (DSMEM). Every element of y_h has at most one non-zero padded input (n <= m/2). CTA h then owns
// the spectra Z[2k+h]: the Hermitian separation pairs Z[k] with Z[-k], same parity, same CTA.
// Q: 4n == M (quarter-pruned first pass).
template <int M, int RB, typename R, bool Q, int IN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(M / 2 / RB, 2)
k_t2_rows_pk_dif(OpDev<R> d, const void* __restrict__ in, PUpd<R> pu) {
  namespace cgr = cooperative_groups;
  constexpr int MH = M / 2;
  using S = FftShape<MH, RB>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* row = reinterpret_cast<C2*>(smraw);
  C2* xs = row + S::STRIDE;  // this CTA's half of the packed, updated, deapodised input (n/2 entries)
  const int b = blockIdx.y;
  double beta = 0.0, alpha = 0.0;
  if constexpr (IN == 3) {
    const SliceScalars& sc = pu.red.sc[b];
    if (sc.done || sc.frozen) return;  // cluster-uniform (same slice)
    beta = sc.cg_beta;
    alpha = sc.cg_alpha;
  } else if constexpr (IN == 2) {
    if (!cg_step_live(pu.red, b, pu.step, beta)) return;
  } else {
    if (pu.red.sc && pu.red.sc[b].frozen) return;
  }
  const int n = Q ? M / 4 : d.n, npair = n >> 1, nh = n / 2;
  const int q = blockIdx.x >> 1, h = blockIdx.x & 1, t = threadIdx.x;
  if (q >= npair) return;  // cluster-uniform
  cgr::cluster_group cluster = cgr::this_cluster();
  const size_t base = (static_cast<size_t>(b) * n + 2 * q) * n;  // row 2q; row 2q+1 at + n
  const R a1a = d.apod[2 * q], a1b = d.apod[2 * q + 1];
  const R bt = static_cast<R>(beta), al = static_cast<R>(alpha);
  auto value = [&](size_t o) -> R {
    if constexpr (IN == 3) {
      R rv = pu.r[o];
      if (pu.step > 0) {
        R pv = rv, sv = pu.w[o];
        if (pu.step > 1) {
          pv += bt * pu.p[o];
          sv += bt * pu.s[o];
        }
        const R xv = pu.x[o] + al * pv;
        rv -= al * sv;
        pu.p[o] = pv;
        pu.s[o] = sv;
        pu.x[o] = xv;
        pu.r[o] = rv;
        if (!finite_r(xv)) pu.red.sc[b].nonfinite = 1;
      }
      return rv;
    } else if constexpr (IN == 2) {
      R pv = pu.p[o];
      if (pu.step > 0) {
        pv = pu.r[o] + bt * pv;
        pu.p[o] = pv;
      }
      return pv;
    } else {
      return reinterpret_cast<const R*>(in)[o];
    }
  };
  // CTA 0: t2 = nh + j (padded positions j in [0, n/2)); CTA 1: t2 = j (positions M - n/2 + j)
  for (int j = t; j < nh; j += blockDim.x) {
    const int t2 = h == 0 ? nh + j : j;
    const R ap = __ldg(&d.apod[t2]);
    const R va = value(base + t2) * (a1a * ap);
    const R vb = value(base + n + t2) * (a1b * ap);
    xs[j] = mk<C2>(va, -vb);  // inverse transform: conj in, conj out
  }
  cluster.sync();
  const C2* xa = cluster.map_shared_rank(xs, 0);  // positions [0, n/2)
  const C2* xb = cluster.map_shared_rank(xs, 1);  // positions [M - n/2, M)
  auto load = [&](int i) -> C2 {
    C2 v = czero<C2>();
    if (i < nh) {
      v = xa[i];
    } else if (i >= MH - nh) {
      v = xb[i - (MH - nh)];
      if (h == 1) v = mk<C2>(-v.x, -v.y);
    }
    return h == 0 ? v : cmul(v, __ldg(&d.tw[i]));
  };
  auto store = [&](int k, C2 v) { row[pad16(k)] = cconj(v); };
  fft_row<MH, RB, true, C2, Q ? 1 : 0>(row, d.tw_half, t, true, load, store);
  cluster.sync();  // the peer's reads of this CTA's xs are done before either CTA exits
  // spectra of the two rows at k = 2k' + h in [0, M/2]: Z[k] = row[k'], Z[M - k] = row[(MH - k' - h) % MH]
  C2* H = d.H + static_cast<size_t>(b) * M * n + 2 * q;
  const R hf = R(0.5);
  for (int idx = t; idx < 2 * (MH / 2 + 1); idx += blockDim.x) {
    const int kp = idx >> 1, c = idx & 1;
    const int k = 2 * kp + h;
    if (k > M / 2) continue;
    const C2 z = row[pad16(kp)], zm = row[pad16((MH - kp - h) & (MH - 1))];
    H[static_cast<size_t>(k) * n + c] = c ? mk<C2>(hf * (z.y + zm.y), hf * (zm.x - z.x))
                                          : mk<C2>(hf * (z.x + zm.x), hf * (z.y - zm.y));
  }
}

// P2: inverse FFT along ix of the H row (conj in / conj out), natural stores g[iy][2k+h].
// Q: 4n == M, the non-zero inputs of y are its first and last quarter (compile-time pruning).
template <int M, int RB, typename R, bool Q>
__global__ void __launch_bounds__(M / 2 / RB, 2) k_t2_cols_dif(OpDev<R> d, int nrows, const SliceScalars* skip) {
  constexpr int MH = M / 2;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* row = reinterpret_cast<C2*>(smraw);
  const int b = blockIdx.y;
  if (skip && (skip[b].done || skip[b].frozen)) return;
  const int iy = blockIdx.x >> 1, h = blockIdx.x & 1;
  if (iy >= nrows) return;  // CTA-uniform
  const int n = Q ? M / 4 : d.n, t = threadIdx.x;
  const C2* H = d.H + (static_cast<size_t>(b) * M + iy) * n;
  C2* g = d.g + (static_cast<size_t>(b) * M + iy) * M;
  auto in = [&](int p) -> C2 {  // conj(x[p]): H at t1 = (p + n/2) mod M < n (pruned padding)
    const int t1 = (p + n / 2) & (M - 1);
    return t1 < n ? cconj(H[t1]) : czero<C2>();
  };
  auto load = [&](int i) -> C2 {
    const C2 xa = in(i), xb = in(i + MH);
    return h == 0 ? cadd(xa, xb) : cmul(csub(xa, xb), __ldg(&d.tw[i]));
  };
  auto store = [&](int k, C2 v) { g[2 * k + h] = cconj(v); };
  fft_row<MH, RB, false, C2, Q ? 1 : 0>(row, d.tw_half, t, true, load, store);
}

// PA: forward FFT along ix of the spread-grid row; the kept bins of half h are t1 = 2q + par,
// par = (h + n/2) & 1, staged at q and stored transposed to K[t1][iy].
template <int M, int RB, typename R>
__global__ void __launch_bounds__(M / 2 / RB, 2) k_t1_cols_dif(OpDev<R> d, int nrows, const SliceScalars* skip) {
  constexpr int MH = M / 2;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* row = reinterpret_cast<C2*>(smraw);
  const int b = blockIdx.y;
  if (skip && (skip[b].done || skip[b].frozen)) return;
  const int iy = blockIdx.x >> 1, h = blockIdx.x & 1;
  if (iy >= nrows) return;  // CTA-uniform
  const int n = d.n, t = threadIdx.x;
  const C2* Gr = d.Gt + (static_cast<size_t>(b) * M + iy) * M;
  auto load = [&](int i) -> C2 {
    const C2 xa = Gr[i], xb = Gr[i + MH];
    return h == 0 ? cadd(xa, xb) : cmul(csub(xa, xb), __ldg(&d.tw[i]));
  };
  auto store = [&](int kh, C2 v) {
    const int t1 = (2 * kh + h + n / 2) & (M - 1);
    if (t1 < n) row[pad16(t1 >> 1)] = v;
  };
  fft_row<MH, RB, true, C2, 0>(row, d.tw_half, t, true, load, store);
  const int par = (h + n / 2) & 1;
  C2* K = d.K + static_cast<size_t>(b) * n * M + iy;
  for (int q = t; q < n / 2; q += blockDim.x) K[static_cast<size_t>(2 * q + par) * M] = row[pad16(q)];
}

template <int M, int RB, typename R>
__global__ void k_fft_rows_test(const cplx<R>* tw, const cplx<R>* in, cplx<R>* out, int rows, int inverse) {
  using S = FftShape<M, RB>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  const int r = blockIdx.x;
  const int t = threadIdx.x;
  const C2* src = in + static_cast<size_t>(r) * M;
  C2* dst = out + static_cast<size_t>(r) * M;
  auto load = [&](int i) -> C2 { return inverse ? cconj(src[i]) : src[i]; };
  auto store = [&](int k, C2 v) { dst[k] = inverse ? cconj(v) : v; };
  fft_row<M, RB, false, C2>(sm, tw, t, true, load, store);
}

// ---------------------------------------------------------------- dispatch helpers
// rows-per-CTA: transposed stores need >= 32 B per row segment (rpc >= 32 / sizeof(C2)),
// enough threads per CTA, bounded smem, and as many CTAs as possible above that.
int choose_rpc(int T, int m, int rows_per_slice, int B, size_t elem, bool transposed) {
  const int min_rpc = transposed ? std::max(1, static_cast<int>(32 / elem)) : 1;
  int rpc = std::max(min_rpc, std::max(1, 128 / T));
  while (rpc > 1 && (rpc * T > kFftThreads || static_cast<size_t>(rpc) * padded_len(m) * elem > 110 * 1024)) rpc >>= 1;
  while (rpc > min_rpc && rpc * T > 256 && static_cast<int64_t>((rows_per_slice + rpc - 1) / rpc) * B < 2 * 148) rpc >>= 1;
  while (rpc > 1 && rpc > rows_per_slice) rpc >>= 1;  // small grids (m = 32): never more rows than exist
  return std::max(rpc, 1);
}

// Base radix of the FFT rows. Measured on B200 (c2 fp64 / c3 fp32): radix 8 and 4 (more
// threads per row, one more smem pass) were 1.3-1.9x slower than radix 16 even where radix 16
// leaves the GPU under-occupied, so radix 16 is used throughout (fft.cuh keeps the others).
int choose_rb(int, int64_t, size_t) { return 16; }

template <typename F>
void dispatch_m(int m, F&& f) {
  switch (m) {
    case 32: f(std::integral_constant<int, 32>{}); break;
    case 64: f(std::integral_constant<int, 64>{}); break;
    case 128: f(std::integral_constant<int, 128>{}); break;
    case 256: f(std::integral_constant<int, 256>{}); break;
    case 512: f(std::integral_constant<int, 512>{}); break;
    case 1024: f(std::integral_constant<int, 1024>{}); break;
    case 2048: f(std::integral_constant<int, 2048>{}); break;
    case 4096: f(std::integral_constant<int, 4096>{}); break;
    case 8192: f(std::integral_constant<int, 8192>{}); break;
    default: throw std::runtime_error("grid side m must be a power of two in [32, 8192], got " + std::to_string(m));
  }
}

template <typename F>
void dispatch_m_rb(int m, int rb, F&& f) {
  dispatch_m(m, [&](auto MC) {
    (void)rb;
    f(MC, std::integral_constant<int, 16>{});
  });
}

// The n-row passes (P1, PB) run on n of the m rows only. For fp64 rows up to m = 2048 that
// leaves the GPU short of warps (126-register threads, ~7 warps/SM at c2), and radix-8 rows
// (twice the threads per row, one more smem pass) measured faster: c2 t2_rows 10.5 -> 9.9 us,
// t1_rows 11.7 -> 10.7 us. fp32 (c3: 17 -> 23 us) and m = 8192 keep radix 16.
// TOMO_ROW_RB=8|16 overrides (A/B runs, TOMO_AB=1).
int env_int(const char* name, int dflt) { return ab_int(name, dflt); }

// `rows` = transforms per launch (image rows, or row pairs on the half grid, times slices): fp64
// launches of at most 256 rows at m = 512 / 1024 take radix 4 (twice radix 8's threads per row; c2,
// 256 row pairs: 32.3 -> 32.6 slices/s, PB 10.3 -> 9.9 us over 3 runs each; c1's 896 pairs per lane
// are slower at radix 4).
int row_rb(int m, size_t elem, int64_t rows) {
  static const int forced = env_int("TOMO_ROW_RB", 0);
  if (forced == 4 || forced == 8 || forced == 16) return forced;
  if (elem == 16 && (m == 512 || m == 1024) && rows <= 256) return 4;
  return elem == 16 && m <= 2048 ? 8 : 16;
}

template <typename F>
void dispatch_m_rows(int m, size_t elem, int64_t rows, F&& f) {
  dispatch_m(m, [&](auto MC) {
    constexpr int M = decltype(MC)::value;
    if constexpr (M == 512 || M == 1024) {  // radix 4 (A/B, TOMO_ROW_RB=4): c1 / c2 grid sizes only
      if (row_rb(m, elem, rows) == 4) {
        f(MC, std::integral_constant<int, 4>{});
        return;
      }
    }
    if (row_rb(m, elem, rows) == 8 && M / 8 <= kFftThreads)
      f(MC, std::integral_constant<int, 8>{});
    else
      f(MC, std::integral_constant<int, 16>{});
  });
}

// fp64 8192-point grid rows split over two CTAs by one decimation-in-frequency step (k_t2_cols_dif /
// k_t1_cols_dif); TOMO_DIF=0 restores the whole-row kernels (A/B runs).
bool dif_on() {
  static const bool v = env_int("TOMO_DIF", 1) != 0;
  return v;
}

// Grid-row passes (P2, PA): radix 16 unless TOMO_COL_RB=8 (A/B runs; one-shot kernels only).
int col_rb(int m, size_t elem) {
  static const int forced = ab_int("TOMO_COL_RB", 0);
  (void)m;
  (void)elem;
  return forced == 8 ? 8 : 16;
}

template <typename F>
void dispatch_m_cols(int m, size_t elem, F&& f) {
  dispatch_m(m, [&](auto MC) {
    constexpr int M = decltype(MC)::value;
    if constexpr (M < kPersistMinM) {
      if (col_rb(m, elem) == 8) {
        f(MC, std::integral_constant<int, 8>{});
        return;
      }
    }
    f(MC, std::integral_constant<int, 16>{});
  });
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
  // Opt in to > 48 KB dynamic smem once per kernel (and per larger size).
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> granted;
  if (bytes <= 48 * 1024) return;
  std::lock_guard<std::mutex> lk(mu);
  size_t& g = granted[reinterpret_cast<const void*>(kernel)];
  if (g >= bytes) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  g = bytes;
}

}  // namespace

template <typename R>
void launch_t2_rows(const OpDev<R>& d, int B, const void* in, bool in_complex, const PUpd<R>& pu, cudaStream_t st) {
  if constexpr (sizeof(R) == 8) {
    if (d.herm_in && !in_complex && d.m == 8192 && dif_on()) {  // fp64 8192: a CTA-pair cluster per row pair
      constexpr int M = 8192, RB = 16;
      using SH = FftShape<M / 2, RB>;
      const size_t smem = (static_cast<size_t>(SH::STRIDE) + d.n / 2) * sizeof(cplx<R>);
      const int mode = !pu.enabled ? 1 : pu.cgcg ? 3 : 2;
      auto go = [&](auto kern) {
        set_smem(kern, smem);
        CK_LAUNCH(launch_k(kern, dim3(2 * (d.n / 2), B), SH::T, smem, st, d, in, pu));
      };
      auto go_q = [&](auto QC) {
        constexpr bool QQ = decltype(QC)::value;
        switch (mode) {
          case 1: go(k_t2_rows_pk_dif<M, RB, R, QQ, 1>); break;
          case 2: go(k_t2_rows_pk_dif<M, RB, R, QQ, 2>); break;
          default: go(k_t2_rows_pk_dif<M, RB, R, QQ, 3>); break;
        }
      };
      if (4 * d.n == M) go_q(std::true_type{});
      else go_q(std::false_type{});
      note_launch();
      return;
    }
  }
  if (d.herm_in && !in_complex) {  // real image: two rows per complex transform, H rows [0, m/2]
    dispatch_m_rows(d.m, sizeof(cplx<R>), static_cast<int64_t>(d.n / 2) * B, [&](auto MC, auto RC) {
      constexpr int M = decltype(MC)::value, RB = decltype(RC)::value;
      using S = FftShape<M, RB>;
      // 2 rpc t1 values per H row segment: >= 32 B segments need rpc >= 16 / sizeof(C2)
      const int rpc = choose_rpc(S::T, M, d.n / 2, B, 2 * sizeof(cplx<R>), true);
      const size_t smem = static_cast<size_t>(rpc) * S::STRIDE * sizeof(cplx<R>);
      dim3 grid((d.n / 2 + rpc - 1) / rpc, B);
      auto go = [&](auto kern) {
        set_smem(kern, smem);
        CK_LAUNCH(launch_k(kern, grid, rpc * S::T, smem, st, d, in, pu, rpc));
      };
      const int mode = !pu.enabled ? 1 : pu.cgcg ? 3 : 2;
      auto go_mode = [&](auto HC) {
        constexpr bool H = decltype(HC)::value;
        switch (mode) {
          case 1: go(k_t2_rows_pk<M, RB, R, H, 1>); break;
          case 2: go(k_t2_rows_pk<M, RB, R, H, 2>); break;
          default: go(k_t2_rows_pk<M, RB, R, H, 3>); break;
        }
      };
      if (2 * d.n == M) go_mode(std::true_type{});
      else go_mode(std::false_type{});
      note_launch();
    });
    return;
  }
  dispatch_m_rows(d.m, sizeof(cplx<R>), static_cast<int64_t>(d.n) * B, [&](auto MC, auto RC) {
    constexpr int M = decltype(MC)::value, RB = decltype(RC)::value;
    using S = FftShape<M, RB>;
    const int rpc = choose_rpc(S::T, M, d.n, B, sizeof(cplx<R>), true);
    const size_t smem = static_cast<size_t>(rpc) * S::STRIDE * sizeof(cplx<R>);
    dim3 grid((d.n + rpc - 1) / rpc, B);
    auto go = [&](auto kern) {
      set_smem(kern, smem);
      CK_LAUNCH(launch_k(kern, grid, rpc * S::T, smem, st, d, in, pu, rpc));
    };
    const int mode = in_complex ? 0 : !pu.enabled ? 1 : pu.cgcg ? 3 : 2;
    auto go_mode = [&](auto HC) {
      constexpr bool H = decltype(HC)::value;
      switch (mode) {
        case 0: go(k_t2_rows<M, RB, R, H, 0>); break;
        case 1: go(k_t2_rows<M, RB, R, H, 1>); break;
        case 2: go(k_t2_rows<M, RB, R, H, 2>); break;
        default: go(k_t2_rows<M, RB, R, H, 3>); break;
      }
    };
    if (2 * d.n == M) go_mode(std::true_type{});
    else go_mode(std::false_type{});
    note_launch();
  });
}

template <typename K>
int persistent_ctas(K kernel, int threads, size_t smem, int rows_per_slice, int B) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> occ_cache;
  int occ = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = occ_cache.find(reinterpret_cast<const void*>(kernel));
    if (it != occ_cache.end()) {
      occ = it->second;
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
      occ_cache[reinterpret_cast<const void*>(kernel)] = occ;
    }
  }
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t slots = static_cast<int64_t>(std::max(occ, 1)) * sms;
  const int64_t per_slice = std::max<int64_t>(1, slots / std::max(B, 1));
  return static_cast<int>(std::min<int64_t>(rows_per_slice, per_slice));
}

template <typename R>
void launch_t2_cols(const OpDev<R>& d, int B, const SliceScalars* skip, cudaStream_t st) {
  dispatch_m_cols(d.m, sizeof(cplx<R>), [&](auto MC, auto RC) {
    constexpr int M = decltype(MC)::value, RB = decltype(RC)::value;
    using S = FftShape<M, RB>;
    const int nrows = d.herm_in ? M / 2 + 1 : M;  // Hermitian spectrum: rows [0, m/2]
    if constexpr (M == 8192 && sizeof(R) == 8) {  // fp64 8192-point rows split over two CTAs
      if (dif_on()) {
        using SH = FftShape<M / 2, RB>;
        const size_t smem = static_cast<size_t>(SH::STRIDE) * sizeof(cplx<R>);
        auto go = [&](auto kern) {
          set_smem(kern, smem);
          CK_LAUNCH(launch_k(kern, dim3(2 * nrows, B), SH::T, smem, st, d, nrows, skip));
        };
        if (4 * d.n == M) go(k_t2_cols_dif<M, RB, R, true>);
        else go(k_t2_cols_dif<M, RB, R, false>);
        note_launch();
        return;
      }
    }
    if constexpr (M >= kPersistMinM) {
      const size_t smem = (static_cast<size_t>(S::STRIDE) + d.n) * sizeof(cplx<R>);
      set_smem(k_t2_cols_p<M, RB, R>, smem);
      const int ctas = persistent_ctas(k_t2_cols_p<M, RB, R>, S::T, smem, nrows, B);
      CK_LAUNCH(launch_k(k_t2_cols_p<M, RB, R>, dim3(ctas, B), S::T, smem, st, d, nrows, skip));
    } else {
      const int rpc = choose_rpc(S::T, M, nrows, B, sizeof(cplx<R>), false);
      const size_t smem = static_cast<size_t>(rpc) * S::STRIDE * sizeof(cplx<R>);
      auto go = [&](auto kern) {
        set_smem(kern, smem);
        CK_LAUNCH(launch_k(kern, dim3((nrows + rpc - 1) / rpc, B), rpc * S::T, smem, st, d, rpc, nrows, skip));
      };
      if (2 * d.n == M) go(k_t2_cols<M, RB, R, true>);
      else go(k_t2_cols<M, RB, R, false>);
    }
    note_launch();
  });
}

template <typename R>
void launch_wt_rows(const OpDev<R>& d, int B, const SliceScalars* skip, cudaStream_t st) {
  launch_wt_spread<R>(d, B, d.s, d.Gt, skip, st);
  launch_t1_cols_only<R>(d, B, skip, st);
}

template <typename R>
void launch_t1_cols_only(const OpDev<R>& d, int B, const SliceScalars* skip, cudaStream_t st) {
  dispatch_m_cols(d.m, sizeof(cplx<R>), [&](auto MC, auto RC) {
    constexpr int M = decltype(MC)::value, RB = decltype(RC)::value;
    using S = FftShape<M, RB>;
    const int nrows = d.herm_out ? M / 2 + 1 : M;  // the folded (Hermitian) grid: rows [0, m/2]
    if constexpr (M == 8192 && sizeof(R) == 8) {  // fp64 8192-point rows split over two CTAs
      if (dif_on()) {
        using SH = FftShape<M / 2, RB>;
        const size_t smem = static_cast<size_t>(SH::STRIDE) * sizeof(cplx<R>);
        set_smem(k_t1_cols_dif<M, RB, R>, smem);
        CK_LAUNCH(launch_k(k_t1_cols_dif<M, RB, R>, dim3(2 * nrows, B), SH::T, smem, st, d, nrows, skip));
        note_launch();
        return;
      }
    }
    if constexpr (M >= kPersistMinM) {
      // transposed K stores need >= 32 B per row segment; staging holds rpc full rows
      int rpc = std::max(1, static_cast<int>(32 / sizeof(cplx<R>)));
      while (rpc > 1 && (rpc * S::T > kFftThreads ||
                         static_cast<size_t>(rpc) * (S::STRIDE + M) * sizeof(cplx<R>) > 200 * 1024))
        rpc >>= 1;
      const size_t smem = static_cast<size_t>(rpc) * (S::STRIDE + M) * sizeof(cplx<R>);
      if (smem <= kMaxSmem) {
        set_smem(k_t1_cols_p<M, RB, R>, smem);
        const int ctas = persistent_ctas(k_t1_cols_p<M, RB, R>, rpc * S::T, smem, (nrows + rpc - 1) / rpc, B);
        CK_LAUNCH(launch_k(k_t1_cols_p<M, RB, R>, dim3(ctas, B), rpc * S::T, smem, st, d, rpc, nrows, skip));
        note_launch();
        return;
      }
    }
    // one-shot CTAs (also when row + staging do not fit: fp64, m = 8192)
    const int rpc1 = choose_rpc(S::T, M, nrows, B, sizeof(cplx<R>), true);
    const size_t smem1 = static_cast<size_t>(rpc1) * S::STRIDE * sizeof(cplx<R>);
    auto go = [&](auto kern) {
      set_smem(kern, smem1);
      CK_LAUNCH(launch_k(kern, dim3((nrows + rpc1 - 1) / rpc1, B), rpc1 * S::T, smem1, st, d, rpc1, nrows, skip));
    };
    if (2 * d.n == M) go(k_t1_cols<M, RB, R, true>);
    else go(k_t1_cols<M, RB, R, false>);
    note_launch();
  });
}

template <typename R>
void launch_t1_rows(const OpDev<R>& d, int B, const PbEpi<R>& e, cudaStream_t st) {
  if (d.herm_out) {  // real-part output from the folded grid: two image rows per complex transform
    if (e.mode == PB_COMPLEX) throw std::runtime_error("launch_t1_rows: complex output from a folded grid");
    if constexpr (sizeof(R) == 8) {
    if (d.m == 8192 && dif_on()) {  // fp64 8192-point rows split over two CTAs
      using SH = FftShape<4096, 16>;
      const size_t smem = static_cast<size_t>(SH::STRIDE) * sizeof(cplx<R>);
      const int np = d.n / 2;
      if (2 * np > MAX_PART_BLOCKS) throw std::runtime_error("launch_t1_rows: too many row pairs for one reduction");
      auto go = [&](auto kern) {
        set_smem(kern, smem);
        CK_LAUNCH(launch_k(kern, dim3(2 * np, B), SH::T, smem, st, d, e));
      };
      if (e.mode == PB_REAL) go(k_t1_rows_pk_dif<8192, 16, R, 1>);
      else go(k_t1_rows_pk_dif<8192, 16, R, 2>);
      note_launch();
      return;
    }
    }
    dispatch_m_rows(d.m, sizeof(cplx<R>), static_cast<int64_t>(d.n / 2) * B, [&](auto MC, auto RC) {
      constexpr int M = decltype(MC)::value, RB = decltype(RC)::value;
      using S = FftShape<M, RB>;
      const int np = d.n / 2;
      int rpc = choose_rpc(S::T, M, np, B, sizeof(cplx<R>), false);
      while ((rpc * S::T) % 32) rpc <<= 1;
      while (rpc > 1 && (np + rpc - 1) / rpc > MAX_PART_BLOCKS) rpc <<= 1;
      const size_t smem = static_cast<size_t>(rpc) * S::STRIDE * sizeof(cplx<R>);
      dim3 grid((np + rpc - 1) / rpc, B);
      auto go = [&](auto kern) {
        set_smem(kern, smem);
        CK_LAUNCH(launch_k(kern, grid, rpc * S::T, smem, st, d, e, rpc));
      };
      auto go_epi = [&](auto HC) {
        constexpr bool H = decltype(HC)::value;
        if (e.mode == PB_REAL) go(k_t1_rows_pk<M, RB, R, H, 1>);
        else go(k_t1_rows_pk<M, RB, R, H, 2>);
      };
      if (2 * d.n == M) go_epi(std::true_type{});
      else go_epi(std::false_type{});
      note_launch();
    });
    return;
  }
  dispatch_m_rows(d.m, sizeof(cplx<R>), static_cast<int64_t>(d.n) * B, [&](auto MC, auto RC) {
    constexpr int M = decltype(MC)::value, RB = decltype(RC)::value;
    using S = FftShape<M, RB>;
    constexpr size_t smem_p = (static_cast<size_t>(S::STRIDE) + M) * sizeof(cplx<R>);
    if constexpr (S::T % 32 == 0 && smem_p <= kMaxSmem && M >= kPersistMinM) {
      const size_t smem = smem_p;
      set_smem(k_t1_rows_p<M, RB, R>, smem);
      const int ctas = std::min(MAX_PART_BLOCKS, persistent_ctas(k_t1_rows_p<M, RB, R>, S::T, smem, d.n, B));
      CK_LAUNCH(launch_k(k_t1_rows_p<M, RB, R>, dim3(ctas, B), S::T, smem, st, d, e));
    } else {  // rows shorter than 512: whole warps need several rows per CTA
      int rpc = choose_rpc(S::T, M, d.n, B, sizeof(cplx<R>), false);
      while ((rpc * S::T) % 32) rpc <<= 1;
      while (rpc > 1 && (d.n + rpc - 1) / rpc > MAX_PART_BLOCKS) rpc <<= 1;
      const size_t smem = static_cast<size_t>(rpc) * S::STRIDE * sizeof(cplx<R>);
      dim3 grid((d.n + rpc - 1) / rpc, B);
      auto go = [&](auto kern) {
        set_smem(kern, smem);
        CK_LAUNCH(launch_k(kern, grid, rpc * S::T, smem, st, d, e, rpc));
      };
      const int epi = e.mode == PB_COMPLEX ? 0 : e.mode == PB_REAL ? 1 : 2;
      auto go_epi = [&](auto HC) {
        constexpr bool H = decltype(HC)::value;
        if (epi == 0) go(k_t1_rows<M, RB, R, H, 0>);
        else if (epi == 1) go(k_t1_rows<M, RB, R, H, 1>);
        else go(k_t1_rows<M, RB, R, H, 2>);
      };
      if (2 * d.n == M) go_epi(std::true_type{});
      else go_epi(std::false_type{});
    }
    note_launch();
  });
}

template <typename R>
void launch_fft_rows_test(int m, int rows, const cplx<R>* tw, const cplx<R>* in, cplx<R>* out, bool inverse,
                          cudaStream_t st) {
  dispatch_m_rb(m, choose_rb(m, rows, sizeof(cplx<R>)), [&](auto MC, auto RC) {
    constexpr int M = decltype(MC)::value, RB = decltype(RC)::value;
    using S = FftShape<M, RB>;
    const size_t smem = S::STRIDE * sizeof(cplx<R>);
    set_smem(k_fft_rows_test<M, RB, R>, smem);
    CK_LAUNCH(launch_k(k_fft_rows_test<M, RB, R>, rows, S::T, smem, st, tw, in, out, rows, inverse ? 1 : 0));
    note_launch();
  });
}

#define TOMO_INST_NUFFT(R)                                                                                   \
  template void launch_t2_rows<R>(const OpDev<R>&, int, const void*, bool, const PUpd<R>&, cudaStream_t);   \
  template void launch_t2_cols<R>(const OpDev<R>&, int, const SliceScalars*, cudaStream_t);                 \
  template void launch_wt_rows<R>(const OpDev<R>&, int, const SliceScalars*, cudaStream_t);                 \
  template void launch_t1_cols_only<R>(const OpDev<R>&, int, const SliceScalars*, cudaStream_t);            \
  template void launch_t1_rows<R>(const OpDev<R>&, int, const PbEpi<R>&, cudaStream_t);                     \
  template void launch_fft_rows_test<R>(int, int, const cplx<R>*, const cplx<R>*, cplx<R>*, bool, cudaStream_t);

TOMO_INST_NUFFT(float)
TOMO_INST_NUFFT(double)

}  // namespace tomo_b200
