// nufft.cu — the normal-operator hot path on sm_100a:
//
//   type-2 (F_NU^*, proj/src/nufft.cpp:261-286):  P1 deapod+pad+row iFFT  ->  P2 column iFFT
//                                                  -> W  (SELL-32 ELL SpMV, interpolate :160-202)
//   type-1 (F_NU,   proj/src/nufft.cpp:236-259):  W^T (SELL-32 SpMV over the precomputed
//                                                  transpose, spread :119-158) fused into the
//                                                  first FFT pass -> PB row FFT + crop + deapod
//
// The 2-D transforms (fft.cpp:26-50) are split into a pass over the n non-zero image rows and
// a pass over the m grid rows; zero padding and cropping (coeff_bin, nufft.cpp:232) are
// pruned: only n of m inputs are loaded and only n of m outputs are stored. The spatial grid
// is kept transposed ([iy][ix]) so every pass reads and writes contiguous rows; W's column
// indices are built for that layout. All kernels are templated on the real type R.
#include <algorithm>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.h"

namespace tomo_b200 {

namespace {

__device__ __forceinline__ int bin_of(int t, int n, int M) { return (t - n / 2 + M) & (M - 1); }

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

template <typename T>
__device__ __forceinline__ T ldg(const T* p) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ Quad<float> ldg(const Quad<float>* p) {
  const float4 v = __ldg(reinterpret_cast<const float4*>(p));
  return Quad<float>{{v.x, v.y, v.z, v.w}};
}
template <>
__device__ __forceinline__ Quad<double> ldg(const Quad<double>* p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return Quad<double>{{a.x, a.y, b.x, b.y}};
}
template <>
__device__ __forceinline__ WtEnt<float> ldg(const WtEnt<float>* p) {
  const int2 v = __ldg(reinterpret_cast<const int2*>(p));
  return WtEnt<float>{v.x, __int_as_float(v.y)};
}
template <>
__device__ __forceinline__ WtEnt<double> ldg(const WtEnt<double>* p) {
  const int4 v = __ldg(reinterpret_cast<const int4*>(p));
  return WtEnt<double>{v.x, 0, __hiloint2double(v.w, v.z)};
}

// ---------------------------------------------------------------- P1: image rows
template <int M, typename R>
__global__ void k_t2_rows(OpDev<R> d, const void* __restrict__ in, int in_complex, PUpd<R> pu, int rpc) {
  using S = FftShape<M>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  const int b = blockIdx.y;
  double beta = 0.0;
  if (pu.enabled && !cg_step_live(pu.red, b, pu.step, beta)) return;
  if (!pu.enabled && pu.red.sc && pu.red.sc[b].frozen) return;
  const int rr = threadIdx.x / S::T, t = threadIdx.x % S::T;
  const int n = d.n;
  const int t1 = blockIdx.x * rpc + rr;
  const bool active = rr < rpc && t1 < n;
  C2* row = sm + rr * S::STRIDE;
  if (active) {
    const R a1 = d.apod[t1];
    const size_t base = (static_cast<size_t>(b) * n + t1) * n;
    const R bt = static_cast<R>(beta);
    for (int i = t; i < M; i += S::T) {
      const int t2 = (i + n / 2) & (M - 1);
      C2 v = czero<C2>();
      if (t2 < n) {
        const R sc = a1 * d.apod[t2];
        if (in_complex) {
          v = reinterpret_cast<const C2*>(in)[base + t2];
        } else if (pu.enabled) {
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
      row[pad16(i)] = v;
    }
  }
  fft_row_smem<M, C2>(row, d.tw, t, active);
  // transposed store H[b][k][t1]: rpc consecutive t1 per k
  const int t10 = blockIdx.x * rpc;
  C2* H = d.H + static_cast<size_t>(b) * M * n;
  for (int idx = threadIdx.x; idx < M * rpc; idx += blockDim.x) {
    const int k = idx / rpc, q = idx - k * rpc;
    if (t10 + q < n) H[static_cast<size_t>(k) * n + t10 + q] = cconj(sm[q * S::STRIDE + pad16(k)]);
  }
}

// ---------------------------------------------------------------- P2: grid rows (iy)
template <int M, typename R>
__global__ void k_t2_cols(OpDev<R> d, int rpc, const SliceScalars* skip) {
  using S = FftShape<M>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  const int b = blockIdx.y;
  if (skip && (skip[b].done || skip[b].frozen)) return;
  const int rr = threadIdx.x / S::T, t = threadIdx.x % S::T;
  const int n = d.n;
  const int iy = blockIdx.x * rpc + rr;
  const bool active = rr < rpc;
  C2* row = sm + rr * S::STRIDE;
  if (active) {
    const C2* H = d.H + (static_cast<size_t>(b) * M + iy) * n;
    for (int i = t; i < M; i += S::T) {
      const int t1 = (i + n / 2) & (M - 1);
      row[pad16(i)] = t1 < n ? cconj(H[t1]) : czero<C2>();
    }
  }
  fft_row_smem<M, C2>(row, d.tw, t, active);
  if (active) {
    C2* g = d.g + (static_cast<size_t>(b) * M + iy) * M;
    for (int i = t; i < M; i += S::T) g[i] = cconj(row[pad16(i)]);
  }
}

// ---------------------------------------------------------------- W: SELL-32 ELL SpMV
// One thread per slice sample (row of W); entries streamed as int4 column / value quads,
// coalesced across the warp (lane = row within the 32-row slice). The batch of slices
// shares the matrix stream (SpMM over BT slices per pass).
template <int BT, typename R>
__global__ void __launch_bounds__(256) k_w(OpDev<R> d, int B, const cplx<R>* __restrict__ grid,
                                            cplx<R>* __restrict__ out, const SliceScalars* skip) {
  using C2 = cplx<R>;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d.Ppad) return;
  const int blk = j >> 5, lane = j & 31;
  const size_t G = static_cast<size_t>(d.m) * d.m;
  for (int b0 = 0; b0 < B; b0 += BT) {
    C2 acc[BT];
#pragma unroll
    for (int q = 0; q < BT; ++q) acc[q] = czero<C2>();
    const int4* cp = d.w_cols + static_cast<size_t>(blk) * d.nq * 32 + lane;
    const Quad<R>* vp = d.w_vals + static_cast<size_t>(blk) * d.nq * 32 + lane;
    for (int q4 = 0; q4 < d.nq; ++q4) {
      const int4 c = __ldg(cp + q4 * 32);
      const Quad<R> v = ldg(vp + q4 * 32);
#pragma unroll
      for (int q = 0; q < BT; ++q) {
        if (b0 + q < B) {
          const C2* gb = grid + G * (b0 + q);
          const C2 g0 = gb[c.x], g1 = gb[c.y], g2 = gb[c.z], g3 = gb[c.w];
          acc[q].x += v.v[0] * g0.x + v.v[1] * g1.x + v.v[2] * g2.x + v.v[3] * g3.x;
          acc[q].y += v.v[0] * g0.y + v.v[1] * g1.y + v.v[2] * g2.y + v.v[3] * g3.y;
        }
      }
    }
    if (j < d.P) {
#pragma unroll
      for (int q = 0; q < BT; ++q)
        if (b0 + q < B && !(skip && (skip[b0 + q].done || skip[b0 + q].frozen)))
          out[static_cast<size_t>(b0 + q) * d.P + j] = acc[q];
    }
  }
}

// W^T SpMV of one 32-node SELL block: lane's node value.
template <typename R>
__device__ __forceinline__ cplx<R> wt_node(const OpDev<R>& d, const cplx<R>* __restrict__ s, int gb, int lane) {
  using C2 = cplx<R>;
  const uint32_t c0 = __ldg(&d.wt_chunk[gb]), c1 = __ldg(&d.wt_chunk[gb + 1]);
  C2 a0 = czero<C2>(), a1 = czero<C2>();
  const WtEnt<R>* e = d.wt_ent + static_cast<size_t>(c0) * 32 + lane;
  uint32_t c = c0;
  for (; c + 1 < c1; c += 2, e += 64) {
    const WtEnt<R> x0 = ldg(e), x1 = ldg(e + 32);
    const C2 s0 = __ldg(&s[x0.j]), s1 = __ldg(&s[x1.j]);
    a0.x += x0.w * s0.x;
    a0.y += x0.w * s0.y;
    a1.x += x1.w * s1.x;
    a1.y += x1.w * s1.y;
  }
  if (c < c1) {
    const WtEnt<R> x0 = ldg(e);
    const C2 s0 = __ldg(&s[x0.j]);
    a0.x += x0.w * s0.x;
    a0.y += x0.w * s0.y;
  }
  return cadd(a0, a1);
}

// ---------------------------------------------------------------- W^T + first type-1 pass
template <int M, typename R>
__global__ void k_wt_rows(OpDev<R> d, int rpc, const SliceScalars* skip) {
  using S = FftShape<M>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  const int b = blockIdx.y;
  if (skip && (skip[b].done || skip[b].frozen)) return;
  const int n = d.n;
  const int iy0 = blockIdx.x * rpc;
  const C2* s = d.s + static_cast<size_t>(b) * d.P;
  // W^T rows of the CTA's grid rows: SELL blocks [iy0*M/32, (iy0+rpc)*M/32)
  const int nblocks = rpc * (M / 32);
  const int gb0 = iy0 * (M / 32);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int q = warp; q < nblocks; q += nwarps) {
    const C2 v = wt_node<R>(d, s, gb0 + q, lane);
    const int local = q * 32 + lane;  // node index within the CTA's rows
    const int rr = local / M, ix = local - rr * M;
    sm[rr * S::STRIDE + pad16(ix)] = v;
  }
  const int rr = threadIdx.x / S::T, t = threadIdx.x % S::T;
  fft_row_smem<M, C2>(sm + rr * S::STRIDE, d.tw, t, rr < rpc);
  // pruned transposed store K[b][t1][iy0 + q] = X[bin(t1)]
  C2* K = d.K + static_cast<size_t>(b) * n * M;
  for (int idx = threadIdx.x; idx < n * rpc; idx += blockDim.x) {
    const int t1 = idx / rpc, q = idx - t1 * rpc;
    K[static_cast<size_t>(t1) * M + iy0 + q] = sm[q * S::STRIDE + pad16(bin_of(t1, n, M))];
  }
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

// ---------------------------------------------------------------- PB: image rows (t1)
template <int M, typename R>
__global__ void k_t1_rows(OpDev<R> d, PbEpi<R> e, int rpc) {
  using S = FftShape<M>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  __shared__ double red_scratch[32];
  const int b = blockIdx.y;
  if (e.mode == PB_CG_STEP && (e.red.sc[b].done || e.red.sc[b].frozen)) return;
  if (e.mode == PB_CG_INIT && e.red.sc[b].frozen) return;
  const int n = d.n;
  const int rr = threadIdx.x / S::T, t = threadIdx.x % S::T;
  const int t1 = blockIdx.x * rpc + rr;
  const bool active = rr < rpc && t1 < n;
  C2* row = sm + rr * S::STRIDE;
  if (active) {
    const C2* K = d.K + (static_cast<size_t>(b) * n + t1) * M;
    for (int i = t; i < M; i += S::T) row[pad16(i)] = K[i];
  }
  fft_row_smem<M, C2>(row, d.tw, t, active);
  double acc0 = 0.0, acc1 = 0.0;
  if (active) {
    const R a1 = d.apod[t1] * e.scale;
    const size_t base = (static_cast<size_t>(b) * n + t1) * n;
    const R lam = static_cast<R>(e.sys.lambda), shift = static_cast<R>(e.sys.shift);
    for (int t2 = t; t2 < n; t2 += S::T) {
      const C2 X = row[pad16(bin_of(t2, n, M))];
      const R sc = a1 * d.apod[t2];
      const size_t o = base + t2;
      if (e.mode == PB_COMPLEX) {
        e.out_c[o] = cscale(X, sc);
      } else if (e.mode == PB_REAL) {
        e.out_r[o] = X.x * sc;
      } else {
        const R* p = e.p + static_cast<size_t>(b) * n * n;
        const R pv = p[static_cast<size_t>(t1) * n + t2];
        R ax = X.x * sc;
        if (lam != R(0)) ax += lam * ktk_at<R>(p, n, t1, t2, pv);
        ax += shift * pv;
        if (e.mode == PB_CG_STEP) {
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
    }
  }
  if (e.mode >= PB_CG_STEP) {
    double t0s, t1s;
    SliceScalars& sc = e.red.sc[b];
    double* part = e.red.part + static_cast<size_t>(b) * MAX_PART_BLOCKS * 2;
    if (reduce2_last(acc0, acc1, part, gridDim.x, blockIdx.x, &sc.counter[0], red_scratch, t0s, t1s) &&
        threadIdx.x == 0) {
      if (e.mode == PB_CG_STEP) {
        sc.pap = t0s;
        sc.pp = t1s;
      } else {
        sc.rr[0] = t0s;
        sc.bb = t1s;
        sc.done = 0;
        sc.steps_run = 0;
        sc.min_ritz = __longlong_as_double(0x7ff0000000000000LL);  // +inf
      }
    }
  }
}

// ---------------------------------------------------------------- standalone W^T (tests)
template <typename R>
__global__ void k_wt_grid(OpDev<R> d, int B, const cplx<R>* __restrict__ s, cplx<R>* __restrict__ grid) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= d.G32) return;
  const size_t G = static_cast<size_t>(d.m) * d.m;
  for (int b = 0; b < B; ++b)
    grid[G * b + static_cast<size_t>(gw) * 32 + lane] = wt_node<R>(d, s + static_cast<size_t>(b) * d.P, gw, lane);
}

// Radial density weights |k_r| (DC: 1/4), normal_ops.cpp:208-219, applied to samples.
template <typename R>
__global__ void k_weight_samples(cplx<R>* s, int B, int P, int nb) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(B) * P) return;
  const int j = static_cast<int>(i % P);
  const int kr = (j % nb) - nb / 2;
  const R w = kr == 0 ? R(0.25) : static_cast<R>(kr < 0 ? -kr : kr);
  s[i] = cscale(s[i], w);
}

template <int M, typename R>
__global__ void k_fft_rows_test(const cplx<R>* tw, const cplx<R>* in, cplx<R>* out, int rows, int inverse) {
  using S = FftShape<M>;
  using C2 = cplx<R>;
  extern __shared__ __align__(16) unsigned char smraw[];
  C2* sm = reinterpret_cast<C2*>(smraw);
  const int r = blockIdx.x;
  const int t = threadIdx.x;
  for (int i = t; i < M; i += S::T) {
    C2 v = in[static_cast<size_t>(r) * M + i];
    sm[pad16(i)] = inverse ? cconj(v) : v;
  }
  fft_row_smem<M, C2>(sm, tw, t, true);
  for (int i = t; i < M; i += S::T) {
    C2 v = sm[pad16(i)];
    out[static_cast<size_t>(r) * M + i] = inverse ? cconj(v) : v;
  }
}

// ---------------------------------------------------------------- dispatch helpers
// rows-per-CTA: enough threads per CTA, bounded smem, and at least ~2 waves of CTAs.
int choose_rpc(int m, int rows_per_slice, int B, size_t elem) {
  const int T = m / 16;
  int rpc = std::max(1, 256 / T);
  while (rpc > 1 && (rpc * T > 1024 || static_cast<size_t>(rpc) * padded_len(m) * elem > 100 * 1024)) rpc >>= 1;
  while (rpc > 1 && static_cast<int64_t>((rows_per_slice + rpc - 1) / rpc) * B < 2 * 148) rpc >>= 1;
  return rpc;
}

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
  dispatch_m(d.m, [&](auto MC) {
    constexpr int M = decltype(MC)::value;
    using S = FftShape<M>;
    const int rpc = choose_rpc(M, d.n, B, sizeof(cplx<R>));
    const size_t smem = static_cast<size_t>(rpc) * S::STRIDE * sizeof(cplx<R>);
    set_smem(k_t2_rows<M, R>, smem);
    dim3 grid((d.n + rpc - 1) / rpc, B);
    k_t2_rows<M, R><<<grid, rpc * S::T, smem, st>>>(d, in, in_complex ? 1 : 0, pu, rpc);
    note_launch();
  });
}

template <typename R>
void launch_t2_cols(const OpDev<R>& d, int B, const SliceScalars* skip, cudaStream_t st) {
  dispatch_m(d.m, [&](auto MC) {
    constexpr int M = decltype(MC)::value;
    using S = FftShape<M>;
    const int rpc = choose_rpc(M, M, B, sizeof(cplx<R>));
    const size_t smem = static_cast<size_t>(rpc) * S::STRIDE * sizeof(cplx<R>);
    set_smem(k_t2_cols<M, R>, smem);
    dim3 grid(M / rpc, B);
    k_t2_cols<M, R><<<grid, rpc * S::T, smem, st>>>(d, rpc, skip);
    note_launch();
  });
}

template <typename R>
void launch_w(const OpDev<R>& d, int B, const cplx<R>* grid, cplx<R>* samples, const SliceScalars* skip,
              cudaStream_t st) {
  const int threads = 256;
  const int blocks = (d.Ppad + threads - 1) / threads;
  if (B >= 4)
    k_w<4, R><<<blocks, threads, 0, st>>>(d, B, grid, samples, skip);
  else if (B >= 2)
    k_w<2, R><<<blocks, threads, 0, st>>>(d, B, grid, samples, skip);
  else
    k_w<1, R><<<blocks, threads, 0, st>>>(d, B, grid, samples, skip);
  note_launch();
}

template <typename R>
void launch_wt_rows(const OpDev<R>& d, int B, const SliceScalars* skip, cudaStream_t st) {
  dispatch_m(d.m, [&](auto MC) {
    constexpr int M = decltype(MC)::value;
    using S = FftShape<M>;
    const int rpc = choose_rpc(M, M, B, sizeof(cplx<R>));
    const size_t smem = static_cast<size_t>(rpc) * S::STRIDE * sizeof(cplx<R>);
    set_smem(k_wt_rows<M, R>, smem);
    dim3 grid(M / rpc, B);
    k_wt_rows<M, R><<<grid, std::max(32, rpc * S::T), smem, st>>>(d, rpc, skip);
    note_launch();
  });
}

template <typename R>
void launch_t1_rows(const OpDev<R>& d, int B, const PbEpi<R>& e, cudaStream_t st) {
  dispatch_m(d.m, [&](auto MC) {
    constexpr int M = decltype(MC)::value;
    using S = FftShape<M>;
    int rpc = choose_rpc(M, d.n, B, sizeof(cplx<R>));
    while (rpc > 1 && (d.n + rpc - 1) / rpc > MAX_PART_BLOCKS) rpc <<= 1;
    const size_t smem = static_cast<size_t>(rpc) * S::STRIDE * sizeof(cplx<R>);
    set_smem(k_t1_rows<M, R>, smem);
    dim3 grid((d.n + rpc - 1) / rpc, B);
    const int threads = std::max(32, rpc * S::T);
    k_t1_rows<M, R><<<grid, threads, smem, st>>>(d, e, rpc);
    note_launch();
  });
}

template <typename R>
void launch_wt_grid(const OpDev<R>& d, int B, const cplx<R>* samples, cplx<R>* grid, cudaStream_t st) {
  const int threads = 256;
  const int blocks = (d.G32 * 32 + threads - 1) / threads;
  k_wt_grid<R><<<blocks, threads, 0, st>>>(d, B, samples, grid);
  note_launch();
}

template <typename R>
void launch_weight_samples(cplx<R>* s, int B, int P, int nb, cudaStream_t st) {
  // angle blocks hold whole angles: t = j % nb is unchanged by a shard offset
  const int64_t total = static_cast<int64_t>(B) * P;
  k_weight_samples<R><<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(s, B, P, nb);
  note_launch();
}

template <typename R>
void launch_fft_rows_test(int m, int rows, const cplx<R>* tw, const cplx<R>* in, cplx<R>* out, bool inverse,
                          cudaStream_t st) {
  dispatch_m(m, [&](auto MC) {
    constexpr int M = decltype(MC)::value;
    using S = FftShape<M>;
    const size_t smem = S::STRIDE * sizeof(cplx<R>);
    set_smem(k_fft_rows_test<M, R>, smem);
    k_fft_rows_test<M, R><<<rows, S::T, smem, st>>>(tw, in, out, rows, inverse ? 1 : 0);
    note_launch();
  });
}

#define TOMO_INST_NUFFT(R)                                                                                   \
  template void launch_t2_rows<R>(const OpDev<R>&, int, const void*, bool, const PUpd<R>&, cudaStream_t);   \
  template void launch_t2_cols<R>(const OpDev<R>&, int, const SliceScalars*, cudaStream_t);                 \
  template void launch_w<R>(const OpDev<R>&, int, const cplx<R>*, cplx<R>*, const SliceScalars*, cudaStream_t); \
  template void launch_wt_rows<R>(const OpDev<R>&, int, const SliceScalars*, cudaStream_t);                 \
  template void launch_t1_rows<R>(const OpDev<R>&, int, const PbEpi<R>&, cudaStream_t);                     \
  template void launch_wt_grid<R>(const OpDev<R>&, int, const cplx<R>*, cplx<R>*, cudaStream_t);            \
  template void launch_weight_samples<R>(cplx<R>*, int, int, int, cudaStream_t);                            \
  template void launch_fft_rows_test<R>(int, int, const cplx<R>*, const cplx<R>*, cplx<R>*, bool, cudaStream_t);

TOMO_INST_NUFFT(float)
TOMO_INST_NUFFT(double)

}  // namespace tomo_b200
