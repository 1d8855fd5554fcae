// spmv.cu — the sparse interpolation of the normal-operator hot path on sm_100a:
//
//   W   (interpolate, proj/src/nufft.cpp:160-202): k_w_sep, the separable window SpMV
//   W^T (spread, nufft.cpp:119-158): k_task_spmv over the precomputed, count-sorted transpose
//       (also the fused backend's Gram W^T W and the Hermitian fold of W^T)
//   sample-vector kernels (radial weights, reference-order gathers, split-Bregman feedback)
//
// The FFT passes around them are in nufft.cu.
#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "kernels.h"

namespace tomo_b200 {

namespace {

int env_int(const char* name, int dflt) { return ab_int(name, dflt); }

template <typename T>
__device__ __forceinline__ T ldg(const T* p) {
  return __ldg(p);
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
// Streaming (evict-first) loads of the once-read W^T entry stream, so it does not evict the
// gathered slice samples from L2 (c5: 613 MB of entries vs 16 MB of samples).
__device__ __forceinline__ WtEnt<float> ldcs(const WtEnt<float>* p) {
  const int2 v = __ldcs(reinterpret_cast<const int2*>(p));
  return WtEnt<float>{v.x, __int_as_float(v.y)};
}
__device__ __forceinline__ WtEnt<double> ldcs(const WtEnt<double>* p) {
  const int4 v = __ldcs(reinterpret_cast<const int4*>(p));
  return WtEnt<double>{v.x, 0, __hiloint2double(v.w, v.z)};
}

// ---------------------------------------------------------------- W, separable storage
// Same matrix as k_w, stored as its rank-1 blocks: per row j the base node (ix0, iy0) and the
// two window factor vectors (SoA, coalesced): 4 + 2w*sizeof(R) bytes per row instead of
// w^2*(4 + sizeof(R)). The inner loop walks a grid row (b fixed, ix0+a consecutive).
// HERM: the grid holds rows iy in [0, m/2] of a Hermitian spectrum (real image); row iy > m/2 is
// read as the conjugate of row m - iy at mirrored columns.
template <int BT, int WMAX, int RU, typename R, bool BY = false, bool HERM = false>  // BY: slice groups across grid.y
__global__ void __launch_bounds__(256) k_w_sep(OpDev<R> d, int B, const cplx<R>* __restrict__ grid,
                                                cplx<R>* __restrict__ out, const SliceScalars* skip) {
  using C2 = cplx<R>;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;  // table position
  if (t >= d.P) return;
  const int j = d.w_perm && !d.w_out_pos ? __ldg(&d.w_perm[t]) : t;  // output index
  const int m = d.m, w = d.w;
  const int base = __ldg(&d.w_base[t]);
  const int ix0 = base & 0xffff, iy0 = base >> 16;
  R wx[WMAX];
  int ix[WMAX];
#pragma unroll
  for (int a = 0; a < WMAX; ++a) {
    if (a < w) {
      wx[a] = __ldg(&d.w_x[static_cast<size_t>(a) * d.Ppad + t]);
      const int u = ix0 + a;
      ix[a] = u >= m ? u - m : u;
    }
  }
  const size_t G = static_cast<size_t>(m) * m;
  for (int b0 = BY ? static_cast<int>(blockIdx.y) * BT : 0; b0 < B; b0 += (BY ? static_cast<int>(gridDim.y) : 1) * BT) {
    C2 acc[BT];
#pragma unroll
    for (int q = 0; q < BT; ++q) acc[q] = czero<C2>();
    // RU grid rows per step: RU*w gathers in flight per thread (registers vs. occupancy)
#pragma unroll 1
    for (int bb0 = 0; bb0 < w; bb0 += RU) {
#pragma unroll
      for (int k = 0; k < RU; ++k) {
        const int bb = bb0 + k;
        if (bb < w) {
          const R wyv = __ldg(&d.w_y[static_cast<size_t>(bb) * d.Ppad + t]);
          const int u0 = iy0 + bb;
          const int u = u0 >= m ? u0 - m : u0;
          const bool mir = HERM && u > (m >> 1);
          const size_t rowoff = static_cast<size_t>(mir ? m - u : u) * m;
#pragma unroll
          for (int q = 0; q < BT; ++q) {
            if (b0 + q < B) {
              const C2* row = grid + G * (b0 + q) + rowoff;
              C2 ra = czero<C2>();
#pragma unroll
              for (int a = 0; a < WMAX; ++a) {
                if (a < w) {
                  const C2 gv = row[mir ? ((m - ix[a]) & (m - 1)) : ix[a]];
                  ra.x += wx[a] * gv.x;
                  ra.y += wx[a] * gv.y;
                }
              }
              if (mir) ra.y = -ra.y;  // conj(sum w g) = sum w conj(g)
              acc[q].x += wyv * ra.x;
              acc[q].y += wyv * ra.y;
            }
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < BT; ++q)
      if (b0 + q < B && !(skip && (skip[b0 + q].done || skip[b0 + q].frozen)))
        out[static_cast<size_t>(b0 + q) * d.s_stride + j] = acc[q];
  }
}

// fp32, width-6 windows (c3, c4): the same separable product with each window row fetched as
// 16-byte vectors (3 or 4 float4 = the 6 nodes, two per vector) instead of 6 scalar 8-byte
// gathers: W is bound by L1 request / sector throughput (32 samples per warp request, one node each),
// and a vector carries two nodes of the same row. Rows that wrap around the grid edge take the
// scalar gathers. Same arithmetic, same order as k_w_sep (bit-identical).
template <int BT, bool BY, bool HERM>
__global__ void __launch_bounds__(256) k_w_sep_v6(OpDev<float> d, int B, const float2* __restrict__ grid,
                                                   float2* __restrict__ out, const SliceScalars* skip) {
  constexpr int W = 6;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;  // table position
  if (t >= d.P) return;
  const int j = d.w_perm && !d.w_out_pos ? __ldg(&d.w_perm[t]) : t;  // output index
  const int m = d.m;
  const int base = __ldg(&d.w_base[t]);
  const int ix0 = base & 0xffff, iy0 = base >> 16;
  float wx[W];
#pragma unroll
  for (int a = 0; a < W; ++a) wx[a] = __ldg(&d.w_x[static_cast<size_t>(a) * d.Ppad + t]);
  // contiguous (no wrap) node ranges: plain rows [ix0, ix0 + 5], mirrored rows [m - ix0 - 5, m - ix0]
  const bool plain_ok = ix0 + W <= m, mir_ok = ix0 >= 1 && ix0 <= m - W + 1;
  const size_t G = static_cast<size_t>(m) * m;
  for (int b0 = BY ? static_cast<int>(blockIdx.y) * BT : 0; b0 < B; b0 += (BY ? static_cast<int>(gridDim.y) : 1) * BT) {
    float2 acc[BT];
#pragma unroll
    for (int q = 0; q < BT; ++q) acc[q] = make_float2(0.f, 0.f);
#pragma unroll 1
    for (int bb = 0; bb < W; ++bb) {
      const float wyv = __ldg(&d.w_y[static_cast<size_t>(bb) * d.Ppad + t]);
      const int u0 = iy0 + bb;
      const int u = u0 >= m ? u0 - m : u0;
      const bool mir = HERM && u > (m >> 1);
      const size_t rowoff = static_cast<size_t>(mir ? m - u : u) * m;
      const int lo = mir ? m - ix0 - (W - 1) : ix0;
      const bool vec = mir ? mir_ok : plain_ok;
      const bool odd = lo & 1;
#pragma unroll
      for (int q = 0; q < BT; ++q) {
        if (b0 + q < B) {
          const float2* row = grid + G * (b0 + q) + rowoff;
          float2 ra = make_float2(0.f, 0.f);
          if (vec) {
            const float4* p4 = reinterpret_cast<const float4*>(row + (lo & ~1));
            const float4 v0 = __ldg(p4), v1 = __ldg(p4 + 1), v2 = __ldg(p4 + 2);
            const float4 v3 = odd ? __ldg(p4 + 3) : make_float4(0.f, 0.f, 0.f, 0.f);
            const float2 nd[8] = {make_float2(v0.x, v0.y), make_float2(v0.z, v0.w), make_float2(v1.x, v1.y),
                                  make_float2(v1.z, v1.w), make_float2(v2.x, v2.y), make_float2(v2.z, v2.w),
                                  make_float2(v3.x, v3.y), make_float2(v3.z, v3.w)};
#pragma unroll
            for (int a = 0; a < W; ++a) {
              // tap a is node a of the range (plain) or node W-1-a (mirrored), shifted by odd
              const float2 e = mir ? (odd ? nd[W - a] : nd[W - 1 - a]) : (odd ? nd[a + 1] : nd[a]);
              ra.x += wx[a] * e.x;
              ra.y += wx[a] * e.y;
            }
          } else {
#pragma unroll
            for (int a = 0; a < W; ++a) {
              const int v0 = ix0 + a;
              const int v = v0 >= m ? v0 - m : v0;
              const float2 gv = row[mir ? ((m - v) & (m - 1)) : v];
              ra.x += wx[a] * gv.x;
              ra.y += wx[a] * gv.y;
            }
          }
          if (mir) ra.y = -ra.y;  // conj(sum w g) = sum w conj(g)
          acc[q].x += wyv * ra.x;
          acc[q].y += wyv * ra.y;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < BT; ++q)
      if (b0 + q < B && !(skip && (skip[b0 + q].done || skip[b0 + q].frozen)))
        out[static_cast<size_t>(b0 + q) * d.s_stride + j] = acc[q];
  }
}

// Wide windows (w > 8, e.g. the digits12 preset's 25 taps): the same separable product with the
// factor vectors read in the loops (L1-resident per thread) instead of held in registers.
template <typename R>
__global__ void __launch_bounds__(256) k_w_sep_wide(OpDev<R> d, int B, const cplx<R>* __restrict__ grid,
                                                     cplx<R>* __restrict__ out, const SliceScalars* skip) {
  using C2 = cplx<R>;
  const int tp = blockIdx.x * blockDim.x + threadIdx.x;  // table position
  if (tp >= d.P) return;
  const int j = d.w_perm && !d.w_out_pos ? __ldg(&d.w_perm[tp]) : tp;  // output index
  const int m = d.m, w = d.w;
  const int base = __ldg(&d.w_base[tp]);
  const int ix0 = base & 0xffff, iy0 = base >> 16;
  const size_t G = static_cast<size_t>(m) * m;
  for (int b = 0; b < B; ++b) {
    if (skip && (skip[b].done || skip[b].frozen)) continue;
    const C2* gb = grid + G * b;
    C2 acc = czero<C2>();
    for (int bb = 0; bb < w; ++bb) {
      const int t0 = iy0 + bb;
      const int t = t0 >= m ? t0 - m : t0;
      const bool mir = d.herm_in && t > (m >> 1);
      const C2* row = gb + static_cast<size_t>(mir ? m - t : t) * m;
      C2 ra = czero<C2>();
      for (int a = 0; a < w; ++a) {
        const int u0 = ix0 + a;
        const int u = u0 >= m ? u0 - m : u0;
        const R wx = __ldg(&d.w_x[static_cast<size_t>(a) * d.Ppad + tp]);
        const C2 gv = row[mir ? ((m - u) & (m - 1)) : u];
        ra.x += wx * gv.x;
        ra.y += wx * gv.y;
      }
      if (mir) ra.y = -ra.y;
      const R wy = __ldg(&d.w_y[static_cast<size_t>(bb) * d.Ppad + tp]);
      acc.x += wy * ra.x;
      acc.y += wy * ra.y;
    }
    out[static_cast<size_t>(b) * d.s_stride + j] = acc;
  }
}

// ---------------------------------------------------------------- W^T / Gram: balanced task SpMV
// The same kernel applies W^T (input = slice samples, stride P) and, for the fused backend, the
// Gram operator W^T W (input = the grid, stride m^2; grid_in must not alias grid).
// One warp per task {block, chunk0, nchunks, slot}: lane l accumulates node (block, l) over
// the task's chunks (coalesced 32-entry chunks, 4 in flight), then writes either the grid node
// (iy*m + perm) or, for a split block, its partial slot.
// BY: slices across grid.y (batched launches with a small task grid); BY = false keeps the
// in-warp slice loop with fp32's 32 registers (the grid.y form needs 34: 6 instead of 8 CTAs
// per SM, c3 W^T 31.6 -> 34.6 us)
// HERM: the Hermitian fold of W^T (entry .j bit 31 = use conj(s_j)).
template <bool HERM, typename C2>
__device__ __forceinline__ C2 gather_s(const C2* __restrict__ s, int j) {
  if constexpr (HERM) {
    C2 v = __ldg(&s[j & 0x7fffffff]);
    if (j < 0) v.y = -v.y;
    return v;
  } else {
    return __ldg(&s[j]);
  }
}

template <int GRP, bool PIPE, typename R, bool BY = false, bool HERM = false>
__global__ void __launch_bounds__(256) k_task_spmv(TaskSpmv<R> ts, int m, int B, const cplx<R>* __restrict__ s_all,
                                                    size_t in_stride, cplx<R>* __restrict__ grid,
                                                    const SliceScalars* skip) {
  using C2 = cplx<R>;
  const int task = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (task >= ts.n_tasks) return;
  const int4 tk = __ldg(&ts.tasks[task]);
  const int blk = tk.x, c0 = tk.y, nc = tk.z, slot = tk.w;
  const int bpr = m / 32;  // blocks per grid row
  const int iy = blk / bpr;
  const int ix = __ldg(&ts.perm[static_cast<size_t>(blk) * 32 + lane]);
  const size_t G = static_cast<size_t>(m) * m;
  const WtEnt<R>* e = ts.ent + static_cast<size_t>(c0) * 32 + lane;
  for (int b = BY ? static_cast<int>(blockIdx.y) : 0; b < B; b += BY ? static_cast<int>(gridDim.y) : 1) {
    if (skip && (skip[b].done || skip[b].frozen)) continue;
    const C2* s = s_all + static_cast<size_t>(b) * in_stride;
    C2 a0 = czero<C2>(), a1 = czero<C2>();
    if constexpr (PIPE) {
    // software pipeline: the entries of group c+GRP are loaded while group c's gathers are in
    // flight, so a group costs max(entry stream, L2 gather) latency instead of their sum
    WtEnt<R> q[GRP];
#pragma unroll
    for (int k = 0; k < GRP; ++k) {
      if (k < nc) {
        q[k] = ldcs(e + k * 32);
      } else {
        q[k].j = 0;
        q[k].w = R(0);
      }
    }
    for (int c = 0; c < nc; c += GRP) {
      C2 v[GRP];
#pragma unroll
      for (int k = 0; k < GRP; ++k) v[k] = q[k].w != R(0) ? gather_s<HERM>(s, q[k].j) : czero<C2>();
      WtEnt<R> qn[GRP];
#pragma unroll
      for (int k = 0; k < GRP; ++k) {
        if (c + GRP + k < nc) {
          qn[k] = ldcs(e + (c + GRP + k) * 32);
        } else {
          qn[k].j = 0;
          qn[k].w = R(0);
        }
      }
#pragma unroll
      for (int k = 0; k < GRP; k += 2) {
        a0.x += q[k].w * v[k].x;
        a0.y += q[k].w * v[k].y;
        a1.x += q[k + 1].w * v[k + 1].x;
        a1.y += q[k + 1].w * v[k + 1].y;
      }
#pragma unroll
      for (int k = 0; k < GRP; ++k) q[k] = qn[k];
    }
    } else {
    // groups of GRP chunks with predicated tails (all loads of a group in flight at once)
    for (int c = 0; c < nc; c += GRP) {
      WtEnt<R> q[GRP];
      C2 v[GRP];
#pragma unroll
      for (int k = 0; k < GRP; ++k) {
        if (c + k < nc) {
          q[k] = ldcs(e + (c + k) * 32);
        } else {
          q[k].j = 0;
          q[k].w = R(0);
        }
      }
#pragma unroll
      for (int k = 0; k < GRP; ++k) v[k] = q[k].w != R(0) ? gather_s<HERM>(s, q[k].j) : czero<C2>();
#pragma unroll
      for (int k = 0; k < GRP; k += 2) {
        a0.x += q[k].w * v[k].x;
        a0.y += q[k].w * v[k].y;
        a1.x += q[k + 1].w * v[k + 1].x;
        a1.y += q[k + 1].w * v[k + 1].y;
      }
    }
    }
    const C2 v = cadd(a0, a1);
    if (slot < 0) {
      grid[G * b + static_cast<size_t>(iy) * m + ix] = v;
    } else {
      // split block: publish the partial; the warp that finishes the block's last task sums
      // all of its partials in slot order (deterministic) and writes the node values
      C2* part = ts.part + static_cast<size_t>(b) * ts.n_slots * 32;
      part[static_cast<size_t>(slot) * 32 + lane] = v;
      __threadfence();
      __syncwarp();  // every lane's partial is fenced before lane 0 takes the ticket
      const int h = __ldg(&ts.slot_heavy[slot]);
      unsigned* cnt = ts.heavy_cnt + static_cast<size_t>(b) * ts.n_heavy + h;
      unsigned ticket = 0;
      if (lane == 0) ticket = atomicAdd(cnt, 1u);
      ticket = __shfl_sync(0xffffffffu, ticket, 0);
      const int4 hv = __ldg(&ts.heavy[h]);
      if (ticket == static_cast<unsigned>(hv.z - 1)) {
        __threadfence();
        C2 acc = czero<C2>();
        for (int k = 0; k < hv.z; ++k) acc = cadd(acc, __ldcg(&part[static_cast<size_t>(hv.y + k) * 32 + lane]));
        grid[G * b + static_cast<size_t>(iy) * m + ix] = acc;
        if (lane == 0) *cnt = 0u;
      }
    }
  }
}

// Radial density weights |k_r| (DC: 1/4), normal_ops.cpp:208-219, applied to samples.
template <typename R>
__global__ void k_weight_samples(cplx<R>* s, int B, int P, int nb, const int* __restrict__ perm) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(B) * P) return;
  const int t = static_cast<int>(i % P);
  const int j = perm ? perm[t] : t;  // reference sample index
  const int kr = (j % nb) - nb / 2;
  const R w = kr == 0 ? R(0.25) : static_cast<R>(kr < 0 ? -kr : kr);
  s[i] = cscale(s[i], w);
}

template <typename R>
__global__ void k_gather_samples(const cplx<R>* __restrict__ in, cplx<R>* __restrict__ out, const int* __restrict__ perm,
                                 int B, int P) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(B) * P) return;
  const int64_t b = i / P, t = i - b * P;
  out[i] = in[b * P + (perm ? perm[t] : t)];
}

// split-Bregman data feedback (solver.cpp:283-286): fk += f - F_NU^* mu, and s = fk for the
// back-projection that follows
template <typename R>
__global__ void k_feedback_samples(int64_t n, cplx<R>* __restrict__ fk, const cplx<R>* __restrict__ f,
                                   cplx<R>* __restrict__ s) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const cplx<R> v = cadd(fk[i], csub(f[i], s[i]));
  fk[i] = v;
  s[i] = v;
}

// ---------------------------------------------------------------- W by mirror-pair units (overlap pairs)
// LN lanes per unit. The primary's window is taps [0, w) of the (w + 1)-wide union window, the
// partner's conjugate-mirrored window taps [1, w]; the two share the factors of taps [1, w): each
// grid row is read once, its common part summed once.
//   s_primary = sum_{b < w} fy[b] (sum_{a < w} fx[a] g[b][a])
//   t         = sum_{b >= 1} fy[b] (sum_{a >= 1} fx[a] g[b][a])      (= conj(s_partner))
// Outputs s[pos] = s_primary, s[ppos] = conj(t), s[P + pos] = s_primary + t (the pair sum the
// overlap-pair fold reads). HERM as in k_w_sep (this path is used on the half grid only).
template <int WMAX, int LN, typename R>
__global__ void __launch_bounds__(256) k_w_pair(OpDev<R> d, PairW<R> pw, int B, const cplx<R>* __restrict__ grid,
                                                 cplx<R>* __restrict__ out, const SliceScalars* skip) {
  using C2 = cplx<R>;
  // LN lanes per unit: lane h sums the union window's rows [h * nr, (h + 1) * nr), nr = ceil((w + 1) / LN)
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int u = tid / LN, h = tid % LN;
  if (u >= pw.Upad) return;  // Upad is a multiple of 32: both lanes of a unit stay (padding units: zero factors)
  const int m = d.m, w = d.w;  // union window: w + 1 <= WMAX taps
  const int nr = (w + LN) / LN;
  const int base = __ldg(&pw.base[u]);
  const int ix0 = base & 0xffff, iy0 = base >> 16;
  const int po = __ldg(&pw.pos[u]), pp = __ldg(&pw.ppos[u]);
  R fx[WMAX];
  int ix[WMAX];
#pragma unroll
  for (int a = 0; a < WMAX; ++a) {
    if (a <= w) {
      fx[a] = __ldg(&pw.fx[static_cast<size_t>(a) * pw.Upad + u]);
      const int v = ix0 + a;
      ix[a] = v >= m ? v - m : v;
    }
  }
  const size_t G = static_cast<size_t>(m) * m;
  for (int b = static_cast<int>(blockIdx.y); b < B; b += static_cast<int>(gridDim.y)) {
    if (skip && (skip[b].done || skip[b].frozen)) continue;
    C2 s = czero<C2>(), t = czero<C2>();
#pragma unroll 1
    for (int bb = h * nr; bb < min((h + 1) * nr, w + 1); ++bb) {
      const R fyv = __ldg(&pw.fy[static_cast<size_t>(bb) * pw.Upad + u]);
      const int v0 = iy0 + bb;
      const int v = v0 >= m ? v0 - m : v0;
      const bool mir = v > (m >> 1);
      const C2* row = grid + G * b + static_cast<size_t>(mir ? m - v : v) * m;
      C2 g0 = czero<C2>(), gw = czero<C2>(), mid = czero<C2>();
#pragma unroll
      for (int a = 0; a < WMAX; ++a) {
        if (a <= w) {
          const C2 gv = row[mir ? ((m - ix[a]) & (m - 1)) : ix[a]];
          if (a == 0) {
            g0 = mk<C2>(fx[0] * gv.x, fx[0] * gv.y);
          } else if (a == w) {
            gw = mk<C2>(fx[a] * gv.x, fx[a] * gv.y);
          } else {
            mid.x += fx[a] * gv.x;
            mid.y += fx[a] * gv.y;
          }
        }
      }
      if (mir) {  // conj(sum f g) = sum f conj(g)
        g0.y = -g0.y;
        gw.y = -gw.y;
        mid.y = -mid.y;
      }
      if (bb < w) {
        s.x += fyv * (g0.x + mid.x);
        s.y += fyv * (g0.y + mid.y);
      }
      if (bb >= 1) {
        t.x += fyv * (mid.x + gw.x);
        t.y += fyv * (mid.y + gw.y);
      }
    }
#pragma unroll
    for (int o = 1; o < LN; o <<= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
      t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
      t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
    }
    if (po < 0) continue;  // padding unit
    C2* sb = out + static_cast<size_t>(b) * d.s_stride;
    if (h == 0) {
      sb[po] = s;
    } else if (h == 1 && pp >= 0) {
      sb[pp] = mk<C2>(t.x, -t.y);
      sb[d.P + po] = mk<C2>(s.x + t.x, s.y + t.y);
    }
  }
}

}  // namespace

// Batched calls (B slices per launch) of the small-grid SpMVs: slice groups go to grid.y
// until the launch has about 8 CTAs of 256 threads per SM, instead of each thread / warp
// looping over all B slices (c1: 86-CTA W and ~110-CTA W^T grids with B = 7 per lane).
// TOMO_BATCH_Y=0 restores the in-thread loop (A/B runs).
unsigned batch_ydim(int blocks, int groups) {
  static const int env_on = env_int("TOMO_BATCH_Y", 1);
  if (!env_on || groups <= 1) return 1u;
  const int target = 148 * 8;
  return static_cast<unsigned>(std::max(1, std::min(groups, (target + blocks - 1) / std::max(blocks, 1))));
}

template <typename R>
void launch_w(const OpDev<R>& d, int B, const cplx<R>* grid, cplx<R>* samples, const SliceScalars* skip,
              cudaStream_t st) {
  static const int env_thr = env_int("TOMO_W_THREADS", 256);
  const int threads = env_thr == 64 || env_thr == 128 ? env_thr : 256;
  const int blocks = (d.Ppad + threads - 1) / threads;
  {
    // compile-time window bound: registers scale with it (6/7 are the configs' windows)
    // one grid row (w gathers) per step: rows-in-flight 1, 2, 3 and w measured equal on B200
    // (c2 8.8-9.2 us, c3 16-19 us); 1 needs the fewest registers
    auto go2 = [&](auto WC, auto HC) {
      constexpr int WM = decltype(WC)::value;
      constexpr bool HM = decltype(HC)::value;
      const unsigned ydim = batch_ydim(blocks, (B + 1) / 2);
      if (B >= 2 && ydim > 1)
        CK_LAUNCH(launch_k(k_w_sep<2, WM, 1, R, true, HM>, dim3(blocks, ydim), threads, 0, st, d, B, grid, samples,
                           skip));
      else if (B >= 2)
        CK_LAUNCH(launch_k(k_w_sep<2, WM, 1, R, false, HM>, blocks, threads, 0, st, d, B, grid, samples, skip));
      else
        CK_LAUNCH(launch_k(k_w_sep<1, WM, 1, R, false, HM>, blocks, threads, 0, st, d, B, grid, samples, skip));
    };
    auto go = [&](auto WC) {
      if (d.herm_in)
        go2(WC, std::true_type{});
      else
        go2(WC, std::false_type{});
    };
    static const int vec_on = env_int("TOMO_W_VEC", 1);  // A/B: 0 = scalar gathers
    if constexpr (sizeof(R) == 4) {
      if (vec_on && d.w == 6) {
        auto gov = [&](auto HC) {
          constexpr bool HM = decltype(HC)::value;
          const unsigned ydim = batch_ydim(blocks, (B + 1) / 2);
          if (B >= 2 && ydim > 1)
            CK_LAUNCH(launch_k(k_w_sep_v6<2, true, HM>, dim3(blocks, ydim), threads, 0, st, d, B, grid, samples, skip));
          else if (B >= 2)
            CK_LAUNCH(launch_k(k_w_sep_v6<2, false, HM>, blocks, threads, 0, st, d, B, grid, samples, skip));
          else
            CK_LAUNCH(launch_k(k_w_sep_v6<1, false, HM>, blocks, threads, 0, st, d, B, grid, samples, skip));
        };
        if (d.herm_in) gov(std::true_type{});
        else gov(std::false_type{});
        note_launch();
        return;
      }
    }
    if (d.w <= 6)
      go(std::integral_constant<int, 6>{});
    else if (d.w <= 8)
      go(std::integral_constant<int, 8>{});
    else
      CK_LAUNCH(launch_k(k_w_sep_wide<R>, blocks, threads, 0, st, d, B, grid, samples, skip));
  }
  note_launch();
}

template <typename R>
void launch_task_spmv(const TaskSpmv<R>& ts, int m, int B, const cplx<R>* x, size_t in_stride, cplx<R>* grid,
                      const SliceScalars* skip, cudaStream_t st, bool herm = false) {
  if (ts.n_tasks <= 0) return;
  // CTA size (a warp per task either way), measured: c2 35.0 / 34.7 / 34.6 slices/s and c1 81k / 81k /
  // 76k applies/s at 256 / 128 / 64 threads; c5 (m = 8192, row-ordered tasks) 959 / 965 / 967 applies/s
  // (W^T 177 -> 170 us); c3 equal. TOMO_WT_THREADS overrides (A/B).
  static const int env_wt_thr = env_int("TOMO_WT_THREADS", 0);
  const int threads = env_wt_thr == 64 || env_wt_thr == 128 || env_wt_thr == 256 ? env_wt_thr : (m >= 4096 ? 64 : 256);
  const int blocks = (ts.n_tasks * 32 + threads - 1) / threads;
  // group depth and software pipelining measured on B200 (c2/c3/c5): fp32 6 chunks, not
  // pipelined (32 registers, full occupancy); fp64 4 chunks, pipelined for m <= 2048 (c2 W^T
  // 16.8 -> 14.8 us; c5's m = 8192 W^T got slower, 342 -> 375 us). TOMO_WT_GRP (2/4/6/8) /
  // TOMO_WT_PIPE override for A/B runs.
  static const int env_grp = env_int("TOMO_WT_GRP", 0), env_pipe = env_int("TOMO_WT_PIPE", -1);
  const bool pipe = env_pipe >= 0 ? env_pipe != 0 : (sizeof(R) == 8 && m <= 2048);
  const int grp = env_grp > 0 ? env_grp : (sizeof(R) == 4 ? 6 : 4);
  const unsigned ydim = batch_ydim(blocks, B);
  auto go = [&](auto kern, auto kern_by) {
    if (ydim > 1)
      CK_LAUNCH(launch_k(kern_by, dim3(blocks, ydim), threads, 0, st, ts, m, B, x, in_stride, grid, skip));
    else
      CK_LAUNCH(launch_k(kern, blocks, threads, 0, st, ts, m, B, x, in_stride, grid, skip));
  };
  // group depth x pipelining x Hermitian fold, all compiled; the defaults above, others by A/B knobs
  auto go_h = [&](auto GC, auto PC, auto HC) {
    constexpr int G = decltype(GC)::value;
    constexpr bool P = decltype(PC)::value, H = decltype(HC)::value;
    go(k_task_spmv<G, P, R, false, H>, k_task_spmv<G, P, R, true, H>);
  };
  auto go_p = [&](auto GC, auto HC) {
    if (pipe) go_h(GC, std::true_type{}, HC);
    else go_h(GC, std::false_type{}, HC);
  };
  auto go_g = [&](auto HC) {
    if (grp == 2) go_p(std::integral_constant<int, 2>{}, HC);
    else if (grp == 4) go_p(std::integral_constant<int, 4>{}, HC);
    else if (grp == 8) go_p(std::integral_constant<int, 8>{}, HC);
    else go_p(std::integral_constant<int, 6>{}, HC);
  };
  if (herm) go_g(std::true_type{});
  else go_g(std::false_type{});
  note_launch();
}

template <typename R>
void launch_wt_spread(const OpDev<R>& d, int B, const cplx<R>* samples, cplx<R>* grid, const SliceScalars* skip,
                      cudaStream_t st) {
  if (d.herm_out)
    launch_task_spmv<R>(d.wth, d.m, B, samples, static_cast<size_t>(d.s_stride), grid, skip, st, true);
  else
    launch_task_spmv<R>(d.wt_view(), d.m, B, samples, static_cast<size_t>(d.s_stride), grid, skip, st);
}

template <typename R>
void launch_w_pair(const OpDev<R>& d, const PairW<R>& pw, int B, const cplx<R>* grid, cplx<R>* samples,
                   const SliceScalars* skip, cudaStream_t st) {
  // measured at c2 (slices/s): 1 lane per unit 30.2, 2 lanes 33.9, 4 lanes in 128-thread CTAs 35.2
  // (64 threads 34.8, 256 threads 33.5), 8 lanes 33.1; the pair-sum pass behind the plain W 33.5
  constexpr int kLanes = 4, kThreads = 128;
  const int blocks = (kLanes * pw.Upad + kThreads - 1) / kThreads;
  const unsigned ydim = batch_ydim(blocks, B);
  CK_LAUNCH(launch_k(k_w_pair<8, kLanes, R>, dim3(blocks, ydim), kThreads, 0, st, d, pw, B, grid, samples, skip));
  note_launch();
}

// Overlap pairs: the pair sums s_j + conj(s_partner) behind the samples of each slice.
template <typename R>
__global__ void k_pair_sigma(cplx<R>* __restrict__ s, int B, int P, int stride, const int* __restrict__ ppos) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P) return;
  const int q = __ldg(&ppos[t]);
  if (q < 0) return;
  for (int b = 0; b < B; ++b) {
    cplx<R>* sb = s + static_cast<size_t>(b) * stride;
    const cplx<R> a = sb[t], c = sb[q];
    sb[P + t] = mk<cplx<R>>(a.x + c.x, a.y - c.y);
  }
}

template <typename R>
void launch_pair_sigma(cplx<R>* s, int B, int P, int stride, const int* ppos, cudaStream_t st) {
  CK_LAUNCH(launch_k(k_pair_sigma<R>, static_cast<unsigned>((P + 255) / 256), 256, 0, st, s, B, P, stride, ppos));
  note_launch();
}

template <typename R>
void launch_gram(const OpDev<R>& d, int B, const cplx<R>* grid_in, cplx<R>* grid_out, const SliceScalars* skip,
                 cudaStream_t st) {
  launch_task_spmv<R>(d.gram, d.m, B, grid_in, static_cast<size_t>(d.m) * d.m, grid_out, skip, st);
}

template <typename R>
void launch_wt_grid(const OpDev<R>& d, int B, const cplx<R>* samples, cplx<R>* grid, cudaStream_t st) {
  cudaMemsetAsync(grid, 0, sizeof(cplx<R>) * static_cast<size_t>(B) * d.m * d.m, st);
  launch_wt_spread<R>(d, B, samples, grid, nullptr, st);
}

template <typename R>
void launch_weight_samples(cplx<R>* s, int B, int P, int nb, const int* perm, cudaStream_t st) {
  // angle blocks hold whole angles: t = j % nb is unchanged by a shard offset
  const int64_t total = static_cast<int64_t>(B) * P;
  CK_LAUNCH(launch_k(k_weight_samples<R>, static_cast<unsigned>((total + 255) / 256), 256, 0, st, s, B, P, nb, perm));
  note_launch();
}

template <typename R>
void launch_feedback_samples(int64_t n, cplx<R>* fk, const cplx<R>* f, cplx<R>* s, cudaStream_t st) {
  CK_LAUNCH(launch_k(k_feedback_samples<R>, static_cast<unsigned>((n + 255) / 256), 256, 0, st, n, fk, f, s));
  note_launch();
}

template <typename R>
void launch_gather_samples(const cplx<R>* in, cplx<R>* out, const int* perm, int B, int P, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(B) * P;
  CK_LAUNCH(launch_k(k_gather_samples<R>, static_cast<unsigned>((total + 255) / 256), 256, 0, st, in, out, perm, B, P));
  note_launch();
}


#define TOMO_INST_SPMV(R)                                                                                    \
  template void launch_w<R>(const OpDev<R>&, int, const cplx<R>*, cplx<R>*, const SliceScalars*, cudaStream_t); \
  template void launch_wt_spread<R>(const OpDev<R>&, int, const cplx<R>*, cplx<R>*, const SliceScalars*,    \
                                    cudaStream_t);                                                          \
  template void launch_gram<R>(const OpDev<R>&, int, const cplx<R>*, cplx<R>*, const SliceScalars*, cudaStream_t); \
  template void launch_pair_sigma<R>(cplx<R>*, int, int, int, const int*, cudaStream_t);                         \
  template void launch_w_pair<R>(const OpDev<R>&, const PairW<R>&, int, const cplx<R>*, cplx<R>*, const SliceScalars*, \
                                 cudaStream_t);                                                                  \
  template void launch_wt_grid<R>(const OpDev<R>&, int, const cplx<R>*, cplx<R>*, cudaStream_t);            \
  template void launch_weight_samples<R>(cplx<R>*, int, int, int, const int*, cudaStream_t);               \
  template void launch_gather_samples<R>(const cplx<R>*, cplx<R>*, const int*, int, int, cudaStream_t);     \
  template void launch_feedback_samples<R>(int64_t, cplx<R>*, const cplx<R>*, cplx<R>*, cudaStream_t);

TOMO_INST_SPMV(float)
TOMO_INST_SPMV(double)

}  // namespace tomo_b200
