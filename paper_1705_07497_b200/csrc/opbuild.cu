// opbuild.cu — operator construction on the GPU: plan_spreading
// (proj/src/nufft.cpp:71-101, weights :56-69) and the W / W^T tables of tomo_capi.cu's host
// build_tables, produced on the device so that setup no longer dominates at large sizes.
//
//   k_plan        one thread per slice sample: nearest grid index, e1/e2 recurrence (fp64, the
//                 host formula with the products rounded exactly as on the host), the separable
//                 W storage (base node + factor vectors) and the (node, sample) pairs of W^T
//   radix sorts   (node, sample) pairs -> W^T rows in ascending sample order (= the host fill);
//                 nodes of every grid row by (count desc, ix) (= the host stable_sort)
//   k_blocks ...  32-node blocks, chunk offsets, warp tasks (split above kWtMaxChunks), the
//                 stable longest-first task order, and the chunk-major entry stream
//
// The result is the same table layout (and, up to 1-ulp differences of exp(), the same values)
// as the host build; tests/test_gpu_build.py compares the two.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <vector>
#include <string>

#include "common.cuh"
#include "kernels.h"

namespace tomo_b200 {

namespace {

#define BK(x)                                                                   \
  do {                                                                          \
    const cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string("opbuild: ") + cudaGetErrorString(e_)); \
  } while (0)

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  void alloc(size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    BK(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)));
  }
};

__device__ __forceinline__ int wrapd(int i, int m) { return i < 0 ? i + m : (i >= m ? i - m : i); }

__device__ __forceinline__ double reduce_2pi(double v) {
  const double two_pi = 2.0 * M_PI;
  double r = fmod(v, two_pi);
  if (r < 0.0) r += two_pi;
  if (r >= two_pi) r = 0.0;
  return r;
}

// plan + separable W + W^T pairs; j in [0, Ppad)
template <typename R>
__global__ void k_plan(BuildArgs a, const double* __restrict__ cs, const double* __restrict__ e3, int* base,
                       R* wxr, R* wyr, unsigned long long* keys, R* vals, int* cnt) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= a.Ppad) return;
  const int w = a.w;
  if (j >= a.P) {
    base[j] = 0;
    for (int q = 0; q < w; ++q) {
      wxr[static_cast<size_t>(q) * a.Ppad + j] = R(0);
      wyr[static_cast<size_t>(q) * a.Ppad + j] = R(0);
    }
    return;
  }
  const int al = static_cast<int>(j / a.nb), t = static_cast<int>(j % a.nb);
  const double c = cs[2 * al], s = cs[2 * al + 1];
  const double big_m = a.m / 2.0, h = M_PI / big_m;
  const double k_r = (2.0 * M_PI / a.nb) * (t - a.nb / 2);
  const double xy[2] = {reduce_2pi(__dmul_rn(k_r, c)), reduce_2pi(__dmul_rn(k_r, s))};
  const int reach = max(a.hi, -a.lo);
  double wd[2][64];
  int i0[2];
  for (int dd = 0; dd < 2; ++dd) {
    int mj = static_cast<int>(floor(xy[dd] / h));
    if (mj >= a.m) mj = a.m - 1;
    const double xi = __dsub_rn(xy[dd], __dmul_rn(h, static_cast<double>(mj)));  // no FMA contraction
    const double f1 = exp(-__dmul_rn(xi, xi) / (4.0 * a.tau));
    const double f2 = exp(__dmul_rn(xi, M_PI) / (big_m * 2.0 * a.tau));
    const double f2inv = 1.0 / f2;
    double* wv = wd[dd];
    wv[-a.lo] = f1;
    double p = f1, q = f1;
    for (int l = 1; l <= reach; ++l) {
      p = __dmul_rn(p, f2);
      q = __dmul_rn(q, f2inv);
      if (l <= a.hi) wv[l - a.lo] = __dmul_rn(p, e3[l - a.lo]);
      if (-l >= a.lo) wv[-l - a.lo] = __dmul_rn(q, e3[-l - a.lo]);
    }
    i0[dd] = wrapd(mj + a.lo, a.m);
  }
  base[j] = i0[0] | (i0[1] << 16);
  for (int q = 0; q < w; ++q) {
    wxr[static_cast<size_t>(q) * a.Ppad + j] = static_cast<R>(wd[0][q]);
    wyr[static_cast<size_t>(q) * a.Ppad + j] = static_cast<R>(wd[1][q]);
  }
  // W^T pairs: entry (a, b) of row j -> node ((iy0+b) mod m, (ix0+a) mod m), value wx[a]wy[b]
  const size_t e0 = static_cast<size_t>(j) * w * w;
  for (int qa = 0; qa < w; ++qa) {
    const int ix = wrapd(i0[0] + qa, a.m);
    for (int qb = 0; qb < w; ++qb) {
      const int iy = wrapd(i0[1] + qb, a.m);
      const int node = iy * a.m + ix;
      keys[e0 + qa * w + qb] = (static_cast<unsigned long long>(node) << 32) | static_cast<unsigned long long>(j);
      vals[e0 + qa * w + qb] = static_cast<R>(__dmul_rn(wd[0][qa], wd[1][qb]));
      atomicAdd(&cnt[node], 1);
    }
  }
}

// per node: key (iy, count descending, ix) for the per-row stable order; touched-node count
__global__ void k_node_keys(int m, int64_t G, int maxc, const int* __restrict__ cnt, unsigned long long* keys,
                            unsigned long long* touched) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= G) return;
  const int iy = static_cast<int>(i / m), ix = static_cast<int>(i % m);
  const int c = cnt[i];
  keys[i] = (static_cast<unsigned long long>(iy) << 32) | (static_cast<unsigned long long>(maxc - c) << 16) |
            static_cast<unsigned long long>(ix);
  if (c > 0) atomicAdd(touched, 1ull);
}

// per 32-node block: perm, chunk count L, task / slot / heavy counts
__global__ void k_blocks(int m, int64_t G32, int maxch, const unsigned long long* __restrict__ sorted,
                         const int* __restrict__ cnt, uint16_t* perm, int* L, int* ntask, int* nslot, int* nheavy) {
  const int64_t bk = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (bk >= G32) return;
  const int ix = static_cast<int>(sorted[bk * 32 + lane] & 0xFFFFull);
  perm[bk * 32 + lane] = static_cast<uint16_t>(ix);
  if (lane == 0) {
    const int iy = static_cast<int>((bk * 32) / m);
    const int l = cnt[static_cast<int64_t>(iy) * m + ix];
    L[bk] = l;
    const int nt = l == 0 ? 0 : (l <= maxch ? 1 : (l + maxch - 1) / maxch);
    ntask[bk] = nt;
    nslot[bk] = l > maxch ? nt : 0;
    nheavy[bk] = l > maxch ? 1 : 0;
  }
}

__global__ void k_tasks(int64_t G32, int maxch, const int* __restrict__ L, const int64_t* __restrict__ chunk0,
                        const int* __restrict__ toff, const int* __restrict__ soff, const int* __restrict__ hoff,
                        int4* tasks, int* tkey, int4* heavy, int* slot_heavy) {
  const int64_t bk = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (bk >= G32) return;
  const int l = L[bk];
  if (!l) return;
  const int c0 = static_cast<int>(chunk0[bk]);
  if (l <= maxch) {
    tasks[toff[bk]] = make_int4(static_cast<int>(bk), c0, l, -1);
    tkey[toff[bk]] = maxch - l;
    return;
  }
  const int ns = (l + maxch - 1) / maxch, s0 = soff[bk], h = hoff[bk];
  heavy[h] = make_int4(static_cast<int>(bk), s0, ns, 0);
  for (int k = 0; k < ns; ++k) {
    const int nc = min(maxch, l - k * maxch);
    tasks[toff[bk] + k] = make_int4(static_cast<int>(bk), c0 + k * maxch, nc, s0 + k);
    tkey[toff[bk] + k] = maxch - nc;
    slot_heavy[s0 + k] = h;
  }
}

template <typename R>
__global__ void k_gather_tasks(int n, const int* __restrict__ idx, const int4* __restrict__ in, int4* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[idx[i]];
}

// chunk-major entries: block bk, lane l, chunk k < L; padding re-reads the last sample
template <typename R>
__global__ void k_entries(int m, int64_t G32, const uint16_t* __restrict__ perm, const int* __restrict__ L,
                          const int64_t* __restrict__ chunk0, const int* __restrict__ cnt, const int* __restrict__ off,
                          const int* __restrict__ sj, const R* __restrict__ svals, WtEnt<R>* ent) {
  const int64_t bk = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (bk >= G32) return;
  const int l = L[bk];
  if (!l) return;
  const int64_t row = (bk * 32) / m * m;
  const int64_t node = row + perm[bk * 32 + lane];
  const int64_t first = row + perm[bk * 32];
  const int c = cnt[node];
  const int o = off[node];
  int lastj = c > 0 ? sj[o] : sj[off[first]];
  for (int k = 0; k < l; ++k) {
    WtEnt<R> e{};
    if (k < c) {
      lastj = sj[o + k];
      e.j = lastj;
      e.w = svals[o + k];
    } else {
      e.j = lastj;
      e.w = R(0);
    }
    ent[(static_cast<size_t>(chunk0[bk]) + k) * 32 + lane] = e;
  }
}

}  // namespace

// Warp-task order of W^T. Longest tasks first balances small grids (c2/c3: 24.9 vs 23.4
// slices/s, 30 vs 40 us); for large grids (m >= 4096) grid-row order keeps the samples that
// concurrently running tasks gather in cache (c5: 440 -> 346 us). TOMO_TASK_ORDER=rows|len.
bool wt_row_order(int m) {
  const std::string ord = ab_knob("TOMO_TASK_ORDER");
  if (ord == "rows") return true;
  if (ord == "len" || ord == "band") return false;
  return m >= 4096;
}

int wt_task_band(int m);

// Rows per task band (0: no bands) — see gpu_build_finish. Measured (B200, same box): bands of 32
// rows, heaviest band first, c2 W^T 17.9 -> 15.8 us (31.1 -> 32.4 slices/s), c3 30.2 -> 26.7 us
// (12.27k -> 12.63k applies/s); c1 (m = 512, batched lanes) 71.1k -> 69.6k and c5 (m = 8192, row
// order) unchanged, so bands are the default for 1024 <= m <= 2048 only. TOMO_TASK_ORDER=band|rows|len
// and TOMO_TASK_BAND=<rows> override (A/B runs).
int wt_task_band(int m) {
  const std::string ord = ab_knob("TOMO_TASK_ORDER");
  if (ord == "rows" || ord == "len") return 0;
  if (ord == "band") return std::max(1, ab_int("TOMO_TASK_BAND", 32));
  return m >= 1024 && m <= 2048 ? 32 : 0;
}

namespace {

int bits_for(uint64_t v) {
  int b = 1;
  while ((uint64_t(1) << b) <= v && b < 64) ++b;
  return b;
}

}  // namespace

__global__ void k_low32(int64_t n, const unsigned long long* __restrict__ keys, int* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = static_cast<int>(keys[i] & 0xFFFFFFFFull);
}

struct GpuBuild {
  BuildArgs a{};
  int rows = 0;  // grid rows of the node set: m, or m/2 + 1 for the Hermitian fold
  int64_t nnz = 0, G = 0, G32 = 0;
  DBuf<int> sj;  // entry columns (sample / grid node) in final entry order
  DBuf<int> cnt, off, L, ntask, nslot, nheavy, toff, soff, hoff, tkey, tkey2, tidx, tidx2;
  DBuf<int64_t> chunk0;
  DBuf<int4> tasks_raw;
  DBuf<unsigned char> vals_sorted;  // R values, type-erased
  DBuf<uint16_t> perm;
  GpuBuildSizes sz{};
};

void build_structure(GpuBuild* b, cudaStream_t st);

template <typename R>
GpuBuild* gpu_build_begin(const BuildArgs& a, const double* h_cs, const double* h_e3, int* base, R* wx, R* wy,
                          cudaStream_t st, GpuBuildSizes* sizes) {
  auto b = std::make_unique<GpuBuild>();
  b->a = a;
  const int m = a.m, w = a.w;
  b->nnz = a.P * w * w;
  b->G = static_cast<int64_t>(m) * m;
  b->G32 = b->G / 32;
  if (b->nnz >= (int64_t(1) << 31)) throw std::runtime_error("opbuild: W^T too large for 32-bit offsets");
  const int n_ang = static_cast<int>(a.P / a.nb);
  DBuf<double> cs(2 * static_cast<size_t>(n_ang)), e3(w);
  BK(cudaMemcpyAsync(cs.p, h_cs, sizeof(double) * 2 * n_ang, cudaMemcpyHostToDevice, st));
  BK(cudaMemcpyAsync(e3.p, h_e3, sizeof(double) * w, cudaMemcpyHostToDevice, st));
  DBuf<unsigned long long> keys(b->nnz), skeys(b->nnz);
  DBuf<R> vals(b->nnz);
  b->vals_sorted.alloc(sizeof(R) * b->nnz);
  b->cnt.alloc(b->G);
  BK(cudaMemsetAsync(b->cnt.p, 0, sizeof(int) * b->G, st));
  k_plan<R><<<static_cast<unsigned>((a.Ppad + 127) / 128), 128, 0, st>>>(a, cs.p, e3.p, base, wx, wy, keys.p, vals.p,
                                                                        b->cnt.p);
  BK(cudaGetLastError());
  // W^T rows: sort the (node, sample) pairs; ascending sample order within a node = the host fill
  const int key_bits = 32 + bits_for(static_cast<uint64_t>(b->G));
  size_t tmp_bytes = 0;
  BK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, skeys.p, vals.p,
                                     reinterpret_cast<R*>(b->vals_sorted.p), static_cast<int>(b->nnz), 0, key_bits,
                                     st));
  {
    DBuf<unsigned char> tmp(tmp_bytes);
    BK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, skeys.p, vals.p,
                                       reinterpret_cast<R*>(b->vals_sorted.p), static_cast<int>(b->nnz), 0, key_bits,
                                       st));
  }
  b->sj.alloc(b->nnz);
  k_low32<<<static_cast<unsigned>((b->nnz + 255) / 256), 256, 0, st>>>(b->nnz, skeys.p, b->sj.p);
  BK(cudaGetLastError());
  build_structure(b.get(), st);
  *sizes = b->sz;
  return b.release();
}

// Task structure from entries already in final order (b->sj, b->vals_sorted) and the per-node
// counts b->cnt: node offsets, per-row node order, 32-node blocks, warp tasks, totals.
int wt_max_chunks() {
  static const int v = std::min(std::max(ab_int("TOMO_WT_MAXCH", kWtMaxChunks), 1), 1024);
  return v;
}

void build_structure(GpuBuild* b, cudaStream_t st) {
  const int m = b->a.m;
  size_t tmp_bytes = 0;
  DBuf<unsigned char> tmp;
  b->off.alloc(b->G);
  tmp_bytes = 0;
  BK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, b->cnt.p, b->off.p, static_cast<int>(b->G), st));
  tmp.alloc(tmp_bytes);
  BK(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, b->cnt.p, b->off.p, static_cast<int>(b->G), st));
  // per-row node order: (count desc, ix asc) = the host's stable_sort by count
  const int maxc = 65535;
  DBuf<unsigned long long> nkeys(b->G), nsorted(b->G), touched(1);
  BK(cudaMemsetAsync(touched.p, 0, sizeof(unsigned long long), st));
  k_node_keys<<<static_cast<unsigned>((b->G + 255) / 256), 256, 0, st>>>(m, b->G, maxc, b->cnt.p, nkeys.p, touched.p);
  BK(cudaGetLastError());
  tmp_bytes = 0;
  const int nbits = 32 + bits_for(static_cast<uint64_t>(m));
  BK(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, nkeys.p, nsorted.p, static_cast<int>(b->G), 0, nbits, st));
  tmp.alloc(tmp_bytes);
  BK(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, nkeys.p, nsorted.p, static_cast<int>(b->G), 0, nbits, st));
  // blocks
  b->perm.alloc(b->G);
  b->L.alloc(b->G32);
  b->ntask.alloc(b->G32);
  b->nslot.alloc(b->G32);
  b->nheavy.alloc(b->G32);
  k_blocks<<<static_cast<unsigned>((b->G32 + 7) / 8), 256, 0, st>>>(m, b->G32, wt_max_chunks(), nsorted.p, b->cnt.p, b->perm.p,
                                                                   b->L.p, b->ntask.p, b->nslot.p, b->nheavy.p);
  BK(cudaGetLastError());
  b->chunk0.alloc(b->G32 + 1);
  b->toff.alloc(b->G32 + 1);
  b->soff.alloc(b->G32 + 1);
  b->hoff.alloc(b->G32 + 1);
  auto scan = [&](const int* in, auto* out) {
    size_t tb = 0;
    BK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, static_cast<int>(b->G32), st));
    DBuf<unsigned char> t2(tb);
    BK(cub::DeviceScan::ExclusiveSum(t2.p, tb, in, out, static_cast<int>(b->G32), st));
  };
  scan(b->L.p, b->chunk0.p);
  scan(b->ntask.p, b->toff.p);
  scan(b->nslot.p, b->soff.p);
  scan(b->nheavy.p, b->hoff.p);
  // totals = last exclusive sum + last count
  int64_t c_last = 0;
  int l_last = 0, t_last = 0, nt_last = 0, s_last = 0, ns_last = 0, h_last = 0, nh_last = 0;
  unsigned long long tch = 0;
  BK(cudaMemcpyAsync(&c_last, b->chunk0.p + b->G32 - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  BK(cudaMemcpyAsync(&l_last, b->L.p + b->G32 - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaMemcpyAsync(&t_last, b->toff.p + b->G32 - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaMemcpyAsync(&nt_last, b->ntask.p + b->G32 - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaMemcpyAsync(&s_last, b->soff.p + b->G32 - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaMemcpyAsync(&ns_last, b->nslot.p + b->G32 - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaMemcpyAsync(&h_last, b->hoff.p + b->G32 - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaMemcpyAsync(&nh_last, b->nheavy.p + b->G32 - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaMemcpyAsync(&tch, touched.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  BK(cudaStreamSynchronize(st));
  b->sz.chunks = c_last + l_last;
  b->sz.n_tasks = t_last + nt_last;
  b->sz.n_slots = s_last + ns_last;
  b->sz.n_heavy = h_last + nh_last;
  b->sz.touched = static_cast<int64_t>(tch);
  b->sz.nnz = b->nnz;
  if (b->sz.chunks > (int64_t(1) << 31) - 1) throw std::runtime_error("opbuild: W^T too large");
}

template <typename R>
void gpu_build_finish(GpuBuild* b, WtEnt<R>* ent, int4* tasks, uint16_t* perm, int4* heavy, int* slot_heavy,
                      cudaStream_t st) {
  const int m = b->a.m;
  const int nt = b->sz.n_tasks;
  DBuf<int4> traw(nt);
  DBuf<int> tkey(nt), tkey2(nt), tidx(nt), tidx2(nt);
  k_tasks<<<static_cast<unsigned>((b->G32 + 255) / 256), 256, 0, st>>>(
      b->G32, wt_max_chunks(), b->L.p, b->chunk0.p, b->toff.p, b->soff.p, b->hoff.p, traw.p, tkey.p, heavy, slot_heavy);
  BK(cudaGetLastError());
  const int band = wt_task_band(m);
  if (nt > 0 && band > 0) {
    // bands of `band` grid rows; the bands heaviest first (by their longest task), row order between
    // equal bands, longest tasks first within a band: one band's tasks gather the same samples
    // (L1 / L2 reuse) and the heavy bands around the zero frequency do not form the tail
    std::vector<int4> h(nt);
    BK(cudaMemcpyAsync(h.data(), traw.p, sizeof(int4) * nt, cudaMemcpyDeviceToHost, st));
    BK(cudaStreamSynchronize(st));
    const int bpr = m / 32;
    std::vector<int> bmax((b->rows > 0 ? b->rows : m) / band + 1, 0);
    for (const int4& t : h) bmax[(t.x / bpr) / band] = std::max(bmax[(t.x / bpr) / band], t.z);
    std::vector<int> ord(nt);
    for (int i = 0; i < nt; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) {
      const int bx = (h[x].x / bpr) / band, by = (h[y].x / bpr) / band;
      if (bmax[bx] != bmax[by]) return bmax[bx] > bmax[by];
      if (bx != by) return bx < by;
      return h[x].z > h[y].z;
    });
    std::vector<int4> sorted(nt);
    for (int i = 0; i < nt; ++i) sorted[i] = h[ord[i]];
    BK(cudaMemcpyAsync(tasks, sorted.data(), sizeof(int4) * nt, cudaMemcpyHostToDevice, st));
    BK(cudaStreamSynchronize(st));
  } else if (nt > 0 && wt_row_order(m)) {
    BK(cudaMemcpyAsync(tasks, traw.p, sizeof(int4) * nt, cudaMemcpyDeviceToDevice, st));
  } else if (nt > 0) {
    // longest tasks first, stable (LSD radix sort) = the host's stable_sort by nchunks desc
    std::vector<int> iota(nt);
    for (int i = 0; i < nt; ++i) iota[i] = i;
    BK(cudaMemcpyAsync(tidx.p, iota.data(), sizeof(int) * nt, cudaMemcpyHostToDevice, st));
    size_t tb = 0;
    BK(cub::DeviceRadixSort::SortPairs(nullptr, tb, tkey.p, tkey2.p, tidx.p, tidx2.p, nt, 0,
                                       bits_for(wt_max_chunks()), st));
    DBuf<unsigned char> t2(tb);
    BK(cub::DeviceRadixSort::SortPairs(t2.p, tb, tkey.p, tkey2.p, tidx.p, tidx2.p, nt, 0, bits_for(wt_max_chunks()),
                                       st));
    k_gather_tasks<R><<<(nt + 255) / 256, 256, 0, st>>>(nt, tidx2.p, traw.p, tasks);
    BK(cudaGetLastError());
    BK(cudaStreamSynchronize(st));  // iota must outlive the copy
  }
  BK(cudaMemcpyAsync(perm, b->perm.p, sizeof(uint16_t) * b->G, cudaMemcpyDeviceToDevice, st));
  k_entries<R><<<static_cast<unsigned>((b->G32 + 7) / 8), 256, 0, st>>>(
      m, b->G32, b->perm.p, b->L.p, b->chunk0.p, b->cnt.p, b->off.p, b->sj.p,
      reinterpret_cast<const R*>(b->vals_sorted.p), ent);
  BK(cudaGetLastError());
  BK(cudaStreamSynchronize(st));
}

void gpu_build_free(GpuBuild* b) { delete b; }

// ---- Hermitian fold of W^T (real-subspace applies) -------------------------------------------
// Re(F_NU s) = IFFT2 of the Hermitian part of the spread grid Gt, so a real-output type-1 needs
// only F[node] = Gt[node] + conj(Gt[-node]) (= 2 x the Hermitian part) on the grid rows
// iy in [0, m/2]. Entry (node (iy, ix), sample j, w) of W^T contributes w s_j to F[iy][ix] when
// iy <= m/2 and w conj(s_j) to F[-iy][-ix] when iy >= m/2 or iy == 0 (rows 0 and m/2 are their
// own mirror rows: both). The conj flag is bit 31 of the entry's sample index.
namespace {
// `pair` (mirror-pair fold, below): entries of a pair's secondary sample (j < pair[j]) are dropped;
// with `base` (overlap pairs) only those inside the pair's common window.
struct PairWin {
  int m, lo, hi;  // window [lo, hi] around floor(x / h)
  // taps q = l - lo of the common window of a sample and its mirror partner: l in [max(lo, 1 - hi), min(hi, 1 - lo)]
  __host__ __device__ int q0() const { return (lo > 1 - hi ? lo : 1 - hi) - lo; }
  __host__ __device__ int q1() const { return (hi < 1 - lo ? hi : 1 - lo) - lo; }
  __device__ bool common(int node, int b) const {
    const int iy = node / m, ix = node - iy * m;
    const int qa = (ix - (b & 0xffff) + m) % m, qb = (iy - ((b >> 16) & 0xffff) + m) % m;
    return qa >= q0() && qa <= q1() && qb >= q0() && qb <= q1();
  }
};

__global__ void k_fold_count(int m, int64_t G, const int* __restrict__ cnt, const int* __restrict__ off,
                             const int* __restrict__ sj, const int* __restrict__ pair, const int* __restrict__ base,
                             PairWin pw, int* ecnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= G) return;
  const int iy = static_cast<int>(i / m);
  const int mult = (iy == 0 || iy == m / 2) ? 2 : 1;
  int c = cnt[i];
  if (pair) {
    const int o = off[i];
    int kept = 0;
    for (int k = 0; k < c; ++k) {
      const int j = sj[o + k];
      const bool secondary = pair[j] >= 0 && j < pair[j];
      kept += !(secondary && (!base || pw.common(static_cast<int>(i), base[j])));
    }
    c = kept;
  }
  ecnt[i] = c * mult;
}

template <typename R>
__global__ void k_fold_emit(int m, int64_t G, const int* __restrict__ cnt, const int* __restrict__ off,
                            const int* __restrict__ eoff, const int* __restrict__ sj, const R* __restrict__ vals,
                            const int* __restrict__ pair, const int* __restrict__ base, PairWin pw, unsigned P,
                            unsigned long long* keys, R* fvals) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= G) return;
  const int iy = static_cast<int>(i / m), ix = static_cast<int>(i - static_cast<int64_t>(iy) * m);
  const int c = cnt[i];
  int o = eoff[i];
  const unsigned long long mnode =
      static_cast<unsigned long long>((m - iy) & (m - 1)) * m + static_cast<unsigned long long>((m - ix) & (m - 1));
  for (int k = 0; k < c; ++k) {
    unsigned j = static_cast<unsigned>(sj[off[i] + k]);
    R v = vals[off[i] + k];
    if (pair && !base) {
      const int pr = pair[j];
      if (pr >= 0 && static_cast<int>(j) < pr) continue;  // secondary: carried by its primary
      if (pr >= 0) v = v + v;                             // primary: its own and its mirror's share
    } else if (pair) {
      // overlap pairs: inside the common window the primary's entry reads the pair sum
      // s_j + conj(s_partner) (index P + j) and the secondary's is dropped
      const int pr = pair[j];
      if (pr >= 0 && pw.common(static_cast<int>(i), base[j])) {
        if (static_cast<int>(j) < pr) continue;
        j += P;
      }
    }
    if (iy <= m / 2) {
      keys[o] = (static_cast<unsigned long long>(i) << 32) | j;
      fvals[o++] = v;
    }
    if (iy >= m / 2 || iy == 0) {
      keys[o] = (mnode << 32) | 0x80000000ull | j;
      fvals[o++] = v;
    }
  }
}

__global__ void k_fold_cnt(int64_t n, const unsigned long long* __restrict__ keys, int* cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&cnt[keys[i] >> 32], 1);
}
}  // namespace

template <typename R>
GpuBuild* gpu_build_fold(const GpuBuild* src, cudaStream_t st, GpuBuildSizes* sizes, const int* pair,
                         const int* base) {
  const int m = src->a.m;
  if (src->G != static_cast<int64_t>(m) * m) throw std::runtime_error("opbuild: fold needs the unfolded W^T");
  auto b = std::make_unique<GpuBuild>();
  b->a = src->a;
  b->rows = m / 2 + 1;
  b->G = static_cast<int64_t>(b->rows) * m;
  b->G32 = b->G / 32;
  const unsigned gs = static_cast<unsigned>((src->G + 255) / 256);
  DBuf<int> ecnt(src->G), eoff(src->G);
  const PairWin pw{m, src->a.lo, src->a.hi};
  if (base && 2 * src->a.P >= (int64_t(1) << 31)) throw std::runtime_error("opbuild: too many samples for pair sums");
  k_fold_count<<<gs, 256, 0, st>>>(m, src->G, src->cnt.p, src->off.p, src->sj.p, pair, base, pw, ecnt.p);
  BK(cudaGetLastError());
  size_t tb = 0;
  BK(cub::DeviceScan::ExclusiveSum(nullptr, tb, ecnt.p, eoff.p, static_cast<int>(src->G), st));
  {
    DBuf<unsigned char> tmp(tb);
    BK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, ecnt.p, eoff.p, static_cast<int>(src->G), st));
  }
  int last_off = 0, last_cnt = 0;
  BK(cudaMemcpyAsync(&last_off, eoff.p + src->G - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaMemcpyAsync(&last_cnt, ecnt.p + src->G - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaStreamSynchronize(st));
  b->nnz = static_cast<int64_t>(last_off) + last_cnt;
  if (b->nnz >= (int64_t(1) << 31)) throw std::runtime_error("opbuild: folded W^T too large for 32-bit offsets");
  DBuf<unsigned long long> keys(b->nnz), skeys(b->nnz);
  DBuf<R> vals(b->nnz);
  k_fold_emit<R><<<gs, 256, 0, st>>>(m, src->G, src->cnt.p, src->off.p, eoff.p, src->sj.p,
                                     reinterpret_cast<const R*>(src->vals_sorted.p), pair, base, pw,
                                     static_cast<unsigned>(src->a.P), keys.p, vals.p);
  BK(cudaGetLastError());
  // (folded node, conj flag, sample): plain entries before conjugated ones, samples ascending
  b->vals_sorted.alloc(sizeof(R) * b->nnz);
  const int key_bits = 32 + bits_for(static_cast<uint64_t>(b->G));
  tb = 0;
  BK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, skeys.p, vals.p, reinterpret_cast<R*>(b->vals_sorted.p),
                                     static_cast<int>(b->nnz), 0, key_bits, st));
  {
    DBuf<unsigned char> tmp(tb);
    BK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, skeys.p, vals.p, reinterpret_cast<R*>(b->vals_sorted.p),
                                       static_cast<int>(b->nnz), 0, key_bits, st));
  }
  b->sj.alloc(b->nnz);
  k_low32<<<static_cast<unsigned>((b->nnz + 255) / 256), 256, 0, st>>>(b->nnz, skeys.p, b->sj.p);
  b->cnt.alloc(b->G);
  BK(cudaMemsetAsync(b->cnt.p, 0, sizeof(int) * b->G, st));
  k_fold_cnt<<<static_cast<unsigned>((b->nnz + 255) / 256), 256, 0, st>>>(b->nnz, skeys.p, b->cnt.p);
  BK(cudaGetLastError());
  build_structure(b.get(), st);
  *sizes = b->sz;
  return b.release();
}

// ---- the fused backend's Gram W^T W on the device (build_btb, normal_ops.cpp:53-173) ------------
namespace {
// one thread per (sample j, tap a, tap b): the w^2 products landing in node (iy0+b, ix0+a)'s band
// cells, fp64, with the host's association (wx[a] wx[a2]) (wy[b] wy[b2])
__global__ void k_gram_tuples(int64_t P, int m, int w, const int* __restrict__ base, const double* __restrict__ wx,
                              const double* __restrict__ wy, unsigned long long* keys, double* vals) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t w2 = static_cast<int64_t>(w) * w;
  if (t >= P * w2) return;
  const int64_t j = t / w2;
  const int ab = static_cast<int>(t - j * w2), a = ab / w, bb = ab - a * w;
  const int ix0 = base[j] & 0xffff, iy0 = base[j] >> 16;
  const int ix = wrapd(ix0 + a, m), iy = wrapd(iy0 + bb, m);
  const unsigned long long row = static_cast<unsigned long long>(iy) * m + ix;
  const int band = 2 * w - 1;
  const double* wxj = wx + j * w;
  const double* wyj = wy + j * w;
  const size_t o = static_cast<size_t>(t) * w2;
  for (int b2 = 0; b2 < w; ++b2) {
    const double py = __dmul_rn(wyj[bb], wyj[b2]);
    for (int a2 = 0; a2 < w; ++a2) {
      const double px = __dmul_rn(wxj[a], wxj[a2]);
      const int cell = (b2 - bb + w - 1) * band + (a2 - a + w - 1);
      keys[o + b2 * w + a2] = (row << 14) | static_cast<unsigned long long>(cell);
      vals[o + b2 * w + a2] = __dmul_rn(px, py);
    }
  }
}

__global__ void k_heads(int64_t n, const unsigned long long* __restrict__ keys, int* head) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void k_seg_starts(int64_t n, const int* __restrict__ head, const int* __restrict__ sid, int* start) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && head[i]) start[sid[i]] = static_cast<int>(i);
}

// one thread per (node, band cell): the sum over samples in ascending j order (the stable sort kept
// it), exactly the host band accumulation; exact zeros dropped like build_btb
__global__ void k_seg_sum(int nseg, int64_t n, int m, int w, const int* __restrict__ start,
                          const unsigned long long* __restrict__ keys, const double* __restrict__ vals, int* row,
                          int* col, double* sum, int* keep) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const int64_t i0 = start[s], i1 = s + 1 < nseg ? start[s + 1] : n;
  double acc = 0.0;
  for (int64_t i = i0; i < i1; ++i) acc += vals[i];
  const unsigned long long k = keys[i0];
  const int r = static_cast<int>(k >> 14), cell = static_cast<int>(k & 0x3fff);
  const int band = 2 * w - 1;
  const int dy = cell / band - (w - 1), dx = cell % band - (w - 1);
  const int iy = r / m, ix = r - iy * m;
  row[s] = r;
  col[s] = wrapd(iy + dy, m) * m + wrapd(ix + dx, m);
  sum[s] = acc;
  keep[s] = acc != 0.0 ? 1 : 0;
}

template <typename R>
__global__ void k_gram_compact(int nseg, const int* __restrict__ keep, const int* __restrict__ pos,
                               const int* __restrict__ row, const int* __restrict__ col, const double* __restrict__ sum,
                               int* sj, R* sv, int* cnt) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg || !keep[s]) return;
  sj[pos[s]] = col[s];
  sv[pos[s]] = static_cast<R>(sum[s]);
  atomicAdd(&cnt[row[s]], 1);
}
}  // namespace

template <typename R>
GpuBuild* gpu_build_gram_begin(int m, int w, int64_t P, const int* h_base, const double* h_wx, const double* h_wy,
                               cudaStream_t st, GpuBuildSizes* sizes, int64_t* nnz_out) {
  const int64_t w2 = static_cast<int64_t>(w) * w;
  const int64_t n = P * w2 * w2;
  if (n >= (int64_t(1) << 31) || 2 * w - 1 > 127) return nullptr;  // the host build handles it
  auto b = std::make_unique<GpuBuild>();
  b->a.m = m;
  b->G = static_cast<int64_t>(m) * m;
  b->G32 = b->G / 32;
  DBuf<int> base(P);
  DBuf<double> wx(P * w), wy(P * w);
  BK(cudaMemcpyAsync(base.p, h_base, sizeof(int) * P, cudaMemcpyHostToDevice, st));
  BK(cudaMemcpyAsync(wx.p, h_wx, sizeof(double) * P * w, cudaMemcpyHostToDevice, st));
  BK(cudaMemcpyAsync(wy.p, h_wy, sizeof(double) * P * w, cudaMemcpyHostToDevice, st));
  DBuf<unsigned long long> keys(n), skeys(n);
  DBuf<double> vals(n), svals(n);
  k_gram_tuples<<<static_cast<unsigned>((P * w2 + 255) / 256), 256, 0, st>>>(P, m, w, base.p, wx.p, wy.p, keys.p,
                                                                            vals.p);
  BK(cudaGetLastError());
  const int key_bits = 14 + bits_for(static_cast<uint64_t>(b->G));
  size_t tb = 0;
  BK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, skeys.p, vals.p, svals.p, static_cast<int>(n), 0, key_bits,
                                     st));
  {
    DBuf<unsigned char> tmp(tb);
    BK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, skeys.p, vals.p, svals.p, static_cast<int>(n), 0,
                                       key_bits, st));
  }
  keys.alloc(1);  // release
  vals.alloc(1);
  DBuf<int> head(n), sid(n);
  const unsigned gn = static_cast<unsigned>((n + 255) / 256);
  k_heads<<<gn, 256, 0, st>>>(n, skeys.p, head.p);
  tb = 0;
  BK(cub::DeviceScan::ExclusiveSum(nullptr, tb, head.p, sid.p, static_cast<int>(n), st));
  {
    DBuf<unsigned char> tmp(tb);
    BK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, head.p, sid.p, static_cast<int>(n), st));
  }
  int last_sid = 0, last_head = 0;
  BK(cudaMemcpyAsync(&last_sid, sid.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaMemcpyAsync(&last_head, head.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaStreamSynchronize(st));
  const int nseg = last_sid + last_head;
  DBuf<int> start(nseg), row(nseg), col(nseg), keep(nseg), pos(nseg);
  DBuf<double> sum(nseg);
  k_seg_starts<<<gn, 256, 0, st>>>(n, head.p, sid.p, start.p);
  const unsigned gs = static_cast<unsigned>((nseg + 255) / 256);
  k_seg_sum<<<gs, 256, 0, st>>>(nseg, n, m, w, start.p, skeys.p, svals.p, row.p, col.p, sum.p, keep.p);
  BK(cudaGetLastError());
  tb = 0;
  BK(cub::DeviceScan::ExclusiveSum(nullptr, tb, keep.p, pos.p, nseg, st));
  {
    DBuf<unsigned char> tmp(tb);
    BK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, keep.p, pos.p, nseg, st));
  }
  int last_pos = 0, last_keep = 0;
  BK(cudaMemcpyAsync(&last_pos, pos.p + nseg - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaMemcpyAsync(&last_keep, keep.p + nseg - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaStreamSynchronize(st));
  const int64_t nnz = static_cast<int64_t>(last_pos) + last_keep;
  b->nnz = nnz;
  b->sj.alloc(nnz);
  b->vals_sorted.alloc(sizeof(R) * nnz);
  b->cnt.alloc(b->G);
  BK(cudaMemsetAsync(b->cnt.p, 0, sizeof(int) * b->G, st));
  k_gram_compact<R><<<gs, 256, 0, st>>>(nseg, keep.p, pos.p, row.p, col.p, sum.p, b->sj.p,
                                        reinterpret_cast<R*>(b->vals_sorted.p), b->cnt.p);
  BK(cudaGetLastError());
  build_structure(b.get(), st);
  *sizes = b->sz;
  *nnz_out = nnz;
  return b.release();
}


namespace {
__global__ void k_tile_keys(int64_t P, int m, const int* __restrict__ base, unsigned long long* keys, int* idx) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= P) return;
  const int b = base[j];
  const int ix0 = b & 0xffff, iy0 = b >> 16;
  const unsigned long long tile = static_cast<unsigned long long>(iy0 / 16) * (m / 16) + ix0 / 16;
  keys[j] = (tile << 32) | static_cast<unsigned long long>(j);
  idx[j] = static_cast<int>(j);
}

template <typename R>
__global__ void k_gather_w(int64_t P, int64_t Ppad, int w, const int* __restrict__ perm, const int* __restrict__ base_in,
                           const R* __restrict__ wx_in, const R* __restrict__ wy_in, int* base_out, R* wx_out,
                           R* wy_out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= P) return;
  const int j = perm[t];
  base_out[t] = base_in[j];
  for (int a = 0; a < w; ++a) {
    wx_out[a * Ppad + t] = wx_in[a * Ppad + j];
    wy_out[a * Ppad + t] = wy_in[a * Ppad + j];
  }
}
__global__ void k_inverse(int64_t P, const int* __restrict__ perm, int* pos) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < P) pos[perm[t]] = static_cast<int>(t);
}

template <typename R>
__global__ void k_remap_ent(int64_t n, const int* __restrict__ pos, WtEnt<R>* ent) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) ent[i].j = pos[ent[i].j & 0x7fffffff] | (ent[i].j & static_cast<int>(0x80000000u));  // keeps the conj flag
}
}  // namespace

template <typename R>
void gpu_sort_w_tables(int m, int64_t P, int64_t Ppad, int w, int* base, R* wx, R* wy, int* perm, WtEnt<R>* ent,
                       int64_t n_ent, WtEnt<R>* ent2, int64_t n_ent2, cudaStream_t st) {
  if (P <= 0) return;
  DBuf<unsigned long long> keys(P), skeys(P);
  DBuf<int> idx(P);
  const unsigned grid = static_cast<unsigned>((P + 255) / 256);
  k_tile_keys<<<grid, 256, 0, st>>>(P, m, base, keys.p, idx.p);
  BK(cudaGetLastError());
  const int tiles = (m / 16) * (m / 16);
  const int key_bits = 32 + bits_for(static_cast<uint64_t>(tiles));
  size_t tb = 0;
  BK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, skeys.p, idx.p, perm, static_cast<int>(P), 0, key_bits, st));
  DBuf<unsigned char> tmp(tb);
  BK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, skeys.p, idx.p, perm, static_cast<int>(P), 0, key_bits, st));
  DBuf<int> b2(Ppad);
  DBuf<R> x2(static_cast<size_t>(w) * Ppad), y2(static_cast<size_t>(w) * Ppad);
  BK(cudaMemcpyAsync(b2.p, base, sizeof(int) * Ppad, cudaMemcpyDeviceToDevice, st));  // padding rows
  BK(cudaMemcpyAsync(x2.p, wx, sizeof(R) * w * Ppad, cudaMemcpyDeviceToDevice, st));
  BK(cudaMemcpyAsync(y2.p, wy, sizeof(R) * w * Ppad, cudaMemcpyDeviceToDevice, st));
  k_gather_w<R><<<grid, 256, 0, st>>>(P, Ppad, w, perm, base, wx, wy, b2.p, x2.p, y2.p);
  BK(cudaGetLastError());
  BK(cudaMemcpyAsync(base, b2.p, sizeof(int) * Ppad, cudaMemcpyDeviceToDevice, st));
  BK(cudaMemcpyAsync(wx, x2.p, sizeof(R) * w * Ppad, cudaMemcpyDeviceToDevice, st));
  BK(cudaMemcpyAsync(wy, y2.p, sizeof(R) * w * Ppad, cudaMemcpyDeviceToDevice, st));
  if (ent && n_ent > 0) {  // W^T entries index samples by position from now on
    DBuf<int> pos(P);
    k_inverse<<<grid, 256, 0, st>>>(P, perm, pos.p);
    k_remap_ent<R><<<static_cast<unsigned>((n_ent + 255) / 256), 256, 0, st>>>(n_ent, pos.p, ent);
    if (ent2 && n_ent2 > 0)
      k_remap_ent<R><<<static_cast<unsigned>((n_ent2 + 255) / 256), 256, 0, st>>>(n_ent2, pos.p, ent2);
    BK(cudaGetLastError());
  }
  BK(cudaStreamSynchronize(st));
}

// ---- mirror pairs of the parallel-beam samples (real-subspace normal operator) ------------------
// Sample (angle a, bin t) sits at frequency k_r (cos, sin) with k_r = (2 pi / nb)(t - nb/2); the bin
// t' = 2 (nb/2) - t of the same angle sits at the mirrored frequency. For a window [lo, hi] with
// lo = 1 - hi around floor(x / h) (the width-6 [-2, 3] of the BASELINE configs) the mirror sample's
// window is the node-for-node mirror image of the sample's own, with the same weights to rounding.
// On the real subspace (Hermitian grid) its W value is then the conjugate of the sample's, so the
// normal operator needs W on one sample per pair only, and the folded W^T needs only the primaries'
// entries, doubled: F[p] = 2 sum_{primary j} (w_pj s_j + w_{-p,j} conj s_j) (+ the unpaired samples'
// entries as before). pair[j] = the mirror sample when the two windows are mirror images (base nodes
// checked exactly, factor vectors to rounding), else -1 (bins without a mirror bin, the zero
// frequency, samples on a grid line whose floor() breaks the symmetry, other windows). The primary
// of a pair is the larger index. The resulting operator is the exact normal operator U^T U of the
// interpolation U whose secondary rows are the conjugate mirrors of the primaries' rows: symmetric
// positive semi-definite, equal to W^T W up to the rounding of the sample positions.
namespace {
template <typename R>
__global__ void k_pairs(int64_t P, int64_t Ppad, int nb, PairWin pw, int w, const int* __restrict__ base,
                        const R* __restrict__ wx, const R* __restrict__ wy, int* pair, unsigned long long* npaired) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= P) return;
  const int m = pw.m;
  const int t = static_cast<int>(j % nb), tm = 2 * (nb / 2) - t;
  int pr = -1;
  if (tm >= 0 && tm < nb && tm != t && pw.q0() <= pw.q1()) {
    const int64_t jm = j - t + tm;
    const int b = base[j], bm = base[jm];
    const int ix0 = b & 0xffff, iy0 = (b >> 16) & 0xffff;
    // node mj + l of the sample <-> node -(mj + l) = (-mj - 1) + (1 - l) of the mirror sample:
    // its base node is -(ix0 - lo) - 1 + lo, its tap of the same node q' = 1 - 2 lo - q
    const int shift = 2 * pw.lo - 1;
    bool ok = (bm & 0xffff) == ((3 * m - ix0 + shift) % m) && ((bm >> 16) & 0xffff) == ((3 * m - iy0 + shift) % m);
    const R tol = sizeof(R) == 8 ? R(1e-9) : R(4e-7);
    for (int q = pw.q0(); ok && q <= pw.q1(); ++q) {
      const int qm = 1 - 2 * pw.lo - q;
      const R x1 = wx[static_cast<size_t>(qm) * Ppad + jm], x2 = wx[static_cast<size_t>(q) * Ppad + j];
      const R y1 = wy[static_cast<size_t>(qm) * Ppad + jm], y2 = wy[static_cast<size_t>(q) * Ppad + j];
      ok = fabs(x1 - x2) <= tol * fmax(fabs(x1), fabs(x2)) && fabs(y1 - y2) <= tol * fmax(fabs(y1), fabs(y2));
    }
    if (ok) {
      pr = static_cast<int>(jm);
      atomicAdd(npaired, 1ull);
    }
  }
  pair[j] = pr;
}

// position (tile order) -> kept by the half W: every sample but the secondaries
__global__ void k_half_flags(int64_t P, const int* __restrict__ perm, const int* __restrict__ pair, int* flag) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= P) return;
  const int j = perm[t];
  flag[t] = !(pair[j] >= 0 && j < pair[j]);
}

template <typename R>
__global__ void k_half_gather(int64_t P, int64_t Ppad, int64_t Ppad_h, int w, const int* __restrict__ perm,
                              const int* __restrict__ pair, const int* __restrict__ flag, const int* __restrict__ hpos,
                              const int* __restrict__ base, const R* __restrict__ wx, const R* __restrict__ wy,
                              int* base_h, R* wx_h, R* wy_h, int* cmap) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= P || !flag[t]) return;
  const int h = hpos[t], j = perm[t];
  base_h[h] = base[t];
  for (int a = 0; a < w; ++a) {
    wx_h[static_cast<size_t>(a) * Ppad_h + h] = wx[static_cast<size_t>(a) * Ppad + t];
    wy_h[static_cast<size_t>(a) * Ppad_h + h] = wy[static_cast<size_t>(a) * Ppad + t];
  }
  cmap[j] = h;
  if (pair[j] >= 0) cmap[pair[j]] = h;  // the secondary reads its primary's value, conjugated
}
}  // namespace

template <typename R>
int64_t gpu_find_pairs(const BuildArgs& a, const int* base, const R* wx, const R* wy, int* pair, cudaStream_t st) {
  if (a.P <= 0) return 0;
  DBuf<unsigned long long> np(1);
  BK(cudaMemsetAsync(np.p, 0, sizeof(unsigned long long), st));
  k_pairs<R><<<static_cast<unsigned>((a.P + 255) / 256), 256, 0, st>>>(a.P, a.Ppad, a.nb, PairWin{a.m, a.lo, a.hi}, a.w,
                                                                        base, wx, wy, pair, np.p);
  BK(cudaGetLastError());
  unsigned long long h = 0;
  BK(cudaMemcpyAsync(&h, np.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  BK(cudaStreamSynchronize(st));
  return static_cast<int64_t>(h);
}

namespace {
// entries: sample j -> position, pair sum P + j -> P + position (conj flag kept)
template <typename R>
__global__ void k_remap_ent_ext(int64_t n, int P, const int* __restrict__ pos, WtEnt<R>* ent) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int e = ent[i].j, flag = e & static_cast<int>(0x80000000u), j = e & 0x7fffffff;
  ent[i].j = (j >= P ? P + pos[j - P] : pos[j]) | flag;
}
__global__ void k_partner_pos(int64_t P, const int* __restrict__ perm, const int* __restrict__ pair,
                              const int* __restrict__ pos, int* ppos) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= P) return;
  const int j = perm[t], pr = pair[j];
  ppos[t] = pr < 0 ? -1 : (j > pr ? pos[pr] : -2 - pos[pr]);  // primary / secondary / unpaired
}
}  // namespace

template <typename R>
void gpu_pair_sigma_setup(int64_t P, const int* perm, const int* pair, WtEnt<R>* ent, int64_t n_ent, int* ppos,
                          cudaStream_t st) {
  DBuf<int> pos(P);
  const unsigned grid = static_cast<unsigned>((P + 255) / 256);
  k_inverse<<<grid, 256, 0, st>>>(P, perm, pos.p);
  k_partner_pos<<<grid, 256, 0, st>>>(P, perm, pair, pos.p, ppos);
  if (n_ent > 0)
    k_remap_ent_ext<R><<<static_cast<unsigned>((n_ent + 255) / 256), 256, 0, st>>>(n_ent, static_cast<int>(P), pos.p, ent);
  BK(cudaGetLastError());
  BK(cudaStreamSynchronize(st));
}

struct HalfWBuild {
  int64_t P = 0, Ph = 0;
  DBuf<int> flag, hpos;
};

HalfWBuild* gpu_half_w_begin(int64_t P, const int* perm, const int* pair, cudaStream_t st, int64_t* Ph) {
  auto hb = std::make_unique<HalfWBuild>();
  hb->P = P;
  hb->flag.alloc(P);
  hb->hpos.alloc(P);
  k_half_flags<<<static_cast<unsigned>((P + 255) / 256), 256, 0, st>>>(P, perm, pair, hb->flag.p);
  BK(cudaGetLastError());
  size_t tb = 0;
  BK(cub::DeviceScan::ExclusiveSum(nullptr, tb, hb->flag.p, hb->hpos.p, static_cast<int>(P), st));
  DBuf<unsigned char> tmp(tb);
  BK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, hb->flag.p, hb->hpos.p, static_cast<int>(P), st));
  int lo = 0, lf = 0;
  BK(cudaMemcpyAsync(&lo, hb->hpos.p + P - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaMemcpyAsync(&lf, hb->flag.p + P - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  BK(cudaStreamSynchronize(st));
  hb->Ph = static_cast<int64_t>(lo) + lf;
  *Ph = hb->Ph;
  return hb.release();
}

template <typename R>
void gpu_half_w_finish(HalfWBuild* hb, int64_t Ppad, int64_t Ppad_h, int w, const int* perm, const int* pair,
                       const int* base, const R* wx, const R* wy, int* base_h, R* wx_h, R* wy_h, WtEnt<R>* ent,
                       int64_t n_ent, cudaStream_t st) {
  const int64_t P = hb->P;
  BK(cudaMemsetAsync(base_h, 0, sizeof(int) * Ppad_h, st));  // padding rows: node 0, zero weights
  BK(cudaMemsetAsync(wx_h, 0, sizeof(R) * w * Ppad_h, st));
  BK(cudaMemsetAsync(wy_h, 0, sizeof(R) * w * Ppad_h, st));
  DBuf<int> cmap(P);
  k_half_gather<R><<<static_cast<unsigned>((P + 255) / 256), 256, 0, st>>>(
      P, Ppad, Ppad_h, w, perm, pair, hb->flag.p, hb->hpos.p, base, wx, wy, base_h, wx_h, wy_h, cmap.p);
  BK(cudaGetLastError());
  if (n_ent > 0)  // the mirror-pair W^T indexes the half W's output positions
    k_remap_ent<R><<<static_cast<unsigned>((n_ent + 255) / 256), 256, 0, st>>>(n_ent, cmap.p, ent);
  BK(cudaGetLastError());
  BK(cudaStreamSynchronize(st));
}

void gpu_half_w_free(HalfWBuild* hb) { delete hb; }

namespace {
template <typename R>
__global__ void k_pair_units(int64_t P, int64_t Ppad, int64_t Upad, int w, const int* __restrict__ flag,
                             const int* __restrict__ hpos, const int* __restrict__ ppos, const int* __restrict__ base,
                             const R* __restrict__ wx, const R* __restrict__ wy, int* ubase, R* ufx, R* ufy, int* upos,
                             int* uppos) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= P || !flag[t]) return;
  const int u = hpos[t], pp = ppos[t] >= 0 ? ppos[t] : -1;
  ubase[u] = base[t];
  for (int a = 0; a < w; ++a) {
    ufx[static_cast<size_t>(a) * Upad + u] = wx[static_cast<size_t>(a) * Ppad + t];
    ufy[static_cast<size_t>(a) * Upad + u] = wy[static_cast<size_t>(a) * Ppad + t];
  }
  // union tap w = the partner's own tap 0 (its node there is the mirror of the primary's node w)
  ufx[static_cast<size_t>(w) * Upad + u] = pp >= 0 ? wx[pp] : R(0);
  ufy[static_cast<size_t>(w) * Upad + u] = pp >= 0 ? wy[pp] : R(0);
  upos[u] = static_cast<int>(t);
  uppos[u] = pp;
}
}  // namespace

template <typename R>
void gpu_pair_w_finish(HalfWBuild* hb, int64_t Ppad, int64_t Upad, int w, const int* ppos, const int* base,
                       const R* wx, const R* wy, int* ubase, R* ufx, R* ufy, int* upos, int* uppos, cudaStream_t st) {
  const int64_t P = hb->P;
  BK(cudaMemsetAsync(ubase, 0, sizeof(int) * Upad, st));  // padding units: node 0, zero factors, no output
  BK(cudaMemsetAsync(ufx, 0, sizeof(R) * (w + 1) * Upad, st));
  BK(cudaMemsetAsync(ufy, 0, sizeof(R) * (w + 1) * Upad, st));
  BK(cudaMemsetAsync(upos, 0xff, sizeof(int) * Upad, st));
  BK(cudaMemsetAsync(uppos, 0xff, sizeof(int) * Upad, st));
  k_pair_units<R><<<static_cast<unsigned>((P + 255) / 256), 256, 0, st>>>(P, Ppad, Upad, w, hb->flag.p, hb->hpos.p, ppos,
                                                                          base, wx, wy, ubase, ufx, ufy, upos, uppos);
  BK(cudaGetLastError());
  BK(cudaStreamSynchronize(st));
}

#define TOMO_INST_BUILD(R)                                                                                     \
  template GpuBuild* gpu_build_begin<R>(const BuildArgs&, const double*, const double*, int*, R*, R*,         \
                                        cudaStream_t, GpuBuildSizes*);                                        \
  template void gpu_build_finish<R>(GpuBuild*, WtEnt<R>*, int4*, uint16_t*, int4*, int*, cudaStream_t); \
  template void gpu_sort_w_tables<R>(int, int64_t, int64_t, int, int*, R*, R*, int*, WtEnt<R>*, int64_t, WtEnt<R>*, \
                                     int64_t, cudaStream_t);                                                   \
  template GpuBuild* gpu_build_fold<R>(const GpuBuild*, cudaStream_t, GpuBuildSizes*, const int*, const int*); \
  template void gpu_pair_sigma_setup<R>(int64_t, const int*, const int*, WtEnt<R>*, int64_t, int*, cudaStream_t); \
  template int64_t gpu_find_pairs<R>(const BuildArgs&, const int*, const R*, const R*, int*, cudaStream_t);  \
  template void gpu_pair_w_finish<R>(HalfWBuild*, int64_t, int64_t, int, const int*, const int*, const R*, const R*, \
                                     int*, R*, R*, int*, int*, cudaStream_t);                                 \
  template void gpu_half_w_finish<R>(HalfWBuild*, int64_t, int64_t, int, const int*, const int*, const int*, \
                                     const R*, const R*, int*, R*, R*, WtEnt<R>*, int64_t, cudaStream_t);    \
  template GpuBuild* gpu_build_gram_begin<R>(int, int, int64_t, const int*, const double*, const double*, cudaStream_t, \
                                             GpuBuildSizes*, int64_t*);

TOMO_INST_BUILD(float)
TOMO_INST_BUILD(double)

}  // namespace tomo_b200
