// common.cuh — shared device helpers for the B200 (sm_100a) normal-operator path.
// Everything is templated on the real type R (float: the complex64 path; double: the
// complex128 path used where CG must track the fp64 reference).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>
#include <utility>

#define TOMO_DEV __device__ __forceinline__

namespace tomo_b200 {

// A/B override knobs (TOMO_ROW_RB, TOMO_COL_RB, TOMO_WT_MAXCH, TOMO_WT_GRP, TOMO_WT_PIPE,
// TOMO_BATCH_Y, TOMO_TASK_ORDER, TOMO_CG, TOMO_BUILD) for measurement runs: honoured only when
// TOMO_AB=1, so a production process cannot change kernel selection by accident. Host only.
inline std::string ab_knob(const char* name) {
  const char* ab = std::getenv("TOMO_AB");
  if (!(ab && std::atoi(ab) != 0)) return std::string();
  const char* v = std::getenv(name);
  return v ? std::string(v) : std::string();
}
inline int ab_int(const char* name, int dflt) {
  const std::string v = ab_knob(name);
  return v.empty() ? dflt : std::atoi(v.c_str());
}


template <typename R>
struct CplxT;
template <>
struct CplxT<float> {
  using T = float2;
};
template <>
struct CplxT<double> {
  using T = double2;
};
template <typename R>
using cplx = typename CplxT<R>::T;

template <typename C2>
TOMO_DEV C2 mk(decltype(C2::x) a, decltype(C2::x) b) {
  C2 r;
  r.x = a;
  r.y = b;
  return r;
}
template <typename C2>
TOMO_DEV C2 cadd(C2 a, C2 b) { return mk<C2>(a.x + b.x, a.y + b.y); }
template <typename C2>
TOMO_DEV C2 csub(C2 a, C2 b) { return mk<C2>(a.x - b.x, a.y - b.y); }
template <typename C2>
TOMO_DEV C2 cmul(C2 a, C2 b) { return mk<C2>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
template <typename C2>
TOMO_DEV C2 cscale(C2 a, decltype(C2::x) s) { return mk<C2>(a.x * s, a.y * s); }
template <typename C2>
TOMO_DEV C2 cconj(C2 a) { return mk<C2>(a.x, -a.y); }
template <typename C2>
TOMO_DEV C2 cmul_negi(C2 a) { return mk<C2>(a.y, -a.x); }  // a * (-i)
template <typename C2>
TOMO_DEV C2 czero() { return mk<C2>(0, 0); }

// complex64 adds / subtracts / real scalings as one packed sm_100 instruction each
// (FADD2 / FMUL2 on an f32x2 register pair) instead of two scalar ones.
template <>
TOMO_DEV float2 cadd<float2>(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 pa, pb, pc;\n\t"
      "mov.b64 pa, {%2, %3};\n\t"
      "mov.b64 pb, {%4, %5};\n\t"
      "add.rn.f32x2 pc, pa, pb;\n\t"
      "mov.b64 {%0, %1}, pc;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
template <>
TOMO_DEV float2 csub<float2>(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 pa, pb, pc;\n\t"
      "mov.b64 pa, {%2, %3};\n\t"
      "mov.b64 pb, {%4, %5};\n\t"
      "sub.rn.f32x2 pc, pa, pb;\n\t"
      "mov.b64 {%0, %1}, pc;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
template <>
TOMO_DEV float2 cscale<float2>(float2 a, float s) {
  float2 r;
  asm("{.reg .b64 pa, ps, pc;\n\t"
      "mov.b64 pa, {%2, %3};\n\t"
      "mov.b64 ps, {%4, %4};\n\t"
      "mul.rn.f32x2 pc, pa, ps;\n\t"
      "mov.b64 {%0, %1}, pc;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(s));
  return r;
}

// Shared-memory padding: one element of slack every 16 so the Stockham stride-16 stores of
// the first radix-16 pass and the transposed row stores are bank-conflict free.
TOMO_DEV int pad16(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded_len(int m) { return m + m / 16 + 4; }

// Warp/block reductions in a fixed order (deterministic: every replica and every CTA that
// re-reduces the same partials gets bit-identical scalars).
TOMO_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of one double per thread; result valid in all threads. blockDim.x must
// be a multiple of 32 and <= 1024. `scratch` needs 32 doubles.
TOMO_DEV double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? scratch[threadIdx.x] : 0.0;
  if (wid == 0) t = warp_sum(t);
  if (threadIdx.x == 0) scratch[0] = t;
  __syncthreads();
  const double r = scratch[0];
  __syncthreads();
  return r;
}

// Block-wide sums of two doubles per thread in one pass (results valid in all threads).
TOMO_DEV void block_sum2(double& a, double& b) {
  __shared__ double sc2[64];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) {
    sc2[wid] = a;
    sc2[32 + wid] = b;
  }
  __syncthreads();
  if (wid == 0) {
    double ta = lane < nw ? sc2[lane] : 0.0, tb = lane < nw ? sc2[32 + lane] : 0.0;
    ta = warp_sum(ta);
    tb = warp_sum(tb);
    if (lane == 0) {
      sc2[0] = ta;
      sc2[32] = tb;
    }
  }
  __syncthreads();
  a = sc2[0];
  b = sc2[32];
  __syncthreads();
}

// Two-value block reduction with "last block finishes": every block writes its partial
// pair to part[2*blk..], takes a ticket; the block that takes the last ticket sums all
// nblk pairs in a fixed order (every thread loads its strided share, then one block tree: one
// round trip for the partials instead of a warp walking them serially), so the result is
// deterministic, resets the ticket counter and returns true with the totals in t0/t1 (valid in
// all of its threads). `scratch` is unused (kept for the callers' signature).
TOMO_DEV bool reduce2_last(double v0, double v1, double* part, int nblk, int blk, unsigned* counter,
                           double* scratch, double& t0, double& t1) {
  (void)scratch;
  __shared__ int s_last;
  block_sum2(v0, v1);
  if (threadIdx.x == 0) {
    part[2 * blk] = v0;
    part[2 * blk + 1] = v1;
    __threadfence();
    const unsigned ticket = atomicAdd(counter, 1u);
    s_last = (ticket == static_cast<unsigned>(nblk - 1));
  }
  __syncthreads();
  const bool last = s_last != 0;
  if (!last) return false;
  __threadfence();
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    a += __ldcg(&part[2 * i]);
    b += __ldcg(&part[2 * i + 1]);
  }
  block_sum2(a, b);
  if (threadIdx.x == 0) *counter = 0u;
  t0 = a;
  t1 = b;
  return true;
}

template <typename R>
TOMO_DEV bool finite_r(R v) { return isfinite(v); }

// Host: launch `kern` on `st` through cudaLaunchKernelEx (status returned for CK_LAUNCH).
// Programmatic dependent launch was measured here (griddepcontrol.wait at kernel entry,
// programmatic stream serialisation on every launch) and gave no gain inside the solver graphs.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(std::forward<Args>(args))...);
}

}  // namespace tomo_b200
