// fft.cuh — in-CTA Stockham FFT over shared memory (sm_100a).
//
// Replaces the reference's per-row Eigen/kissfft calls (proj/src/fft.cpp:26-50). One CTA
// transforms `rows` rows of length M (power of two, 32 <= M <= 8192) that already sit in
// shared memory with the pad16() layout and row stride padded_len(M). Each row is served
// by M/16 threads; passes are radix-16 (registers) with a final radix-2/4/8 pass, one
// smem exchange per pass (Stockham autosort, natural-order output). Twiddles come from a
// per-length table e^{-2 pi i k / M} built on the host in fp64.
//
// Only the forward (e^{-i}) transform is implemented; inverse transforms conjugate on load
// and on store (ifft(x) = conj(fft(conj(x))), unscaled; the 1/m factors are folded into
// the deapodisation table).
#pragma once
#include "common.cuh"

namespace tomo_b200 {

template <int RADIX, typename C2>
struct Dft;

template <typename C2>
struct Dft<2, C2> {
  static TOMO_DEV void run(C2* v) {
    const C2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <typename C2>
struct Dft<4, C2> {
  static TOMO_DEV void run(C2* v) {
    const C2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
    const C2 a2 = cadd(v[1], v[3]), a3 = cmul_negi(csub(v[1], v[3]));
    v[0] = cadd(a0, a2);
    v[2] = csub(a0, a2);
    v[1] = cadd(a1, a3);
    v[3] = csub(a1, a3);
  }
};

template <typename C2>
struct Dft<8, C2> {
  static TOMO_DEV void run(C2* v) {
    using R = decltype(C2::x);
    const R h = R(0.70710678118654752440);
    C2 e[4] = {v[0], v[2], v[4], v[6]};
    C2 o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4, C2>::run(e);
    Dft<4, C2>::run(o);
    // o[k] *= W8^k
    o[1] = mk<C2>(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
    o[2] = cmul_negi(o[2]);
    o[3] = mk<C2>(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = cadd(e[k], o[k]);
      v[k + 4] = csub(e[k], o[k]);
    }
  }
};

template <typename C2>
struct Dft<16, C2> {
  static TOMO_DEV void run(C2* v) {
  // n = n1 + 4 n2, k = k2 + 4 k1:  inner DFT4 over n2, twiddle W16^{n1 k2}, outer DFT4 over n1.
  using R = decltype(C2::x);
  const R c1 = R(0.92387953251128675613), s1 = R(0.38268343236508977173);
  const R h = R(0.70710678118654752440);
  C2 x[4][4];
#pragma unroll
  for (int n1 = 0; n1 < 4; ++n1) {
    x[n1][0] = v[n1];
    x[n1][1] = v[n1 + 4];
    x[n1][2] = v[n1 + 8];
    x[n1][3] = v[n1 + 12];
    Dft<4, C2>::run(x[n1]);
  }
  // twiddles W16^{n1*k2}, n1,k2 in 1..3
  x[1][1] = cmul(x[1][1], mk<C2>(c1, -s1));
  x[1][2] = cmul(x[1][2], mk<C2>(h, -h));
  x[1][3] = cmul(x[1][3], mk<C2>(s1, -c1));
  x[2][1] = cmul(x[2][1], mk<C2>(h, -h));
  x[2][2] = cmul_negi(x[2][2]);
  x[2][3] = cmul(x[2][3], mk<C2>(-h, -h));
  x[3][1] = cmul(x[3][1], mk<C2>(s1, -c1));
  x[3][2] = cmul(x[3][2], mk<C2>(-h, -h));
  x[3][3] = cmul(x[3][3], mk<C2>(-c1, s1));
#pragma unroll
  for (int k2 = 0; k2 < 4; ++k2) {
    C2 y[4] = {x[0][k2], x[1][k2], x[2][k2], x[3][k2]};
    Dft<4, C2>::run(y);
    v[k2] = y[0];
    v[k2 + 4] = y[1];
    v[k2 + 8] = y[2];
    v[k2 + 12] = y[3];
  }
  }
};

template <int M>
struct FftShape {
  static constexpr int LOG = (M >= 8192) ? 13 : (M >= 4096) ? 12 : (M >= 2048) ? 11 : (M >= 1024) ? 10
                           : (M >= 512) ? 9 : (M >= 256) ? 8 : (M >= 128) ? 7 : (M >= 64) ? 6 : 5;
  static constexpr int N16 = LOG / 4;          // number of radix-16 passes
  static constexpr int RL = 1 << (LOG % 4);    // final radix (1 = none)
  static constexpr int T = M / 16;             // threads per row
  static constexpr int STRIDE = padded_len(M); // smem row stride (float2)
  static_assert((1 << LOG) == M, "M must be a power of two in [32, 8192]");
};

// One Stockham pass of radix R with sub-transform size Ns over a row in smem.
// Thread `t` (0..T-1) of the row handles butterflies j = t, t+T, ... (M/R of them).
// Every thread of the CTA executes both barriers; `active` gates the work only.
template <int M, int R, typename C2>
TOMO_DEV void stockham_pass(C2* row, const C2* __restrict__ tw, int Ns, int t, bool active) {
  constexpr int T = M / 16;
  constexpr int NB = M / R;        // butterflies per pass
  constexpr int PER = NB / T;      // butterflies per thread (16/R)
  C2 v[PER][R];
  if (active) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int j = t + q * T;
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = row[pad16(j + r * NB)];
      if (Ns > 1) {
        const int jm = j & (Ns - 1);
        const int step = (M / (Ns * R)) * jm;  // twiddle index increment per r
#pragma unroll
        for (int r = 1; r < R; ++r) v[q][r] = cmul(v[q][r], __ldg(&tw[r * step]));
      }
      Dft<R, C2>::run(v[q]);
    }
  }
  __syncthreads();
  if (active) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int j = t + q * T;
      const int jm = j & (Ns - 1);
      const int base = (j - jm) * R + jm;
#pragma unroll
      for (int r = 0; r < R; ++r) row[pad16(base + r * Ns)] = v[q][r];
    }
  }
  __syncthreads();
}

// Forward FFT of one row per thread group, in place in smem. All threads of the CTA must
// call it (it contains barriers); `t` = thread index within the row (0..M/16-1), and
// threads without a row pass active = false.
template <int M, typename C2>
TOMO_DEV void fft_row_smem(C2* row, const C2* __restrict__ tw, int t, bool active) {
  using S = FftShape<M>;
  __syncthreads();
  int Ns = 1;
#pragma unroll
  for (int p = 0; p < S::N16; ++p) {
    stockham_pass<M, 16, C2>(row, tw, Ns, t, active);
    Ns *= 16;
  }
  if constexpr (S::RL > 1) stockham_pass<M, S::RL, C2>(row, tw, Ns, t, active);
}

}  // namespace tomo_b200
