// fft.cuh — in-CTA Stockham FFT rows (sm_100a).
//
// Replaces the reference's per-row Eigen/kissfft calls (proj/src/fft.cpp:26-50). A CTA
// transforms `rpc` rows of length M (power of two, 32 <= M <= 8192); each row is served by
// M/16 threads. Passes are radix-16 in registers with a final radix-2/4/8 pass (Stockham
// autosort, natural-order output). The FIRST pass loads its 16 inputs per thread straight
// from global memory through a caller-supplied loader (coalesced: thread j reads j + r*M/16)
// and the LAST pass hands its outputs straight to a caller-supplied storer (coalesced for the
// natural-order row stores); only the middle exchanges go through shared memory (pad16
// layout, conflict-free). Twiddles w^1, w^2, w^4, w^8 come from a per-length fp64-built
// table e^{-2 pi i k/M}; the other powers are products of those (<= 3 roundings deep).
//
// Only the forward (e^{-i}) transform is implemented; inverse transforms conjugate on load
// and on store (ifft(x) = conj(fft(conj(x))), unscaled; the 1/m factors are folded into
// the deapodisation table).
#pragma once
#include "common.cuh"

#ifndef TOMO_TW_SPLIT_M
#define TOMO_TW_SPLIT_M 4096  // rows at least this long use split twiddle reads (A/B: 1 << 30 = never)
#endif

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

// Row of length M served by T = M/RB threads: passes of radix RB (16, 8 or 4) and a final
// smaller radix RL. A smaller base radix gives more threads per row and fewer registers per
// thread (more warps for small, latency-bound problems) at the cost of one more smem pass.
template <int M, int RB = 16>
struct FftShape {
  static constexpr int LOG = (M >= 8192) ? 13 : (M >= 4096) ? 12 : (M >= 2048) ? 11 : (M >= 1024) ? 10
                           : (M >= 512) ? 9 : (M >= 256) ? 8 : (M >= 128) ? 7 : (M >= 64) ? 6 : 5;
  static constexpr int LB = RB == 16 ? 4 : RB == 8 ? 3 : 2;  // log2(RB)
  static constexpr int NB = LOG / LB;                          // number of radix-RB passes
  static constexpr int RL = 1 << (LOG % LB);                   // final radix (1 = none)
  static constexpr int NP = NB + (RL > 1 ? 1 : 0);
  static constexpr int T = M / RB;                             // threads per row
  static constexpr int STRIDE = padded_len(M);                 // smem row stride (elements)
  static_assert(RB == 16 || RB == 8 || RB == 4, "base radix");
  static_assert((1 << LOG) == M, "M must be a power of two in [32, 8192]");
  static_assert(NP >= 2, "at least two passes");
};

// Twiddle table entry W^i. SPLIT (long rows, M >= 4096: the 64-128 KB table does not stay in
// L1 next to the CTA's row buffer): W^i = W^(i & ~63) * W^(i & 63), two reads from a 17 KB
// L1-resident subset of the same table, one extra rounding.
template <bool SPLIT, typename C2>
TOMO_DEV C2 tw_at(const C2* __restrict__ tw, int i) {
  if constexpr (SPLIT) {
    const int lo = i & 63;  // tw[0] = 1 exactly: the product is exact for lo = 0
    return cmul(__ldg(&tw[i - lo]), __ldg(&tw[lo]));
  } else {
    return __ldg(&tw[i]);
  }
}

// v[r] *= W^{r * base} for r = 1..R-1, W = e^{-2 pi i / M}: four table loads, the rest by
// products (w3 = w1 w2, w5 = w4 w1, ..., w15 = w8 w7).
template <int R, typename C2, bool SPLIT = false>
TOMO_DEV void twiddle(C2* v, const C2* __restrict__ tw, int base) {
  const C2 w1 = tw_at<SPLIT>(tw, base);
  v[1] = cmul(v[1], w1);
  if constexpr (R >= 4) {
    const C2 w2 = tw_at<SPLIT>(tw, 2 * base);
    const C2 w3 = cmul(w1, w2);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
    if constexpr (R >= 8) {
      const C2 w4 = tw_at<SPLIT>(tw, 4 * base);
      const C2 w5 = cmul(w4, w1), w6 = cmul(w4, w2), w7 = cmul(w4, w3);
      v[4] = cmul(v[4], w4);
      v[5] = cmul(v[5], w5);
      v[6] = cmul(v[6], w6);
      v[7] = cmul(v[7], w7);
      if constexpr (R >= 16) {
        const C2 w8 = tw_at<SPLIT>(tw, 8 * base);
        v[8] = cmul(v[8], w8);
        v[9] = cmul(v[9], cmul(w8, w1));
        v[10] = cmul(v[10], cmul(w8, w2));
        v[11] = cmul(v[11], cmul(w8, w3));
        v[12] = cmul(v[12], cmul(w8, w4));
        v[13] = cmul(v[13], cmul(w8, w5));
        v[14] = cmul(v[14], cmul(w8, w6));
        v[15] = cmul(v[15], cmul(w8, w7));
      }
    }
  }
}

// Compile-time pruning (PR) for rows whose non-zero inputs / kept outputs are exactly the
// first and last quarter of the row (n = M/2, the reference's 2x oversampling): bit 0 — the
// first pass treats inputs M/4 <= i < 3M/4 as zeros (no loads, no arithmetic on them); bit 1 —
// the last pass computes and stores only outputs k < M/4 and k >= 3M/4. Both need radix >= 4
// for that pass (its r-th input / output then lies in the middle half iff R/4 <= r < 3R/4).
template <int R>
TOMO_DEV constexpr bool mid_quarter(int r) { return R >= 4 && r >= R / 4 && r < 3 * R / 4; }

// One Stockham pass (radix R, sub-transform size NS) of the row owned by this thread group.
// FIRST: inputs come from load(i) (global), otherwise from the smem row. LAST: outputs go to
// store(k, value), otherwise back into the smem row. Every thread of the CTA must call each
// pass (barriers inside); `active` gates the work. STORE_SMEM_LAST: the storer writes the smem
// row, so a barrier separates the last reads from those writes.
// NS is a compile-time constant, so whenever the padded (pad16) smem positions of a thread's
// elements differ by compile-time amounts — reads when T and M/R are multiples of 16, writes
// when NS is (or NS = 1 with R = 16) — they are addressed as one base pointer plus immediate
// offsets instead of a pad16 computation per element.
template <int M, int RB, int R, bool FIRST, bool LAST, bool STORE_SMEM_LAST, typename C2, int PR, int NS,
          typename Load, typename Store>
TOMO_DEV void fft_pass(C2* row, const C2* __restrict__ tw, int t, bool active, Load& load, Store& store,
                       const C2* tws = nullptr) {
  constexpr int T = M / RB;
  constexpr int NB = M / R;    // butterflies per pass
  constexpr int PER = NB / T;  // butterflies per thread (RB/R)
  constexpr bool RD_CONST = (T % 16 == 0) && (NB % 16 == 0);
  constexpr bool WR_CONST = (NS % 16 == 0) || (NS == 1 && R == 16);
  C2 v[PER][R];
  if (active) {
    const C2* rd = row + pad16(t);
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int j = t + q * T;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (FIRST && (PR & 1) && mid_quarter<R>(r))
          v[q][r] = czero<C2>();
        else if (FIRST)
          v[q][r] = load(j + r * NB);
        else if constexpr (RD_CONST)
          v[q][r] = rd[q * (T + T / 16) + r * (NB + NB / 16)];
        else
          v[q][r] = row[pad16(j + r * NB)];
      }
      if (!FIRST) {
        const int jm = j & (NS - 1);
        if (jm) {
          if (R == RB && NS == RB && tws) {
            // second pass: the RB - 1 twiddles of sub-transform jm from the CTA's smem table
            // layout [r][jm]: the lanes of a warp (consecutive jm) read consecutive entries
#pragma unroll
            for (int r = 1; r < R; ++r) v[q][r] = cmul(v[q][r], tws[r * RB + jm]);
          } else {
            twiddle<R, C2, (M >= TOMO_TW_SPLIT_M)>(v[q], tw, (M / (NS * R)) * jm);
          }
        }
      }
      Dft<R, C2>::run(v[q]);
    }
  }
  if (!FIRST && (!LAST || STORE_SMEM_LAST)) __syncthreads();
  if (active) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int j = t + q * T;
      const int jm = j & (NS - 1);
      const int base = (j - jm) * R + jm;
      C2* wr = row + pad16(base);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (LAST && (PR & 2) && mid_quarter<R>(r)) continue;
        if (LAST)
          store(base + r * NS, v[q][r]);
        else if constexpr (WR_CONST)
          wr[r * (NS + NS / 16)] = v[q][r];
        else
          row[pad16(base + r * NS)] = v[q][r];
      }
    }
  }
  if (!LAST || STORE_SMEM_LAST) __syncthreads();
}

// Twiddles of the second pass (Ns = RB, radix RB): entry [r][jm] = W^(r * jm * M / RB^2), the same
// for every row of the CTA. Filled before the first pass (whose closing barrier publishes it);
// the pass then reads its RB - 1 twiddles from smem instead of 4 table loads + 11 products.
// TOMO_TWS=0 (A/B) keeps the table-load path.
#ifndef TOMO_TWS
#define TOMO_TWS 1
#endif
template <int M, int RB, typename C2>
TOMO_DEV const C2* fill_tws(const C2* __restrict__ tw) {
  if constexpr (TOMO_TWS && RB * RB <= M) {
    __shared__ __align__(16) C2 tws[RB * RB];
    for (int k = threadIdx.x; k < RB * RB; k += blockDim.x) {
      const int r = k / RB, jm = k % RB;
      tws[k] = __ldg(&tw[(M / (RB * RB)) * jm * r]);
    }
    return tws;
  } else {
    return nullptr;
  }
}

constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

// Passes P, P+1, ... of a row after the first: radix RB with sub-transform size RB^P, then the
// last pass (radix RL, or RB when RL = 1), which hands its outputs to the storer.
template <int M, int RB, bool STORE_SMEM, typename C2, int PR, int P, typename Store>
TOMO_DEV void fft_rest(C2* row, const C2* __restrict__ tw, int t, bool active, Store& store, const C2* tws) {
  using S = FftShape<M, RB>;
  constexpr int NS = ipow(RB, P);
  auto noload = [](int) { return C2{}; };
  if constexpr (S::RL > 1) {
    if constexpr (P < S::NB) {
      fft_pass<M, RB, RB, false, false, false, C2, 0, NS>(row, tw, t, active, noload, store, tws);
      fft_rest<M, RB, STORE_SMEM, C2, PR, P + 1>(row, tw, t, active, store, tws);
    } else {
      fft_pass<M, RB, S::RL, false, true, STORE_SMEM, C2, PR & 2, NS>(row, tw, t, active, noload, store, tws);
    }
  } else {
    if constexpr (P < S::NB - 1) {
      fft_pass<M, RB, RB, false, false, false, C2, 0, NS>(row, tw, t, active, noload, store, tws);
      fft_rest<M, RB, STORE_SMEM, C2, PR, P + 1>(row, tw, t, active, store, tws);
    } else {
      fft_pass<M, RB, RB, false, true, STORE_SMEM, C2, PR & 2, NS>(row, tw, t, active, noload, store, tws);
    }
  }
}

// Forward FFT whose first-pass inputs were loaded earlier into registers: pre[r] holds the
// element at position t + r*M/RB (what load(t + r*M/RB) would return). Lets a persistent
// kernel prefetch the next row while the current one is transformed.
template <int M, int RB, bool STORE_SMEM, typename C2, int PR = 0, typename Store>
TOMO_DEV void fft_row_pre(C2* row, const C2* __restrict__ tw, int t, bool active, const C2 (&pre)[RB],
                          Store&& store) {
  using S = FftShape<M, RB>;
  static_assert(S::T * RB == M, "one first-pass butterfly per thread");
  const C2* tws = fill_tws<M, RB, C2>(tw);
  if (active) {
    C2 v[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) v[r] = pre[r];
    Dft<RB, C2>::run(v);
#pragma unroll
    for (int r = 0; r < RB; ++r) row[pad16(t * RB + r)] = v[r];  // Stockham output of the Ns = 1 pass
  }
  __syncthreads();
  fft_rest<M, RB, STORE_SMEM, C2, PR, 1>(row, tw, t, active, store, tws);
}

// Forward FFT of one row per thread group: load(i) -> ... -> store(k, X[k]).
template <int M, int RB, bool STORE_SMEM, typename C2, int PR = 0, typename Load, typename Store>
TOMO_DEV void fft_row(C2* row, const C2* __restrict__ tw, int t, bool active, Load&& load, Store&& store) {
  const C2* tws = fill_tws<M, RB, C2>(tw);
  fft_pass<M, RB, RB, true, false, false, C2, PR & 1, 1>(row, tw, t, active, load, store);
  fft_rest<M, RB, STORE_SMEM, C2, PR, 1>(row, tw, t, active, store, tws);
}

}  // namespace tomo_b200
