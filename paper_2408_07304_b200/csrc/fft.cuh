// fft.cuh -- FP64 complex FFT passes for CKKS encoding / decoding (C-6, C-10).
//
// Encoding (derivation in DESIGN.md "Encoding"): with M = N/2, g_k = 5^k mod 2N
// = 1 + 4 h_k, and w_j = m_j + i m_{j+M},
//     w_j = (Delta / M) zeta^-j sum_h y_h exp(-2 pi i h j / M),   y_{h_k} = z_k.
// So encode = scatter z_k to brv(h_k), a decimation-in-time FFT (bit-reversed
// input, natural output), a twist by zeta^-j Delta/M and round-half-away of the
// real / imaginary parts into m_j / m_{j+M}.  Decoding is the mirror image:
// twist by zeta^+j, a decimation-in-frequency FFT with the + sign (natural input,
// bit-reversed output), and a gather at brv(h_k).
//
// Passes use the same merged-butterfly structure as the NTT: a pass over stages
// [S0, S0+K) loads groups {base + r 2^S0}, base = beta 2^(S0+K) + o, o < 2^S0.
// The butterfly at stage s between positions x and x + 2^s uses W_M^e,
// e = (x mod 2^s) (M >> (s+1)), W_M = exp(-2 pi i / M) (encode) or its conjugate.
#pragma once

#include "common.cuh"

namespace zinc {

ZINC_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
ZINC_DEV double2 csubd(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
ZINC_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
ZINC_DEV double2 conj2(double2 a) { return make_double2(a.x, -a.y); }

// TWS: twiddle-table stride.  The table holds W_M^e of the full transform; a
// CTA running an M/2-point sub-transform (the split N = 2^15 case) reads it
// with stride 2 (W_{M/2}^e = W_M^{2e}).
// TW_SMEM: 1 the table lives in shared memory (plain loads instead of __ldg), 2 padded (fft_twpad).
template <int LOGM, int S0, int K, int THREADS, bool DIT, bool CONJ, int TWS = 1, int TW_SMEM = 0, class Load,
          class Store>
ZINC_DEV void fft_pass(const double2 *__restrict__ tw, Load load, Store store) {
  constexpr int M = 1 << LOGM;
  constexpr int G = 1 << K;
  constexpr int T = 1 << S0;
  constexpr int NGROUPS = M / G;
#pragma unroll 1
  for (int g = threadIdx.x; g < NGROUPS; g += THREADS) {
    const int beta = g / T, o = g % T;
    const int base = beta * (T << K) + o;
    double2 v[G];
#pragma unroll
    for (int r = 0; r < G; ++r) v[r] = load(base + r * T);
    if constexpr (DIT) {
#pragma unroll
      for (int l = 0; l < K; ++l) {
        const int D = 1 << l;
#pragma unroll
        for (int r = 0; r < G; ++r) {
          if (r & D) continue;
          const int e = (o + (r & (D - 1)) * T) * (M >> (S0 + l + 1)) * TWS;
          double2 w = TW_SMEM == 2 ? tw[fft_twpad(e)] : TW_SMEM ? tw[e] : __ldg(tw + e);
          if (CONJ) w = conj2(w);
          const double2 b = cmul(v[r + D], w);
          v[r + D] = csubd(v[r], b);
          v[r] = cadd(v[r], b);
        }
      }
    } else {
#pragma unroll
      for (int l = K - 1; l >= 0; --l) {
        const int D = 1 << l;
#pragma unroll
        for (int r = 0; r < G; ++r) {
          if (r & D) continue;
          const int e = (o + (r & (D - 1)) * T) * (M >> (S0 + l + 1)) * TWS;
          double2 w = TW_SMEM == 2 ? tw[fft_twpad(e)] : TW_SMEM ? tw[e] : __ldg(tw + e);
          if (CONJ) w = conj2(w);
          const double2 a = v[r], b = v[r + D];
          v[r] = cadd(a, b);
          v[r + D] = cmul(csubd(a, b), w);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < G; ++r) store(base + r * T, v[r]);
  }
}

// Three-pass plans (stages 0..LOGM-1 split as 4 + 4 + rest), 256 threads.
template <int LOGM> struct FftPlan {
  static constexpr int THREADS = 256, K1 = 4, K2 = 4, K3 = LOGM - 8;
};

}  // namespace zinc
