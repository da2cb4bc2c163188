// ntt.cuh -- block-level negacyclic NTT / INTT over one RNS limb (C-3).
//
// One CTA transforms one limb of N = 2^LOGN words.  The 14 (for N = 2^14)
// radix-2 stages run as three "merged-butterfly" passes: every thread loads a
// group of 2^K words into registers, runs K stages there, and writes the group
// back; passes exchange data through a padded shared-memory buffer (one pad word
// per 16, which makes every pass's 64-bit accesses bank-conflict free).  The
// first pass reads its inputs through a caller functor (sampling, global loads
// fused in) and the last pass hands its outputs to a caller functor (pointwise
// products, additions, stores fused in), so a full encryption makes exactly one
// trip through HBM.
//
// Indexing.  Forward Cooley-Tukey stage s (0..LOGN-1) splits the array into
// 2^s blocks of N/2^s words; block beta uses the twiddle W[2^s + beta] with
// W[i] = psi^brv(i) (natural-order input, bit-reversed output, exactly C-3).
// A pass over stages [S0, S0+K) works on groups {base + r*T : r < 2^K},
// T = N >> (S0+K), base = beta * (N >> S0) + o, o < T.  The inverse runs the same
// structure backwards with Gentleman-Sande butterflies and W^-1[i] = psi^-brv(i);
// the N^-1 scaling is folded into its last stage.
#pragma once

#include "common.cuh"

namespace zinc {

// Twiddle pair {w, floor(w 2^64 / q)}.
using Tw = ulonglong2;

ZINC_DEV Tw ldtw(const Tw *p) { return __ldg(p); }

// Padded shared-memory index (1 pad word per 16).
ZINC_DEV int pad16(int i) { return i + (i >> 4); }
template <int LOGN>
struct SmemWords { static constexpr int value = (1 << LOGN) + ((1 << LOGN) >> 4); };

// ---------------------------------------------------------------- forward pass
// Load(idx) -> uint64 in [0, 4q); Store(idx, v) with v in [0, 4q).  With
// GROUPED, Store is called once per group as store(base, v) with the 2^K words
// of the group (T == 1: contiguous words base .. base + 2^K - 1).
template <int LOGN, int S0, int K, int THREADS, bool GROUPED = false, class Load, class Store>
ZINC_DEV void ct_pass(const Tw *__restrict__ tw, uint64_t q, Load load, Store store) {
  constexpr int N = 1 << LOGN;
  constexpr int G = 1 << K;
  constexpr int T = N >> (S0 + K);
  constexpr int NGROUPS = N / G;
  const uint64_t two_q = 2 * q;
#pragma unroll 1
  for (int g = threadIdx.x; g < NGROUPS; g += THREADS) {
    const int beta = g / T, o = g % T;
    const int base = beta * (T << K) + o;
    uint64_t v[G];
#pragma unroll
    for (int r = 0; r < G; ++r) v[r] = load(base + r * T);
#pragma unroll
    for (int l = 0; l < K; ++l) {
      const int D = G >> (l + 1);
#pragma unroll
      for (int blk = 0; blk < (1 << l); ++blk) {
        const Tw w = ldtw(tw + (1 << (S0 + l)) + (beta << l) + blk);
#pragma unroll
        for (int j = 0; j < D; ++j) ct_bfly(v[blk * 2 * D + j], v[blk * 2 * D + j + D], w.x, w.y, q, two_q);
      }
    }
    if constexpr (GROUPED) {
      store(base, v);
    } else {
#pragma unroll
      for (int r = 0; r < G; ++r) store(base + r * T, v[r]);
    }
  }
}

// ---------------------------------------------------------------- inverse pass
// Load -> [0, 2q); Store gets [0, 2q).  When LAST (S0 == 0), stage 0 multiplies
// the sum by N^-1 and the difference by N^-1 psi^-brv(1) (folded scaling).
// With GROUPED, Load is called once per group as load(base, v).
template <int LOGN, int S0, int K, int THREADS, bool GROUPED = false, class Load, class Store>
ZINC_DEV void gs_pass(const Tw *__restrict__ itw, const LimbConst &c, Load load, Store store) {
  constexpr int N = 1 << LOGN;
  constexpr int G = 1 << K;
  constexpr int T = N >> (S0 + K);
  constexpr int NGROUPS = N / G;
  const uint64_t q = c.q, two_q = c.two_q;
#pragma unroll 1
  for (int g = threadIdx.x; g < NGROUPS; g += THREADS) {
    const int beta = g / T, o = g % T;
    const int base = beta * (T << K) + o;
    uint64_t v[G];
    if constexpr (GROUPED) {
      load(base, v);
    } else {
#pragma unroll
      for (int r = 0; r < G; ++r) v[r] = load(base + r * T);
    }
#pragma unroll
    for (int l = K - 1; l >= 0; --l) {
      const int D = G >> (l + 1);
      if (S0 == 0 && l == 0) {
        // last stage (single block, twiddle psi^-brv(1)) with N^-1 folded in
#pragma unroll
        for (int j = 0; j < D; ++j) {
          uint64_t X = v[j], Y = v[j + D];
          uint64_t s = X + Y;                 // [0, 4q)
          uint64_t d = X - Y + two_q;         // (0, 4q)
          v[j] = mul_shoup_lazy(s, c.ninv, c.ninv_sh, q);
          v[j + D] = mul_shoup_lazy(d, c.ninv_w, c.ninv_w_sh, q);
        }
      } else {
#pragma unroll
        for (int blk = 0; blk < (1 << l); ++blk) {
          const Tw w = ldtw(itw + (1 << (S0 + l)) + (beta << l) + blk);
#pragma unroll
          for (int j = 0; j < D; ++j) gs_bfly(v[blk * 2 * D + j], v[blk * 2 * D + j + D], w.x, w.y, q, two_q);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < G; ++r) store(base + r * T, v[r]);
  }
}

// ---------------------------------------------------------------- pass plans
// THREADS and the (S0, K) of the three passes per ring degree.  The last
// forward pass (first inverse pass) always has K = 4 and T = 1: groups of 16
// contiguous words (one pad word each), which the fused epilogues rely on.
template <int LOGN> struct Plan;
template <> struct Plan<12> { static constexpr int THREADS = 256, KA = 4, KB = 4, KC = 4; };
template <> struct Plan<13> { static constexpr int THREADS = 256, KA = 5, KB = 4, KC = 4; };
template <> struct Plan<14> { static constexpr int THREADS = 512, KA = 5, KB = 5, KC = 4; };

// Forward NTT: pass A from `load`, passes B, C through smem; `gstore(base, v[16])`
// receives each group of 16 contiguous outputs (bit-reversed NTT order, C-3).
template <int LOGN, class Load, class GStore>
ZINC_DEV void ntt_forward(uint64_t *sm, const Tw *tw, uint64_t q, Load load, GStore gstore) {
  using P = Plan<LOGN>;
  constexpr int SB = P::KA, SC = P::KA + P::KB;
  static_assert(SC + P::KC == LOGN && P::KC == 4, "plan");
  __syncthreads();  // the previous transform may still read sm
  ct_pass<LOGN, 0, P::KA, P::THREADS>(tw, q, load, [&](int i, uint64_t v) { sm[pad16(i)] = v; });
  __syncthreads();
  ct_pass<LOGN, SB, P::KB, P::THREADS>(tw, q, [&](int i) { return sm[pad16(i)]; },
                                        [&](int i, uint64_t v) { sm[pad16(i)] = v; });
  __syncthreads();
  ct_pass<LOGN, SC, P::KC, P::THREADS, true>(tw, q, [&](int i) { return sm[pad16(i)]; }, gstore);
}

// Inverse NTT: `gload(base, v[16])` supplies each group of 16 contiguous inputs
// in [0, 2q); passes B', A' through smem; `store(idx, v)` gets the natural-order
// outputs in [0, 2q) at indices o + r*T with lane-consecutive o (coalesced).
template <int LOGN, class GLoad, class Store>
ZINC_DEV void ntt_inverse(uint64_t *sm, const Tw *itw, const LimbConst &c, GLoad gload, Store store) {
  using P = Plan<LOGN>;
  constexpr int SB = P::KA, SC = P::KA + P::KB;
  __syncthreads();
  gs_pass<LOGN, SC, P::KC, P::THREADS, true>(itw, c, gload, [&](int i, uint64_t v) { sm[pad16(i)] = v; });
  __syncthreads();
  gs_pass<LOGN, SB, P::KB, P::THREADS>(itw, c, [&](int i) { return sm[pad16(i)]; },
                                        [&](int i, uint64_t v) { sm[pad16(i)] = v; });
  __syncthreads();
  gs_pass<LOGN, 0, P::KA, P::THREADS>(itw, c, [&](int i) { return sm[pad16(i)]; }, store);
}

}  // namespace zinc
