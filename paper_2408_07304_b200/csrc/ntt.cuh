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
// Two consecutive twiddle pairs (one 32-byte sector, p 32-byte aligned) in one 256-bit load
// (sm_100's LDG.256): the late stages' groups use 2, 4, 8 consecutive table entries, and two
// 128-bit loads of one sector cost the L1 data pipe two sector accesses.
#ifndef ZINC_TW_LD256
#define ZINC_TW_LD256 1
#endif
ZINC_DEV void ldtw2(const Tw *p, Tw &a, Tw &b) {
#if ZINC_TW_LD256
  asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(a.x), "=l"(a.y), "=l"(b.x), "=l"(b.y) : "l"(p));
#else
  a = __ldg(p);
  b = __ldg(p + 1);
#endif
}

// Padded shared-memory index (1 pad word per 16).
ZINC_DEV int pad16(int i) { return i + (i >> 4); }
template <int LOGN>
struct SmemWords { static constexpr int value = (1 << LOGN) + ((1 << LOGN) >> 4); };

// A two-phase load (`fetch(idx)` -> raw int64 from global memory, `lift(raw, idx)` -> the
// residue) lets a pass issue all of its group's global loads before the first lift, so
// their latencies overlap instead of each one stalling the lift that consumes it.
template <class L, class = void> struct TwoPhase { static constexpr bool value = false; };
template <class L> struct TwoPhase<L, decltype((void)&L::fetch)> { static constexpr bool value = true; };
// A two-phase load may also offer `small(raw)` and `lift_small(raw, idx)`: a cheaper lift valid
// when small() holds for the raw value (e.g. |m| < q/2 for a CKKS plaintext word).  A pass
// takes it when it holds for every word of the whole warp's groups (one vote per group).
template <class L, class = void> struct HasSmallLift { static constexpr bool value = false; };
template <class L> struct HasSmallLift<L, decltype((void)&L::lift_small)> { static constexpr bool value = true; };
// ... or decide it once for every word it will ever load: uniform_small() (a CTA-uniform flag
// the kernel computed up front), which spares the per-word test and the warp vote.
template <class L, class = void> struct HasUniformSmall { static constexpr bool value = false; };
template <class L> struct HasUniformSmall<L, decltype((void)&L::uniform_small)> { static constexpr bool value = true; };

struct NoHook {
  ZINC_DEV void operator()() const {}
};

// ---------------------------------------------------------------- forward pass
// Load(idx) -> uint64 in [0, 4q); Store(idx, v) with v in [0, 8q) (ct_bfly_a), or below 2^64 with NR.  With
// GROUPED, Store is called once per group as store(base, v) with the 2^K words
// of the group (T == 1: contiguous words base .. base + 2^K - 1).
// SMEM_TW: `tw` points to a shared-memory copy of the table (the early passes'
// indices are all < kSmemTw).  pre_store() runs before each group's first store (the
// split transforms, one group per thread, settle a deferred cluster rendezvous there).
template <int LOGN, int S0, int K, int THREADS, bool GROUPED = false, bool SMEM_TW = false, bool NR = false,
          class Load, class Store, class PreStore = NoHook>
ZINC_DEV void ct_pass(const Tw *__restrict__ tw, uint64_t q, int tb, Load load, Store store,
                      PreStore pre_store = PreStore()) {
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
    if constexpr (TwoPhase<Load>::value) {
      int64_t raw[G];
#pragma unroll
      for (int r = 0; r < G; ++r) raw[r] = load.fetch(base + r * T);
      bool small = HasSmallLift<Load>::value;
      if constexpr (HasUniformSmall<Load>::value) {
        small = load.uniform_small();
      } else if constexpr (HasSmallLift<Load>::value) {
#pragma unroll
        for (int r = 0; r < G; ++r) small &= load.small(raw[r]);
        small = __all_sync(0xffffffffu, small);
      }
      if (small) {
        if constexpr (HasSmallLift<Load>::value) {
#pragma unroll
          for (int r = 0; r < G; ++r) v[r] = load.lift_small(raw[r], base + r * T);
        }
      } else {
#pragma unroll
        for (int r = 0; r < G; ++r) v[r] = load.lift(raw[r], base + r * T);
      }
    } else {
#pragma unroll
      for (int r = 0; r < G; ++r) v[r] = load(base + r * T);
    }
    // global-memory twiddles of this group: all 2^K - 1 issued before the first butterfly
    constexpr bool PRE = !SMEM_TW && K <= 4;
    Tw wpre[PRE ? G - 1 : 1];
    if constexpr (PRE) {
#pragma unroll
      for (int l = 0; l < K; ++l) {
        const Tw *p = tw + (tb << (S0 + l)) + (beta << l);  // an even index for l >= 1
        if (l == 0) {
          wpre[0] = ldtw(p);
        } else {
#pragma unroll
          for (int blk = 0; blk < (1 << l); blk += 2) ldtw2(p + blk, wpre[(1 << l) - 1 + blk], wpre[(1 << l) + blk]);
        }
      }
    }
#pragma unroll
    for (int l = 0; l < K; ++l) {
      const int D = G >> (l + 1);
#pragma unroll
      for (int blk = 0; blk < (1 << l); ++blk) {
        const Tw w = PRE ? wpre[(1 << l) - 1 + blk]
                         : SMEM_TW ? tw[(tb << (S0 + l)) + (beta << l) + blk] : ldtw(tw + (tb << (S0 + l)) + (beta << l) + blk);
#pragma unroll
        for (int j = 0; j < D; ++j) {
          if constexpr (NR) ct_bfly_nr(v[blk * 2 * D + j], v[blk * 2 * D + j + D], w.x, w.y, q, two_q);
          else ct_bfly_a(v[blk * 2 * D + j], v[blk * 2 * D + j + D], w.x, w.y, q, 2 * two_q);
        }
      }
    }
    pre_store();
    if constexpr (GROUPED) {
      store(base, v);
    } else {
#pragma unroll
      for (int r = 0; r < G; ++r) store(base + r * T, v[r]);
    }
  }
}

// ---------------------------------------------------------------- inverse pass
// Load -> [0, 4q); intermediate values stay in [0, 4q); Store gets [0, 2q) after the folded last stage (FOLD), [0, 4q) otherwise.  When LAST (S0 == 0), stage 0 multiplies
// the sum by N^-1 and the difference by N^-1 psi^-brv(1) (folded scaling).
// With GROUPED, Load is called once per group as load(base, v).
template <int LOGN, int S0, int K, int THREADS, bool GROUPED = false, bool FOLD = true, bool SMEM_TW = false,
          class Load, class Store>
ZINC_DEV void gs_pass(const Tw *__restrict__ itw, const LimbConst &c, int tb, Load load, Store store) {
  constexpr int N = 1 << LOGN;
  constexpr int G = 1 << K;
  constexpr int T = N >> (S0 + K);
  constexpr int NGROUPS = N / G;
  const uint64_t q = c.q, four_q = 2 * c.two_q;
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
      if (FOLD && S0 == 0 && l == 0) {
        // last stage (single block, twiddle psi^-brv(1)) with N^-1 folded in
#pragma unroll
        for (int j = 0; j < D; ++j) {
          uint64_t X = v[j], Y = v[j + D];
          uint64_t s = X + Y;                 // [0, 8q)
          uint64_t d = X - Y + four_q;        // (0, 8q)
          v[j] = mul_shoup_lazy(s, c.ninv, c.ninv_sh, q);
          v[j + D] = mul_shoup_lazy(d, c.ninv_w, c.ninv_w_sh, q);
        }
      } else {
        const Tw *p = itw + (tb << (S0 + l)) + (beta << l);  // an even index for l >= 1
        if (SMEM_TW || l == 0) {
#pragma unroll
          for (int blk = 0; blk < (1 << l); ++blk) {
            const Tw w = SMEM_TW ? p[blk] : ldtw(p + blk);
#pragma unroll
            for (int j = 0; j < D; ++j) gs_bfly(v[blk * 2 * D + j], v[blk * 2 * D + j + D], w.x, w.y, q, four_q);
          }
        } else {
#pragma unroll
          for (int blk = 0; blk < (1 << l); blk += 2) {
            Tw w0, w1;
            ldtw2(p + blk, w0, w1);
#pragma unroll
            for (int j = 0; j < D; ++j) gs_bfly(v[blk * 2 * D + j], v[blk * 2 * D + j + D], w0.x, w0.y, q, four_q);
#pragma unroll
            for (int j = 0; j < D; ++j) gs_bfly(v[(blk + 1) * 2 * D + j], v[(blk + 1) * 2 * D + j + D], w1.x, w1.y, q, four_q);
          }
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

// ---------------------------------------------------------------- geometry
// N <= 2^14: one CTA holds a whole limb (2^14 words = 128 KiB + padding).
// N = 2^15: a limb (256 KiB) exceeds a CTA's 227 KB of shared memory, so a
// 2-CTA thread-block cluster splits it.  Forward (CT, natural input): stage 0
// pairs j with j + N/2 under one twiddle W[1]; CTA r computes half r of stage 0
// straight from its loads (X + W Y for r = 0, X - W Y for r = 1) and then runs
// the remaining stages as an independent N/2-point transform whose stage-s'
// blocks are the global stage-(s'+1) blocks r 2^s' + beta, i.e. twiddle index
// (2 + r) 2^s' + beta ("tb" below); its outputs are positions [r N/2, (r+1) N/2)
// of the bit-reversed result.  Inverse (GS, bit-reversed input): each CTA runs
// stages LOGN-1 .. 1 on its half, then stage 0 (with N^-1 folded in) exchanges
// halves through distributed shared memory: CTA r finishes j in
// [r N/4, (r+1) N/4) from both CTAs' buffers.
// LM: the largest log2 N one CTA transforms alone (14 fits 128 KiB + padding in one
// CTA's shared memory).  A kernel may choose LM = 13 at N = 2^14: two CTAs of 68 KiB per
// limb, two clusters per SM, so one CTA's barriers and memory phases overlap the
// other's butterflies (measured faster for the INTT-heavy kernels).
template <int LOGN, int LM = 14> struct Geo {
  static constexpr bool SPLIT = LOGN > LM;
  static constexpr int LOGL = SPLIT ? LOGN - 1 : LOGN;  // words per CTA = 2^LOGL
  static constexpr int NL = 1 << LOGL;
  static constexpr int CLUSTER = SPLIT ? 2 : 1;
  static constexpr int THREADS = Plan<LOGL>::THREADS;
  // CTAs per SM the kernels aim for (caps registers so they fit beside shared memory):
  // 2^12-word shares (~34 KiB) three, 2^13 (~68 KiB) two, 2^14 (~136 KiB) one.
  static constexpr int MINB = LOGL <= 12 ? 3 : LOGL == 13 ? 2 : 1;
};

ZINC_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
ZINC_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Generic pointer to the same shared-memory object in cluster CTA `rank`.
template <class T>
ZINC_DEV T *peer_smem(T *p, uint32_t rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(p), "r"(rank));
  return reinterpret_cast<T *>(out);
}
// Index offset of this CTA's share of a limb (0 unless split).
template <int LOGN, int LM = 14> ZINC_DEV int local_off() {
  if constexpr (Geo<LOGN, LM>::SPLIT) return (int)cluster_rank() * Geo<LOGN, LM>::NL;
  else return 0;
}

// Forward NTT: pass A from `load(x)` (x a global index, value in [0, 4q)),
// passes B, C through smem; `gstore(base, v[16])` receives each group of 16
// contiguous outputs (bit-reversed NTT order, C-3) at global position base.
// Entries of the twiddle tables the early passes touch (stages < SB + KB <= 10):
// kernels may stage them in shared memory (STW) and pass the copy as `stw`.
constexpr int kSmemTw = 1024;

// NR: lazy-free butterflies (q < 2^59; outputs < 2^64 instead of [0, 4q), reduce with reduce64).
template <int LOGN, bool STW = false, bool NR = false, int LM = 14, class Load, class GStore>
ZINC_DEV void ntt_forward(uint64_t *sm, const Tw *tw, uint64_t q, Load load, GStore gstore, const Tw *stw = nullptr) {
  using G = Geo<LOGN, LM>;
  using P = Plan<G::LOGL>;
  constexpr int LL = G::LOGL;
  constexpr int SB = P::KA, SC = P::KA + P::KB;
  static_assert(SC + P::KC == LL && P::KC == 4, "plan");
  auto sst = [&](int i, uint64_t v) { sm[pad16(i)] = v; };
  auto sld = [&](int i) { return sm[pad16(i)]; };
  __syncthreads();  // the previous transform may still read sm
  static_assert(!STW || (!G::SPLIT && (1 << (SC)) <= kSmemTw), "smem twiddles cover passes A and B");
  if constexpr (!G::SPLIT) {
    ct_pass<LL, 0, P::KA, P::THREADS, false, STW, NR>(STW ? stw : tw, q, 1, load, sst);
    __syncthreads();
    ct_pass<LL, SB, P::KB, P::THREADS, false, STW, NR>(STW ? stw : tw, q, 1, sld, sst);
    __syncthreads();
    ct_pass<LL, SC, P::KC, P::THREADS, true, false, NR>(tw, q, 1, sld, gstore);
  } else {
    const int r = (int)cluster_rank();
    const Tw w1 = ldtw(tw + 1);
    const uint64_t two_q = 2 * q;
    auto load0 = [&](int x) {
      const uint64_t X = NR ? load(x) : csub(load(x), two_q);
      const uint64_t t = mul_shoup_lazy(load(x + G::NL), w1.x, w1.y, q);
      return r == 0 ? X + t : X - t + two_q;
    };
    const int tb = 2 + r;
    ct_pass<LL, 0, P::KA, P::THREADS, false, false, NR>(tw, q, tb, load0, sst);
    __syncthreads();
    ct_pass<LL, SB, P::KB, P::THREADS, false, false, NR>(tw, q, tb, sld, sst);
    __syncthreads();
    ct_pass<LL, SC, P::KC, P::THREADS, true, false, NR>(tw, q, tb, sld,
        [&](int base, uint64_t (&v)[16]) { gstore(base + r * G::NL, v); });
  }
}

// Forward NTT of one limb by a 2-CTA cluster, split by input parity (no redundant work):
// a(X) = a_e(X^2) + X a_o(X^2), and with k = 2k' + b, C-3's order gives
//   a^[2k' + b] = E[k'] + (-1)^b psi^(2 brv'(k') + 1) O[k'],
// where E, O are the N/2-point transforms of a_e, a_o with root psi^2 in the same order.
// The N/2-point table with root psi^2 is the first half of the N-point table
// (brv_N(i) = 2 brv_{N/2}(i) for i < N/2) and psi^(2 brv'(k') + 1) = W[N/2 + k'], so CTA r
// runs the ordinary passes on inputs x = 2i + r, then the last stage exchanges halves over
// distributed shared memory: CTA r finishes k' in [r N/4, (r+1) N/4) and hands the output
// pair (2k', 2k'+1) -- global positions, values as the one-CTA transform's -- to
// `pair(x, v0, v1)`.  The pair function must not write shared memory (the partner may
// still be reading it); callers stream to global memory.
// after_b(): called by every thread once all threads are past pass B (the last use of stw).
template <int LOGN, bool STW = false, bool NR = false, class Load, class Pair, class AfterB = NoHook>
ZINC_DEV void ntt_forward_dit2(uint64_t *sm, const Tw *tw, uint64_t q, Load load, Pair pair,
                               const Tw *stw = nullptr, AfterB after_b = AfterB()) {
  constexpr int LL = LOGN - 1, NL = 1 << LL, QN = NL / 2;
  using P = Plan<LL>;
  constexpr int SB = P::KA, SC = P::KA + P::KB;
  static_assert(SC + P::KC == LL && P::KC == 4, "plan");
  static_assert(!STW || (1 << SC) <= kSmemTw, "smem twiddles cover passes A and B");
  auto sst = [&](int i, uint64_t v) { sm[pad16(i)] = v; };
  auto sld = [&](int i) { return sm[pad16(i)]; };
  const int r = (int)cluster_rank();
  __syncthreads();
  if constexpr (TwoPhase<Load>::value) {
    if constexpr (HasUniformSmall<Load>::value) {
      struct Parity {  // local index i -> coefficient 2 i + r
        const Load &l;
        int r;
        ZINC_DEV int64_t fetch(int i) const { return l.fetch(2 * i + r); }
        ZINC_DEV uint64_t lift(int64_t raw, int i) const { return l.lift(raw, 2 * i + r); }
        ZINC_DEV bool uniform_small() const { return l.uniform_small(); }
        ZINC_DEV uint64_t lift_small(int64_t raw, int i) const { return l.lift_small(raw, 2 * i + r); }
      };
      ct_pass<LL, 0, P::KA, P::THREADS, false, STW, NR>(STW ? stw : tw, q, 1, Parity{load, r}, sst);
    } else if constexpr (HasSmallLift<Load>::value) {
      struct Parity {  // local index i -> coefficient 2 i + r
        const Load &l;
        int r;
        ZINC_DEV int64_t fetch(int i) const { return l.fetch(2 * i + r); }
        ZINC_DEV uint64_t lift(int64_t raw, int i) const { return l.lift(raw, 2 * i + r); }
        ZINC_DEV bool small(int64_t raw) const { return l.small(raw); }
        ZINC_DEV uint64_t lift_small(int64_t raw, int i) const { return l.lift_small(raw, 2 * i + r); }
      };
      ct_pass<LL, 0, P::KA, P::THREADS, false, STW, NR>(STW ? stw : tw, q, 1, Parity{load, r}, sst);
    } else {
      struct Parity {  // local index i -> coefficient 2 i + r
        const Load &l;
        int r;
        ZINC_DEV int64_t fetch(int i) const { return l.fetch(2 * i + r); }
        ZINC_DEV uint64_t lift(int64_t raw, int i) const { return l.lift(raw, 2 * i + r); }
      };
      ct_pass<LL, 0, P::KA, P::THREADS, false, STW, NR>(STW ? stw : tw, q, 1, Parity{load, r}, sst);
    }
  } else {
    ct_pass<LL, 0, P::KA, P::THREADS, false, STW, NR>(STW ? stw : tw, q, 1, [&](int i) { return load(2 * i + r); },
                                                       sst);
  }
  __syncthreads();
  ct_pass<LL, SB, P::KB, P::THREADS, false, STW, NR>(STW ? stw : tw, q, 1, sld, sst);
  __syncthreads();
  after_b();
  ct_pass<LL, SC, P::KC, P::THREADS, true, false, NR>(tw, q, 1, sld, [&](int base, uint64_t (&v)[16]) {
#pragma unroll
    for (int j = 0; j < 16; ++j) sm[pad16(base + j)] = v[j];
  });
  cluster_sync_all();  // both halves transformed
  const uint64_t *he = peer_smem(sm, 0), *ho = peer_smem(sm, 1);
  const uint64_t two_q = 2 * q;
  constexpr int U = 4;
  static_assert(QN % (P::THREADS * U) == 0, "exchange tiling");
#pragma unroll 1
  for (int k0 = r * QN + threadIdx.x; k0 < (r + 1) * QN; k0 += P::THREADS * U) {
    uint64_t e[U], o[U];
    Tw w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * P::THREADS;
      e[u] = he[pad16(k)];
      o[u] = ho[pad16(k)];
      w[u] = ldtw(tw + NL + k);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * P::THREADS;
      const uint64_t E = NR ? e[u] : csub(csub(e[u], 2 * two_q), two_q);  // [0, 8q) -> [0, 2q)
      const uint64_t t = mul_shoup_lazy(o[u], w[u].x, w[u].y, q);
      pair(2 * k, E + t, E - t + two_q);
    }
  }
  cluster_sync_all();  // the partner finished reading this CTA's half
}

// Inverse NTT: `gload(base, v[16])` supplies each group of 16 contiguous inputs
// in [0, 2q) (global position base); `store(idx, v)` gets the natural-order
// outputs in [0, 2q) at global indices, lane-consecutive (coalesced).  When
// split, every store happens after both CTAs of the pair consumed their inputs
// (in-place use is safe).
template <int LOGN, bool STW = false, int LM = 14, class GLoad, class Store>
ZINC_DEV void ntt_inverse(uint64_t *sm, const Tw *itw, const LimbConst &c, GLoad gload, Store store,
                          const Tw *sitw = nullptr) {
  using G = Geo<LOGN, LM>;
  using P = Plan<G::LOGL>;
  constexpr int LL = G::LOGL;
  constexpr int SB = P::KA, SC = P::KA + P::KB;
  auto sst = [&](int i, uint64_t v) { sm[pad16(i)] = v; };
  auto sld = [&](int i) { return sm[pad16(i)]; };
  __syncthreads();
  static_assert(!STW || (!G::SPLIT && (1 << (SC)) <= kSmemTw), "smem twiddles cover passes B' and A'");
  if constexpr (!G::SPLIT) {
    gs_pass<LL, SC, P::KC, P::THREADS, true>(itw, c, 1, gload, sst);
    __syncthreads();
    gs_pass<LL, SB, P::KB, P::THREADS, false, true, STW>(STW ? sitw : itw, c, 1, sld, sst);
    __syncthreads();
    gs_pass<LL, 0, P::KA, P::THREADS, false, true, STW>(STW ? sitw : itw, c, 1, sld, store);
  } else {
    const int r = (int)cluster_rank();
    const int tb = 2 + r;
    gs_pass<LL, SC, P::KC, P::THREADS, true>(itw, c, tb,
        [&](int base, uint64_t (&v)[16]) { gload(base + r * G::NL, v); }, sst);
    __syncthreads();
    gs_pass<LL, SB, P::KB, P::THREADS>(itw, c, tb, sld, sst);
    __syncthreads();
    gs_pass<LL, 0, P::KA, P::THREADS, false, false>(itw, c, tb, sld, sst);
    cluster_sync_all();  // both halves complete and every input consumed
    const uint64_t *h0 = peer_smem(sm, 0), *h1 = peer_smem(sm, 1);
    const uint64_t four_q = 2 * c.two_q, q = c.q;
    constexpr int QN = G::NL / 2;
#pragma unroll 2
    for (int j = r * QN + threadIdx.x; j < (r + 1) * QN; j += P::THREADS) {
      const uint64_t X = h0[pad16(j)], Y = h1[pad16(j)];  // [0, 4q)
      store(j, mul_shoup_lazy(X + Y, c.ninv, c.ninv_sh, q));
      store(j + G::NL, mul_shoup_lazy(X - Y + four_q, c.ninv_w, c.ninv_w_sh, q));
    }
    cluster_sync_all();  // the partner finished reading this CTA's buffer
  }
}


// ---------------------------------------------------------------- S-CTA cluster transforms
// N = 2^14 and 2^15 as S = N / 2^12 CTAs of one thread-block cluster (4 or 8), each
// holding 2^12 words (34 KiB with padding, 256 threads, one 16-word group per thread per
// pass): small enough for three CTAs per SM, so one CTA's barriers and memory phases
// overlap the butterflies of two others.
//
// Forward (decimation in time at the top).  With F_{c,t} the (N / 2^t)-point transform of
// the subsequence x = c (mod 2^t) of the input (C-3 order, root psi^(2^t)),
//   F_{c,t}[2k + b] = F_{c,t+1}[k] + (-1)^b W[N / 2^(t+1) + k] F_{c + 2^t, t+1}[k],
// because the (N / 2^t)-point table is the first N / 2^t entries of W (brv_N(i) =
// 2^t brv_{N/2^t}(i)).  CTA c (cluster rank) runs the ordinary passes on its subsequence
// x = S i + c, then the last log2 S levels combine the S CTAs' values at one local index k
// into the S contiguous outputs a^[S k .. S k + S) (one register-resident radix-S block per
// k, inputs read over distributed shared memory).  CTA r finishes k in [r NL/S, (r+1) NL/S),
// i.e. the contiguous output range [r NL, (r+1) NL).
//
// Inverse (decimation in frequency at the top, the mirror image).  CTA r takes input
// positions [r NL, (r+1) NL) (bit-reversed order) and runs the GS stages LOGN-1 .. s
// locally (their blocks never straddle a share: twiddle base tb = S + r); stages s-1 .. 0
// pair positions j + c NL across CTAs: stage t pairs c and c + 2^(s-t-1) under
// W^-1[2^t + (c >> (s - t))], stage 0 with N^-1 folded in.  CTA r finishes j in
// [r NL/S, (r+1) NL/S) and stores the natural-order outputs j + c NL.
//
// The forward output range of CTA r is exactly the inverse input range of CTA r, so a
// forward transform, a pointwise product and an inverse transform chain without moving
// data between CTAs (vanilla COEFF form, decryption).
// Cluster-wide rendezvous of the S CTAs on mbarriers (two, alternating; each expects S
// arrivals per phase): every thread fences, a CTA barrier, then one remote arrive on
// every CTA's barrier; wait() polls this CTA's own barrier.  Two alternating barriers make
// a fast CTA's next arrivals land in the other barrier, never in a phase a slow CTA has
// not completed.  barrier.cluster would carry a cluster-scope acquire on every wait
// (CCTL.IVALL: the SM's L1, with the twiddles, invalidated at every exchange); here the
// waits are plain SYNCS polls.  What each rendezvous must order (measured: a stress of
// every variant over 10^5 exchanges, scripts/split_check.py):
//  - sync_raw (peers read this CTA's freshly stored share): the stores must be visible
//    to remote DSMEM readers, which a CTA-scope fence does not guarantee (observed stale
//    reads); a cluster-scope release fence (MEMBAR.GPU) per thread does.  Release only:
//    fence.acq_rel.cluster adds an acquire, i.e. CCTL.IVALL, which invalidated the SM's L1
//    (the cached pass-C and exchange twiddles of all three resident CTAs) at every exchange,
//    while the peers' reads are explicit DSMEM loads that never touch L1.
//  - sync_war (this CTA will overwrite what the peers read): every DSMEM load of the
//    exchange must have completed, which the CTA-scope fence (MEMBAR.CTA) ensures.
//    war_arrive() arrives without waiting and marks the rendezvous pending; settle() waits
//    for it and must run before the next write to the share (the split forward transform
//    calls it in pass A just before the first shared-memory store, so the wait overlaps
//    pass A's loads and butterflies) and before the CTA exits.
struct ClusterBar {
  uint64_t *mbar;  // [2], this CTA's shared memory
  uint32_t k;
  bool pending = false;
  template <int S>
  ZINC_DEV void init() {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(mbar + j)),
                     "r"(S));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    k = 0;
    pending = false;
    // every CTA's barriers are initialised before anyone arrives remotely (once per kernel)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  template <int S>
  ZINC_DEV void arrive() {
    __syncthreads();
    if (threadIdx.x < S) {
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                   : "=r"(ra) : "r"((uint32_t)__cvta_generic_to_shared(mbar + (k & 1))), "r"((uint32_t)threadIdx.x));
      asm volatile("mbarrier.arrive.release.cta.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
    }
  }
  ZINC_DEV void wait() {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar + (k & 1)), par = (k >> 1) & 1u;
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(a), "r"(par) : "memory");
    }
    ++k;
  }
  // The rendezvous before the CTA exits (the peers finished reading this CTA's share): one warp
  // polls and the others block on the CTA barrier.  With every warp polling, this loop was 10 %
  // of the Zinc NTT kernel's executed instructions (ncu source page, profiles/r02e); removing
  // them changed no timing (the scheduler prefers the other CTAs' warps), it keeps the
  // instruction counts honest.
  ZINC_DEV void settle_exit() {
    if (pending) {
      if (threadIdx.x < 32) {
        wait();
      } else {
        ++k;
      }
      pending = false;
    }
    __syncthreads();
  }
  template <int S>
  ZINC_DEV void raw_arrive() {
    settle();
    asm volatile("fence.release.cluster;" ::: "memory");
    arrive<S>();
  }
  template <int S>
  ZINC_DEV void sync_raw() {
    raw_arrive<S>();
    wait();
  }
  template <int S>
  ZINC_DEV void war_arrive() {
    asm volatile("fence.acq_rel.cta;" ::: "memory");
    arrive<S>();
    pending = true;
  }
  ZINC_DEV void settle() {
    if (pending) {
      wait();
      pending = false;
    }
  }
  template <int S>
  ZINC_DEV void sync_war() {
    settle();
    war_arrive<S>();
    settle();
  }
};

// 32-bit shared::cluster address of `p` (this CTA's shared memory) in CTA `rank`, and an
// explicit DSMEM load from it (always the owning SM's shared memory; never an L1 line).
ZINC_DEV uint32_t dsmem_addr(const void *p, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
  return ra;
}
ZINC_DEV uint64_t ld_dsmem(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
  return v;
}

// Makes every DSMEM load whose value feeds `acc` complete before the next rendezvous: a
// shared store of acc (a memory operation, so neither the compiler nor the hardware issues
// the rendezvous before it) that reads every loaded register.  Without it, register-only
// consumers of the loads may be scheduled after the barrier while the loads are in flight,
// and a peer that passed the rendezvous overwrites the words being read (measured:
// scripts/race_check.py, 3 CRT failures in 20480 COEFF-form decryptions).
ZINC_DEV void loads_done(uint64_t acc) {
  __shared__ uint64_t sink;
  asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&sink)), "l"(acc) : "memory");
}

// Passes A, B of the split forward read W[0, 256) from a TMA-staged shared copy (1) or through
// L1 (0; measured 2.6 % slower for the Zinc NTT form at C3, 1 % faster for decryption).
#ifndef ZINC_SPLIT_STW
#define ZINC_SPLIT_STW 1
#endif
constexpr bool SPLIT_STW = ZINC_SPLIT_STW;

template <int LOGN> struct SplitGeo {
  static constexpr int LL = 12, NL = 1 << LL, S = 1 << (LOGN - LL), LOGS = LOGN - LL;
  static constexpr int THREADS = Plan<LL>::THREADS;   // 256
  static constexpr int KPT = NL / S / THREADS;        // exchange indices per thread (4 or 2)
  static constexpr int STW = 1 << (Plan<LL>::KA + Plan<LL>::KB);  // smem-staged twiddles W[0, 256)
  static_assert(KPT >= 1 && NL % (S * THREADS) == 0, "split tiling");
};

// Radix-S combine of the forward transform (register-resident, see above): v[c] = F_{c,s}[k]
// in, v[m] = a^[S k + m] out.  Level t maps the pair (v[p], v[p + S/2]) to (v'[2p], v'[2p+1])
// with twiddle W[N / 2^(t+1) + 2^(s-t-1) k + (p mod 2^(s-t-1))]: 2^(s-t-1) distinct twiddles per
// level, S - 1 per k, held at w[2^(s-t-1) - 1 + j] (split_fwd_tw loads them, so an exchange can
// issue them ahead of the rendezvous or of the previous k's stores).
template <int LOGN>
ZINC_DEV void split_fwd_tw(Tw (&w)[SplitGeo<LOGN>::S - 1], int k, const Tw *tw) {
  using G = SplitGeo<LOGN>;
  constexpr int N = 1 << LOGN;
#pragma unroll
  for (int t = G::LOGS - 1; t >= 0; --t) {
    const int span = 1 << (G::LOGS - t - 1);  // 2^(s-t-1)
    const Tw *p = tw + (N >> (t + 1)) + span * k;  // an even index for span >= 2
    if (span == 1) {
      w[0] = ldtw(p);
    } else {
#pragma unroll
      for (int j = 0; j < span; j += 2) ldtw2(p + j, w[span - 1 + j], w[span + j]);
    }
  }
}
template <int LOGN, bool NR>
ZINC_DEV void split_fwd_combine_w(uint64_t (&v)[SplitGeo<LOGN>::S], const Tw (&w)[SplitGeo<LOGN>::S - 1], uint64_t q) {
  using G = SplitGeo<LOGN>;
  constexpr int S = G::S;
  const uint64_t two_q = 2 * q;
#pragma unroll
  for (int t = G::LOGS - 1; t >= 0; --t) {
    const int span = 1 << (G::LOGS - t - 1);
    uint64_t o[S];
#pragma unroll
    for (int p = 0; p < S / 2; ++p) {
      const Tw ww = w[span - 1 + (p & (span - 1))];
      uint64_t X = v[p], Y = v[p + S / 2];
      if constexpr (NR) ct_bfly_nr(X, Y, ww.x, ww.y, q, two_q);
      else ct_bfly_a(X, Y, ww.x, ww.y, q, 2 * two_q);
      o[2 * p] = X;
      o[2 * p + 1] = Y;
    }
#pragma unroll
    for (int p = 0; p < S; ++p) v[p] = o[p];
  }
}
template <int LOGN, bool NR>
ZINC_DEV void split_fwd_combine(uint64_t (&v)[SplitGeo<LOGN>::S], int k, const Tw *tw, uint64_t q) {
  Tw w[SplitGeo<LOGN>::S - 1];
  split_fwd_tw<LOGN>(w, k, tw);
  split_fwd_combine_w<LOGN, NR>(v, w, q);
}

// An exchange output functor may offer `pre(x0)`: the global loads its store of outputs
// x0 .. x0 + S - 1 needs (e.g. the cache words), issued one k ahead like the twiddles.
template <class O, class = void> struct HasPre { static constexpr bool value = false; };
template <class O> struct HasPre<O, decltype((void)&O::pre)> { static constexpr bool value = true; };
struct NoPre {};
template <class O> ZINC_DEV auto out_pre(const O &o, int x0) {
  if constexpr (HasPre<O>::value) return o.pre(x0);
  else return NoPre{};
}
template <class O, class V, class P> ZINC_DEV void out_call(O &o, int x0, V &v, const P &p) {
  if constexpr (HasPre<O>::value) o(x0, v, p);
  else o(x0, v);
}

// Forward NTT of one limb by the S-CTA cluster.  `load` as ntt_forward (global coefficient
// index x -> value; a TwoPhase load is used as such); `out(x0, v[S])` receives the S
// contiguous outputs at global positions x0 .. x0 + S - 1 (values < 2^64 with NR, [0, 8q)
// otherwise).  With LOAD_ALL the exchange first reads all of the CTA's inputs into
// registers and passes a cluster barrier before any `out` call, so `out` may write this
// CTA's shared memory (the inverse input of a following ntt_inverse_split).
// stw: shared copy of W[0, SplitGeo::STW); after_b() runs once every thread of the CTA is past
// pass C (at the data-ready rendezvous, a CTA barrier), so it may restage stw.
template <int LOGN, bool NR, bool LOAD_ALL = false, class Load, class Out, class AfterB = NoHook>
ZINC_DEV void ntt_forward_split(uint64_t *sm, ClusterBar &cb, const Tw *tw, uint64_t q, Load load, Out out,
                                const Tw *stw, AfterB after_b = AfterB()) {
  using G = SplitGeo<LOGN>;
  using P = Plan<G::LL>;
  constexpr int LL = G::LL, S = G::S, THREADS = G::THREADS;
  constexpr int SB = P::KA, SC = P::KA + P::KB;
  auto sst = [&](int i, uint64_t v) { sm[pad16(i)] = v; };
  auto sld = [&](int i) { return sm[pad16(i)]; };
  const int r = (int)cluster_rank();
  // a deferred buffer-free rendezvous (the previous exchange) settles just before pass A's
  // first shared-memory store: one group per thread, so once per thread
  static_assert(P::THREADS == THREADS && (G::NL >> P::KA) == THREADS, "one pass-A group per thread");
  auto settle = [&]() { cb.settle(); };
  __syncthreads();  // the previous transform may still read sm
  if constexpr (TwoPhase<Load>::value) {
    if constexpr (HasUniformSmall<Load>::value) {
      struct Sub {  // local index i -> coefficient S i + r
        const Load &l;
        int r;
        ZINC_DEV int64_t fetch(int i) const { return l.fetch(S * i + r); }
        ZINC_DEV uint64_t lift(int64_t raw, int i) const { return l.lift(raw, S * i + r); }
        ZINC_DEV bool uniform_small() const { return l.uniform_small(); }
        ZINC_DEV uint64_t lift_small(int64_t raw, int i) const { return l.lift_small(raw, S * i + r); }
      };
      ct_pass<LL, 0, P::KA, THREADS, false, SPLIT_STW, NR>(SPLIT_STW ? stw : tw, q, 1, Sub{load, r}, sst, settle);
    } else if constexpr (HasSmallLift<Load>::value) {
      struct Sub {  // local index i -> coefficient S i + r
        const Load &l;
        int r;
        ZINC_DEV int64_t fetch(int i) const { return l.fetch(S * i + r); }
        ZINC_DEV uint64_t lift(int64_t raw, int i) const { return l.lift(raw, S * i + r); }
        ZINC_DEV bool small(int64_t raw) const { return l.small(raw); }
        ZINC_DEV uint64_t lift_small(int64_t raw, int i) const { return l.lift_small(raw, S * i + r); }
      };
      ct_pass<LL, 0, P::KA, THREADS, false, SPLIT_STW, NR>(SPLIT_STW ? stw : tw, q, 1, Sub{load, r}, sst, settle);
    } else {
      struct Sub {  // local index i -> coefficient S i + r
        const Load &l;
        int r;
        ZINC_DEV int64_t fetch(int i) const { return l.fetch(S * i + r); }
        ZINC_DEV uint64_t lift(int64_t raw, int i) const { return l.lift(raw, S * i + r); }
      };
      ct_pass<LL, 0, P::KA, THREADS, false, SPLIT_STW, NR>(SPLIT_STW ? stw : tw, q, 1, Sub{load, r}, sst, settle);
    }
  } else {
    ct_pass<LL, 0, P::KA, THREADS, false, SPLIT_STW, NR>(SPLIT_STW ? stw : tw, q, 1, [&](int i) { return load(S * i + r); }, sst, settle);
  }
  __syncthreads();
  ct_pass<LL, SB, P::KB, THREADS, false, SPLIT_STW, NR>(SPLIT_STW ? stw : tw, q, 1, sld, sst);
  // Pass B's groups of thread g lie in the 256-word block g / 16 and pass C's in [16 g, 16 g + 16):
  // both passes of warp w touch exactly the words [512 w, 512 w + 512), so a warp hands pass B's
  // output to its own pass C with a warp barrier instead of a CTA barrier, and the warps of a CTA
  // run passes B, C and the exchange prologue out of step with one another.
  static_assert(THREADS == 256 && P::KB == 4 && P::KC == 4 && SB == 4, "warp-local passes B, C");
  __syncwarp();
  ct_pass<LL, SC, P::KC, THREADS, true, false, NR>(tw, q, 1, sld, [&](int base, uint64_t (&v)[16]) {
#pragma unroll
    for (int j = 0; j < 16; ++j) sm[pad16(base + j)] = v[j];
  });
  uint32_t peer[S];
#pragma unroll
  for (int c = 0; c < S; ++c) peer[c] = dsmem_addr(sm, (uint32_t)c);
  const int k0 = r * (G::NL / S) + threadIdx.x;
  if constexpr (LOAD_ALL) {
    cb.raw_arrive<S>();  // every CTA's sub-transform complete
    after_b();
    cb.wait();
    uint64_t v[G::KPT][S];
#pragma unroll
    for (int u = 0; u < G::KPT; ++u)
#pragma unroll
      for (int c = 0; c < S; ++c) v[u][c] = ld_dsmem(peer[c] + 8u * (uint32_t)pad16(k0 + u * THREADS));
    uint64_t acc = 0;
#pragma unroll
    for (int u = 0; u < G::KPT; ++u)
#pragma unroll
      for (int c = 0; c < S; ++c) acc ^= v[u][c];
    loads_done(acc);
    cb.sync_war<S>();  // every CTA has read its inputs: shared memory is free
#pragma unroll
    for (int u = 0; u < G::KPT; ++u) {
      const int k = k0 + u * THREADS;
      split_fwd_combine<LOGN, NR>(v[u], k, tw, q);
      out(S * k, v[u]);
    }
  } else {
    // Software-pipelined exchange, one k per step: the twiddles and the output functor's
    // global loads of k are issued before the rendezvous (k = the first) or before the
    // previous k's stores, and so is k's DSMEM gather, so no global-load latency sits
    // between a store and the next k.  The buffer-free rendezvous is deferred (settle()).
    constexpr int S1 = S - 1;
    constexpr bool DB = S <= 4;  // double-buffered registers (k and k + 1) fit at S = 4
    using PreT = decltype(out_pre(out, 0));
    cb.raw_arrive<S>();  // every CTA's sub-transform complete (wait below)
    after_b();
    Tw wc[S1];
    PreT pc;
    split_fwd_tw<LOGN>(wc, k0, tw);
    pc = out_pre(out, S * k0);
    cb.wait();
    uint64_t vc[S];
#pragma unroll
    for (int c = 0; c < S; ++c) vc[c] = ld_dsmem(peer[c] + 8u * (uint32_t)pad16(k0));
    uint64_t acc = 0;
#pragma unroll
    for (int u = 0; u < G::KPT; ++u) {
      const int k = k0 + u * THREADS;
      if constexpr (DB) {
        Tw wn[S1];
        PreT pn;
        uint64_t vn[S];
        if (u + 1 < G::KPT) {
          split_fwd_tw<LOGN>(wn, k + THREADS, tw);
          pn = out_pre(out, S * (k + THREADS));
#pragma unroll
          for (int c = 0; c < S; ++c) vn[c] = ld_dsmem(peer[c] + 8u * (uint32_t)pad16(k + THREADS));
        }
#pragma unroll
        for (int c = 0; c < S; ++c) acc ^= vc[c];
        split_fwd_combine_w<LOGN, NR>(vc, wc, q);
        out_call(out, S * k, vc, pc);
        if (u + 1 < G::KPT) {
#pragma unroll
          for (int c = 0; c < S; ++c) vc[c] = vn[c];
#pragma unroll
          for (int j = 0; j < S1; ++j) wc[j] = wn[j];
          pc = pn;
        }
      } else {  // S = 8: registers for one k only
        if (u > 0) {
          split_fwd_tw<LOGN>(wc, k, tw);
          pc = out_pre(out, S * k);
#pragma unroll
          for (int c = 0; c < S; ++c) vc[c] = ld_dsmem(peer[c] + 8u * (uint32_t)pad16(k));
        }
#pragma unroll
        for (int c = 0; c < S; ++c) acc ^= vc[c];
        split_fwd_combine_w<LOGN, NR>(vc, wc, q);
        out_call(out, S * k, vc, pc);
      }
    }
    loads_done(acc);
    cb.war_arrive<S>();  // the peers may overwrite their shares once every CTA arrived
  }
}

// An inverse-exchange store functor may offer `pre1(x)`: the global words its store of output
// x needs (a ciphertext or plaintext word), then called as store(x, v, words).  WithPre1 adds
// it to a plain functor pair.
template <class O, class = void> struct HasPre1 { static constexpr bool value = false; };
template <class O> struct HasPre1<O, decltype((void)&O::pre1)> { static constexpr bool value = true; };
template <int S, class T> struct PreW {
  T w[S];
};
template <int S, int NL, class O> ZINC_DEV auto inv_pre(const O &o, int j) {
  if constexpr (HasPre1<O>::value) {
    PreW<S, decltype(o.pre1(0))> p;
#pragma unroll
    for (int cc = 0; cc < S; ++cc) p.w[cc] = o.pre1(j + cc * NL);
    return p;
  } else {
    return NoPre{};
  }
}
template <class O, class P> ZINC_DEV void inv_store(O &o, int x, uint64_t v, const P &p, int cc) {
  if constexpr (HasPre1<O>::value) o(x, v, p.w[cc]);
  else o(x, v);
}
template <class F, class G> struct WithPre1 {
  F f;
  G g;
  ZINC_DEV auto pre1(int x) const { return g(x); }
  template <class W> ZINC_DEV void operator()(int x, uint64_t v, const W &w) const { f(x, v, w); }
};
template <class F, class G> ZINC_DEV WithPre1<F, G> with_pre1(F f, G g) { return WithPre1<F, G>{f, g}; }

// Inverse NTT of one limb by the S-CTA cluster.  With GLOBAL_IN, `gload(base, v[16])`
// supplies the 16 contiguous inputs at global position base (in [r NL, (r+1) NL)) in
// [0, 2q); otherwise the CTA's inputs are already in its shared memory (local position
// i = global - r NL, in [0, 4q)).  `store(x, v)` gets the natural-order output x in [0, 2q).
// Every store happens after all S CTAs consumed their inputs.
template <int LOGN, bool GLOBAL_IN, class GLoad, class Store>
ZINC_DEV void ntt_inverse_split(uint64_t *sm, ClusterBar &cb, const Tw *itw, const LimbConst &c, GLoad gload,
                                Store store) {
  using G = SplitGeo<LOGN>;
  using P = Plan<G::LL>;
  constexpr int LL = G::LL, S = G::S, THREADS = G::THREADS, NL = G::NL;
  constexpr int SB = P::KA, SC = P::KA + P::KB;
  auto sst = [&](int i, uint64_t v) { sm[pad16(i)] = v; };
  auto sld = [&](int i) { return sm[pad16(i)]; };
  const int r = (int)cluster_rank();
  const int tb = S + r;
  cb.settle();  // a deferred buffer-free rendezvous completes before this share is rewritten
  __syncthreads();
  if constexpr (GLOBAL_IN) {
    gs_pass<LL, SC, P::KC, THREADS, true>(itw, c, tb, [&](int base, uint64_t (&v)[16]) { gload(base + r * NL, v); },
                                          sst);
  } else {
    gs_pass<LL, SC, P::KC, THREADS>(itw, c, tb, sld, sst);
  }
  __syncwarp();  // the first two passes of warp w touch only words [512 w, 512 w + 512) (forward)
  gs_pass<LL, SB, P::KB, THREADS>(itw, c, tb, sld, sst);
  __syncthreads();
  gs_pass<LL, 0, P::KA, THREADS, false, false>(itw, c, tb, sld, sst);
  const uint64_t q = c.q, four_q = 2 * c.two_q;
  // the S - 1 cross-share twiddles: stage t uses W^-1[2^t + beta], beta < 2^t
  Tw w[S];
#pragma unroll
  for (int i = 1; i < S; ++i) w[i] = ldtw(itw + i);
  // Software-pipelined exchange as the forward's: the store functor's global words (pre1) of
  // index j are loaded before the rendezvous (the first j) or before the previous j's stores,
  // with j's DSMEM gather.
  cb.raw_arrive<S>();  // every share transformed, every input consumed (wait below)
  uint32_t peer[S];
#pragma unroll
  for (int cc = 0; cc < S; ++cc) peer[cc] = dsmem_addr(sm, (uint32_t)cc);
  const int j0 = r * (NL / S) + threadIdx.x;
  auto pc = inv_pre<S, NL>(store, j0);
  cb.wait();
  uint64_t xc[S];
#pragma unroll
  for (int cc = 0; cc < S; ++cc) xc[cc] = ld_dsmem(peer[cc] + 8u * (uint32_t)pad16(j0));
  uint64_t acc = 0;
  // one index ahead: the pre words when there is one per output, the gather too at S = 4
  constexpr bool PRE_DB = sizeof(decltype(pc)) <= S * sizeof(uint64_t);
  constexpr bool DB = S <= 4 && PRE_DB;
#pragma unroll
  for (int u = 0; u < G::KPT; ++u) {
    const int j = j0 + u * THREADS;
    uint64_t xn[DB ? S : 1];
    decltype(pc) pn;
    if (u > 0) {
      if constexpr (!PRE_DB) pc = inv_pre<S, NL>(store, j);
      if constexpr (!DB) {
#pragma unroll
        for (int cc = 0; cc < S; ++cc) xc[cc] = ld_dsmem(peer[cc] + 8u * (uint32_t)pad16(j));
      }
    }
    if (u + 1 < G::KPT) {
      if constexpr (PRE_DB) pn = inv_pre<S, NL>(store, j + THREADS);
      if constexpr (DB) {
#pragma unroll
        for (int cc = 0; cc < S; ++cc) xn[cc] = ld_dsmem(peer[cc] + 8u * (uint32_t)pad16(j + THREADS));
      }
    }
#pragma unroll
    for (int cc = 0; cc < S; ++cc) acc ^= xc[cc];
#pragma unroll
    for (int t = G::LOGS - 1; t >= 1; --t) {
      const int d = 1 << (G::LOGS - t - 1);
#pragma unroll
      for (int cc = 0; cc < S; ++cc)
        if ((cc & d) == 0) {
          const Tw ww = w[(1 << t) + (cc >> (G::LOGS - t))];
          gs_bfly(xc[cc], xc[cc + d], ww.x, ww.y, q, four_q);
        }
    }
#pragma unroll
    for (int cc = 0; cc < S / 2; ++cc) {  // stage 0: pairs (c, c + S/2), N^-1 folded in
      const uint64_t X = xc[cc], Y = xc[cc + S / 2];
      xc[cc] = mul_shoup_lazy(X + Y, c.ninv, c.ninv_sh, q);
      xc[cc + S / 2] = mul_shoup_lazy(X - Y + four_q, c.ninv_w, c.ninv_w_sh, q);
    }
#pragma unroll
    for (int cc = 0; cc < S; ++cc) inv_store(store, j + cc * NL, xc[cc], pc, cc);
    if (u + 1 < G::KPT) {
      if constexpr (DB) {
#pragma unroll
        for (int cc = 0; cc < S; ++cc) xc[cc] = xn[cc];
      }
      if constexpr (PRE_DB) pc = pn;
    }
  }
  loads_done(acc);
  cb.war_arrive<S>();  // the peers finished reading this CTA's buffer once every CTA arrived
}

}  // namespace zinc
