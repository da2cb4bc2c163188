// k_split.cu -- the transform paths at N = 2^14 and 2^15 on S-CTA thread-block clusters
// (ntt.cuh, ntt_forward_split / ntt_inverse_split): Zinc NTT form,
// vanilla encryption in both forms (Eq. 8) and decryption (Eq. 10,
// PAPER.md:224-227).  Every CTA holds 2^12 words of one limb (34 KiB + samples + 4 KiB of
// staged twiddles, 256 threads), three CTAs per SM.
#include "kcommon.cuh"

namespace zinc {

// resident CTAs per SM the cluster kernels are compiled for: 4 (64 registers, 47 KiB each;
// measured +4-14% over 3 at C3 / C4 despite ~60 B of spills)
#ifndef ZINC_SPLIT_MINB
#define ZINC_SPLIT_MINB 4
#endif

// ============================================================ samplers (C-4) on a share
// CBD samples of the coefficients x = S i + r (the forward split's subsequence), stored at i,
// drawn by the CTA pair (r, r ^ 1) together: x = S i + r and S i + (r ^ 1) are the two halves of
// one Philox block ((S/2) i + (r >> 1)); drawing them per CTA computed every block twice.
// Each CTA draws the blocks of half the indices i and hands the partner's halves over
// distributed shared memory, four samples per 32-bit store.  A cluster barrier must follow
// before either CTA reads its buffer (and one must precede: the partner is running).
template <int THREADS>
ZINC_DEV void sample_cbd_pair(int8_t *dst, int nl, int S, int r, uint64_t seed, uint64_t msg, uint32_t tag) {
  const int h = r & 1, half = nl / 2;
  const uint32_t peer = dsmem_addr(dst, (uint32_t)(r ^ 1));
  for (int i4 = threadIdx.x; i4 < half / 4; i4 += THREADS) {
    const int i0 = h * half + 4 * i4;
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 w = stream_block(seed, msg, tag, 0, (uint32_t)((S / 2) * (i0 + j) + (r >> 1)));
      lo |= ((uint32_t)cbd_lo(w) & 0xFFu) << (8 * j);
      hi |= ((uint32_t)cbd_hi(w) & 0xFFu) << (8 * j);
    }
    // the even rank of the pair owns the even coefficients (the block's low half)
    *reinterpret_cast<uint32_t *>(dst + i0) = h ? hi : lo;
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(peer + (uint32_t)i0), "r"(h ? lo : hi) : "memory");
  }
}
// Ternary samples of x = S i + r (S >= 4: word r & 3 of block x >> 2), packed 2 bits at i.
template <int THREADS>
ZINC_DEV void sample_ternary_sub(uint8_t *dst, int nl, int S, int r, uint64_t seed, uint64_t msg, uint32_t tag) {
  const int wsel = r & 3;
  for (int i4 = threadIdx.x; i4 < nl / 4; i4 += THREADS) {
    uint32_t packed = 0;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int x = S * (4 * i4 + h) + r;
      const uint4 w = stream_block(seed, msg, tag, 0, (uint32_t)(x >> 2));
      const uint32_t word = wsel == 0 ? w.x : wsel == 1 ? w.y : wsel == 2 ? w.z : w.w;
      packed |= (uint32_t)(tern(word) + 1) << (2 * h);
    }
    dst[i4] = (uint8_t)packed;
  }
}
// CBD samples of the inverse split's outputs: positions j + c NL, j in [r NL/S, (r+1) NL/S),
// stored at c (NL/S) + (j - r NL/S).  Pairs of adjacent coefficients share a Philox block.
template <int THREADS>
ZINC_DEV void sample_cbd_inv(int8_t *dst, int nl, int S, int r, uint64_t seed, uint64_t msg, uint32_t tag) {
  const int span = nl / S;
  for (int l2 = threadIdx.x; l2 < nl / 2; l2 += THREADS) {
    const int l = 2 * l2, c = l / span, jj = l % span;
    const int x = c * nl + r * span + jj;  // even
    const uint4 w = stream_block(seed, msg, tag, 0, (uint32_t)(x >> 1));
    dst[l] = (int8_t)cbd_lo(w);
    dst[l + 1] = (int8_t)cbd_hi(w);
  }
}
// index of output position x in the sample_cbd_inv layout of CTA r
template <int LOGN>
ZINC_DEV int inv_sample_idx(int x, int r) {
  using G = SplitGeo<LOGN>;
  constexpr int span = G::NL / G::S;
  return (x >> G::LL) * span + (x & (G::NL - 1)) - r * span;
}

// CKKS plaintext words of this CTA's subsequence (x = S i + r) all below q_min / 2 in absolute
// value (q_min over the CTA's limbs): then every lift of m + e is branch-free (lift_small), for
// every limb, decided once per message instead of per word, limb and transform.
template <int LOGN> struct SplitSmem {
  using G = SplitGeo<LOGN>;
  static constexpr size_t DATA = SmemWords<G::LL>::value * sizeof(uint64_t);  // 34816
  static constexpr size_t TW = SPLIT_STW ? G::STW * sizeof(Tw) : 0;          // 4096
};

// ============================================================ Zinc, NTT form
// Exchange output of the Zinc NTT form: ct = [cache + v] (v the lazy transform output); the
// cache words of an output group are loaded by pre() one k ahead (ntt_forward_split).
template <int S>
struct ZincNttOut {
  struct Pre {
    U64x4 z[S / 4];
  };
  const uint64_t *z;
  uint64_t *ctt;
  const LimbConst &c;
  ZINC_DEV Pre pre(int x0) const {
    Pre p;
#pragma unroll
    for (int u = 0; u < S / 4; ++u) p.z[u] = ld4_nc(z + x0 + 4 * u);
    return p;
  }
  ZINC_DEV void operator()(int x0, uint64_t (&v)[S], const Pre &p) const {
#pragma unroll
    for (int u = 0; u < S / 4; ++u)  // lazy output + canonical cache word < 2^64
      st4_cs(ctt + x0 + 4 * u, reduce_fold(p.z[u].v[0] + v[4 * u], c), reduce_fold(p.z[u].v[1] + v[4 * u + 1], c),
             reduce_fold(p.z[u].v[2] + v[4 * u + 2], c), reduce_fold(p.z[u].v[3] + v[4 * u + 3], c));
  }
};

// c1' = zero1 + NTT(m + e1'), c2' = zero2 + NTT(e2'): both transforms through one copy of
// the transform code (t at run time); the exchange streams cache-added words to HBM.
template <int LOGN, int MODE>
__global__ void __launch_bounds__(256, ZINC_SPLIT_MINB) zinc_ntt_split_kernel(ZincNttArgs a) {
  constexpr bool INTS = MODE == 2, NR = MODE == 0;
  using G = SplitGeo<LOGN>;
  constexpr int N = 1 << LOGN, S = G::S, NL = G::NL, THREADS = G::THREADS;
  extern __shared__ __align__(16) uint64_t sm[];
  Tw *stw = reinterpret_cast<Tw *>(sm + SmemWords<G::LL>::value);
  int8_t *se1 = reinterpret_cast<int8_t *>(stw + (SPLIT_STW ? G::STW : 0)), *se2 = se1 + NL;
  __shared__ __align__(8) uint64_t tw_mbar, cl_mbar[2];
  TwStager tws{&tw_mbar, 0};
  ClusterBar cb{cl_mbar, 0};
  const size_t b = blockIdx.x / S;
  const int r = (int)cluster_rank();
  const uint64_t msg = a.msg_base + b;
  const int L = a.L;
  const int lo = blockIdx.y * a.limbs_per_cta;
  const int hi = min(L, lo + a.limbs_per_cta);
  if constexpr (SPLIT_STW) tws.init();
  cb.init<S>();
  if constexpr (SPLIT_STW) tws.issue_n(stw, a.tw + (size_t)lo * N, G::STW);
  // small batches spread the two transforms over gridDim.z = 2 (t = blockIdx.z)
  const int t_lo = gridDim.z > 1 ? (int)blockIdx.z : 0, t_hi = gridDim.z > 1 ? t_lo + 1 : 2;
  if (t_lo == 0) sample_cbd_pair<THREADS>(se1, NL, S, r, a.seed, msg, TAG_ZINC_E1);
  if (t_hi == 2) sample_cbd_pair<THREADS>(se2, NL, S, r, a.seed, msg, TAG_ZINC_E2);
  cluster_sync_all();  // the partner's halves have landed (once per message)
  pdl_trigger();  // chained after the encode that wrote m: wait before reading it
  pdl_wait();
  const MSub m = m_sub(a.m ? a.m + b * N : nullptr, r, G::LOGS, a.m_deint, LOGN);  // x = S i + r
  const bool all_small = !INTS && t_lo == 0 && plaintext_small_sub<THREADS>(m, NL, a.limbs, lo, hi);
  for (int i = lo; i < hi; ++i) {
    const LimbConst c = a.limbs[i];
    const uint64_t q = c.q;
    const Tw *tw = a.tw + (size_t)i * N;
    uint64_t *ct0 = a.ct + b * 2 * L * N + (size_t)i * N;
    if constexpr (SPLIT_STW) tws.wait();
#pragma unroll 1
    for (int t = t_lo; t < t_hi; ++t) {
      const uint64_t *z = a.cache + (size_t)(t * L + i) * N;
      uint64_t *ctt = ct0 + (size_t)t * L * N;
      ntt_forward_split<LOGN, NR>(sm, cb, tw, q, ZincTLoadU<INTS, G::LOGS>{{m.p, t ? se2 : se1, c, t, m.stride}, all_small},
          ZincNttOut<S>{z, ctt, c}, stw, [&]() {
            if (SPLIT_STW && t == t_hi - 1 && i + 1 < hi) tws.issue_n(stw, tw + N, G::STW);  // lands during pass C + exchange
          });
    }
  }
  cb.settle_exit();  // the peers finished reading this CTA's share
}

// ============================================================ vanilla, NTT form
// NTT(m + e1) -> ct0, NTT(e2) -> ct1, NTT(u) -> ct0 += pk1 u^, ct1 += pk2 u^ (Eq. 8, A1).
// The three transforms of a limb run through one copy of the transform code; every
// exchange thread re-reads only the ciphertext words it wrote itself.
template <int LOGN, int MODE>
__global__ void __launch_bounds__(256, ZINC_SPLIT_MINB) vanilla_ntt_split_kernel(VanillaArgs a) {
  constexpr bool INTS = MODE == 2, NR = MODE == 0;
  using G = SplitGeo<LOGN>;
  constexpr int N = 1 << LOGN, S = G::S, NL = G::NL, THREADS = G::THREADS;
  extern __shared__ __align__(16) uint64_t sm[];
  Tw *stw = reinterpret_cast<Tw *>(sm + SmemWords<G::LL>::value);
  int8_t *se1 = reinterpret_cast<int8_t *>(stw + (SPLIT_STW ? G::STW : 0)), *se2 = se1 + NL;
  uint8_t *su = reinterpret_cast<uint8_t *>(se2 + NL);
  __shared__ __align__(8) uint64_t tw_mbar, cl_mbar[2];
  TwStager tws{&tw_mbar, 0};
  ClusterBar cb{cl_mbar, 0};
  const size_t b = blockIdx.x / S;
  const int r = (int)cluster_rank();
  const uint64_t msg = a.msg_base + b;
  const int L = a.L;
  const int lo = blockIdx.y * a.limbs_per_cta;
  const int hi = min(L, lo + a.limbs_per_cta);
  if constexpr (SPLIT_STW) tws.init();
  cb.init<S>();
  if constexpr (SPLIT_STW) tws.issue_n(stw, a.tw + (size_t)lo * N, G::STW);
  // small batches spread the three transforms over gridDim.z = 3 (t = blockIdx.z; the u
  // transform then writes u^ to a.u_hat and vanilla_combine_kernel forms pk u^)
  const int t_lo = gridDim.z > 1 ? (int)blockIdx.z : 0, t_hi = gridDim.z > 1 ? t_lo + 1 : 3;
  if (t_hi == 3) sample_ternary_sub<THREADS>(su, NL, S, r, a.seed, msg, TAG_ENC_U);
  if (t_lo == 0) sample_cbd_pair<THREADS>(se1, NL, S, r, a.seed, msg, TAG_ENC_E1);
  if (t_lo <= 1 && t_hi >= 2) sample_cbd_pair<THREADS>(se2, NL, S, r, a.seed, msg, TAG_ENC_E2);
  cluster_sync_all();  // the partner's halves have landed (once per message)
  pdl_trigger();
  pdl_wait();
  const MSub m = m_sub(a.m ? a.m + b * N : nullptr, r, G::LOGS, a.m_deint, LOGN);  // x = S i + r
  const bool all_small = !INTS && t_lo == 0 && plaintext_small_sub<THREADS>(m, NL, a.limbs, lo, hi);
  for (int i = lo; i < hi; ++i) {
    const LimbConst c = a.limbs[i];
    const uint64_t q = c.q;
    const Tw *tw = a.tw + (size_t)i * N;
    const uint64_t *pk1 = a.pk + (size_t)i * N, *pk2 = a.pk + (size_t)(L + i) * N;
    const uint64_t *pk1s = a.pk_sh + (size_t)i * N, *pk2s = a.pk_sh + (size_t)(L + i) * N;
    uint64_t *ct0 = a.ct + b * 2 * L * N + (size_t)i * N;
    uint64_t *ct1 = ct0 + (size_t)L * N;
    auto canon = [&](uint64_t v) { return reduce_fold(v, c); };
    if constexpr (SPLIT_STW) tws.wait();
#pragma unroll 1
    for (int t = t_lo; t < t_hi; ++t) {
      ntt_forward_split<LOGN, NR>(sm, cb, tw, q, VanTLoad<INTS, G::LOGS>{m.p, se1, se2, su, c, t, m.stride, all_small || t > 0},
          [&](int x0, uint64_t (&v)[S]) {
            if (t < 2 || gridDim.z > 1) {
              uint64_t *dst = (t == 0 ? ct0 : t == 1 ? ct1 : a.u_hat + (b * L + i) * N) + x0;
#pragma unroll
              for (int u = 0; u < S; u += 4) st4(dst + u, canon(v[u]), canon(v[u + 1]), canon(v[u + 2]), canon(v[u + 3]));
            } else {
#pragma unroll
              for (int u = 0; u < S; u += 4) {
                const U64x4 p1 = ld4_nc(pk1 + x0 + u), p2 = ld4_nc(pk2 + x0 + u);
                const U64x4 s1 = ld4_nc(pk1s + x0 + u), s2 = ld4_nc(pk2s + x0 + u);
                const U64x4 ca = ld4(ct0 + x0 + u), cb2 = ld4(ct1 + x0 + u);
                uint64_t o0[4], o1[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  o0[j] = add_shoup(ca.v[j], v[u + j], p1.v[j], s1.v[j], q);
                  o1[j] = add_shoup(cb2.v[j], v[u + j], p2.v[j], s2.v[j], q);
                }
                st4_cs(ct0 + x0 + u, o0[0], o0[1], o0[2], o0[3]);
                st4_cs(ct1 + x0 + u, o1[0], o1[1], o1[2], o1[3]);
              }
            }
          },
          stw, [&]() {
            if (SPLIT_STW && t == t_hi - 1 && i + 1 < hi) tws.issue_n(stw, tw + N, G::STW);
          });
    }
  }
  cb.settle_exit();  // the peers finished reading this CTA's share
}

// ============================================================ vanilla, COEFF form
// NTT(u) (forward split; its exchange reads every input first, so it can write the
// pointwise product pk1 u^ straight into this CTA's share, and pk2 u^ to ct1 as a
// temporary); INTT(pk1 u^) + e1 + m -> ct0; INTT(ct1) + e2 -> ct1.  The forward output
// range of a CTA is its inverse input range: no data moves between CTAs in between.
template <int LOGN, int MODE>
__global__ void __launch_bounds__(256, ZINC_SPLIT_MINB) vanilla_coeff_split_kernel(VanillaArgs a) {
  constexpr bool INTS = MODE == 2, NR = MODE == 0;
  using G = SplitGeo<LOGN>;
  constexpr int N = 1 << LOGN, S = G::S, NL = G::NL, THREADS = G::THREADS;
  extern __shared__ __align__(16) uint64_t sm[];
  Tw *stw = reinterpret_cast<Tw *>(sm + SmemWords<G::LL>::value);
  int8_t *se1 = reinterpret_cast<int8_t *>(stw + (SPLIT_STW ? G::STW : 0)), *se2 = se1 + NL;
  uint8_t *su = reinterpret_cast<uint8_t *>(se2 + NL);
  __shared__ __align__(8) uint64_t tw_mbar, cl_mbar[2];
  TwStager tws{&tw_mbar, 0};
  ClusterBar cb{cl_mbar, 0};
  const size_t b = blockIdx.x / S;
  const int r = (int)cluster_rank();
  const uint64_t msg = a.msg_base + b;
  const int L = a.L;
  const int lo = blockIdx.y * a.limbs_per_cta;
  const int hi = min(L, lo + a.limbs_per_cta);
  if constexpr (SPLIT_STW) tws.init();
  cb.init<S>();
  if constexpr (SPLIT_STW) tws.issue_n(stw, a.tw + (size_t)lo * N, G::STW);
  sample_ternary_sub<THREADS>(su, NL, S, r, a.seed, msg, TAG_ENC_U);
  sample_cbd_inv<THREADS>(se1, NL, S, r, a.seed, msg, TAG_ENC_E1);
  sample_cbd_inv<THREADS>(se2, NL, S, r, a.seed, msg, TAG_ENC_E2);
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  const int64_t *m = a.m ? a.m + b * N : nullptr;
  for (int i = lo; i < hi; ++i) {
    const LimbConst c = a.limbs[i];
    const uint64_t q = c.q;
    const Tw *tw = a.tw + (size_t)i * N, *itw = a.itw + (size_t)i * N;
    const uint64_t *pk1 = a.pk + (size_t)i * N, *pk2 = a.pk + (size_t)(L + i) * N;
    const uint64_t *pk1s = a.pk_sh + (size_t)i * N, *pk2s = a.pk_sh + (size_t)(L + i) * N;
    uint64_t *ct0 = a.ct + b * 2 * L * N + (size_t)i * N;
    uint64_t *ct1 = ct0 + (size_t)L * N;
    auto canon = [&](uint64_t v) { return reduce_fold(v, c); };
    if constexpr (SPLIT_STW) tws.wait();
    ntt_forward_split<LOGN, NR, true>(sm, cb, tw, q, [&](int x) { return reduce_small(tern_at(su, x >> G::LOGS), q); },
        [&](int x0, uint64_t (&v)[S]) {
#pragma unroll
          for (int u = 0; u < S; u += 4) {
            const U64x4 p1 = ld4_nc(pk1 + x0 + u), p2 = ld4_nc(pk2 + x0 + u);
            const U64x4 s1 = ld4_nc(pk1s + x0 + u), s2 = ld4_nc(pk2s + x0 + u);
            // [0, 2q): the inverse transforms take inputs below 4q
            st4(ct1 + x0 + u, mul_shoup_lazy(v[u], p2.v[0], s2.v[0], q), mul_shoup_lazy(v[u + 1], p2.v[1], s2.v[1], q),
                mul_shoup_lazy(v[u + 2], p2.v[2], s2.v[2], q), mul_shoup_lazy(v[u + 3], p2.v[3], s2.v[3], q));  // temporary
#pragma unroll
            for (int j = 0; j < 4; ++j)  // this CTA's inverse input
              sm[pad16(x0 + u + j - r * NL)] = mul_shoup_lazy(v[u + j], p1.v[j], s1.v[j], q);
          }
        },
        stw, [&]() {
          if (SPLIT_STW && i + 1 < hi) tws.issue_n(stw, tw + N, G::STW);
        });
    ntt_inverse_split<LOGN, false>(sm, cb, itw, c, [](int, uint64_t (&)[16]) {},
        with_pre1(
            [&](int x, uint64_t v, uint64_t mx) {
              const uint64_t e = pt_plus_e<INTS>((int64_t)mx, se1[inv_sample_idx<LOGN>(x, r)], c);
              __stcs(ct0 + x, add_mod(csub(v, q), e, q));
            },
            [&](int x) { return m ? (uint64_t)ldm(m + x) : (uint64_t)0; }));
    ntt_inverse_split<LOGN, true>(sm, cb, itw, c,
        [&](int base, uint64_t (&v)[16]) {
#pragma unroll
          for (int u = 0; u < 16; u += 4) {
            const U64x4 w = ld4(ct1 + base + u);
#pragma unroll
            for (int j = 0; j < 4; ++j) v[u + j] = w.v[j];
          }
        },
        [&](int x, uint64_t v) {
          __stcs(ct1 + x, add_mod(csub(v, q), err_term<INTS>(se2[inv_sample_idx<LOGN>(x, r)], c), q));
        });
  }
  cb.settle_exit();  // the peers finished reading this CTA's share
}

// ============================================================ decrypt (Eq. 10)
// x^(i) = [c1 + c2 s]_{q_i} per limb, limbs in order; limb 0 writes x0 = the centred
// residue mod q_0, every other limb checks x0 mod q_i == x^(i) (C-10); BGV / BFV / wide
// CKKS as decrypt_kernel (k_ntt.cu).  COEFF form: forward split of c2 (its exchange writes
// c2^ s straight into this CTA's share), inverse split, + c1.  NTT form: inverse split of
// c1 + c2 s read from global memory.  Each output position is handled by the same thread
// in every limb, so the CRT check re-reads only words the thread wrote itself.
template <int LOGN, int FORM, bool NR, bool PLAIN = false>
__global__ void __launch_bounds__(256, ZINC_SPLIT_MINB) decrypt_split_kernel(DecryptArgs a) {
  using G = SplitGeo<LOGN>;
  constexpr int N = 1 << LOGN, S = G::S, NL = G::NL;
  extern __shared__ __align__(16) uint64_t sm[];
  __shared__ int bad_flag;
  __shared__ __align__(8) uint64_t cl_mbar[2];
  ClusterBar cb{cl_mbar, 0};
  cb.init<S>();
  const size_t b = blockIdx.x / S;
  const int r = (int)cluster_rank();
  const int L = a.L;
  int bad = 0;
  int64_t *x0 = a.coeff_out + b * N;
  const uint64_t q0 = a.limbs[0].q;
  for (int i = 0; i < L; ++i) {
    const LimbConst c = a.limbs[i];
    const uint64_t q = c.q;
    const uint64_t *c1 = a.ct + b * 2 * L * N + (size_t)i * N;
    const uint64_t *c2 = c1 + (size_t)L * N;
    const uint64_t *s = a.sk_ntt + (size_t)i * N, *ssh = a.sk_sh + (size_t)i * N;
    const Tw *itw = a.itw + (size_t)i * N;
    // w = {c1[x] (COEFF form), x0[x] (limbs > 0)}: loaded one exchange index ahead (pre1)
    auto epilogue = [&](int x, uint64_t v, ulonglong2 w) {
      uint64_t xi = csub(v, q);
      if (FORM == 1) xi = add_mod(xi, w.x, q);
      if (!PLAIN && c.scheme == SCHEME_BFV) {
        a.xl_out[(b * L + i) * N + x] = xi;
        return;
      }
      if (!PLAIN && a.x128_out) {  // wide CKKS: x from limbs 0 and 1, checked on the others
        int64_t *xw = a.x128_out + (b * N + x) * 2;
        if (i == 0) {
          xw[0] = (int64_t)xi;
        } else if (i == 1) {
          const uint64_t xa = (uint64_t)xw[0];
          const uint64_t x0r = reduce_i64q((int64_t)xa, q, c.mu64);
          const uint64_t k = mul_mod(add_mod(xi, x0r ? q - x0r : 0, q), a.q0inv_q1, c);
          unsigned __int128 X = (unsigned __int128)k * q0 + xa;
          const unsigned __int128 Q2 = (unsigned __int128)q0 * q;
          __int128 Xs = (X > Q2 / 2) ? (__int128)X - (__int128)Q2 : (__int128)X;
          xw[0] = (int64_t)(uint64_t)Xs;
          xw[1] = (int64_t)(Xs >> 64);
        } else if (reduce_i128(xw[1], (uint64_t)xw[0], c) != xi) {
          bad = 1;
        }
        return;
      }
      if (i == 0) {
        const int64_t v = xi > q0 / 2 ? -(int64_t)(q0 - xi) : (int64_t)xi;
        x0[x] = (!PLAIN && c.scheme == SCHEME_BGV && L == 1) ? (int64_t)mod_t(v, c.t, c.t_mu) : v;
      } else {
        if (reduce_i64((int64_t)w.y, c) != xi) bad = 1;
        if (!PLAIN && c.scheme == SCHEME_BGV && i == L - 1) x0[x] = (int64_t)mod_t((int64_t)w.y, c.t, c.t_mu);
      }
    };
    // x0 is re-read only by the thread that wrote it (the same output positions every limb)
    auto pre = [&](int x) {
      return make_ulonglong2(FORM == 1 ? (uint64_t)ldm(reinterpret_cast<const int64_t *>(c1) + x) : 0, i > 0 ? (uint64_t)x0[x] : 0);
    };
    if (FORM == 0) {
      ntt_inverse_split<LOGN, true>(sm, cb, itw, c,
          [&](int base, uint64_t (&v)[16]) {
#pragma unroll
            for (int u = 0; u < 16; u += 4) {
              const U64x4 w1 = ld4_nc(c1 + base + u), w2 = ld4_nc(c2 + base + u), ws = ld4_nc(s + base + u),
                          wh = ld4_nc(ssh + base + u);
#pragma unroll
              for (int j = 0; j < 4; ++j) v[u + j] = w1.v[j] + mul_shoup_lazy(w2.v[j], ws.v[j], wh.v[j], q);
            }
          },
          with_pre1(epilogue, pre));
    } else {
      const Tw *tw = a.tw + (size_t)i * N;
      // the forward split reads its early-pass twiddles from global memory here (stw = tw)
      ntt_forward_split<LOGN, NR, true>(sm, cb, tw, q,
          [&](int x) { return (uint64_t)ldm(reinterpret_cast<const int64_t *>(c2) + x); },  // stride S, read once: no L1 allocation
          [&](int x0g, uint64_t (&v)[S]) {
#pragma unroll
            for (int u = 0; u < S; u += 4) {
              const U64x4 ws = ld4_nc(s + x0g + u), wh = ld4_nc(ssh + x0g + u);
#pragma unroll
              for (int j = 0; j < 4; ++j) sm[pad16(x0g + u + j - r * NL)] = mul_shoup_lazy(v[u + j], ws.v[j], wh.v[j], q);
            }
          },
          tw);
      ntt_inverse_split<LOGN, false>(sm, cb, itw, c, [](int, uint64_t (&)[16]) {},
                                     with_pre1(epilogue, pre));
    }
  }
  cb.settle_exit();
  bad = __syncthreads_or(bad);
  // the cluster's verdict: every CTA publishes its flag, rank 0 reads them over DSMEM
  if (threadIdx.x == 0) bad_flag = bad;
  cluster_sync_all();
  if (threadIdx.x == 0 && r == 0 && a.status_out) {
    int any = 0;
    for (int cc = 0; cc < S; ++cc) any |= *peer_smem(&bad_flag, (uint32_t)cc);
    a.status_out[b] = any;
  }
  cluster_sync_all();
}

// ============================================================ launchers
template <int LOGN> static size_t split_smem(int extra) {
  return SplitSmem<LOGN>::DATA + SplitSmem<LOGN>::TW + (size_t)extra;
}
template <int LOGN>
static cudaError_t launch_zinc_ntt_split_t(const ZincNttArgs &a, int mode, size_t batch, int groups, cudaStream_t s) {
  using G = SplitGeo<LOGN>;
  const dim3 grid((unsigned)(batch * G::S), groups, a.t_split ? 2 : 1);
  const size_t smem = split_smem<LOGN>(2 * G::NL);
  if (mode == 2) return launch_ex(zinc_ntt_split_kernel<LOGN, 2>, grid, G::THREADS, smem, G::S, s, a);
  if (mode == 1) return launch_ex(zinc_ntt_split_kernel<LOGN, 1>, grid, G::THREADS, smem, G::S, s, a);
  return launch_ex(zinc_ntt_split_kernel<LOGN, 0>, grid, G::THREADS, smem, G::S, s, a);
}
template <int LOGN>
static cudaError_t launch_vanilla_split_t(const VanillaArgs &a, int form, int mode, size_t batch, int groups,
                                          cudaStream_t s) {
  using G = SplitGeo<LOGN>;
  const dim3 grid((unsigned)(batch * G::S), groups, form == 0 && a.u_hat ? 3 : 1);
  const size_t smem = split_smem<LOGN>(2 * G::NL + G::NL / 4);
#define VS(K, M) launch_ex(K<LOGN, M>, grid, G::THREADS, smem, G::S, s, a)
  if (form == 0) return mode == 2 ? VS(vanilla_ntt_split_kernel, 2) : mode == 1 ? VS(vanilla_ntt_split_kernel, 1)
                                                                            : VS(vanilla_ntt_split_kernel, 0);
  return mode == 2 ? VS(vanilla_coeff_split_kernel, 2) : mode == 1 ? VS(vanilla_coeff_split_kernel, 1)
                                                               : VS(vanilla_coeff_split_kernel, 0);
#undef VS
}
template <int LOGN>
static cudaError_t launch_decrypt_split_t(const DecryptArgs &a, int form, bool nr, size_t batch, cudaStream_t s) {
  using G = SplitGeo<LOGN>;
  const dim3 grid((unsigned)(batch * G::S));
  const size_t smem = SplitSmem<LOGN>::DATA;
#define DS(F, R, P) launch_ex(decrypt_split_kernel<LOGN, F, R, P>, grid, G::THREADS, smem, G::S, s, a)
  if (a.plain_ckks) return form == 0 ? DS(0, false, true) : nr ? DS(1, true, true) : DS(1, false, true);
  return form == 0 ? DS(0, false, false) : nr ? DS(1, true, false) : DS(1, false, false);
#undef DS
}

cudaError_t launch_zinc_ntt_split(int log_n, const ZincNttArgs &a, int mode, size_t batch, int groups, cudaStream_t s) {
  if (log_n == 14) return launch_zinc_ntt_split_t<14>(a, mode, batch, groups, s);
  if (log_n == 15) return launch_zinc_ntt_split_t<15>(a, mode, batch, groups, s);
  return cudaErrorInvalidValue;
}
cudaError_t launch_vanilla_split(int log_n, const VanillaArgs &a, int form, int mode, size_t batch, int groups,
                                 cudaStream_t s) {
  if (log_n == 14) return launch_vanilla_split_t<14>(a, form, mode, batch, groups, s);
  if (log_n == 15) return launch_vanilla_split_t<15>(a, form, mode, batch, groups, s);
  return cudaErrorInvalidValue;
}
cudaError_t launch_decrypt_split(int log_n, const DecryptArgs &a, int form, bool nr, size_t batch, cudaStream_t s) {
  if (log_n == 14) return launch_decrypt_split_t<14>(a, form, nr, batch, s);
  if (log_n == 15) return launch_decrypt_split_t<15>(a, form, nr, batch, s);
  return cudaErrorInvalidValue;
}

}  // namespace zinc
