// zinc_coeff.cuh -- the COEFF-form Zinc add/inject body (S4 S5 S8), shared by
// the standalone kernel (k_stream.cu) and the encode-fused kernel (k_fused.cu).
#pragma once

#include "kcommon.cuh"

namespace zinc {

// ============================================================ Zinc, COEFF form
// Algorithm 1 with cache and output in coefficient form:
//   c1'[i][j] = [zero1[i][j] + m[j] + e1'[j]]_{q_i},  c2'[i][j] = [zero2[i][j] + e2'[j]]_{q_i}.
// CTA (x, y): coefficient tile [x*T, (x+1)*T), messages [y*mpc, (y+1)*mpc).  The
// cache tile [2][L][T] is staged once into shared memory with bulk async copies
// (cp.async.bulk, the 1-D TMA path, completing on an mbarrier) and reused for
// every message; each thread owns 2 coefficients, draws e1'/e2' with one Philox
// call each (C-4 block = j/2), and streams 2L 16-byte stores per message.
//
// Per output word the work is one 64-bit modular add plus a share of the
// limb-independent prologue, so the kernel stays HBM-bound: v = m + e1' is
// formed once per coefficient; when |v| < min_i q_i for the whole warp (every
// CKKS plaintext at these scales) the residue of v mod q_i is v or q_i + v
// (branch-free), otherwise an exact Barrett path runs.  The next message's m
// is loaded while the current one is stored (software pipelining).
ZINC_DEV uint64_t mod_add_signed(uint64_t z, int64_t v, uint64_t q) {
  // z in [0, q), |v| < q  ->  [z + v]_q
  const uint64_t r = (uint64_t)v + (q & (uint64_t)(v >> 63));  // v mod q in [0, q)
  const uint64_t s = z + r;
  return s >= q ? s - q : s;
}

// One CTA's work: coefficient tile `tile_x`, message group `group_y`; `tile`
// is the CTA's dynamic shared memory ([2][L][T] cache words, then q[L], mu64[L]).
template <int LC>
ZINC_DEV void zinc_coeff_body(const ZincCoeffArgs &a, int tile_x, int group_y, uint64_t *tile) {
  __shared__ __align__(8) uint64_t mbar;
  const int T = 2 * blockDim.x;
  const int L = LC > 0 ? LC : a.L;
  const int j0 = tile_x * T;
  uint64_t *sq = tile + (size_t)2 * L * T, *smu = sq + L, *sdel = smu + L, *sdelsh = sdel + L;
  uint64_t *sr64 = sdelsh + L, *sr64sh = sr64 + L, *sfmask = sr64sh + L, *sfcb = sfmask + L;  // wide path
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    sr64[i] = a.limbs[i].r64;
    sr64sh[i] = a.limbs[i].r64_sh;
    sfmask[i] = a.limbs[i].fold_mask;
    sfcb[i] = (uint64_t)a.limbs[i].fold_c | ((uint64_t)a.limbs[i].b << 32) | ((uint64_t)a.limbs[i].fold_n << 40);
    sq[i] = a.limbs[i].q;
    smu[i] = a.limbs[i].mu64;
    sdel[i] = a.limbs[i].delta;
    sdelsh[i] = a.limbs[i].delta_sh;
  }
  const uint32_t scheme = a.limbs[0].scheme;
  const uint64_t tpl = a.limbs[0].t, tmu = a.limbs[0].t_mu;
  if (threadIdx.x == 0) {
    uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    const uint32_t bytes = (uint32_t)(T * sizeof(uint64_t));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes * 2 * L) : "memory");
    for (int r = 0; r < 2 * L; ++r) {
      const uint64_t *src = a.cache + (size_t)r * a.n + j0;
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(tile + (size_t)r * T);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(src), "r"(bytes), "r"(mb) : "memory");
    }
  }
  if (threadIdx.x == 32 && a.prefetch_bytes) {
    // warm this CTA's share of the next chunk's slots into L2 (the next encode reads them)
    const size_t nblk = (size_t)gridDim.x * gridDim.y;
    const size_t share = ((a.prefetch_bytes + nblk - 1) / nblk + 15) & ~(size_t)15;
    const size_t lo = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * share;
    if (lo < a.prefetch_bytes) {
      const uint32_t sz = (uint32_t)min(share, a.prefetch_bytes - lo);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.prefetch + lo), "r"(sz) : "memory");
    }
  }
  const int jl = 2 * threadIdx.x;       // local coefficient pair
  const int j = j0 + jl;
  const size_t b_begin = (size_t)group_y * a.msgs_per_cta;
  size_t b_end = b_begin + a.msgs_per_cta;
  if (b_end > a.batch) b_end = a.batch;
  const size_t lnn = (size_t)L * a.n;
  // under a programmatic dependent launch the encode kernel that wrote m may still be
  // running: everything above overlaps it; m is read only after its grid completed
  pdl_trigger();
  pdl_wait();
  // first message's plaintext words, fetched while the tile is in flight
  ulonglong2 mv = make_ulonglong2(0, 0);
  if (a.m && b_begin < b_end) mv = ld2_nc(a.m + b_begin * a.m_stride + j);
  {
    uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(mb) : "memory");
    }
  }
  const uint64_t qmin = a.qmin;
  if (a.m128) {
    // 128-bit plaintexts (f3, the paper's Delta = 2^55): per limb, [z + hi 2^64 + lo + e1']_q.
    // Fast path (the whole warp has |hi| < qmin and every limb folds once): hi 2^64 = hi r64 as
    // a Shoup product by the constant r64 = 2^64 mod q, lo folded once (below 2q), one fold of
    // the sum finishes -- per-limb constants from shared memory.  Otherwise reduce_i128.
    pdl_wait();
    bool fold1 = true;
    for (int i = 0; i < L; ++i) fold1 &= ((sfcb[i] >> 40) & 0xff) == 1;
    for (size_t b = b_begin; b < b_end; ++b) {
      const uint64_t msg = a.msg_base + b;
      const int64_t *mp = a.m128 + (b * a.n + j) * 2;
      const ulonglong2 p0 = ld2_nc(mp), p1 = ld2_nc(mp + 2);  // (lo, hi) of coefficients j, j + 1
      const uint4 w1 = stream_block(a.seed, msg, TAG_ZINC_E1, 0, (uint32_t)(j >> 1));
      const uint4 w2 = stream_block(a.seed, msg, TAG_ZINC_E2, 0, (uint32_t)(j >> 1));
      const int e0 = cbd_lo(w1), e1 = cbd_hi(w1), f0 = cbd_lo(w2), f1 = cbd_hi(w2);
      const int64_t h0 = (int64_t)p0.y, h1 = (int64_t)p1.y;
      const bool hsmall = (uint64_t)(h0 < 0 ? -h0 : h0) < qmin && (uint64_t)(h1 < 0 ? -h1 : h1) < qmin;
      uint64_t *out = a.ct + b * 2 * lnn + j;
      // Tiny high words (the paper's value ranges put |m| a few bits past 2^64): V = hi 2^64 + lo +
      // e1' is formed once per coefficient as a signed 128-bit value (hh, ll); with |hh| < 2^hb,
      // hb = 63 - bits(q_max), the term hh 2^64 = hh r64 (mod q) is one 32 x 64-bit product below
      // 2^hb q < 2^63 (2^hb q minus it when hh < 0): no Shoup product, no per-limb residue of e1'.
      // The sum with fold(ll) and the cache word stays below 2^64 and one fold finishes.
      const int hb = a.wide_hb;
      const uint64_t ee0 = (uint64_t)(int64_t)e0, ee1 = (uint64_t)(int64_t)e1;
      const uint64_t ll0 = p0.x + ee0, ll1 = p1.x + ee1;
      const int64_t hh0 = h0 + (e0 < 0 ? -1 : 0) + (ll0 < p0.x ? 1 : 0), hh1 = h1 + (e1 < 0 ? -1 : 0) + (ll1 < p1.x ? 1 : 0);
      const uint64_t ah0 = (uint64_t)(hh0 < 0 ? -hh0 : hh0), ah1 = (uint64_t)(hh1 < 0 ? -hh1 : hh1);
      const bool tiny = hb > 0 && ((ah0 | ah1) >> hb) == 0;
      if (fold1 && __all_sync(0xffffffffu, tiny)) {
        const uint32_t a0 = (uint32_t)ah0, a1 = (uint32_t)ah1;
#pragma unroll 2
        for (int i = 0; i < L; ++i) {
          const uint64_t q = sq[i], r64 = sr64[i], fm = sfmask[i], fcb = sfcb[i];
          const uint32_t fc = (uint32_t)fcb, fb = (uint32_t)(fcb >> 32) & 0xff;
          uint64_t z10, z11, z20, z21;
          ld2(tile + (size_t)i * T + jl, z10, z11);
          ld2(tile + (size_t)(L + i) * T + jl, z20, z21);
          auto fold = [&](uint64_t x) { return fold_once(x, fb - 32, (uint32_t)(fm >> 32), fc); };
          const uint64_t qk = q << hb;
          const uint64_t t0 = (uint64_t)a0 * r64, t1 = (uint64_t)a1 * r64;  // below 2^hb q
          // term below 2^63, fold(ll) below 2q, the cache word below q
          const uint64_t s0 = (hh0 < 0 ? qk - t0 : t0) + fold(ll0) + z10;
          const uint64_t s1 = (hh1 < 0 ? qk - t1 : t1) + fold(ll1) + z11;
          st2_cs(out + (size_t)i * a.n, csub(fold(s0), q), csub(fold(s1), q));
          st2_cs(out + lnn + (size_t)i * a.n, mod_add_signed(z20, f0, q), mod_add_signed(z21, f1, q));
        }
      } else if (fold1 && __all_sync(0xffffffffu, hsmall)) {
#pragma unroll 2
        for (int i = 0; i < L; ++i) {
          const uint64_t q = sq[i], r64 = sr64[i], r64s = sr64sh[i], fm = sfmask[i], fcb = sfcb[i];
          const uint32_t fc = (uint32_t)fcb, fb = (uint32_t)(fcb >> 32) & 0xff;
          uint64_t z10, z11, z20, z21;
          ld2(tile + (size_t)i * T + jl, z10, z11);
          ld2(tile + (size_t)(L + i) * T + jl, z20, z21);
          auto fold = [&](uint64_t x) { return fold_once(x, fb - 32, (uint32_t)(fm >> 32), fc); };
          // each term below 2q, the sum below 6q < 2^64
          const uint64_t s0 = mul_shoup_lazy(reduce_small(h0, q), r64, r64s, q) + fold(p0.x) + z10 + reduce_small(e0, q);
          const uint64_t s1 = mul_shoup_lazy(reduce_small(h1, q), r64, r64s, q) + fold(p1.x) + z11 + reduce_small(e1, q);
          st2_cs(out + (size_t)i * a.n, csub(fold(s0), q), csub(fold(s1), q));
          st2_cs(out + lnn + (size_t)i * a.n, mod_add_signed(z20, f0, q), mod_add_signed(z21, f1, q));
        }
      } else {
#pragma unroll 1
        for (int i = 0; i < L; ++i) {
          const LimbConst &c = a.limbs[i];
          const uint64_t q = sq[i];
          uint64_t z10, z11, z20, z21;
          ld2(tile + (size_t)i * T + jl, z10, z11);
          ld2(tile + (size_t)(L + i) * T + jl, z20, z21);
          const uint64_t r0 = reduce_i128(h0, p0.x, c), r1 = reduce_i128(h1, p1.x, c);
          st2_cs(out + (size_t)i * a.n, mod_add_signed(add_mod(z10, r0, q), e0, q),
                 mod_add_signed(add_mod(z11, r1, q), e1, q));
          st2_cs(out + lnn + (size_t)i * a.n, mod_add_signed(z20, f0, q), mod_add_signed(z21, f1, q));
        }
      }
    }
    return;
  }
  for (size_t b = b_begin; b < b_end; ++b) {
    const uint64_t msg = a.msg_base + b;
    const int64_t m0 = (int64_t)mv.x, m1 = (int64_t)mv.y;
    if (a.m && b + 1 < b_end) mv = ld2_nc(a.m + (b + 1) * a.m_stride + j);  // prefetch
    const uint4 w1 = stream_block(a.seed, msg, TAG_ZINC_E1, 0, (uint32_t)(j >> 1));
    const uint4 w2 = stream_block(a.seed, msg, TAG_ZINC_E2, 0, (uint32_t)(j >> 1));
    const int e0 = cbd_lo(w1), e1 = cbd_hi(w1);
    const int f0 = cbd_lo(w2), f1 = cbd_hi(w2);
    uint64_t *out = a.ct + b * 2 * lnn + j;
    if (scheme == SCHEME_BFV) {
      // Eq. 12, Zinc "without modification": c1' = zero1 + Delta (m mod t) + e1' (per limb)
      const uint64_t mt0 = mod_t(m0, tpl, tmu), mt1 = mod_t(m1, tpl, tmu);
#pragma unroll 1
      for (int i = 0; i < L; ++i) {
        const uint64_t q = sq[i];
        uint64_t z10, z11, z20, z21;
        ld2(tile + (size_t)i * T + jl, z10, z11);
        ld2(tile + (size_t)(L + i) * T + jl, z20, z21);
        const uint64_t d0 = csub(mul_shoup_lazy(mt0, sdel[i], sdelsh[i], q), q);
        const uint64_t d1 = csub(mul_shoup_lazy(mt1, sdel[i], sdelsh[i], q), q);
        st2_cs(out + (size_t)i * a.n, mod_add_signed(add_mod(z10, d0, q), e0, q),
               mod_add_signed(add_mod(z11, d1, q), e1, q));
        st2_cs(out + lnn + (size_t)i * a.n, mod_add_signed(z20, f0, q), mod_add_signed(z21, f1, q));
      }
      // the library's own encode scratch is dead once read (the stores above consumed it):
      // drop its L2 lines without a write-back.  Lanes 8r..8r+7 share a 128-byte line.
      if (a.discard_m && (threadIdx.x & 7) == 0)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(a.m + b * a.m_stride + j) : "memory");
      continue;
    }
    // CKKS: v = m + e1' (|m| < 2^62 rules out int64 overflow); BGV (Eq. 13): v = (m mod t) +
    // t e1', g = t e2'.  Either way v is limb-independent and |v| < qmin is the fast path.
    int64_t v0, v1, g0 = f0, g1 = f1;
    bool in_range = true;
    if (scheme == SCHEME_BGV) {
      v0 = (int64_t)mod_t(m0, tpl, tmu) + (int64_t)tpl * e0;
      v1 = (int64_t)mod_t(m1, tpl, tmu) + (int64_t)tpl * e1;
      g0 = (int64_t)tpl * f0;
      g1 = (int64_t)tpl * f1;
    } else {
      v0 = m0 + e0;
      v1 = m1 + e1;
      in_range = (m0 > -(1ll << 62)) && (m0 < (1ll << 62)) && (m1 > -(1ll << 62)) && (m1 < (1ll << 62));
    }
    const uint64_t a0 = v0 < 0 ? (uint64_t)0 - (uint64_t)v0 : (uint64_t)v0;
    const uint64_t a1 = v1 < 0 ? (uint64_t)0 - (uint64_t)v1 : (uint64_t)v1;
    const uint64_t ag = (uint64_t)(g0 < 0 ? -g0 : g0) | (uint64_t)(g1 < 0 ? -g1 : g1);
    const bool small = in_range && a0 < qmin && a1 < qmin && ag < qmin;
    if (__all_sync(0xffffffffu, small)) {
#pragma unroll
      for (int i = 0; i < L; ++i) {
        const uint64_t q = sq[i];
        uint64_t z10, z11, z20, z21;
        ld2(tile + (size_t)i * T + jl, z10, z11);
        ld2(tile + (size_t)(L + i) * T + jl, z20, z21);
        st2_cs(out + (size_t)i * a.n, mod_add_signed(z10, v0, q), mod_add_signed(z11, v1, q));
        st2_cs(out + lnn + (size_t)i * a.n, mod_add_signed(z20, g0, q), mod_add_signed(z21, g1, q));
      }
    } else {
#pragma unroll 1
      for (int i = 0; i < L; ++i) {
        const LimbConst &c = a.limbs[i];
        const uint64_t q = c.q;
        uint64_t z10, z11, z20, z21;
        ld2(tile + (size_t)i * T + jl, z10, z11);
        ld2(tile + (size_t)(L + i) * T + jl, z20, z21);
        st2_cs(out + (size_t)i * a.n, add_mod(z10, pt_plus_e(m0, e0, c), q), add_mod(z11, pt_plus_e(m1, e1, c), q));
        st2_cs(out + lnn + (size_t)i * a.n, add_mod(z20, err_term(f0, c), q), add_mod(z21, err_term(f1, c), q));
      }
    }
    // the library's own encode scratch is dead once read (the stores above consumed it):
    // drop its L2 lines without a write-back.  Lanes 8r..8r+7 share a 128-byte line.
    if (a.discard_m && (threadIdx.x & 7) == 0)
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(a.m + b * a.m_stride + j) : "memory");
  }
}

}  // namespace zinc
