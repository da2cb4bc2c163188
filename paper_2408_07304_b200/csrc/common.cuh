// common.cuh -- device building blocks of the B200 Zinc path (sm_100a).
//
// 64-bit modular arithmetic (Shoup twiddle products, Barrett for
// variable x variable, lazy Harvey butterflies), the Philox4x32-10 counter-based
// generator and the ternary / CBD / uniform samplers of docs/CONVENTIONS.md C-4.
// Nothing here is shared with oracle/ (which uses plain `unsigned __int128 %`).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define ZINC_DEV __device__ __forceinline__

namespace zinc {

// Per-limb constants, uploaded once per context (device array of L).
struct LimbConst {
  uint64_t q;        // prime modulus, q = 1 mod 2N, q < 2^61
  uint64_t two_q;
  uint64_t mu64;     // floor(2^64 / q): reduction of a 64-bit value
  uint64_t bmu;      // floor(2^(2b) / q), b = bitlen(q): Barrett of a 128-bit product
  uint32_t b;        // bit length of q
  uint32_t pad;
  uint64_t ninv;     // N^-1 mod q
  uint64_t ninv_sh;  // Shoup companion of ninv
  uint64_t ninv_w;   // N^-1 * psi^-brv(1) mod q (last GS stage, folded scaling)
  uint64_t ninv_w_sh;
  // scheme (section 4.2): the same in every limb's entry
  uint32_t scheme;   // SCHEME_CKKS / SCHEME_BFV / SCHEME_BGV
  uint32_t pad2;
  uint64_t t;        // plaintext modulus (BFV, BGV), 2 <= t < 2^32
  uint64_t t_mu;     // floor(2^64 / t)
  uint64_t delta;    // BFV: floor(Q/t) mod q;  Shoup companion below
  uint64_t delta_sh;
  uint64_t dec_i;    // BFV decrypt: floor(t Q~_i / q_i) mod t, Q~_i = (Q/q_i)^-1 mod q_i
  uint64_t dec_f;    // BFV decrypt: round(frac(t Q~_i / q_i) 2^64)
  uint64_t r64;      // 2^64 mod q (128-bit plaintext residues)
  // q = 2^b - fold_c with fold_c < 2^32 (the C-1 primes sit just below 2^b): reduce_fold
  uint64_t fold_mask;  // 2^b - 1
  uint32_t fold_c;
  uint32_t fold_n;     // folds that bring any 64-bit value below 2q (1 or 2); 0: use reduce64
  uint64_t qinv_hi, qinv_lo;  // floor(2^128 / q): Shoup companions on the device (shoup_prep_kernel)
  uint64_t r64_sh;   // Shoup companion of r64 = 2^64 mod q
  uint32_t fold_sh;  // b - 32 (reduce_fold works on the high word: b > 32 whenever fold_n > 0)
  uint32_t fold_mhi; // 2^(b-32) - 1
};
enum : uint32_t { SCHEME_CKKS = 0, SCHEME_BFV = 1, SCHEME_BGV = 2 };

// Random stream tags (C-4).
enum Tag : uint32_t {
  TAG_SK = 1, TAG_PK_E = 2, TAG_PK_A = 3, TAG_ENC_U = 4, TAG_ENC_E1 = 5, TAG_ENC_E2 = 6,
  TAG_ZINC_E1 = 7, TAG_ZINC_E2 = 8
};

// ------------------------------------------------------------------ modular
// w*y mod q in [0, 2q) for any y < 2^64, given wp = floor(w 2^64 / q), w < q.
ZINC_DEV uint64_t mul_shoup_lazy(uint64_t y, uint64_t w, uint64_t wp, uint64_t q) {
  return w * y - __umul64hi(wp, y) * q;
}
ZINC_DEV uint64_t csub(uint64_t x, uint64_t m) { return x >= m ? x - m : x; }
ZINC_DEV uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) { return csub(a + b, q); }  // a,b < q
// a*b mod q, a, b < q < 2^61 (Barrett with mu = floor(2^(2b)/q); remainder < 3q)
ZINC_DEV uint64_t mul_mod(uint64_t a, uint64_t b, const LimbConst &c) {
  uint64_t lo = a * b, hi = __umul64hi(a, b);
  uint64_t x1 = (hi << (65 - c.b)) | (lo >> (c.b - 1));
  uint64_t ph = __umul64hi(x1, c.bmu), pl = x1 * c.bmu;
  uint64_t q3 = (ph << (63 - c.b)) | (pl >> (c.b + 1));
  uint64_t r = lo - q3 * c.q;
  r = csub(r, c.q);
  return csub(r, c.q);
}
// [a + w y]_q for canonical a, a key word w < q with Shoup companion wp, and any y < 2^64
// (the lazy output of a transform): the Shoup product is in [0, 2q), the sum below 3q.
ZINC_DEV uint64_t add_shoup(uint64_t a, uint64_t y, uint64_t w, uint64_t wp, uint64_t q) {
  return csub(csub(a + mul_shoup_lazy(y, w, wp, q), 2 * q), q);
}
// Canonical residue of a signed 64-bit integer (reading A15); mu = floor(2^64/q).
ZINC_DEV uint64_t reduce_i64q(int64_t v, uint64_t q, uint64_t mu) {
  uint64_t a = v < 0 ? (uint64_t)0 - (uint64_t)v : (uint64_t)v;
  uint64_t r;
  if (a < q) {
    r = a;
  } else {
    r = a - __umul64hi(a, mu) * q;  // [0, 2q)
    r = csub(r, q);
  }
  return (v < 0 && r != 0) ? q - r : r;
}
ZINC_DEV uint64_t reduce_i64(int64_t v, const LimbConst &c) { return reduce_i64q(v, c.q, c.mu64); }
// Residue of m + e for an int64 plaintext coefficient m and a small error e,
// exact even when m + e overflows int64 (then both are reduced separately).
ZINC_DEV uint64_t reduce_m_plus_e(int64_t m, int e, uint64_t q, uint64_t mu) {
  const int64_t v = (int64_t)((uint64_t)m + (uint64_t)(int64_t)e);
  const bool ovf = ((m ^ v) & ((int64_t)e ^ v)) < 0;
  if (!ovf) return reduce_i64q(v, q, mu);
  const uint64_t r = reduce_i64q(m, q, mu), f = e < 0 ? (uint64_t)((int64_t)q + e) : (uint64_t)e;
  return csub(r + f, q);
}
// Residue of a small signed value |v| < q.
ZINC_DEV uint64_t reduce_small(int64_t v, uint64_t q) {
  return v < 0 ? (uint64_t)(v + (int64_t)q) : (uint64_t)v;
}

// ------------------------------------------------------------------ wide plaintexts
// A 128-bit plaintext coefficient is stored as an int64 pair (lo, hi): v = hi 2^64 + lo.
// Integral double -> pair (round half away from zero first, as llround does).
ZINC_DEV void store_i128(int64_t *p, double v) {
  const double r = round(v);
  if (fabs(r) < 9.0e18) {
    const int64_t x = (int64_t)r;
    p[0] = x;
    p[1] = x < 0 ? -1 : 0;
  } else {  // |r| >= 2^63: r has at most 53 significant bits, both parts are exact
    const double hi = floor(r * 0x1p-64);
    const double lo = r - hi * 0x1p64;  // [0, 2^64)
    p[0] = (int64_t)(uint64_t)lo;
    p[1] = (int64_t)hi;
  }
}
ZINC_DEV double load_i128(const int64_t *p) { return (double)p[1] * 0x1p64 + (double)(uint64_t)p[0]; }
// Canonical residue of hi 2^64 + lo (hi signed, lo unsigned).
ZINC_DEV uint64_t reduce_i128(int64_t hi, uint64_t lo, const LimbConst &c) {
  uint64_t l = lo - __umul64hi(lo, c.mu64) * c.q;  // [0, 2q)
  l = csub(l, c.q);
  return add_mod(mul_mod(reduce_i64q(hi, c.q, c.mu64), c.r64, c), l, c.q);
}

// ------------------------------------------------------------------ schemes
// m mod t in [0, t) for any int64 m (t < 2^32, t_mu = floor(2^64 / t)).
ZINC_DEV uint64_t mod_t(int64_t m, uint64_t t, uint64_t t_mu) {
  const uint64_t a = m < 0 ? (uint64_t)0 - (uint64_t)m : (uint64_t)m;
  uint64_t r = a - __umul64hi(a, t_mu) * t;  // [0, 2t)
  r = csub(r, t);
  return (m < 0 && r != 0) ? t - r : r;
}
// Residue of the scheme's c1 plaintext-plus-error term for plaintext coefficient
// m and error e: CKKS m + e (Eq. 8); BFV Delta (m mod t) + e (Eq. 12);
// BGV (m mod t) + t e (Eq. 13).
// INTS = false compiles the CKKS term only (the kernels' CKKS instantiations).
template <bool INTS = true>
ZINC_DEV uint64_t pt_plus_e(int64_t m, int e, const LimbConst &c) {
  if (!INTS || c.scheme == SCHEME_CKKS) return reduce_m_plus_e(m, e, c.q, c.mu64);
  const uint64_t mt = mod_t(m, c.t, c.t_mu);
  if (c.scheme == SCHEME_BFV)
    return add_mod(csub(mul_shoup_lazy(mt, c.delta, c.delta_sh, c.q), c.q), reduce_small(e, c.q), c.q);
  return reduce_i64q((int64_t)mt + (int64_t)c.t * e, c.q, c.mu64);
}
// A plaintext word read by a transform's first pass.  Each is used once per limb by one thread
// and the cluster kernels read them with stride S (8 of every 32 bytes): with ZINC_M_NOALLOC
// the load bypasses L1 allocation, which leaves L1 to the twiddles.
#ifndef ZINC_M_NOALLOC
#define ZINC_M_NOALLOC 1
#endif
ZINC_DEV int64_t ldm(const int64_t *p) {
#if ZINC_M_NOALLOC
  // volatile: callers guard this load with a null check (m = 0 encryptions), and a plain asm is a
  // pure function the compiler may hoist above its guard (seen once: a fault in an experimental
  // build of the N = 2^15 vanilla kernel, profiles/r02d_experiments.txt)
  int64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}
// Index of twiddle e in the padded shared-memory copy of a table (TW_SMEM = 2): one 16-byte pad per
// 8, 64 and 512 entries.  The passes read entries (o + c) 2^k for consecutive o; unpadded, every
// stride of 8 entries or more puts a warp's loads in one 128-byte bank row (measured 8x the ideal
// wavefronts on 15 of the second pass's loads); padded, strides 2^0 .. 2^9 spread evenly.
__host__ __device__ constexpr int fft_twpad(int e) { return e + (e >> 3) + (e >> 6) + (e >> 9); }
// Entries of the padded copy of an n-entry table.
__host__ __device__ constexpr int fft_twpad_size(int n) { return fft_twpad(n - 1) + 1; }

// Index of coefficient x in a plaintext de-interleaved by 2^d (EncodeArgs::deint_log), d = 0: x.
ZINC_DEV int deint_idx(int x, int d, int log_n) { return ((x & ((1 << d) - 1)) << (log_n - d)) + (x >> d); }
// The words x = 2^log_s i + r (i = 0, 1, ...) of a plaintext stored in natural order (d = 0) or
// de-interleaved by 2^d = 2^log_s (deint_idx): word i of the subsequence sits at p[i stride].
struct MSub {
  const int64_t *p;
  int stride;
};
ZINC_DEV MSub m_sub(const int64_t *m, int r, int log_s, int d, int log_n) {
  if (!m) return MSub{nullptr, 1};
  return d ? MSub{m + ((size_t)r << (log_n - d)), 1} : MSub{m + r, 1 << log_s};
}
// Residue of the scheme's error term: e (CKKS, BFV) or t e (BGV).
// The plaintext-plus-error input of the first forward transform as a two-phase load
// (ntt.cuh TwoPhase): fetch(x) reads m[x] from global memory, lift(raw, x) adds the sample
// (stored at x >> SHIFT: 1 for parity-split sample buffers) and reduces.
template <bool INTS, int SHIFT = 0>
struct PtLoad {
  const int64_t *m;  // the CTA's subsequence (m_sub): word x sits at m[(x >> SHIFT) ms]
  const int8_t *se1;
  const LimbConst &c;
  int ms = 1;
  ZINC_DEV int64_t fetch(int x) const { return m ? ldm(m + (x >> SHIFT) * ms) : 0; }
  ZINC_DEV uint64_t lift(int64_t raw, int x) const { return pt_plus_e<INTS>(raw, se1[x >> SHIFT], c); }
  ZINC_DEV uint64_t operator()(int x) const { return lift(fetch(x), x); }
};

template <bool INTS = true>
ZINC_DEV uint64_t err_term(int e, const LimbConst &c) {
  return (INTS && c.scheme == SCHEME_BGV) ? reduce_i64q((int64_t)c.t * e, c.q, c.mu64) : reduce_small(e, c.q);
}

// Input of either Zinc NTT-form transform as one two-phase load, so both transforms run
// through one copy of the transform code: t = 0 gives m + e1' (fetching m), t = 1 gives
// e2' (no global load).  Samples are stored at x >> SHIFT (1: parity-split buffers).
template <bool INTS, int SHIFT = 1>
struct ZincTLoad {
  const int64_t *m;
  const int8_t *se;
  const LimbConst &c;
  int t;
  int ms = 1;  // m is the CTA's subsequence (m_sub): word x sits at m[(x >> SHIFT) ms]
  ZINC_DEV int64_t fetch(int x) const { return (t == 0 && m) ? ldm(m + (x >> SHIFT) * ms) : 0; }
  ZINC_DEV uint64_t lift(int64_t raw, int x) const {
    return t == 0 ? pt_plus_e<INTS>(raw, se[x >> SHIFT], c) : err_term<INTS>(se[x >> SHIFT], c);
  }
  ZINC_DEV uint64_t operator()(int x) const { return lift(fetch(x), x); }
  // CKKS: |m| < q/2 makes |m + e| < q, and the residue is branch-free
  ZINC_DEV bool small(int64_t raw) const { return !INTS && (uint64_t)raw + (c.q >> 1) < c.q; }
  ZINC_DEV uint64_t lift_small(int64_t raw, int x) const {
    const int64_t v = raw + se[x >> SHIFT];
    return (uint64_t)v + (c.q & (uint64_t)(v >> 63));
  }
};

// ZincTLoad with the smallness of m decided once per message (plaintext_small, k_split.cu):
// t = 1 (e2', no plaintext) is always small.
template <bool INTS, int SHIFT = 1>
struct ZincTLoadU : ZincTLoad<INTS, SHIFT> {
  bool all_small;
  ZINC_DEV bool uniform_small() const { return !INTS && (all_small || this->t != 0); }
};

// t = w Y - umulhi_approx(w', Y) q (mod 2^64), the lazy Shoup product of the butterflies below
// (w Y mod q plus at most 3q), in PTX on 32-bit halves: Q = w'_h Y_h + (hi(w'_l Y_h) + hi(w'_h Y_l))
// as one wide multiply and a 32-bit add with carry, w Y and Q q mod 2^64 as one wide multiply and
// two 32-bit multiply-adds each.  The C form of the same arithmetic compiles to ~22 SASS
// instructions per butterfly, about 4 of them register moves that set up 64-bit addend pairs;
// this one to ~18 (K11 probe, scripts/probes: 905 -> 1111 G butterflies/s).  Bit-identical.
ZINC_DEV uint64_t shoup3(uint64_t Y, uint64_t w, uint64_t wp, uint64_t q) {
  uint64_t t;
  asm("{\n\t.reg .u32 yl, yh, wl, wh, pl, ph, ql, qh, h1, h2, Ql, Qh, tl, th, ul, uh;\n\t.reg .u64 Q, T, U;\n\t"
      "mov.b64 {yl, yh}, %1;\n\tmov.b64 {wl, wh}, %2;\n\tmov.b64 {pl, ph}, %3;\n\tmov.b64 {ql, qh}, %4;\n\t"
      "mul.hi.u32 h1, pl, yh;\n\t"
      "mul.hi.u32 h2, ph, yl;\n\t"
      "mul.wide.u32 Q, ph, yh;\n\t"
      "mov.b64 {Ql, Qh}, Q;\n\t"
      "add.cc.u32 Ql, Ql, h1;\n\t"
      "addc.u32 Qh, Qh, 0;\n\t"
      "add.cc.u32 Ql, Ql, h2;\n\t"
      "addc.u32 Qh, Qh, 0;\n\t"
      "mul.wide.u32 T, wl, yl;\n\t"
      "mov.b64 {tl, th}, T;\n\t"
      "mad.lo.u32 th, wl, yh, th;\n\t"
      "mad.lo.u32 th, wh, yl, th;\n\t"
      "mul.wide.u32 U, Ql, ql;\n\t"
      "mov.b64 {ul, uh}, U;\n\t"
      "mad.lo.u32 uh, Ql, qh, uh;\n\t"
      "mad.lo.u32 uh, Qh, ql, uh;\n\t"
      "sub.cc.u32 tl, tl, ul;\n\t"
      "subc.u32 th, th, uh;\n\t"
      "mov.b64 %0, {tl, th};\n\t}"
      : "=l"(t) : "l"(Y), "l"(w), "l"(wp), "l"(q));
  return t;
}

// Forward Cooley-Tukey butterfly, lazy (Harvey): X, Y in [0, 4q) -> [0, 4q).
ZINC_DEV void ct_bfly(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wp, uint64_t q, uint64_t two_q) {
  uint64_t x = csub(X, two_q);
  uint64_t t = mul_shoup_lazy(Y, w, wp, q);
  X = x + t;
  Y = x - t + two_q;
}
// Inverse Gentleman-Sande butterfly, lazy: X, Y in [0, 4q) -> [0, 4q) (every q < 2^60 here,
// so 8q < 2^64).  The sum comes back below 4q with one conditional subtraction; the product
// uses the 3-partial-product Shoup quotient (umulhi_approx below: w d mod q plus at most 3q).
ZINC_DEV uint64_t umulhi_approx(uint64_t a, uint64_t b);
ZINC_DEV uint64_t shoup3(uint64_t Y, uint64_t w, uint64_t wp, uint64_t q);
ZINC_DEV void gs_bfly(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wp, uint64_t q, uint64_t four_q) {
  const uint64_t s = X + Y;
  const uint64_t d = X - Y + four_q;
  Y = shoup3(d, w, wp, q);
  X = s >= four_q ? s - four_q : s;
}
// [0, 4q) -> [0, q)
ZINC_DEV uint64_t canon4(uint64_t x, uint64_t q, uint64_t two_q) { return csub(csub(x, two_q), q); }
// [0, 8q) -> [0, q): outputs of the forward transforms with conditional subtractions
ZINC_DEV uint64_t canon8(uint64_t x, uint64_t q, uint64_t two_q) { return canon4(csub(x, 2 * two_q), q, two_q); }
// High word of a 64 x 64-bit product from three 32-bit partial products (a_hi b_hi exact, the
// cross terms' high halves; the low x low product and the cross terms' low halves dropped):
// exact - 2 <= result <= exact.
ZINC_DEV uint64_t umulhi_approx(uint64_t a, uint64_t b) {
  const uint32_t al = (uint32_t)a, ah = (uint32_t)(a >> 32), bl = (uint32_t)b, bh = (uint32_t)(b >> 32);
  return (uint64_t)ah * bh + __umulhi(al, bh) + __umulhi(ah, bl);
}
// Forward butterfly for moduli up to 2^60 (no lazy-free headroom): X, Y in [0, 8q) -> [0, 8q)
// with one conditional subtraction and the 3-partial-product Shoup quotient (T < 4q).
ZINC_DEV uint64_t umulhi_approx(uint64_t a, uint64_t b);
ZINC_DEV void ct_bfly_a(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wp, uint64_t q, uint64_t four_q) {
  const uint64_t x = csub(X, four_q);
  const uint64_t t = shoup3(Y, w, wp, q);
  X = x + t;
  Y = x - t + four_q;
}
// Forward butterfly without the conditional subtraction and with the cheaper Shoup quotient:
// T = w Y - umulhi_approx(w', Y) q is w Y mod q plus at most 3q (the quotient is at most 2
// short of Shoup's, which is itself within 1), so T < 4q and X, Y < B q -> X', Y' < (B + 4) q.
// Canonical inputs stay below (1 + 4 s) q after s stages: a whole transform (plus one exact
// split stage) fits in 64 bits while q < 2^58 for N <= 2^15 ("lazy-free" transforms: no
// subtraction, one 32 x 32 -> 64 and two high-half multiplies instead of four for w'Y).
ZINC_DEV void ct_bfly_nr(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wp, uint64_t q, uint64_t two_q) {
  const uint64_t t = shoup3(Y, w, wp, q);
  Y = X - t + 2 * two_q;
  X = X + t;
}
// Any 64-bit value -> [0, q) (mu = floor(2^64 / q)): the end of a lazy-free transform.
ZINC_DEV uint64_t reduce64(uint64_t x, uint64_t q, uint64_t mu) { return csub(x - __umul64hi(x, mu) * q, q); }
// Any 64-bit value -> [0, q) for q = 2^b - c: 2^b = c (mod q), so x = xh 2^b + xl = xh c + xl.
// One fold is one IMAD.WIDE.U32 (xh c with the masked x as its addend) plus a shift and a
// mask; fold_n folds leave a value below 2q (checked on the host), one csub finishes.
// About half the instructions of reduce64's 64 x 64 high product, mostly off the fma pipe.
// With b > 32 a fold touches only the high word: (hi >> (b-32)) c with {lo, hi & (2^(b-32)-1)}
// as the addend -- a shift, a mask and one IMAD.WIDE.U32.
ZINC_DEV uint64_t fold_once(uint64_t x, uint32_t sh, uint32_t mhi, uint32_t c) {
  const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  return (((uint64_t)(hi & mhi) << 32) | lo) + (uint64_t)(hi >> sh) * c;
}
ZINC_DEV uint64_t reduce_fold(uint64_t x, const LimbConst &c) {
  if (c.fold_n == 1) return csub(fold_once(x, c.fold_sh, c.fold_mhi, c.fold_c), c.q);
  if (c.fold_n == 2) return csub(fold_once(fold_once(x, c.fold_sh, c.fold_mhi, c.fold_c), c.fold_sh, c.fold_mhi, c.fold_c), c.q);
  return reduce64(x, c.q, c.mu64);
}

// ------------------------------------------------------------------ Philox4x32-10
// Salmon et al., SC'11.  Counter (block, msg_lo, msg_hi, tag<<16|limb),
// key (seed_lo, seed_hi)  (C-4).
ZINC_DEV uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}
ZINC_DEV uint4 stream_block(uint64_t seed, uint64_t msg, uint32_t tag, uint32_t limb, uint32_t block) {
  return philox(make_uint4(block, (uint32_t)msg, (uint32_t)(msg >> 32), (tag << 16) | limb),
                (uint32_t)seed, (uint32_t)(seed >> 32));
}
// CBD(eta = 21): coefficients 2*block + {0, 1}
ZINC_DEV int cbd_lo(uint4 w) { return __popc(w.x & 0x1FFFFFu) - __popc(w.y & 0x1FFFFFu); }
ZINC_DEV int cbd_hi(uint4 w) { return __popc(w.z & 0x1FFFFFu) - __popc(w.w & 0x1FFFFFu); }
// ternary: coefficient 4*block + r, value ((w_r * 3) >> 32) - 1
ZINC_DEV int tern(uint32_t w) { return (int)__umulhi(w, 3u) - 1; }
// uniform mod q: (w3:w2:w1:w0) mod q, q < 2^61, via Horner on 32-bit digits
ZINC_DEV uint64_t uniform_mod(uint4 w, uint64_t q) {
  // r = ((w3 * 2^32 + w2) mod q) ... exact 128-bit remainder by repeated 96/64 steps
  uint64_t r = (((uint64_t)w.w << 32) | w.z) % q;
  r = (uint64_t)(((unsigned __int128)r << 32 | w.y) % q);
  r = (uint64_t)(((unsigned __int128)r << 32 | w.x) % q);
  return r;
}

}  // namespace zinc
