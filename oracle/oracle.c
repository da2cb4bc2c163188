/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the Zinc hot path
 * computes (arXiv 2408.07304, /root/reference/PAPER.md).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  It shares no code, header, table or constant
 * generator with the CUDA library under paper_2408_07304_b200/csrc/.
 *
 * Style rules (kept on purpose): plain loops, `unsigned __int128` with `%` for
 * every modular product, no Shoup/Barrett/Montgomery, no lazy reduction, no
 * SIMD, long double for the CKKS encoding.  Every function names the passage
 * it follows.  Numeric conventions C-1 .. C-10 are written out in
 * docs/CONVENTIONS.md.
 *
 * Pins (tests/test_oracle_*.py): Miller-Rabin primes re-checked with Python
 * big ints; psi minimality by exhaustive scan; Philox known-answer vectors;
 * exact sampler pmfs; NTT against evaluation at the odd powers of psi and the
 * convolution theorem against a Python schoolbook product; encode closed forms
 * and a numpy-FFT cross-check; Theorem 1 residual identity; Zinc == vanilla
 * with summed errors.  No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

/* ------------------------------------------------------------------------ */
/* Operation counters ("each call increments a global NTT-  */
/* count statistic"; PAPER.md:308-317 transform accounting).                 */
/* ------------------------------------------------------------------------ */
static uint64_t g_transforms = 0; /* forward + inverse NTTs on one limb      */
static uint64_t g_pointwise = 0;  /* pointwise modular products (poly mults) */

void orc_counters_reset(void) { g_transforms = 0; g_pointwise = 0; }
void orc_counters_get(uint64_t *transforms, uint64_t *pointwise) {
  *transforms = g_transforms;
  *pointwise = g_pointwise;
}

/* ------------------------------------------------------------------------ */
/* Plain modular arithmetic, [.]_q of PAPER.md:138.                          */
/* ------------------------------------------------------------------------ */
static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) {
  return (uint64_t)(((u128)a * (u128)b) % q);
}
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) {
  return (uint64_t)(((u128)a + (u128)b) % q);
}
static uint64_t submod(uint64_t a, uint64_t b, uint64_t q) {
  /* a, b in [0, q) */
  return (uint64_t)(((u128)a + (u128)q - (u128)b) % q);
}
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = mulmod(r, a, q);
    a = mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}
/* The mathematical non-negative residue of a signed integer (reading A15). */
static uint64_t residue_i64(int64_t v, uint64_t q) {
  i128 r = (i128)v % (i128)q;
  if (r < 0) r += (i128)q;
  return (uint64_t)r;
}
/* Centered representative in (-q/2, q/2] (infinity norm). */
static int64_t centered(uint64_t x, uint64_t q) {
  if (x > q / 2) return -(int64_t)(q - x);
  return (int64_t)x;
}

/* ------------------------------------------------------------------------ */
/* C-1 primes: deterministic Miller-Rabin with the first 12 primes as bases  */
/* (exact for n < 3.3e24).  PAPER.md:351 ("prime numbers ... chosen").       */
/* ------------------------------------------------------------------------ */
int orc_is_prime(uint64_t n) {
  static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; i++) {
    if (n == bases[i]) return 1;
    if (n % bases[i] == 0) return 0;
  }
  uint64_t d = n - 1;
  int s = 0;
  while ((d & 1) == 0) { d >>= 1; s++; }
  for (int i = 0; i < 12; i++) {
    uint64_t x = powmod(bases[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int witness = 1;
    for (int r = 1; r < s; r++) {
      x = mulmod(x, x, n);
      if (x == n - 1) { witness = 0; break; }
    }
    if (witness) return 0;
  }
  return 1;
}

/* For each listed bit size b (in the listed order), the largest prime
 * q < 2^b with q = 1 mod 2N that was not already used for an earlier limb of
 * the same size (C-1).  Returns 0 on success, -1 if no prime was found. */
int orc_find_primes(int log_n, int num_limbs, const int *bits, uint64_t *q_out) {
  uint64_t two_n = 2ull << log_n;
  for (int i = 0; i < num_limbs; i++) {
    int b = bits[i];
    if (b < 2 || b > 62) return -1;
    /* start just below the smallest prime already taken at this size */
    uint64_t start = 1ull << b;
    for (int j = 0; j < i; j++)
      if (bits[j] == b && q_out[j] < start) start = q_out[j];
    /* largest candidate < start with candidate = 1 mod 2N */
    uint64_t c = start - 1;
    c -= (c - 1) % two_n;
    if (c >= start) c -= two_n;
    int found = 0;
    while (c > two_n) {
      if (orc_is_prime(c)) { found = 1; break; }
      c -= two_n;
    }
    if (!found) return -1;
    q_out[i] = c;
  }
  return 0;
}

/* C-2: psi = the smallest primitive 2N-th root of unity mod q.  Find any g
 * with g^N = -1 (g = x^((q-1)/2N) for x = 2, 3, ...), then the primitive
 * 2N-th roots are exactly g^k for odd k; return their minimum. */
uint64_t orc_min_psi(uint64_t q, int log_n) {
  uint64_t n = 1ull << log_n, two_n = 2 * n;
  uint64_t g = 0;
  for (uint64_t x = 2; x < q; x++) {
    uint64_t cand = powmod(x, (q - 1) / two_n, q);
    if (powmod(cand, n, q) == q - 1) { g = cand; break; }
  }
  if (g == 0) return 0;
  uint64_t g2 = mulmod(g, g, q);
  uint64_t p = g, best = g;
  for (uint64_t k = 1; k < two_n; k += 2) {
    if (p < best) best = p;
    p = mulmod(p, g2, q);
  }
  return best;
}

/* ------------------------------------------------------------------------ */
/* C-4 Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), written from the   */
/* published round function.  Pinned by its known-answer vectors.           */
/* ------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; round++) {
    if (round > 0) { k0 += W0; k1 += W1; }
    uint64_t p0 = (uint64_t)M0 * c0;
    uint64_t p1 = (uint64_t)M1 * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Tags of C-4. */
enum { TAG_SK = 1, TAG_PK_E = 2, TAG_PK_A = 3, TAG_ENC_U = 4, TAG_ENC_E1 = 5,
       TAG_ENC_E2 = 6, TAG_ZINC_E1 = 7, TAG_ZINC_E2 = 8 };

/* One Philox block of the stream (seed, msg, tag, limb): counter
 * (block, msg_lo32, msg_hi32, tag<<16 | limb), key (seed_lo32, seed_hi32). */
static void stream_block(uint64_t seed, uint64_t msg, uint32_t tag, uint32_t limb,
                         uint32_t block, uint32_t w[4]) {
  uint32_t ctr[4] = {block, (uint32_t)msg, (uint32_t)(msg >> 32), (tag << 16) | limb};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  orc_philox4x32_10(ctr, key, w);
}

static int popcount32(uint32_t x) {
  int c = 0;
  for (int i = 0; i < 32; i++) c += (x >> i) & 1u;
  return c;
}

/* R_2 of PAPER.md:136 -- coefficients uniform in {-1, 0, 1}.  Coefficient c
 * comes from block c/4, word c%4: t = (w*3) >> 32 in {0,1,2}, value t-1. */
void orc_sample_ternary(uint64_t seed, uint64_t msg, uint32_t tag, int n, int64_t *out) {
  for (int c = 0; c < n; c++) {
    uint32_t w[4];
    stream_block(seed, msg, tag, 0, (uint32_t)(c / 4), w);
    uint64_t t = ((uint64_t)w[c % 4] * 3u) >> 32;
    out[c] = (int64_t)t - 1;
  }
}

/* chi of PAPER.md:135, read as the centered binomial CBD(eta=21) fixed by
 * BASELINE.json (reading A3).  Coefficient c comes from block c/2, words
 * 2r and 2r+1 with r = c%2: popc(w_2r & (2^21-1)) - popc(w_2r+1 & (2^21-1)). */
void orc_sample_cbd(uint64_t seed, uint64_t msg, uint32_t tag, int n, int64_t *out) {
  const uint32_t mask = (1u << 21) - 1u;
  for (int c = 0; c < n; c++) {
    uint32_t w[4];
    stream_block(seed, msg, tag, 0, (uint32_t)(c / 2), w);
    int r = c % 2;
    out[c] = (int64_t)popcount32(w[2 * r] & mask) - (int64_t)popcount32(w[2 * r + 1] & mask);
  }
}

/* R_q of PAPER.md:134 on limb `limb`: coefficient c comes from block c,
 * (w3:w2:w1:w0 as a 128-bit integer) mod q. */
void orc_sample_uniform(uint64_t seed, uint64_t msg, uint32_t tag, uint32_t limb, uint64_t q,
                        int n, uint64_t *out) {
  for (int c = 0; c < n; c++) {
    uint32_t w[4];
    stream_block(seed, msg, tag, limb, (uint32_t)c, w);
    u128 v = ((u128)w[3] << 96) | ((u128)w[2] << 64) | ((u128)w[1] << 32) | (u128)w[0];
    out[c] = (uint64_t)(v % q);
  }
}

/* ------------------------------------------------------------------------ */
/* C-3 negacyclic NTT: a_hat[k] = sum_j a_j psi^((2 brv(k) + 1) j) mod q.    */
/* PAPER.md:306 ("performs a discrete Fourier transform (DFT) on the         */
/* polynomials").                                              */
/* ------------------------------------------------------------------------ */
static uint64_t bitrev(uint64_t x, int bits) {
  uint64_t r = 0;
  for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
  return r;
}

/* The definition, O(N^2). */
void orc_ntt_definition(const uint64_t *a, int log_n, uint64_t q, uint64_t psi, uint64_t *out) {
  uint64_t n = 1ull << log_n, two_n = 2 * n;
  uint64_t *pw = (uint64_t *)malloc(sizeof(uint64_t) * two_n);
  pw[0] = 1;
  for (uint64_t r = 1; r < two_n; r++) pw[r] = mulmod(pw[r - 1], psi, q);
  for (uint64_t k = 0; k < n; k++) {
    uint64_t e = 2 * bitrev(k, log_n) + 1;
    uint64_t acc = 0;
    for (uint64_t j = 0; j < n; j++) acc = addmod(acc, mulmod(a[j] % q, pw[(e * j) % two_n], q), q);
    out[k] = acc;
  }
  free(pw);
}

/* The textbook iterative Cooley-Tukey form of the same transform (natural-
 * order input, bit-reversed output, table psi^brv(i)).  Stage with m blocks:
 * block i uses S = psi^brv(m+i); U = a[j], V = a[j+t] S; a[j] = U+V,
 * a[j+t] = U-V. */
void orc_ntt(uint64_t *a, int log_n, uint64_t q, uint64_t psi) {
  uint64_t n = 1ull << log_n;
  uint64_t *psi_rev = (uint64_t *)malloc(sizeof(uint64_t) * n);
  for (uint64_t i = 0; i < n; i++) psi_rev[i] = powmod(psi, bitrev(i, log_n), q);
  for (uint64_t i = 0; i < n; i++) a[i] %= q;
  uint64_t t = n;
  for (uint64_t m = 1; m < n; m <<= 1) {
    t >>= 1;
    for (uint64_t i = 0; i < m; i++) {
      uint64_t j1 = 2 * i * t;
      uint64_t S = psi_rev[m + i];
      for (uint64_t j = j1; j < j1 + t; j++) {
        uint64_t U = a[j], V = mulmod(a[j + t], S, q);
        a[j] = addmod(U, V, q);
        a[j + t] = submod(U, V, q);
      }
    }
  }
  free(psi_rev);
  g_transforms++;
}

/* Exact inverse of orc_ntt (Gentleman-Sande with psi^-1, then times N^-1). */
void orc_intt(uint64_t *a, int log_n, uint64_t q, uint64_t psi) {
  uint64_t n = 1ull << log_n;
  uint64_t psi_inv = powmod(psi, q - 2, q);
  uint64_t *ipsi_rev = (uint64_t *)malloc(sizeof(uint64_t) * n);
  for (uint64_t i = 0; i < n; i++) ipsi_rev[i] = powmod(psi_inv, bitrev(i, log_n), q);
  uint64_t t = 1;
  for (uint64_t m = n; m > 1; m >>= 1) {
    uint64_t h = m / 2, j1 = 0;
    for (uint64_t i = 0; i < h; i++) {
      uint64_t S = ipsi_rev[h + i];
      for (uint64_t j = j1; j < j1 + t; j++) {
        uint64_t U = a[j], V = a[j + t];
        a[j] = addmod(U, V, q);
        a[j + t] = mulmod(submod(U, V, q), S, q);
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
  uint64_t n_inv = powmod(n % q, q - 2, q);
  for (uint64_t i = 0; i < n; i++) a[i] = mulmod(a[i], n_inv, q);
  free(ipsi_rev);
  g_transforms++;
}

/* Schoolbook product in Z_q[X]/(X^N+1) (X^N = -1). */
void orc_polymul_schoolbook(const uint64_t *a, const uint64_t *b, int log_n, uint64_t q,
                            uint64_t *out) {
  uint64_t n = 1ull << log_n;
  for (uint64_t k = 0; k < n; k++) out[k] = 0;
  for (uint64_t i = 0; i < n; i++)
    for (uint64_t j = 0; j < n; j++) {
      uint64_t p = mulmod(a[i] % q, b[j] % q, q);
      if (i + j < n) out[i + j] = addmod(out[i + j], p, q);
      else out[i + j - n] = submod(out[i + j - n], p, q);
    }
}

/* ------------------------------------------------------------------------ */
/* C-6 CKKS encoding (canonical embedding; the paper defers encoding to the  */
/* CKKS paper).  zeta = exp(i pi / N), g_k = 5^k mod 2N:  */
/*   m_j = round_half_away( (2 Delta / N) Re sum_{k<N/2} z_k zeta^(-g_k j) ) */
/* ------------------------------------------------------------------------ */
static void root_table(int log_n, long double *c, long double *s) {
  uint64_t n = 1ull << log_n, two_n = 2 * n;
  const long double pi = 3.141592653589793238462643383279502884L;
  for (uint64_t r = 0; r < two_n; r++) {
    c[r] = cosl(pi * (long double)r / (long double)n);
    s[r] = sinl(pi * (long double)r / (long double)n);
  }
}

/* The definition, O(N^2), exact exponent reduction, long double sums. */
void orc_encode_definition(const double *z_re, const double *z_im, int log_n, int log_scale,
                           int64_t *m) {
  uint64_t n = 1ull << log_n, two_n = 2 * n, slots = n / 2;
  long double *c = (long double *)malloc(sizeof(long double) * two_n);
  long double *s = (long double *)malloc(sizeof(long double) * two_n);
  uint64_t *g = (uint64_t *)malloc(sizeof(uint64_t) * slots);
  root_table(log_n, c, s);
  uint64_t gk = 1;
  for (uint64_t k = 0; k < slots; k++) { g[k] = gk; gk = (gk * 5) % two_n; }
  long double scale = ldexpl(2.0L, log_scale) / (long double)n;
  for (uint64_t j = 0; j < n; j++) {
    long double acc = 0.0L;
    for (uint64_t k = 0; k < slots; k++) {
      /* Re( z_k * zeta^(-r) ) with r = g_k j mod 2N: zeta^(-r) = cos r - i sin r */
      uint64_t r = (g[k] * j) % two_n;
      long double zr = (long double)z_re[k], zi = z_im ? (long double)z_im[k] : 0.0L;
      acc += zr * c[r] + zi * s[r];
    }
    m[j] = llroundl(scale * acc);
  }
  free(c); free(s); free(g);
}

/* Decode (inverse of the canonical embedding, C-10):
 *   z_k = (1/Delta) sum_j x_j zeta^(g_k j), O(N^2). */
void orc_decode_definition(const int64_t *x, int log_n, int log_scale, double *z_re,
                           double *z_im) {
  uint64_t n = 1ull << log_n, two_n = 2 * n, slots = n / 2;
  long double *c = (long double *)malloc(sizeof(long double) * two_n);
  long double *s = (long double *)malloc(sizeof(long double) * two_n);
  root_table(log_n, c, s);
  long double inv_scale = ldexpl(1.0L, -log_scale);
  uint64_t gk = 1;
  for (uint64_t k = 0; k < slots; k++) {
    long double ar = 0.0L, ai = 0.0L;
    for (uint64_t j = 0; j < n; j++) {
      uint64_t r = (gk * j) % two_n;
      ar += (long double)x[j] * c[r];
      ai += (long double)x[j] * s[r];
    }
    z_re[k] = (double)(ar * inv_scale);
    z_im[k] = (double)(ai * inv_scale);
    gk = (gk * 5) % two_n;
  }
  free(c); free(s);
}

/* The same encode in O(N log N).  With M = N/2, g_k = 1 + 4 h_k and
 * w_j = m_j + i m_{j+M}, the definition is equivalent to
 *   w_j = (Delta / M) zeta^(-j) sum_h y_h exp(-2 pi i h j / M),  y_{h_k} = z_k
 * (derivation in DESIGN.md, "Encoding").  A plain recursive-free radix-2
 * DFT in long double evaluates the inner sum. */
static void fft_ld(long double *re, long double *im, uint64_t len, int sign) {
  int bits = 0;
  while ((1ull << bits) < len) bits++;
  for (uint64_t i = 0; i < len; i++) {
    uint64_t j = bitrev(i, bits);
    if (j > i) {
      long double t = re[i]; re[i] = re[j]; re[j] = t;
      t = im[i]; im[i] = im[j]; im[j] = t;
    }
  }
  const long double pi = 3.141592653589793238462643383279502884L;
  for (uint64_t size = 2; size <= len; size <<= 1) {
    uint64_t half = size / 2;
    for (uint64_t start = 0; start < len; start += size)
      for (uint64_t k = 0; k < half; k++) {
        long double ang = (long double)sign * 2.0L * pi * (long double)k / (long double)size;
        long double wr = cosl(ang), wi = sinl(ang);
        uint64_t a = start + k, b = start + k + half;
        long double tr = re[b] * wr - im[b] * wi, ti = re[b] * wi + im[b] * wr;
        re[b] = re[a] - tr; im[b] = im[a] - ti;
        re[a] += tr; im[a] += ti;
      }
  }
}

void orc_encode_fft(const double *z_re, const double *z_im, int log_n, int log_scale,
                    int64_t *m) {
  uint64_t n = 1ull << log_n, two_n = 2 * n, M = n / 2;
  long double *re = (long double *)calloc(M, sizeof(long double));
  long double *im = (long double *)calloc(M, sizeof(long double));
  uint64_t gk = 1;
  for (uint64_t k = 0; k < M; k++) {
    uint64_t h = (gk - 1) / 4;
    re[h] = (long double)z_re[k];
    im[h] = z_im ? (long double)z_im[k] : 0.0L;
    gk = (gk * 5) % two_n;
  }
  fft_ld(re, im, M, -1);
  const long double pi = 3.141592653589793238462643383279502884L;
  long double scale = ldexpl(1.0L, log_scale) / (long double)M;
  for (uint64_t j = 0; j < M; j++) {
    long double ang = -pi * (long double)j / (long double)n; /* zeta^(-j) */
    long double cr = cosl(ang), ci = sinl(ang);
    long double wr = (re[j] * cr - im[j] * ci) * scale;
    long double wi = (re[j] * ci + im[j] * cr) * scale;
    m[j] = llroundl(wr);
    m[j + M] = llroundl(wi);
  }
  free(re); free(im);
}

/* Wide plaintexts (the paper's own parameters: Delta = 2^55
 * makes |m_j| exceed 2^63 for the paper's value ranges).  Coefficient j is the
 * 128-bit integer hi.2^64 + lo, stored as int64 pairs m[2j] = lo, m[2j+1] = hi. */
static void ld_to_i128(long double r, int64_t *out) {
  /* r integral; long double carries 64 significant bits, so both parts are exact */
  long double hi = floorl(ldexpl(r, -64));
  long double lo = r - ldexpl(hi, 64); /* [0, 2^64) */
  out[0] = (int64_t)(uint64_t)lo;
  out[1] = (int64_t)hi;
}
static long double i128_to_ld(const int64_t *x) {
  return ldexpl((long double)x[1], 64) + (long double)(uint64_t)x[0];
}
/* C-6 encode with 128-bit integer output: the same transform as orc_encode_fft,
 * rounded half away from zero into m[2N] (lo, hi pairs). */
void orc_encode_fft_i128(const double *z_re, const double *z_im, int log_n, int log_scale,
                         int64_t *m) {
  uint64_t n = 1ull << log_n, two_n = 2 * n, M = n / 2;
  long double *re = (long double *)calloc(M, sizeof(long double));
  long double *im = (long double *)calloc(M, sizeof(long double));
  uint64_t gk = 1;
  for (uint64_t k = 0; k < M; k++) {
    uint64_t h = (gk - 1) / 4;
    re[h] = (long double)z_re[k];
    im[h] = z_im ? (long double)z_im[k] : 0.0L;
    gk = (gk * 5) % two_n;
  }
  fft_ld(re, im, M, -1);
  const long double pi = 3.141592653589793238462643383279502884L;
  long double scale = ldexpl(1.0L, log_scale) / (long double)M;
  for (uint64_t j = 0; j < M; j++) {
    long double ang = -pi * (long double)j / (long double)n;
    long double cr = cosl(ang), ci = sinl(ang);
    ld_to_i128(roundl((re[j] * cr - im[j] * ci) * scale), m + 2 * j);
    ld_to_i128(roundl((re[j] * ci + im[j] * cr) * scale), m + 2 * (j + M));
  }
  free(re); free(im);
}
/* C-10 decode of a 128-bit integer polynomial x[2N] (lo, hi pairs). */
void orc_decode_fft_i128(const int64_t *x, int log_n, int log_scale, double *z_re,
                         double *z_im) {
  uint64_t n = 1ull << log_n, two_n = 2 * n, M = n / 2;
  long double *re = (long double *)malloc(sizeof(long double) * M);
  long double *im = (long double *)malloc(sizeof(long double) * M);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (uint64_t j = 0; j < M; j++) {
    long double ang = pi * (long double)j / (long double)n;
    long double cr = cosl(ang), ci = sinl(ang);
    long double vr = i128_to_ld(x + 2 * j), vi = i128_to_ld(x + 2 * (j + M));
    re[j] = vr * cr - vi * ci;
    im[j] = vr * ci + vi * cr;
  }
  fft_ld(re, im, M, +1);
  long double inv_scale = ldexpl(1.0L, -log_scale);
  uint64_t gk = 1;
  for (uint64_t k = 0; k < M; k++) {
    uint64_t h = (gk - 1) / 4;
    z_re[k] = (double)(re[h] * inv_scale);
    z_im[k] = (double)(im[h] * inv_scale);
    gk = (gk * 5) % two_n;
  }
  free(re); free(im);
}

/* Decode in O(N log N): z_k = (1/Delta) sum_j v_j zeta^j exp(+2 pi i h_k j / M)
 * with v_j = x_j + i x_{j+M}. */
void orc_decode_fft(const int64_t *x, int log_n, int log_scale, double *z_re, double *z_im) {
  uint64_t n = 1ull << log_n, two_n = 2 * n, M = n / 2;
  long double *re = (long double *)malloc(sizeof(long double) * M);
  long double *im = (long double *)malloc(sizeof(long double) * M);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (uint64_t j = 0; j < M; j++) {
    long double ang = pi * (long double)j / (long double)n; /* zeta^j */
    long double cr = cosl(ang), ci = sinl(ang);
    long double vr = (long double)x[j], vi = (long double)x[j + M];
    re[j] = vr * cr - vi * ci;
    im[j] = vr * ci + vi * cr;
  }
  fft_ld(re, im, M, +1);
  long double inv_scale = ldexpl(1.0L, -log_scale);
  uint64_t gk = 1;
  for (uint64_t k = 0; k < M; k++) {
    uint64_t h = (gk - 1) / 4;
    z_re[k] = (double)(re[h] * inv_scale);
    z_im[k] = (double)(im[h] * inv_scale);
    gk = (gk * 5) % two_n;
  }
  free(re); free(im);
}

/* ------------------------------------------------------------------------ */
/* C-5 keygen, Eq. 7: sk <- R_2,           */
/* a <- R_q, e <- chi; pk1 = [-a.sk + e]_q, pk2 = a.  Stored in NTT form.    */
/* Outputs: sk_coeff [N] (int64 in {-1,0,1}), sk_ntt [L][N], pk_ntt [2][L][N]*/
/* ------------------------------------------------------------------------ */
/* e_scale = 1 (CKKS, BFV) or t (BGV, reading A17: pk1 = [-a.sk + t.e]_q). */
void orc_keygen_scaled(int log_n, int num_limbs, const uint64_t *q, const uint64_t *psi,
                       uint64_t seed, int64_t e_scale, int64_t *sk_coeff, uint64_t *sk_ntt,
                       uint64_t *pk_ntt);
void orc_keygen(int log_n, int num_limbs, const uint64_t *q, const uint64_t *psi, uint64_t seed,
                int64_t *sk_coeff, uint64_t *sk_ntt, uint64_t *pk_ntt) {
  orc_keygen_scaled(log_n, num_limbs, q, psi, seed, 1, sk_coeff, sk_ntt, pk_ntt);
}
void orc_keygen_scaled(int log_n, int num_limbs, const uint64_t *q, const uint64_t *psi,
                       uint64_t seed, int64_t e_scale, int64_t *sk_coeff, uint64_t *sk_ntt,
                       uint64_t *pk_ntt) {
  uint64_t n = 1ull << log_n;
  int64_t *e = (int64_t *)malloc(sizeof(int64_t) * n);
  uint64_t *a = (uint64_t *)malloc(sizeof(uint64_t) * n);
  uint64_t *s_l = (uint64_t *)malloc(sizeof(uint64_t) * n);
  uint64_t *e_l = (uint64_t *)malloc(sizeof(uint64_t) * n);
  orc_sample_ternary(seed, 0, TAG_SK, (int)n, sk_coeff);
  orc_sample_cbd(seed, 0, TAG_PK_E, (int)n, e);
  for (int i = 0; i < num_limbs; i++) {
    uint64_t qi = q[i];
    orc_sample_uniform(seed, 0, TAG_PK_A, (uint32_t)i, qi, (int)n, a);
    for (uint64_t j = 0; j < n; j++) {
      s_l[j] = residue_i64(sk_coeff[j], qi);
      e_l[j] = residue_i64(e[j] * e_scale, qi);
    }
    orc_ntt(a, log_n, qi, psi[i]);
    orc_ntt(s_l, log_n, qi, psi[i]);
    orc_ntt(e_l, log_n, qi, psi[i]);
    uint64_t *pk1 = pk_ntt + (uint64_t)i * n;
    uint64_t *pk2 = pk_ntt + ((uint64_t)num_limbs + i) * n;
    for (uint64_t j = 0; j < n; j++) {
      /* NTT(-a.s + e) = -NTT(a) (.) NTT(s) + NTT(e)  (convolution theorem) */
      pk1[j] = addmod(submod(0, mulmod(a[j], s_l[j], qi), qi), e_l[j], qi);
      g_pointwise++;
      pk2[j] = a[j];
      sk_ntt[(uint64_t)i * n + j] = s_l[j];
    }
  }
  free(e); free(a); free(s_l); free(e_l);
}

/* ------------------------------------------------------------------------ */
/* C-7 vanilla encryption, Eq. 8 with the c2 typo fixed   */
/* (reading A1: c2 = [pk2.u + e2]_q, per the proof at PAPER.md:239, 245):    */
/*   c1 = [pk1.u + e1 + m]_q,  c2 = [pk2.u + e2]_q.                          */
/* Explicit-randomness form: u, e1, e2, m are signed integer polynomials.    */
/* form 0 = NTT (ciphertext stored as NTT(c1), NTT(c2)); form 1 = COEFF.     */
/* ct layout [2][L][N]; component 0 = paper c1, component 1 = paper c2.      */
/* ------------------------------------------------------------------------ */
void orc_vanilla_encrypt_explicit(int log_n, int num_limbs, const uint64_t *q,
                                  const uint64_t *psi, const uint64_t *pk_ntt, const int64_t *m,
                                  const int64_t *u, const int64_t *e1, const int64_t *e2,
                                  int form, uint64_t *ct) {
  uint64_t n = 1ull << log_n;
  uint64_t *u_l = (uint64_t *)malloc(sizeof(uint64_t) * n);
  uint64_t *a1 = (uint64_t *)malloc(sizeof(uint64_t) * n);
  uint64_t *a2 = (uint64_t *)malloc(sizeof(uint64_t) * n);
  for (int i = 0; i < num_limbs; i++) {
    uint64_t qi = q[i];
    const uint64_t *pk1 = pk_ntt + (uint64_t)i * n;
    const uint64_t *pk2 = pk_ntt + ((uint64_t)num_limbs + i) * n;
    uint64_t *c1 = ct + (uint64_t)i * n;
    uint64_t *c2 = ct + ((uint64_t)num_limbs + i) * n;
    for (uint64_t j = 0; j < n; j++) u_l[j] = residue_i64(u[j], qi);
    orc_ntt(u_l, log_n, qi, psi[i]);
    /* pk1.u and pk2.u as NTT-domain products */
    for (uint64_t j = 0; j < n; j++) {
      a1[j] = mulmod(pk1[j], u_l[j], qi);
      a2[j] = mulmod(pk2[j], u_l[j], qi);
      g_pointwise += 2;
    }
    if (form == 0) {
      /* c1_hat = pk1_hat.u_hat + NTT(e1 + m); c2_hat = pk2_hat.u_hat + NTT(e2) */
      for (uint64_t j = 0; j < n; j++) {
        c1[j] = addmod(residue_i64(e1[j], qi), residue_i64(m[j], qi), qi);
        c2[j] = residue_i64(e2[j], qi);
      }
      orc_ntt(c1, log_n, qi, psi[i]);
      orc_ntt(c2, log_n, qi, psi[i]);
      for (uint64_t j = 0; j < n; j++) {
        c1[j] = addmod(a1[j], c1[j], qi);
        c2[j] = addmod(a2[j], c2[j], qi);
      }
    } else {
      /* c1 = INTT(pk1_hat.u_hat) + e1 + m; c2 = INTT(pk2_hat.u_hat) + e2 */
      orc_intt(a1, log_n, qi, psi[i]);
      orc_intt(a2, log_n, qi, psi[i]);
      for (uint64_t j = 0; j < n; j++) {
        c1[j] = addmod(addmod(a1[j], residue_i64(e1[j], qi), qi), residue_i64(m[j], qi), qi);
        c2[j] = addmod(a2[j], residue_i64(e2[j], qi), qi);
      }
    }
  }
  free(u_l); free(a1); free(a2);
}

/* Seeded vanilla encryption of message index `msg` (C-4 tags ENC_U/E1/E2). */
void orc_vanilla_encrypt(int log_n, int num_limbs, const uint64_t *q, const uint64_t *psi,
                         const uint64_t *pk_ntt, const int64_t *m, uint64_t seed, uint64_t msg,
                         int form, uint64_t *ct) {
  uint64_t n = 1ull << log_n;
  int64_t *u = (int64_t *)malloc(sizeof(int64_t) * n);
  int64_t *e1 = (int64_t *)malloc(sizeof(int64_t) * n);
  int64_t *e2 = (int64_t *)malloc(sizeof(int64_t) * n);
  orc_sample_ternary(seed, msg, TAG_ENC_U, (int)n, u);
  orc_sample_cbd(seed, msg, TAG_ENC_E1, (int)n, e1);
  orc_sample_cbd(seed, msg, TAG_ENC_E2, (int)n, e2);
  orc_vanilla_encrypt_explicit(log_n, num_limbs, q, psi, pk_ntt, m, u, e1, e2, form, ct);
  free(u); free(e1); free(e2);
}

/* C-8 cache precompute, PAPER.md:164-166 ("caches a single Enc(0)"):
 * vanilla encryption of m = 0 with msg = 2^64 - 1 under the cache seed. */
void orc_precompute_cache(int log_n, int num_limbs, const uint64_t *q, const uint64_t *psi,
                          const uint64_t *pk_ntt, uint64_t cache_seed, int form,
                          uint64_t *cache) {
  uint64_t n = 1ull << log_n;
  int64_t *zero = (int64_t *)calloc(n, sizeof(int64_t));
  orc_vanilla_encrypt(log_n, num_limbs, q, psi, pk_ntt, zero, cache_seed, UINT64_MAX, form,
                      cache);
  free(zero);
}

/* ------------------------------------------------------------------------ */
/* C-9 Zinc, Algorithm 1, Eq. 4 + Eq. 9:                  */
/*   line 1: c = zero + m         (m added to c1 only, reading A2)           */
/*   line 2: e1', e2' <- chi                                                 */
/*   line 3: c' = ([c1 + e1']_q, [c2 + e2']_q)                               */
/* In NTT form the added polynomials are transformed first.   */
/* ------------------------------------------------------------------------ */
void orc_zinc_encrypt_explicit(int log_n, int num_limbs, const uint64_t *q, const uint64_t *psi,
                               const uint64_t *cache, int form, const int64_t *m,
                               const int64_t *e1p, const int64_t *e2p, uint64_t *ct) {
  uint64_t n = 1ull << log_n;
  uint64_t *mp = (uint64_t *)malloc(sizeof(uint64_t) * n);
  uint64_t *ep1 = (uint64_t *)malloc(sizeof(uint64_t) * n);
  uint64_t *ep2 = (uint64_t *)malloc(sizeof(uint64_t) * n);
  for (int i = 0; i < num_limbs; i++) {
    uint64_t qi = q[i];
    const uint64_t *z1 = cache + (uint64_t)i * n;
    const uint64_t *z2 = cache + ((uint64_t)num_limbs + i) * n;
    uint64_t *c1 = ct + (uint64_t)i * n;
    uint64_t *c2 = ct + ((uint64_t)num_limbs + i) * n;
    for (uint64_t j = 0; j < n; j++) {
      mp[j] = residue_i64(m[j], qi);
      ep1[j] = residue_i64(e1p[j], qi);
      ep2[j] = residue_i64(e2p[j], qi);
    }
    if (form == 0) {
      /* the plaintext in NTT form (the "suitable plaintext format" the paper
         assumes) plus the DFT "on both e1' and e2'"
         (PAPER.md:315): 3 transforms per limb here; the CUDA path transforms
         m + e1' together (2 per limb), equal by linearity. */
      orc_ntt(mp, log_n, qi, psi[i]);
      orc_ntt(ep1, log_n, qi, psi[i]);
      orc_ntt(ep2, log_n, qi, psi[i]);
    }
    for (uint64_t j = 0; j < n; j++) {
      uint64_t c1j = addmod(z1[j], mp[j], qi); /* line 1 */
      c1[j] = addmod(c1j, ep1[j], qi);         /* line 3 */
      c2[j] = addmod(z2[j], ep2[j], qi);
    }
  }
  free(mp); free(ep1); free(ep2);
}

void orc_zinc_encrypt(int log_n, int num_limbs, const uint64_t *q, const uint64_t *psi,
                      const uint64_t *cache, int form, const int64_t *m, uint64_t seed,
                      uint64_t msg, uint64_t *ct) {
  uint64_t n = 1ull << log_n;
  int64_t *e1p = (int64_t *)malloc(sizeof(int64_t) * n);
  int64_t *e2p = (int64_t *)malloc(sizeof(int64_t) * n);
  orc_sample_cbd(seed, msg, TAG_ZINC_E1, (int)n, e1p); /* line 2 */
  orc_sample_cbd(seed, msg, TAG_ZINC_E2, (int)n, e2p);
  orc_zinc_encrypt_explicit(log_n, num_limbs, q, psi, cache, form, m, e1p, e2p, ct);
  free(e1p); free(e2p);
}

/* ------------------------------------------------------------------------ */
/* C-10 decryption, Eq. 10: x = [c1 + c2.sk]_q per limb.  */
/* x_out = the centered residue mod q_0 (limb 0, the largest prime); the     */
/* status is 0 if x_0 mod q_i == x^(i) for every limb i (a CRT consistency   */
/* check, valid while |m + v| < q_0 / 2), else 1.  x_limbs (optional, may be */
/* NULL) receives the canonical residues [L][N].                             */
/* ------------------------------------------------------------------------ */
int orc_decrypt(int log_n, int num_limbs, const uint64_t *q, const uint64_t *psi,
                const uint64_t *sk_ntt, const uint64_t *ct, int form, int64_t *x_out,
                uint64_t *x_limbs) {
  uint64_t n = 1ull << log_n;
  uint64_t *x = (uint64_t *)malloc(sizeof(uint64_t) * n * (uint64_t)num_limbs);
  uint64_t *t = (uint64_t *)malloc(sizeof(uint64_t) * n);
  for (int i = 0; i < num_limbs; i++) {
    uint64_t qi = q[i];
    const uint64_t *c1 = ct + (uint64_t)i * n;
    const uint64_t *c2 = ct + ((uint64_t)num_limbs + i) * n;
    const uint64_t *s = sk_ntt + (uint64_t)i * n;
    uint64_t *xi = x + (uint64_t)i * n;
    if (form == 0) {
      for (uint64_t j = 0; j < n; j++) xi[j] = addmod(c1[j], mulmod(c2[j], s[j], qi), qi);
      orc_intt(xi, log_n, qi, psi[i]);
    } else {
      for (uint64_t j = 0; j < n; j++) t[j] = c2[j];
      orc_ntt(t, log_n, qi, psi[i]);
      for (uint64_t j = 0; j < n; j++) t[j] = mulmod(t[j], s[j], qi);
      orc_intt(t, log_n, qi, psi[i]);
      for (uint64_t j = 0; j < n; j++) xi[j] = addmod(c1[j], t[j], qi);
    }
  }
  int status = 0;
  for (uint64_t j = 0; j < n; j++) {
    int64_t v = centered(x[j], q[0]);
    x_out[j] = v;
    for (int i = 1; i < num_limbs; i++)
      if (residue_i64(v, q[i]) != x[(uint64_t)i * n + j]) status = 1;
  }
  if (x_limbs) memcpy(x_limbs, x, sizeof(uint64_t) * n * (uint64_t)num_limbs);
  free(x); free(t);
  return status;
}

/* ------------------------------------------------------------------------ */
/* Scheme variants, PAPER.md:319-343 (section 4.2).  The plaintext space is  */
/* Z_t/(X^N+1); a plaintext coefficient is taken as its residue m mod t in   */
/* [0, t) (reading A18).                                                     */
/*   BFV, Eq. 12:  c1 = [pk1.u + e1 + Delta.m]_Q, Delta = floor(Q/t);        */
/*                 Zinc "without modification".               */
/*   BGV, Eq. 13:  c1 = [pk1.u + t.e1 + m]_Q, c2 = [pk2.u + t.e2]_Q;          */
/*                 Zinc adds t.e1', t.e2'.                     */
/* (c2 uses pk2, reading A1, as for CKKS.)  scheme: 0 CKKS, 1 BFV, 2 BGV.    */
/* ------------------------------------------------------------------------ */
static uint64_t mod_t(int64_t m, uint64_t t) {
  i128 r = (i128)m % (i128)t;
  if (r < 0) r += (i128)t;
  return (uint64_t)r;
}
/* Delta mod q_i with Delta = floor(Q/t), Q = prod q_k, exactly and without big
 * integers: Q = Delta.t + (Q mod t) and q_i | Q give
 * Delta = -(Q mod t) . t^{-1}  (mod q_i). */
uint64_t orc_bfv_delta_mod(int num_limbs, const uint64_t *q, uint64_t t, int i) {
  uint64_t qmod_t = 1 % t;
  for (int k = 0; k < num_limbs; k++) qmod_t = (uint64_t)(((u128)qmod_t * (q[k] % t)) % t);
  uint64_t tinv = powmod(t % q[i], q[i] - 2, q[i]); /* q_i prime, t < q_i */
  return mulmod(submod(0, qmod_t % q[i], q[i]), tinv, q[i]);
}
/* Residues [L][N] of the scheme's plaintext term: CKKS m; BFV Delta.(m mod t); BGV m mod t. */
void orc_plaintext_residues(int scheme, uint64_t t, int log_n, int num_limbs, const uint64_t *q,
                            const int64_t *m, uint64_t *out) {
  uint64_t n = 1ull << log_n;
  for (int i = 0; i < num_limbs; i++) {
    uint64_t delta = scheme == 1 ? orc_bfv_delta_mod(num_limbs, q, t, i) : 1;
    for (uint64_t j = 0; j < n; j++) {
      uint64_t v;
      if (scheme == 0) v = residue_i64(m[j], q[i]);
      else v = mulmod(delta, mod_t(m[j], t) % q[i], q[i]);
      out[(uint64_t)i * n + j] = v;
    }
  }
}
/* General explicit encryption: c1 = [pk1.u + es.e1 + pt]_q, c2 = [pk2.u + es.e2]_q
 * with pt given as residues [L][N] and es the error scale (1, or t for BGV). */
void orc_encrypt_general_explicit(int log_n, int num_limbs, const uint64_t *q,
                                  const uint64_t *psi, const uint64_t *pk_ntt,
                                  const uint64_t *pt_res, const int64_t *u, const int64_t *e1,
                                  const int64_t *e2, int64_t es, int form, uint64_t *ct) {
  uint64_t n = 1ull << log_n;
  int64_t *zero = (int64_t *)calloc(n, sizeof(int64_t));
  int64_t *se1 = (int64_t *)malloc(sizeof(int64_t) * n);
  int64_t *se2 = (int64_t *)malloc(sizeof(int64_t) * n);
  for (uint64_t j = 0; j < n; j++) {
    se1[j] = e1[j] * es;
    se2[j] = e2[j] * es;
  }
  /* Eq. 8 structure with m = 0, then + pt (same ring element in either form) */
  orc_vanilla_encrypt_explicit(log_n, num_limbs, q, psi, pk_ntt, zero, u, se1, se2, form, ct);
  uint64_t *p = (uint64_t *)malloc(sizeof(uint64_t) * n);
  for (int i = 0; i < num_limbs; i++) {
    memcpy(p, pt_res + (uint64_t)i * n, sizeof(uint64_t) * n);
    if (form == 0) orc_ntt(p, log_n, q[i], psi[i]);
    for (uint64_t j = 0; j < n; j++) ct[(uint64_t)i * n + j] = addmod(ct[(uint64_t)i * n + j], p[j], q[i]);
  }
  free(zero); free(se1); free(se2); free(p);
}
void orc_encrypt_scheme(int scheme, uint64_t t, int log_n, int num_limbs, const uint64_t *q,
                        const uint64_t *psi, const uint64_t *pk_ntt, const int64_t *m,
                        uint64_t seed, uint64_t msg, int form, uint64_t *ct) {
  uint64_t n = 1ull << log_n;
  int64_t *u = (int64_t *)malloc(sizeof(int64_t) * n);
  int64_t *e1 = (int64_t *)malloc(sizeof(int64_t) * n);
  int64_t *e2 = (int64_t *)malloc(sizeof(int64_t) * n);
  uint64_t *pt = (uint64_t *)malloc(sizeof(uint64_t) * n * (uint64_t)num_limbs);
  orc_sample_ternary(seed, msg, TAG_ENC_U, (int)n, u);
  orc_sample_cbd(seed, msg, TAG_ENC_E1, (int)n, e1);
  orc_sample_cbd(seed, msg, TAG_ENC_E2, (int)n, e2);
  orc_plaintext_residues(scheme, t, log_n, num_limbs, q, m, pt);
  orc_encrypt_general_explicit(log_n, num_limbs, q, psi, pk_ntt, pt, u, e1, e2,
                               scheme == 2 ? (int64_t)t : 1, form, ct);
  free(u); free(e1); free(e2); free(pt);
}
/* Cache of a scheme: its Enc(0), msg = 2^64 - 1. */
void orc_precompute_cache_scheme(int scheme, uint64_t t, int log_n, int num_limbs,
                                 const uint64_t *q, const uint64_t *psi, const uint64_t *pk_ntt,
                                 uint64_t cache_seed, int form, uint64_t *cache) {
  uint64_t n = 1ull << log_n;
  int64_t *zero = (int64_t *)calloc(n, sizeof(int64_t));
  orc_encrypt_scheme(scheme, t, log_n, num_limbs, q, psi, pk_ntt, zero, cache_seed, UINT64_MAX,
                     form, cache);
  free(zero);
}
/* Zinc of a scheme: Algorithm 1 with the plaintext term of the scheme (line 1)
 * and, for BGV, the injected errors scaled by t (line 3). */
void orc_zinc_encrypt_scheme(int scheme, uint64_t t, int log_n, int num_limbs, const uint64_t *q,
                             const uint64_t *psi, const uint64_t *cache, int form,
                             const int64_t *m, uint64_t seed, uint64_t msg, uint64_t *ct) {
  uint64_t n = 1ull << log_n;
  int64_t *e1p = (int64_t *)malloc(sizeof(int64_t) * n);
  int64_t *e2p = (int64_t *)malloc(sizeof(int64_t) * n);
  uint64_t *pt = (uint64_t *)malloc(sizeof(uint64_t) * n * (uint64_t)num_limbs);
  uint64_t *ep = (uint64_t *)malloc(sizeof(uint64_t) * n);
  orc_sample_cbd(seed, msg, TAG_ZINC_E1, (int)n, e1p); /* line 2 */
  orc_sample_cbd(seed, msg, TAG_ZINC_E2, (int)n, e2p);
  orc_plaintext_residues(scheme, t, log_n, num_limbs, q, m, pt);
  int64_t es = scheme == 2 ? (int64_t)t : 1;
  for (int i = 0; i < num_limbs; i++) {
    uint64_t qi = q[i];
    uint64_t *p = pt + (uint64_t)i * n;
    uint64_t *c1 = ct + (uint64_t)i * n;
    uint64_t *c2 = ct + ((uint64_t)num_limbs + i) * n;
    const uint64_t *z1 = cache + (uint64_t)i * n;
    const uint64_t *z2 = cache + ((uint64_t)num_limbs + i) * n;
    for (uint64_t j = 0; j < n; j++) ep[j] = residue_i64(e1p[j] * es, qi);
    if (form == 0) { orc_ntt(p, log_n, qi, psi[i]); orc_ntt(ep, log_n, qi, psi[i]); }
    for (uint64_t j = 0; j < n; j++) c1[j] = addmod(addmod(z1[j], p[j], qi), ep[j], qi);
    for (uint64_t j = 0; j < n; j++) ep[j] = residue_i64(e2p[j] * es, qi);
    if (form == 0) orc_ntt(ep, log_n, qi, psi[i]);
    for (uint64_t j = 0; j < n; j++) c2[j] = addmod(z2[j], ep[j], qi);
  }
  free(e1p); free(e2p); free(pt); free(ep);
}

/* ------------------------------------------------------------------------ */
/* Eq. 2: Enc(a) (+) Enc(b) is the componentwise sum, and   */
/* aggregation of a batch is the repeated sum.  Either form (the NTT is      */
/* linear).  ct arrays [count][2][L][N].                                     */
/* ------------------------------------------------------------------------ */
void orc_ct_add(int log_n, int num_limbs, const uint64_t *q, const uint64_t *a, const uint64_t *b,
                uint64_t count, uint64_t *out) {
  uint64_t n = 1ull << log_n;
  for (uint64_t k = 0; k < count; k++)
    for (int c = 0; c < 2; c++)
      for (int i = 0; i < num_limbs; i++)
        for (uint64_t j = 0; j < n; j++) {
          uint64_t w = ((k * 2 + c) * (uint64_t)num_limbs + i) * n + j;
          out[w] = addmod(a[w], b[w], q[i]);
        }
}
void orc_ct_sum(int log_n, int num_limbs, const uint64_t *q, const uint64_t *ct, uint64_t count,
                uint64_t *out) {
  uint64_t n = 1ull << log_n, words = 2ull * num_limbs * n;
  for (uint64_t w = 0; w < words; w++) out[w] = 0;
  for (uint64_t k = 0; k < count; k++)
    for (uint64_t w = 0; w < words; w++) {
      int i = (int)((w / n) % (uint64_t)num_limbs);
      out[w] = addmod(out[w], ct[k * words + w], q[i]);
    }
}

/* Plain helpers exposed for tests: forward/inverse NTT of [L][N] in place. */
void orc_ntt_limbs(uint64_t *a, int log_n, int num_limbs, const uint64_t *q, const uint64_t *psi) {
  uint64_t n = 1ull << log_n;
  for (int i = 0; i < num_limbs; i++) orc_ntt(a + (uint64_t)i * n, log_n, q[i], psi[i]);
}
void orc_intt_limbs(uint64_t *a, int log_n, int num_limbs, const uint64_t *q,
                    const uint64_t *psi) {
  uint64_t n = 1ull << log_n;
  for (int i = 0; i < num_limbs; i++) orc_intt(a + (uint64_t)i * n, log_n, q[i], psi[i]);
}
