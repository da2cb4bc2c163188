// k_ntt.cu -- Zinc NTT form, keygen (Eq. 7), decrypt (Eq. 10) and the standalone NTT / INTT.
#include "kcommon.cuh"

namespace zinc {

// ============================================================ Zinc, NTT form
// c1' = zero1 + NTT(m + e1'), c2' = zero2 + NTT(e2') (two DFTs,
// no multiplication).  N <= 2^13: one CTA per (message, limb group).  N >= 2^14: a 2-CTA
// cluster per message splits every transform by input parity (ntt_forward_dit2), each
// CTA holding half a limb (68 KiB at 2^14: two clusters per SM) and only its parity's
// samples; the transform's last stage streams the ciphertext pairs straight to HBM.
template <int LOGN> struct ZincNttGeo {
  static constexpr bool DIT = LOGN >= 14;
  static constexpr int LOGL = DIT ? LOGN - 1 : LOGN, NL = 1 << LOGL;
  static constexpr int THREADS = Plan<LOGL>::THREADS, CLUSTER = DIT ? 2 : 1;
  static constexpr int MINB = LOGL <= 12 ? 3 : LOGL == 13 ? 2 : 1;
  static constexpr size_t SMEM = SmemWords<LOGL>::value * sizeof(uint64_t) + 2 * NL + kSmemTw * sizeof(Tw);
};

// MODE 0: CKKS, lazy-free butterflies (every q < 2^59); 1: CKKS with conditional
// subtractions; 2: BFV / BGV terms (with subtractions).
template <int LOGN, int MODE>
__global__ void __launch_bounds__(ZincNttGeo<LOGN>::THREADS, ZincNttGeo<LOGN>::MINB) zinc_ntt_kernel(ZincNttArgs a) {
  constexpr bool INTS = MODE == 2, NR = MODE == 0;
  using G = ZincNttGeo<LOGN>;
  constexpr int N = 1 << LOGN;
  constexpr int THREADS = G::THREADS;
  extern __shared__ __align__(16) uint64_t sm[];
  int8_t *se1 = reinterpret_cast<int8_t *>(sm + SmemWords<G::LOGL>::value);  // [NL]: this CTA's samples
  int8_t *se2 = se1 + G::NL;
  Tw *stw = reinterpret_cast<Tw *>(se2 + G::NL);
  __shared__ __align__(8) uint64_t tw_mbar;
  TwStager tws{&tw_mbar, 0};
  const size_t b = blockIdx.x / G::CLUSTER;
  const int r = G::DIT ? (int)cluster_rank() : 0;
  const uint64_t msg = a.msg_base + b;
  const int L = a.L;
  const int lo = blockIdx.y * a.limbs_per_cta;
  const int hi = min(L, lo + a.limbs_per_cta);
  tws.init();
  __syncthreads();
  tws.issue(stw, a.tw + (size_t)lo * N);
  if constexpr (G::DIT) {
    sample_cbd_parity<THREADS>(se1, N, a.seed, msg, TAG_ZINC_E1, r);
    sample_cbd_parity<THREADS>(se2, N, a.seed, msg, TAG_ZINC_E2, r);
  } else {
    sample_cbd_smem<THREADS>(se1, N, a.seed, msg, TAG_ZINC_E1);
    sample_cbd_smem<THREADS>(se2, N, a.seed, msg, TAG_ZINC_E2);
  }
  __syncthreads();
  // chained after the encode that wrote m (programmatic dependent launch): the prologue
  // above overlapped its tail; m is read only after its grid completed
  pdl_trigger();
  pdl_wait();
  const int64_t *m = a.m ? a.m + b * N : nullptr;
  for (int i = lo; i < hi; ++i) {
    const LimbConst c = a.limbs[i];
    const uint64_t q = c.q;
    const Tw *tw = a.tw + (size_t)i * N;
    const uint64_t *z1 = a.cache + (size_t)i * N, *z2 = a.cache + (size_t)(L + i) * N;
    uint64_t *ct0 = a.ct + b * 2 * L * N + (size_t)i * N;
    uint64_t *ct1 = ct0 + (size_t)L * N;
    // the lazy transform output plus the canonical cache word stays below 2^64
    tws.wait();
    if constexpr (G::DIT) {
      // both transforms through one copy of the transform code (the kernel is instruction-
      // fetch bound otherwise); sample of coefficient x = 2 i' + r sits at i' = x >> 1
#pragma unroll 1
      for (int t = 0; t < 2; ++t) {
        const uint64_t *z = t ? z2 : z1;
        uint64_t *ctt = t ? ct1 : ct0;
        ntt_forward_dit2<LOGN, true, NR>(sm, tw, q, ZincTLoad<INTS>{m ? m + r : nullptr, t ? se2 : se1, c, t, 2},  // x = 2 i + r
            [&](int x, uint64_t v0, uint64_t v1) {
              const ulonglong2 zz = ld2_nc(z + x);
              st2_cs(ctt + x, reduce_fold(zz.x + v0, c), reduce_fold(zz.y + v1, c));
            },
            stw, [&]() {
              if (t == 1 && i + 1 < hi) tws.issue(stw, tw + N);  // lands during pass C + exchange
            });
      }
    } else {
      // one copy of the transform code for both transforms at N = 2^13 (+6 %); at 2^12 the
      // 80-register budget favours two specialised copies (measured)
      constexpr bool ONE = LOGN >= 13;
#pragma unroll 1
      for (int t = 0; t < 2; ++t) {
        const uint64_t *z = t ? z2 : z1;
        uint64_t *ctt = t ? ct1 : ct0;
        auto out = [&](int x, uint64_t v0, uint64_t v1) {
          const ulonglong2 zz = ld2_nc(z + x);
          st2_cs(ctt + x, reduce_fold(zz.x + v0, c), reduce_fold(zz.y + v1, c));
        };
        if constexpr (ONE) {
          ntt_forward<LOGN, true, NR>(sm, tw, q, ZincTLoad<INTS, 0>{m, t ? se2 : se1, c, t}, to_smem<LOGN>(sm), stw);
        } else if (t == 0) {
          ntt_forward<LOGN, true, NR>(sm, tw, q, PtLoad<INTS>{m, se1, c}, to_smem<LOGN>(sm), stw);
        } else {
          ntt_forward<LOGN, true, NR>(sm, tw, q, [&](int x) { return err_term<INTS>(se2[x], c); }, to_smem<LOGN>(sm), stw);
        }
        __syncthreads();
        if (t == 1 && i + 1 < hi) tws.issue(stw, tw + N);  // next limb's table lands during this epilogue
        stream_pairs<LOGN>(sm, out);
      }
    }
  }
}

// ============================================================ keygen (Eq. 7)
// One CTA per limb: a <- U(R_qi) (tag PK_A, limb i), s <- R_2 (SK), e <- chi (PK_E);
// pk2 = a^, sk = s^, pk1 = -a^ s^ + e^ (NTT domain; C-5).
template <int LOGN>
__global__ void __launch_bounds__(Geo<LOGN>::THREADS, Geo<LOGN>::MINB) keygen_kernel(KeygenArgs a) {
  using G = Geo<LOGN>;
  constexpr int N = 1 << LOGN;
  constexpr int THREADS = G::THREADS;
  extern __shared__ __align__(16) uint64_t sm[];
  int8_t *ss = reinterpret_cast<int8_t *>(sm + SmemWords<G::LOGL>::value);
  int8_t *se = ss + N;
  sample_ternary_smem<THREADS>(ss, N, a.seed, 0, TAG_SK);
  sample_cbd_smem<THREADS>(se, N, a.seed, 0, TAG_PK_E);
  __syncthreads();
  const int i = blockIdx.x / G::CLUSTER, L = a.L;
  if (i == 0 && local_off<LOGN>() == 0 && a.sk_coeff)
    for (int x = threadIdx.x; x < N; x += THREADS) a.sk_coeff[x] = ss[x];
  const LimbConst c = a.limbs[i];
  const uint64_t q = c.q, two_q = c.two_q;
  const Tw *tw = a.tw + (size_t)i * N;
  uint64_t *pk1 = a.pk + (size_t)i * N, *pk2 = a.pk + (size_t)(L + i) * N;
  uint64_t *sk = a.sk_ntt + (size_t)i * N;
  ntt_forward<LOGN>(sm, tw, q, [&](int x) { return uniform_mod(stream_block(a.seed, 0, TAG_PK_A, i, x), q); },
      [&](int base, uint64_t (&v)[16]) {
#pragma unroll
        for (int r = 0; r < 16; ++r) pk2[base + r] = canon8(v[r], q, two_q);
      });
  ntt_forward<LOGN>(sm, tw, q, [&](int x) { return reduce_small(ss[x], q); },
      [&](int base, uint64_t (&v)[16]) {
#pragma unroll
        for (int r = 0; r < 16; ++r) sk[base + r] = canon8(v[r], q, two_q);
      });
  ntt_forward<LOGN>(sm, tw, q, [&](int x) { return err_term(se[x], c); },  // BGV: t e (reading A17)
      [&](int base, uint64_t (&v)[16]) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          uint64_t as = mul_mod(pk2[base + r], sk[base + r], c);
          pk1[base + r] = add_mod(q - as == q ? 0 : q - as, canon8(v[r], q, two_q), q);
        }
      });
}

// ============================================================ decrypt (Eq. 10)
// One CTA per message, limbs in order 0..L-1: x^(i) = [c1 + c2 s]_{q_i} (an INTT,
// plus an NTT of c2 in COEFF form).  Limb 0 writes x0 = centred residue mod q_0
// to coeff_out; every other limb checks x0 mod q_i == x^(i) (C-10).  BGV then
// replaces x0 by m = x0 mod t (Eq. 13's decoder; valid while |x| < q_0 / 2, the
// same condition as CKKS's check).  BFV needs every residue: each limb's x^(i)
// goes to a scratch [B][L][N] and bfv_scale_kernel forms round(t x / Q) mod t.
template <int LOGN, int FORM>
__global__ void __launch_bounds__(Geo<LOGN, 13>::THREADS, Geo<LOGN, 13>::MINB) decrypt_kernel(DecryptArgs a) {
  using G = Geo<LOGN, 13>;
  constexpr int N = 1 << LOGN;
  extern __shared__ __align__(16) uint64_t sm[];
  __shared__ int bad_flag;
  const size_t b = blockIdx.x / G::CLUSTER;
  const int loff = local_off<LOGN, 13>();
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
    auto epilogue = [&](int x, uint64_t v) {
      uint64_t xi = csub(v, q);
      if (FORM == 1) xi = add_mod(xi, __ldg(c1 + x), q);  // read-only: may be hoisted above the stores
      if (c.scheme == SCHEME_BFV) {
        a.xl_out[(b * L + i) * N + x] = xi;
        return;
      }
      if (a.x128_out) {  // wide CKKS: x from limbs 0 and 1, checked on the others
        int64_t *xw = a.x128_out + (b * N + x) * 2;
        if (i == 0) {
          xw[0] = (int64_t)xi;
        } else if (i == 1) {
          const uint64_t x0 = (uint64_t)xw[0];
          const uint64_t x0r = reduce_i64q((int64_t)x0, q, c.mu64);
          const uint64_t k = mul_mod(add_mod(xi, x0r ? q - x0r : 0, q), a.q0inv_q1, c);  // (x1 - x0) / q0 mod q1
          unsigned __int128 X = (unsigned __int128)k * q0 + x0;  // [0, q0 q1)
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
        x0[x] = xi > q0 / 2 ? -(int64_t)(q0 - xi) : (int64_t)xi;
      } else {
        if (reduce_i64(x0[x], c) != xi) bad = 1;
      }
      if (c.scheme == SCHEME_BGV && i == L - 1) x0[x] = (int64_t)mod_t(x0[x], c.t, c.t_mu);
    };
    if (FORM == 0) {
      ntt_inverse<LOGN, false, 13>(sm, itw, c,
          [&](int base, uint64_t (&v)[16]) {
#pragma unroll
            for (int r = 0; r < 16; ++r)
              v[r] = __ldg(c1 + base + r) + mul_shoup_lazy(__ldg(c2 + base + r), __ldg(s + base + r), __ldg(ssh + base + r), q);
          },
          epilogue);
    } else {
      const Tw *tw = a.tw + (size_t)i * N;
      ntt_forward<LOGN, false, false, 13>(sm, tw, q, [&](int x) { return __ldg(c2 + x); },
          [&](int base, uint64_t (&v)[16]) {
#pragma unroll
            for (int r = 0; r < 16; ++r)
              sm[pad16(base - loff + r)] = mul_shoup_lazy(v[r], __ldg(s + base + r), __ldg(ssh + base + r), q);
          });
      ntt_inverse<LOGN, false, 13>(sm, itw, c,
          [&](int base, uint64_t (&v)[16]) {
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = sm[pad16(base - loff + r)];
          },
          epilogue);
    }
  }
  bad = __syncthreads_or(bad);
  if constexpr (G::SPLIT) {
    // the pair's verdict: rank 1 publishes its flag, rank 0 reads it over DSMEM
    if (threadIdx.x == 0) bad_flag = bad;
    cluster_sync_all();
    if (threadIdx.x == 0 && loff == 0 && a.status_out) a.status_out[b] = bad | *peer_smem(&bad_flag, 1);
    cluster_sync_all();
  } else {
    if (threadIdx.x == 0 && a.status_out) a.status_out[b] = bad;
  }
}

// ============================================================ BFV decryption scaling
// m = round(t x / Q) mod t from the residues x_i = x mod q_i (Eq. 12's decoder):
// with Q~_i = (Q/q_i)^-1 mod q_i, t x / Q = sum_i x_i t Q~_i / q_i - t k, so mod t
// only the sum matters.  t Q~_i / q_i = I_i + F_i; the integer parts enter mod t,
// the fractions as 64-bit fixed point f_i = round(F_i 2^64): the 128-bit sum's
// high word (mod t) plus a rounding bit from the low word.  The fixed-point
// error is < sum_i x_i / 2^65 <= L q / 2^65 (<= 1/8 at L = 4, 60-bit q), far
// inside the 1/2 rounding margin for a decryptable ciphertext.
__global__ void __launch_bounds__(256) bfv_scale_kernel(BfvScaleArgs a) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= a.batch * (size_t)a.n) return;
  const size_t b = idx / a.n, j = idx % a.n;
  const uint64_t t = a.limbs[0].t, tmu = a.limbs[0].t_mu;
  uint64_t lo = 0, hi = 0, ip = 0;  // hi, ip kept mod t
  for (int i = 0; i < a.L; ++i) {
    const uint64_t x = a.xl[(b * a.L + i) * a.n + j];
    const LimbConst &c = a.limbs[i];
    const uint64_t plo = x * c.dec_f, phi = __umul64hi(x, c.dec_f);
    const uint64_t nlo = lo + plo;
    hi = (hi + mod_t((int64_t)phi, t, tmu) + (nlo < lo ? 1 : 0)) % t;
    lo = nlo;
    ip = (ip + mod_t((int64_t)x, t, tmu) * c.dec_i) % t;
  }
  a.m_out[idx] = (int64_t)((ip + hi + (lo >> 63)) % t);
}

// ============================================================ standalone NTT
template <int LOGN, int INV>
__global__ void __launch_bounds__(Geo<LOGN, 13>::THREADS, Geo<LOGN, 13>::MINB) ntt_kernel(NttArgs a) {
  constexpr int N = 1 << LOGN;
  extern __shared__ __align__(16) uint64_t sm[];
  const size_t poly = blockIdx.x / Geo<LOGN, 13>::CLUSTER;
  const int i = (int)(poly % a.L);
  uint64_t *p = a.data + poly * N;
  const LimbConst c = a.limbs[i];
  const uint64_t q = c.q, two_q = c.two_q;
  if (INV == 0) {
    ntt_forward<LOGN, false, false, 13>(sm, a.tw + (size_t)i * N, q, [&](int x) { return p[x]; },
        [&](int base, uint64_t (&v)[16]) {
#pragma unroll
          for (int r = 0; r < 16; ++r) p[base + r] = canon8(v[r], q, two_q);
        });
  } else {
    ntt_inverse<LOGN, false, 13>(sm, a.itw + (size_t)i * N, c,
        [&](int base, uint64_t (&v)[16]) {
#pragma unroll
          for (int r = 0; r < 16; ++r) v[r] = p[base + r];
        },
        [&](int x, uint64_t v) { p[x] = csub(v, q); });
  }
}

template <int LOGN>
static cudaError_t launch_zinc_ntt_t(const ZincNttArgs &a, int mode, size_t batch, int groups, cudaStream_t s) {
  using G = ZincNttGeo<LOGN>;
  const dim3 grid((unsigned)(batch * G::CLUSTER), groups);
  if (mode == 2) return launch_ex(zinc_ntt_kernel<LOGN, 2>, grid, G::THREADS, G::SMEM, G::CLUSTER, s, a);
  if (mode == 1) return launch_ex(zinc_ntt_kernel<LOGN, 1>, grid, G::THREADS, G::SMEM, G::CLUSTER, s, a);
  return launch_ex(zinc_ntt_kernel<LOGN, 0>, grid, G::THREADS, G::SMEM, G::CLUSTER, s, a);
}
cudaError_t launch_zinc_ntt(int log_n, const ZincNttArgs &a, int mode, size_t batch, int groups, cudaStream_t s) {
#define CALL(K) launch_zinc_ntt_t<K>(a, mode, batch, groups, s)
  ZINC_LOGN_SWITCH(log_n, CALL)
#undef CALL
}

template <int LOGN>
static cudaError_t launch_keygen_t(const KeygenArgs &a, cudaStream_t s) {
  using G = Geo<LOGN>;
  const size_t smem = ntt_smem_bytes<LOGN>() + 2 * (1 << LOGN);
  return launch_ex(keygen_kernel<LOGN>, msg_grid<LOGN>(a.L), G::THREADS, smem, G::CLUSTER, s, a);
}
cudaError_t launch_keygen(int log_n, const KeygenArgs &a, cudaStream_t s) {
#define CALL(K) launch_keygen_t<K>(a, s)
  ZINC_LOGN_SWITCH(log_n, CALL)
#undef CALL
}

template <int LOGN>
static cudaError_t launch_decrypt_t(const DecryptArgs &a, int form, size_t batch, cudaStream_t s) {
  using G = Geo<LOGN, 13>;
  const size_t smem = ntt_smem_bytes<LOGN, 13>();
  if (form == 0) return launch_ex(decrypt_kernel<LOGN, 0>, msg_grid<LOGN, 13>(batch), G::THREADS, smem, G::CLUSTER, s, a);
  return launch_ex(decrypt_kernel<LOGN, 1>, msg_grid<LOGN, 13>(batch), G::THREADS, smem, G::CLUSTER, s, a);
}
cudaError_t launch_bfv_scale(const BfvScaleArgs &a, cudaStream_t s) {
  const size_t n = a.batch * (size_t)a.n;
  bfv_scale_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_decrypt(int log_n, const DecryptArgs &a, int form, size_t batch, cudaStream_t s) {
#define CALL(K) launch_decrypt_t<K>(a, form, batch, s)
  ZINC_LOGN_SWITCH(log_n, CALL)
#undef CALL
}

template <int LOGN>
static cudaError_t launch_ntt_t(const NttArgs &a, int inv, size_t polys, cudaStream_t s) {
  using G = Geo<LOGN, 13>;
  const size_t smem = ntt_smem_bytes<LOGN, 13>();
  if (inv == 0) return launch_ex(ntt_kernel<LOGN, 0>, msg_grid<LOGN, 13>(polys), G::THREADS, smem, G::CLUSTER, s, a);
  return launch_ex(ntt_kernel<LOGN, 1>, msg_grid<LOGN, 13>(polys), G::THREADS, smem, G::CLUSTER, s, a);
}
cudaError_t launch_ntt(int log_n, const NttArgs &a, int inv, size_t polys, cudaStream_t s) {
#define CALL(K) launch_ntt_t<K>(a, inv, polys, s)
  ZINC_LOGN_SWITCH(log_n, CALL)
#undef CALL
}


}  // namespace zinc
