// k_vanilla.cu -- vanilla encryption (Eq. 8), both forms.
#include "kcommon.cuh"

namespace zinc {

// ============================================================ vanilla encryption
// Eq. 8 with reading A1: c1 = [pk1.u + e1 + m]_q, c2 = [pk2.u + e2]_q (BFV Eq. 12 /
// BGV Eq. 13 through pt_plus_e / err_term).  CTA =
// (message b, limb group); u, e1, e2 are sampled once per CTA into smem (int8),
// then per limb:
//  NTT form:   NTT(e1 + m) -> ct0;  NTT(e2) -> ct1;
//              NTT(u) -> epilogue ct0 += pk1 u^, ct1 += pk2 u^.
//  COEFF form: NTT(u) -> epilogue: ct1 <- pk2 u^ (temporary), smem <- pk1 u^;
//              INTT(smem) + e1 + m -> ct0;  INTT(ct1) + e2 -> ct1.
// 3 transforms per limb either way.
// MODE as zinc_ntt_kernel: 0 CKKS lazy-free forward transforms (q < 2^59), 1 CKKS, 2 BFV / BGV.
// COEFF form (1 forward + 2 inverse transforms per limb) runs N = 2^14 as 2-CTA clusters.
template <int FORM> __host__ __device__ constexpr int vanilla_lm() { return FORM == 1 ? 13 : 14; }

template <int LOGN, int FORM, int MODE>
__global__ void __launch_bounds__(Geo<LOGN, vanilla_lm<FORM>()>::THREADS, Geo<LOGN, vanilla_lm<FORM>()>::MINB)
    vanilla_kernel(VanillaArgs a) {
  constexpr bool INTS = MODE == 2, NR = MODE == 0;
  constexpr int LM = vanilla_lm<FORM>();
  using G = Geo<LOGN, LM>;
  constexpr int N = 1 << LOGN;
  constexpr int THREADS = G::THREADS;
  extern __shared__ __align__(16) uint64_t sm[];
  uint8_t *su = reinterpret_cast<uint8_t *>(sm + SmemWords<G::LOGL>::value);
  int8_t *se1 = reinterpret_cast<int8_t *>(su + N / 4), *se2 = se1 + N;
  // early forward passes read shared-memory copies of W[0, kSmemTw); the inverse twiddles stay
  // in L1/L2: staging them too (16 KiB more) would cost the COEFF form a CTA per SM at N <= 2^13
  constexpr bool STW = !G::SPLIT;
  Tw *stw = reinterpret_cast<Tw *>(se2 + N);
  __shared__ __align__(8) uint64_t tw_mbar;
  TwStager tws{&tw_mbar, 0};
  const size_t b = blockIdx.x / G::CLUSTER;
  const int loff = local_off<LOGN, LM>();
  const uint64_t msg = a.msg_base + b;
  const int L = a.L;
  const int lo = blockIdx.y * a.limbs_per_cta;
  const int hi = min(L, lo + a.limbs_per_cta);
  if constexpr (STW) tws.init();
  __syncthreads();
  if constexpr (STW) tws.issue(stw, a.tw + (size_t)lo * N);
  sample_ternary_packed<THREADS>(su, N, a.seed, msg, TAG_ENC_U);
  sample_cbd_smem<THREADS>(se1, N, a.seed, msg, TAG_ENC_E1);
  sample_cbd_smem<THREADS>(se2, N, a.seed, msg, TAG_ENC_E2);
  __syncthreads();
  pdl_trigger();  // chained after the encode that wrote m: wait before reading it
  pdl_wait();
  const int64_t *m = a.m ? a.m + b * N : nullptr;
  for (int i = lo; i < hi; ++i) {
    const LimbConst c = a.limbs[i];
    const uint64_t q = c.q;
    const Tw *tw = a.tw + (size_t)i * N;
    const uint64_t *pk1 = a.pk + (size_t)i * N, *pk2 = a.pk + (size_t)(L + i) * N;
    const uint64_t *pk1s = a.pk_sh + (size_t)i * N, *pk2s = a.pk_sh + (size_t)(L + i) * N;
    uint64_t *ct0 = a.ct + b * 2 * L * N + (size_t)i * N;
    uint64_t *ct1 = ct0 + (size_t)L * N;
    if constexpr (STW) tws.wait();
    auto canon = [&](uint64_t v) { return reduce_fold(v, c); };
    if (FORM == 0) {
      ntt_forward<LOGN, STW, NR, LM>(sm, tw, q, PtLoad<INTS>{m, se1, c},
                             to_smem<LOGN, LM>(sm), stw);
      __syncthreads();
      stream_pairs<LOGN, 4, LM>(sm, [&](int x, uint64_t v0, uint64_t v1) {
        st2(ct0 + x, canon(v0), canon(v1));
      });
      ntt_forward<LOGN, STW, NR, LM>(sm, tw, q, [&](int x) { return err_term<INTS>(se2[x], c); }, to_smem<LOGN, LM>(sm), stw);
      __syncthreads();
      stream_pairs<LOGN, 4, LM>(sm, [&](int x, uint64_t v0, uint64_t v1) {
        st2(ct1 + x, canon(v0), canon(v1));
      });
      ntt_forward<LOGN, STW, NR, LM>(sm, tw, q, [&](int x) { return reduce_small(tern_at(su, x), q); }, to_smem<LOGN, LM>(sm),
                             stw);
      __syncthreads();
      if constexpr (STW) {
        if (i + 1 < hi) tws.issue(stw, tw + N);
      }
      stream_pairs<LOGN, 2, LM>(sm, [&](int x, uint64_t v0, uint64_t v1) {
        const ulonglong2 p1 = ld2_nc(pk1 + x), p2 = ld2_nc(pk2 + x), s1 = ld2_nc(pk1s + x), s2 = ld2_nc(pk2s + x);
        uint64_t a0, a1, b0, b1;
        ld2(ct0 + x, a0, a1);
        ld2(ct1 + x, b0, b1);
        st2_cs(ct0 + x, add_shoup(a0, v0, p1.x, s1.x, q), add_shoup(a1, v1, p1.y, s1.y, q));
        st2_cs(ct1 + x, add_shoup(b0, v0, p2.x, s2.x, q), add_shoup(b1, v1, p2.y, s2.y, q));
      });
    } else {
      ntt_forward<LOGN, STW, NR, LM>(sm, tw, q, [&](int x) { return reduce_small(tern_at(su, x), q); }, to_smem<LOGN, LM>(sm),
                             stw);
      __syncthreads();
      if constexpr (STW) {
        if (i + 1 < hi) tws.issue(stw, tw + N);
      }
      stream_pairs<LOGN, 2, LM>(sm, [&](int x, uint64_t v0, uint64_t v1) {
        const ulonglong2 p1 = ld2_nc(pk1 + x), p2 = ld2_nc(pk2 + x), s1 = ld2_nc(pk1s + x), s2 = ld2_nc(pk2s + x);
        // [0, 2q): the inverse transforms take inputs below 4q
        st2(ct1 + x, mul_shoup_lazy(v0, p2.x, s2.x, q), mul_shoup_lazy(v1, p2.y, s2.y, q));  // temporary: pk2 u^
        sm[pad16(x - loff)] = mul_shoup_lazy(v0, p1.x, s1.x, q);                             // in place: pk1 u^
        sm[pad16(x - loff + 1)] = mul_shoup_lazy(v1, p1.y, s1.y, q);
      });
      const Tw *itw = a.itw + (size_t)i * N;
      ntt_inverse<LOGN, false, LM>(sm, itw, c,
          [&](int base, uint64_t (&v)[16]) {
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = sm[pad16(base - loff + r)];
          },
          [&](int x, uint64_t v) {
            uint64_t e = pt_plus_e<INTS>(m ? __ldg(m + x) : 0, se1[x], c);  // read-only: hoistable above the stores
            __stcs(ct0 + x, add_mod(csub(v, q), e, q));
          }, nullptr);
      __syncthreads();  // the inverse's last stores may still read sm (split exchange) -- and ct1 temp visibility
      load_share<LOGN, 4, LM>(sm, ct1);
      ntt_inverse<LOGN, false, LM>(sm, itw, c,
          [&](int base, uint64_t (&v)[16]) {
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = sm[pad16(base - loff + r)];
          },
          [&](int x, uint64_t v) { __stcs(ct1 + x, add_mod(csub(v, q), err_term<INTS>(se2[x], c), q)); }, nullptr);
    }
  }
}

// NTT form at N >= 2^14: a 2-CTA cluster per message splits each of the three transforms by
// input parity (ntt_forward_dit2, as zinc_ntt_kernel): 68 KiB halves, two clusters per SM at
// 2^14, only this parity's samples, early-pass twiddles in shared memory, and the last stage
// streams straight into the ciphertext.
template <int LOGN> struct VanillaDitGeo {
  static constexpr int LOGL = LOGN - 1, NL = 1 << LOGL;
  static constexpr int THREADS = Plan<LOGL>::THREADS, MINB = LOGL == 13 ? 2 : 1;
  static constexpr size_t SMEM = SmemWords<LOGL>::value * sizeof(uint64_t) + NL / 4 + 2 * NL + kSmemTw * sizeof(Tw);
};
template <int LOGN, int MODE>
__global__ void __launch_bounds__(VanillaDitGeo<LOGN>::THREADS, VanillaDitGeo<LOGN>::MINB)
    vanilla_ntt_dit_kernel(VanillaArgs a) {
  constexpr bool INTS = MODE == 2, NR = MODE == 0;
  using G = VanillaDitGeo<LOGN>;
  constexpr int N = 1 << LOGN, THREADS = G::THREADS;
  extern __shared__ __align__(16) uint64_t sm[];
  uint8_t *su = reinterpret_cast<uint8_t *>(sm + SmemWords<G::LOGL>::value);  // this parity's samples
  int8_t *se1 = reinterpret_cast<int8_t *>(su + G::NL / 4), *se2 = se1 + G::NL;
  Tw *stw = reinterpret_cast<Tw *>(se2 + G::NL);
  __shared__ __align__(8) uint64_t tw_mbar;
  TwStager tws{&tw_mbar, 0};
  const size_t b = blockIdx.x / 2;
  const int r = (int)cluster_rank();
  const uint64_t msg = a.msg_base + b;
  const int L = a.L;
  const int lo = blockIdx.y * a.limbs_per_cta;
  const int hi = min(L, lo + a.limbs_per_cta);
  tws.init();
  cluster_sync_all();  // both CTAs run: the samplers below store into the partner's buffers
  tws.issue(stw, a.tw + (size_t)lo * N);
  sample_ternary_parity_pair<THREADS>(su, N, a.seed, msg, TAG_ENC_U, r);
  sample_cbd_parity_pair<THREADS>(se1, N, a.seed, msg, TAG_ENC_E1, r);
  sample_cbd_parity_pair<THREADS>(se2, N, a.seed, msg, TAG_ENC_E2, r);
  cluster_sync_all();  // the partner's halves have landed (once per message)
  pdl_trigger();  // chained after the encode that wrote m: wait before reading it
  pdl_wait();
  const MSub m = m_sub(a.m ? a.m + b * N : nullptr, r, 1, a.m_deint, LOGN);  // x = 2 i + r
  const bool all_small = !INTS && plaintext_small_sub<THREADS>(m, G::NL, a.limbs, lo, hi);
  for (int i = lo; i < hi; ++i) {
    const LimbConst c = a.limbs[i];
    const uint64_t q = c.q;
    const Tw *tw = a.tw + (size_t)i * N;
    const uint64_t *pk1 = a.pk + (size_t)i * N, *pk2 = a.pk + (size_t)(L + i) * N;
    const uint64_t *pk1s = a.pk_sh + (size_t)i * N, *pk2s = a.pk_sh + (size_t)(L + i) * N;
    uint64_t *ct0 = a.ct + b * 2 * L * N + (size_t)i * N;
    uint64_t *ct1 = ct0 + (size_t)L * N;
    auto canon = [&](uint64_t v) { return reduce_fold(v, c); };
    tws.wait();
    // the three transforms through one copy of the transform code (t at run time: a third of
    // the instruction footprint); the sample of coefficient x = 2 i' + r sits at i' = x >> 1
#pragma unroll 1
    for (int t = 0; t < 3; ++t) {
      ntt_forward_dit2<LOGN, true, NR>(sm, tw, q, VanTLoad<INTS, 1>{m.p, se1, se2, su, c, t, m.stride, all_small || t > 0},
          [&](int x, uint64_t v0, uint64_t v1) {
            if (t < 2) {
              st2((t == 0 ? ct0 : ct1) + x, canon(v0), canon(v1));
            } else {
              const ulonglong2 p1 = ld2_nc(pk1 + x), p2 = ld2_nc(pk2 + x), s1 = ld2_nc(pk1s + x), s2 = ld2_nc(pk2s + x);
              uint64_t a0, a1, b0, b1;
              ld2(ct0 + x, a0, a1);
              ld2(ct1 + x, b0, b1);
              st2_cs(ct0 + x, add_shoup(a0, v0, p1.x, s1.x, q), add_shoup(a1, v1, p1.y, s1.y, q));
              st2_cs(ct1 + x, add_shoup(b0, v0, p2.x, s2.x, q), add_shoup(b1, v1, p2.y, s2.y, q));
            }
          },
          stw, [&]() {
            if (t == 2 && i + 1 < hi) tws.issue(stw, tw + N);  // lands during pass C + exchange
          });
    }
  }
}

template <int LOGN, int F>
static size_t vanilla_smem() {
  using G = Geo<LOGN, vanilla_lm<F>()>;
  const size_t twb = G::SPLIT ? 0 : (size_t)kSmemTw * sizeof(Tw);
  return ntt_smem_bytes<LOGN, vanilla_lm<F>()>() + (1 << LOGN) / 4 + 2 * (1 << LOGN) + twb;
}

template <int LOGN>
static cudaError_t launch_vanilla_t(const VanillaArgs &a, int form, int mode, size_t batch, int groups,
                                    cudaStream_t s) {
#define VK(F, M)                                                                                              \
  launch_ex(vanilla_kernel<LOGN, F, M>, msg_grid<LOGN, vanilla_lm<F>()>(batch, groups),                      \
            Geo<LOGN, vanilla_lm<F>()>::THREADS, vanilla_smem<LOGN, F>(), Geo<LOGN, vanilla_lm<F>()>::CLUSTER, s, a)
  if constexpr (LOGN >= 14) {
    if (form == 0) {
      using D = VanillaDitGeo<LOGN>;
      const dim3 grid((unsigned)(batch * 2), groups);
#define VD(M) launch_ex(vanilla_ntt_dit_kernel<LOGN, M>, grid, D::THREADS, D::SMEM, 2, s, a)
      return mode == 2 ? VD(2) : mode == 1 ? VD(1) : VD(0);
#undef VD
    }
  }
  if (mode == 2) return form == 0 ? VK(0, 2) : VK(1, 2);
  if (mode == 1) return form == 0 ? VK(0, 1) : VK(1, 1);
  return form == 0 ? VK(0, 0) : VK(1, 0);
#undef VK
}
cudaError_t launch_vanilla(int log_n, const VanillaArgs &a, int form, int mode, size_t batch, int groups,
                           cudaStream_t s) {
#define CALL(K) launch_vanilla_t<K>(a, form, mode, batch, groups, s)
  ZINC_LOGN_SWITCH(log_n, CALL)
#undef CALL
}


}  // namespace zinc
