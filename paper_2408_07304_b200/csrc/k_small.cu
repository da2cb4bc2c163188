// k_small.cu -- the small-batch latency path: one real-slot CKKS encode (S3, C-6) spread over
// a C-CTA thread-block cluster, optionally fused with the COEFF-form Zinc add/inject (S4 S5 S8,
// Algorithm 1) in the same launch.
//
// The throughput encode (encode_real.cuh) runs one message per CTA: at a batch of one that is
// one SM doing 12 dependent FFT passes and streaming every output word.  Here the M/2 = H-point
// DIT FFT of one message is split over C CTAs the way the transform kernels split a limb:
//  - the bit-reversed input positions [c B, (c+1) B), B = H / C, are CTA c's; the first
//    log2 B stages pair positions inside that block, so CTA c runs them alone on the slots it
//    gathered (slot k lands at brv(h_k >> 1), h_k = (5^k mod 2N - 1) / 4, and the block of k
//    depends on k mod 2C only);
//  - the last log2 C stages pair the C CTAs' values at one local offset o: CTA c finishes the
//    offsets [c B/C, (c+1) B/C) as radix-C DIT blocks over distributed shared memory;
//  - the split step needs X_j and X_{H-j}: X_{H-j} is one DSMEM load from the CTA that owns it.
// Every butterfly is the same operation on the same twiddle W_H^e, e = (x mod 2^s) (H >> (s+1)),
// and the split step is the same function (encode_post_y) as the one-CTA encode: the plaintext
// coefficients are bit-identical to it (tests/test_gpu_parity.py).
//
// SINK 0 writes the plaintext coefficients to m_out (the vanilla and Zinc NTT-form paths read
// them).  SINK 1 keeps them in shared memory and streams the Zinc ciphertext words of exactly
// those coefficients: ct[t][i][j] = [cache[t][i][j] + (m_j + e1'_j if t = 0 else e2'_j)]_{q_i},
// the values zinc_coeff_body computes.  With few messages the cluster is replicated R times per
// message: every replica encodes (latency is what bounds it, the copies run side by side) and
// streams its own share of the 2L ciphertext polynomials, so a single message still writes from
// R x C SMs.
#include "encode_real.cuh"
#include "zinc_coeff.cuh"

namespace zinc {

// one C-CTA cluster per (message, replica); THREADS per CTA
constexpr int kSmallThreads = 256;

template <int LOGM, int LC> struct SmallGeo {
  static constexpr int M = 1 << LOGM, LH = LOGM - 1, H = 1 << LH;
  static constexpr int C = 1 << LC, LB = LH - LC, B = 1 << LB;  // B points per CTA
  static constexpr int OC = B / C;                               // cross-stage offsets per CTA
  static constexpr int NPT = encode_post_tw_entries<LOGM>();
  // local passes: K1 + K2 + K3 = LB stages
  static constexpr int K3 = 3, K2 = LB >= 8 ? 3 : 2, K1 = LB - K2 - K3;
  // shared memory (double2 units): buf [B + B/16], obuf [B], ltw [B/2], xtw [(C-1) OC], ptw [NPT],
  // then (SINK 1) the plaintext words [4 B] as int64
  static constexpr int D2 = B + B / 16 + B + B / 2 + (C - 1) * OC + NPT;
  static constexpr size_t smem(int sink) { return D2 * sizeof(double2) + (sink ? 4 * B * sizeof(int64_t) : 0); }
  static_assert(OC >= 2 && OC % 2 == 0, "cross-stage offsets come in pairs");
  static_assert(K1 >= 1, "local pass plan");
  static_assert(M % (C * kSmallThreads) == 0, "scatter tiling");
};

template <int LOGM, int LC, int SINK>
__global__ void __launch_bounds__(kSmallThreads) encode_cluster_kernel(EncodeArgs e, ZincCoeffArgs z, int R, int PP) {
  using G = SmallGeo<LOGM, LC>;
  constexpr int M = G::M, LH = G::LH, H = G::H, C = G::C, LB = G::LB, B = G::B, OC = G::OC, THREADS = kSmallThreads;
  extern __shared__ __align__(16) double2 sb[];
  double2 *buf = sb, *obuf = buf + B + B / 16, *ltw = obuf + B, *xtw = ltw + B / 2, *ptw = xtw + (C - 1) * OC;
  int64_t *mloc = reinterpret_cast<int64_t *>(ptw + G::NPT);
  double *bufd = reinterpret_cast<double *>(buf);
  const int tid = threadIdx.x;
  const int c = (int)cluster_rank();
  const unsigned cid = blockIdx.x / C;
  const size_t b = cid / (unsigned)R;
  const int g = (int)(cid % (unsigned)R);

  // ---- 1. gather: slots of block c, twiddles of the local and cross stages, split tables
  // The block of slot k is brv_LC(((5^k mod 2N) >> 3) mod C), a function of k mod 2C: exactly
  // two residues r0 < r1 of k mod 2C land in block c.
  constexpr uint32_t MASK = 4u * M - 1u;
  int r0 = -1, r1 = -1;
  {
    uint32_t gg = 1;
#pragma unroll 1
    for (int kk = 0; kk < 2 * C; ++kk, gg = (gg * 5u) & MASK) {
      const int blk = (int)(__brev((gg >> 3) & (C - 1)) >> (32 - LC));
      if (blk == c) {
        if (r0 < 0) r0 = kk;
        else r1 = kk;
      }
    }
  }
  constexpr int U = M / (C * THREADS);  // slots per thread
  const int res = (tid & 1) ? r1 : r0;
  const uint32_t step = pow5_mod_pow2(2u * C * (THREADS / 2), MASK);
  uint32_t gk = pow5_mod_pow2((uint32_t)(res + 2 * C * (tid >> 1)), MASK);
  const double *slots = e.slots + b * M;
  double zv[U];
#pragma unroll
  for (int u = 0; u < U; ++u) zv[u] = __ldg(slots + res + 2 * C * ((tid >> 1) + u * (THREADS / 2)));
  for (int i = tid; i < B / 2; i += THREADS) ltw[i] = __ldg(e.fft_tw_h + (size_t)i * C);
  for (int i = tid; i < (C - 1) * OC; i += THREADS) {
    const int row = i / OC, ol = i % OC;
    const int l = 31 - __clz(row + 1), kk = row + 1 - (1 << l);
    const int o = c * OC + ol;
    xtw[i] = __ldg(e.fft_tw_h + (size_t)(o + B * kk) * (H >> (LB + l + 1)));
  }
  for (int i = tid; i < G::NPT; i += THREADS) ptw[i] = __ldg(e.post_tw + i);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t h = gk >> 2;
    const int pos = (int)(__brev(h >> 1) >> (32 - LH)) - c * B;
    bufd[2 * pad16(pos) + (h & 1)] = zv[u];
    gk = (gk * step) & MASK;
  }
  __syncthreads();

  // ---- 2. stages 0 .. LB-1 inside the block (table ltw[e] = W_H^(e C))
  auto lds = [&](int i) { return buf[pad16(i)]; };
  auto sts = [&](int i, double2 v) { buf[pad16(i)] = v; };
  fft_pass<LB, 0, G::K1, THREADS, true, false, 1, true>(ltw, lds, sts);
  __syncthreads();
  fft_pass<LB, G::K1, G::K2, THREADS, true, false, 1, true>(ltw, lds, sts);
  __syncthreads();
  fft_pass<LB, G::K1 + G::K2, G::K3, THREADS, true, false, 1, true>(ltw, lds, sts);
  cluster_sync_all();  // every block's local stages are visible cluster-wide

  // ---- 3. stages LB .. LH-1 across the cluster: offset o = c OC + tid, x = o + B k
  if (tid < OC) {
    const int o = c * OC + tid;
    double2 v[C];
#pragma unroll
    for (int k = 0; k < C; ++k) v[k] = peer_smem(buf, (uint32_t)k)[pad16(o)];
#pragma unroll
    for (int l = 0; l < LC; ++l) {
      const int D = 1 << l;
#pragma unroll
      for (int k = 0; k < C; ++k) {
        if (k & D) continue;
        const double2 w = xtw[((D - 1) + (k & (D - 1))) * OC + tid];
        const double2 t = cmul(v[k + D], w);
        v[k + D] = csubd(v[k], t);
        v[k] = cadd(v[k], t);
      }
    }
#pragma unroll
    for (int k = 0; k < C; ++k) obuf[k * OC + tid] = v[k];
  }
  cluster_sync_all();  // X is complete: obuf[k OC + ol] = X_{c OC + ol + B k}

  // ---- 4. split step, twist and rounding (encode_post_y) of this CTA's B indices j
  pdl_trigger();
  const double scale = e.scale;
  const double2 *tA = ptw, *tB = ptw + H / 64, *tA5 = tB + 64, *tB5 = tA5 + H / 64;
  int64_t *mg = SINK == 0 ? e.m_out + b * e.m_stride : nullptr;
  if (SINK == 0 && e.wait_mode == 0) pdl_wait();
#pragma unroll 2
  for (int jl = tid; jl < B; jl += THREADS) {
    const int j = c * OC + (jl % OC) + B * (jl / OC);
    const int jr = (H - j) & (H - 1);
    const int orr = jr & (B - 1);
    const double2 xh = peer_smem(obuf, (uint32_t)(orr / OC))[(jr >> LB) * OC + (orr % OC)];
    double2 y0, y1;
    encode_post_y(obuf[jl], xh, tA[j >> 6], tB[j & 63], tA5[j >> 6], tB5[j & 63], y0, y1);
    const int64_t v0 = llround(y0.x * scale), v1 = llround(y0.y * scale);
    const int64_t v2 = llround(y1.x * scale), v3 = llround(y1.y * scale);
    if constexpr (SINK == 0) {
      mg[j] = v0;
      mg[j + M] = v1;
      mg[j + H] = v2;
      mg[j + H + M] = v3;
    } else {
      mloc[jl] = v0;
      mloc[B + jl] = v1;
      mloc[2 * B + jl] = v2;
      mloc[3 * B + jl] = v3;
    }
  }
  // peers may still read this CTA's obuf: arrive now, wait before exiting
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  if constexpr (SINK == 1) {
    __syncthreads();
    // ---- 5. Zinc add/inject of this CTA's 4 B coefficients for polynomials [p_lo, p_hi):
    // every pair's samples first (limb-independent), then per polynomial all of the thread's
    // cache loads in flight before its stores
    const int L = z.L, n = z.n;
    const int p_lo = g * PP, p_hi = min(2 * L, p_lo + PP);
    const bool need_e1 = p_lo < L, need_e2 = p_hi > L;
    const uint64_t msg = z.msg_base + b;
    const uint64_t qmin = z.qmin;
    uint64_t *ctb = z.ct + b * 2 * (size_t)L * n;
    constexpr int NP = 2 * B / THREADS;  // coefficient pairs per thread
    int jj[NP];
    int64_t v[NP][2];
    int8_t f[NP][2], ee[NP][2];  // e2' (t = 1) and e1' (the exact path of t = 0)
    bool sm[NP][2];
#pragma unroll
    for (int u = 0; u < NP; ++u) {
      const int pi = tid + u * THREADS;
      const int qd = pi / (B / 2), rem = pi % (B / 2);
      const int k = rem / (OC / 2), ol = 2 * (rem % (OC / 2));
      const int jl = k * OC + ol;
      jj[u] = (qd & 1 ? M : 0) + (qd & 2 ? H : 0) + c * OC + ol + B * k;  // even
      const int64_t m0 = mloc[qd * B + jl], m1 = mloc[qd * B + jl + 1];
      int e0 = 0, e1 = 0;
      f[u][0] = f[u][1] = 0;
      if (need_e1) {
        const uint4 w1 = stream_block(z.seed, msg, TAG_ZINC_E1, 0, (uint32_t)(jj[u] >> 1));
        e0 = cbd_lo(w1);
        e1 = cbd_hi(w1);
      }
      if (need_e2) {
        const uint4 w2 = stream_block(z.seed, msg, TAG_ZINC_E2, 0, (uint32_t)(jj[u] >> 1));
        f[u][0] = (int8_t)cbd_lo(w2);
        f[u][1] = (int8_t)cbd_hi(w2);
      }
      // CKKS: v = m + e1' (|m| < 2^62 rules out int64 overflow); |v| < q_min: branch-free
      // residue; otherwise v keeps m and the exact residue of m + e1' is taken per limb
      const bool in0 = m0 > -(1ll << 62) && m0 < (1ll << 62), in1 = m1 > -(1ll << 62) && m1 < (1ll << 62);
      const int64_t a0 = m0 + e0, a1 = m1 + e1;
      sm[u][0] = in0 && (uint64_t)(a0 < 0 ? -a0 : a0) < qmin;
      sm[u][1] = in1 && (uint64_t)(a1 < 0 ? -a1 : a1) < qmin;
      v[u][0] = sm[u][0] ? a0 : m0;
      v[u][1] = sm[u][1] ? a1 : m1;
      ee[u][0] = (int8_t)e0;
      ee[u][1] = (int8_t)e1;
    }
#pragma unroll 1
    for (int p = p_lo; p < p_hi; ++p) {
      const int t = p >= L, i = p - t * L;
      const LimbConst &lc = z.limbs[i];
      const uint64_t q = __ldg(&lc.q);
      const uint64_t *zp = z.cache + (size_t)p * n;
      uint64_t *op = ctb + (size_t)p * n;
      ulonglong2 zz[NP];
#pragma unroll
      for (int u = 0; u < NP; ++u) zz[u] = ld2_nc(zp + jj[u]);
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        uint64_t o[2];
        const uint64_t zw[2] = {zz[u].x, zz[u].y};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (t == 0)
            o[h] = sm[u][h] ? mod_add_signed(zw[h], v[u][h], q) : add_mod(zw[h], pt_plus_e<false>(v[u][h], ee[u][h], lc), q);
          else
            o[h] = mod_add_signed(zw[h], f[u][h], q);
        }
        st2_cs(op + jj[u], o[0], o[1]);
      }
    }
  }
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (SINK == 0 && e.wait_mode == 1) pdl_wait();  // completion implies the previous kernel's
}

// clusters of C = 2^LC CTAs: 8 (portable) at every N
constexpr int kSmallLC = 3;

template <int LOGM, int SINK>
static cudaError_t launch_small_t(const EncodeArgs &e, const ZincCoeffArgs &z, size_t batch, int R, int PP,
                                  cudaStream_t s) {
  using G = SmallGeo<LOGM, kSmallLC>;
  return launch_ex(encode_cluster_kernel<LOGM, kSmallLC, SINK>, dim3((unsigned)(batch * R * G::C)), kSmallThreads,
                   G::smem(SINK), G::C, s, e, z, R, PP);
}

int small_cluster_ctas() { return 1 << kSmallLC; }

cudaError_t launch_encode_cluster(int log_n, const EncodeArgs &e, size_t batch, cudaStream_t s) {
  const ZincCoeffArgs z{};
  switch (log_n) {
    case 12: return launch_small_t<11, 0>(e, z, batch, 1, 0, s);
    case 13: return launch_small_t<12, 0>(e, z, batch, 1, 0, s);
    case 14: return launch_small_t<13, 0>(e, z, batch, 1, 0, s);
    case 15: return launch_small_t<14, 0>(e, z, batch, 1, 0, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_zinc_coeff_small(int log_n, const EncodeArgs &e, const ZincCoeffArgs &z, size_t batch, int R,
                                    int PP, cudaStream_t s) {
  switch (log_n) {
    case 12: return launch_small_t<11, 1>(e, z, batch, R, PP, s);
    case 13: return launch_small_t<12, 1>(e, z, batch, R, PP, s);
    case 14: return launch_small_t<13, 1>(e, z, batch, R, PP, s);
    case 15: return launch_small_t<14, 1>(e, z, batch, R, PP, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace zinc
