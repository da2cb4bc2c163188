// encode_real.cuh -- the real-slot CKKS encode body (S3, C-6), shared by the
// standalone encode kernel (k_fft.cu) and the encode-fused Zinc kernel (k_fused.cu).
#pragma once

#include "kcommon.cuh"

namespace zinc {

// ============================================================ encode, real slots
// Real slots make the FFT input y (y_{h_k} = z_k) real, so the M-point
// transform Y = FFT_M(y) is Hermitian and is obtained from ONE M/2-point complex
// FFT of x_h = y_{2h} + i y_{2h+1} (the standard real-input split):
//   X = FFT_{M/2}(x),  E_j = (X_j + conj X_{M/2-j}) / 2,  O_j = -i (X_j - conj X_{M/2-j}) / 2,
//   Y_j = E_j + W_M^j O_j,  Y_{j+M/2} = E_j - W_M^j O_j   (j < M/2).
// Half the FP64 work and half the shared memory of the complex path, and one
// CTA covers N = 2^15.  Latency is what bounds a one-message-per-CTA FFT, so:
// the message's slots (64 KiB at N = 2^14) and the W_{M/2} twiddle table arrive
// by TMA bulk copies on one mbarrier; the slot order g_k = 5^k mod 2N is
// generated in registers (2N is a power of two) instead of loaded; the FFT
// reads its twiddles from shared memory.  The twist and rounding to m_j /
// m_{j+M} are the same as encode_kernel's.
ZINC_DEV uint32_t pow5_mod_pow2(uint32_t e, uint32_t mask) {
  uint32_t r = 1, b = 5;
  for (; e; e >>= 1, b = (b * b) & mask)
    if (e & 1) r = (r * b) & mask;
  return r;
}

// Split step, twist and rounding of one message's half-length FFT result `buf`
// into the plaintext coefficients m[0, 2M) (C-6).  For j < H = M/2:
//   E = (X_j + conj X_{H-j}) / 2,  O = -i (X_j - conj X_{H-j}) / 2,
//   y0 = (E + W_M^j O) zeta^-j = E t_j + O p_j,   y1 = (E - W_M^j O) zeta^-(j+H) = (E t_j - O p_j) c
// with t_j = zeta^-j = e^{-i pi j / N}, p_j = W_M^j t_j = e^{-5 i pi j / N} and the constant
// c = zeta^-H = e^{-i pi / 4} (H = N/4).  t_j and p_j come from two split tables each
// (j = 64 a + b: t_j = A[a] B[b], p_j = A5[a] B5[b]; `ptw` = [A | B | A5 | B5], H/64 + 64
// entries per pair, 4 KiB at N = 2^14) instead of 48 bytes of L2-resident tables per j.
// One output index j of the split step: y0, y1 from X_j, X_{H-j} (unconjugated) and the four
// table entries A[j/64], B[j%64], A5[j/64], B5[j%64].  Shared by encode_real_post and the
// cluster encode (k_small.cu), so both round the same doubles.
ZINC_DEV void encode_post_y(double2 xj, double2 xh, double2 ta, double2 tb, double2 t5a, double2 t5b, double2 &y0,
                            double2 &y1) {
  constexpr double R = 0.70710678118654752440;  // c = R (1 - i)
  const double2 t = cmul(ta, tb);
  const double2 pj = cmul(t5a, t5b);
  const double2 xr = conj2(xh);
  const double2 e = make_double2(0.5 * (xj.x + xr.x), 0.5 * (xj.y + xr.y));
  const double2 d = make_double2(0.5 * (xj.x - xr.x), 0.5 * (xj.y - xr.y));
  const double2 o = make_double2(d.y, -d.x);  // -i d
  const double2 U = cmul(e, t), W = cmul(o, pj);
  y0 = cadd(U, W);
  const double2 df = csubd(U, W);
  y1 = make_double2(R * (df.x + df.y), R * (df.y - df.x));
}

template <int LOGM, bool WIDE, int THREADS = 256, bool PT_SMEM = true>
ZINC_DEV void encode_real_post(const EncodeArgs &a, int64_t *m, const double2 *buf, const double2 *ptw) {
  constexpr int M = 1 << LOGM, H = M / 2, NA = H / 64;
  const double2 *tA = ptw, *tB = ptw + NA, *tA5 = tB + 64, *tB5 = tA5 + NA;
  auto ld = [](const double2 *p) { return PT_SMEM ? *p : __ldg(p); };
  const int tid = threadIdx.x;
  const double scale = a.scale;  // Delta / M
  constexpr int V = 4;  // independent post-processing iterations per batch
  static_assert(H % (THREADS * V) == 0, "post tiling");
#pragma unroll 1
  for (int j0 = tid; j0 < H; j0 += THREADS * V) {
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const int j = j0 + u * THREADS;
      double2 y0, y1;
      encode_post_y(buf[pad16(j)], buf[pad16((H - j) & (H - 1))], ld(tA + (j >> 6)), ld(tB + (j & 63)),
                    ld(tA5 + (j >> 6)), ld(tB5 + (j & 63)), y0, y1);
      if constexpr (WIDE) {  // 128-bit coefficients (f3: Delta = 2^55 and large slots)
        store_i128(m + 2 * j, y0.x * scale);
        store_i128(m + 2 * (j + M), y0.y * scale);
        store_i128(m + 2 * (j + H), y1.x * scale);
        store_i128(m + 2 * (j + H + M), y1.y * scale);
      } else {  // plain stores: the path kernel re-reads m from L2 (de-interleaved by 2^d for it)
        const int d = a.deint_log;
        m[deint_idx(j, d, LOGM + 1)] = llround(y0.x * scale);
        m[deint_idx(j + M, d, LOGM + 1)] = llround(y0.y * scale);
        m[deint_idx(j + H, d, LOGM + 1)] = llround(y1.x * scale);
        m[deint_idx(j + H + M, d, LOGM + 1)] = llround(y1.y * scale);
      }
    }
  }
}

// Entries of the split post tables (A, B, A5, B5).
template <int LOGM> __host__ __device__ constexpr int encode_post_tw_entries() { return 2 * ((1 << (LOGM - 1)) / 64 + 64); }

// Shared memory bytes of one real-slot encode CTA (FFT buffer + twiddles).
template <int LOGM> constexpr size_t encode_real_smem() {
  return ((1 << (LOGM - 1)) + (1 << (LOGM - 1)) / 16 + fft_twpad_size((1 << (LOGM - 1)) / 2) + encode_post_tw_entries<LOGM>()) *
         sizeof(double2);
}

// The half-length DIT FFT of the encode: NPASS = 3 radix-16 passes (FftPlan) or
// NPASS = 4 radix-8 passes (3 + 3 + 3 + rest; half the registers per thread).
template <int LH, int THREADS, int NPASS, int TW_SMEM, class Ld, class St>
ZINC_DEV void encode_fft(const double2 *tw, Ld lds, St sts) {
  using P = FftPlan<LH>;
  if constexpr (NPASS == 3) {
    fft_pass<LH, 0, P::K1, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
    __syncthreads();
    fft_pass<LH, P::K1, P::K2, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
    __syncthreads();
    fft_pass<LH, P::K1 + P::K2, P::K3, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
  } else if constexpr (NPASS == 6) {  // radix-4 passes: 1024 threads on one message (latency)
    static_assert(LH >= 11, "six-pass plan");
    fft_pass<LH, 0, 2, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
    __syncthreads();
    fft_pass<LH, 2, 2, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
    __syncthreads();
    fft_pass<LH, 4, 2, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
    __syncthreads();
    fft_pass<LH, 6, 2, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
    __syncthreads();
    fft_pass<LH, 8, 2, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
    __syncthreads();
    fft_pass<LH, 10, LH - 10, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
  } else {
    static_assert(LH >= 10, "four-pass plan");
    fft_pass<LH, 0, 3, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
    __syncthreads();
    fft_pass<LH, 3, 3, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
    __syncthreads();
    fft_pass<LH, 6, 3, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
    __syncthreads();
    fft_pass<LH, 9, LH - 9, THREADS, true, false, 1, TW_SMEM>(tw, lds, sts);
  }
}

// One CTA's work: encode message `b`; `buf` is the CTA's dynamic shared memory.
// THREADS = 256 with radix-16 passes, or 512 with radix-8 passes (NPASS = 4): twice
// the warps on one message's latency-bound phases at the same shared memory.
template <int LOGM, bool WIDE = false, int THREADS = 256, int NPASS = 3>
ZINC_DEV void encode_real_body(const EncodeArgs &a, size_t b, double2 *buf) {
  constexpr int M = 1 << LOGM, LH = LOGM - 1, H = 1 << LH;
  constexpr int PER = M / THREADS;
  static_assert(NPASS != 3 || FftPlan<LH>::THREADS == THREADS, "plan");
  double2 *stw = buf + H + H / 16;  // FFT buffer [H + H/16], then twiddles [H/2, padded], then post tables
  constexpr int TWP = fft_twpad_size(H / 2);
  double2 *sptw = stw + TWP;
  constexpr int NPT = encode_post_tw_entries<LOGM>();
  double *bufd = reinterpret_cast<double *>(buf);
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x;
  if (tid == 0) mbar_init(&mbar, 1);
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(&mbar, (uint32_t)(M * sizeof(double) + (TWP + NPT) * sizeof(double2)));
    bulk_g2s(buf, a.slots + b * M, M * sizeof(double), &mbar);  // raw slots into the buffer prefix
    bulk_g2s(stw, a.fft_tw_hp, TWP * sizeof(double2), &mbar);
    bulk_g2s(sptw, a.post_tw, NPT * sizeof(double2), &mbar);
  }
  constexpr uint32_t MASK = 4u * M - 1u;  // mod 2N
  uint32_t g = pow5_mod_pow2((uint32_t)tid, MASK);
  const uint32_t step = pow5_mod_pow2((uint32_t)THREADS, MASK);
  mbar_wait(&mbar, 0);
  double zv[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) zv[i] = bufd[tid + i * THREADS];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const uint32_t h = g >> 2;  // h_k = (g_k - 1) / 4
    const int pos = (int)(__brev(h >> 1) >> (32 - LH));
    bufd[2 * pad16(pos) + (h & 1)] = zv[i];
    g = (g * step) & MASK;
  }
  __syncthreads();
  auto lds = [&](int i) { return buf[pad16(i)]; };
  auto sts = [&](int i, double2 v) { buf[pad16(i)] = v; };
  encode_fft<LH, THREADS, NPASS, 2>(stw, lds, sts);
  __syncthreads();
  // Under a programmatic dependent launch the previous Zinc kernel may still read the scratch
  // this encode overwrites: the loads and the FFT above overlapped it, the stores wait.
  pdl_trigger();
  if (a.wait_mode == 0) pdl_wait();
  encode_real_post<LOGM, WIDE, THREADS>(a, a.m_out + b * a.m_stride, buf, sptw);
  if (a.wait_mode == 1) pdl_wait();  // completion still implies the previous kernel's (stream order)
}

}  // namespace zinc
