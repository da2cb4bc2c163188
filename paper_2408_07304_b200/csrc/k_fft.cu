// k_fft.cu -- CKKS encode (C-6) and decode (C-10): FP64 FFT kernels.
#include "kcommon.cuh"

namespace zinc {

// ============================================================ encode (C-6)
// One CTA per message (M = N/2 <= 2^13 complex points in smem), or, at
// M = 2^14 (N = 2^15), a 2-CTA cluster: CTA r gathers the slots whose
// bit-reversed position lies in half r, runs the first LOGM-1 DIT stages on
// its M/2 points, and the last stage (pairs x, x + M/2 with W_M^x) reads both
// halves over distributed shared memory; CTA r finishes x in [r M/4, (r+1) M/4).
template <int LOGM>
__global__ void __launch_bounds__(FftPlan<(LOGM > 13 ? LOGM - 1 : LOGM)>::THREADS) encode_kernel(EncodeArgs a) {
  constexpr bool SPLIT = LOGM > 13;
  constexpr int LL = SPLIT ? LOGM - 1 : LOGM;
  constexpr int M = 1 << LOGM, ML = 1 << LL;
  constexpr int TWS = SPLIT ? 2 : 1;
  using P = FftPlan<LL>;
  extern __shared__ __align__(16) double2 buf[];
  const size_t b = blockIdx.x / (SPLIT ? 2 : 1);
  const int r = SPLIT ? (int)cluster_rank() : 0;
  for (int k = threadIdx.x; k < M; k += P::THREADS) {
    const int pos = a.perm[k] - r * ML;
    if (SPLIT && (unsigned)pos >= (unsigned)ML) continue;
    double2 z;
    if (a.complex_slots) {
      z = reinterpret_cast<const double2 *>(a.slots)[b * M + k];
    } else {
      z = make_double2(a.slots[b * M + k], 0.0);
    }
    buf[pad16(pos)] = z;
  }
  __syncthreads();
  auto lds = [&](int i) { return buf[pad16(i)]; };
  auto sts = [&](int i, double2 v) { buf[pad16(i)] = v; };
  fft_pass<LL, 0, P::K1, P::THREADS, true, false, TWS>(a.fft_tw, lds, sts);
  __syncthreads();
  fft_pass<LL, P::K1, P::K2, P::THREADS, true, false, TWS>(a.fft_tw, lds, sts);
  __syncthreads();
  int64_t *m = a.m_out + b * (2 * M);
  const double scale = a.scale;  // Delta / M, a power of two
  auto emit = [&](int j, double2 v) {
    const double2 w = cmul(v, __ldg(a.twist + j));
    m[j] = llround(w.x * scale);
    m[j + M] = llround(w.y * scale);
  };
  if constexpr (!SPLIT) {
    fft_pass<LL, P::K1 + P::K2, P::K3, P::THREADS, true, false>(a.fft_tw, lds, emit);
  } else {
    fft_pass<LL, P::K1 + P::K2, P::K3, P::THREADS, true, false, TWS>(a.fft_tw, lds, sts);
    cluster_sync_all();
    const double2 *h0 = peer_smem(buf, 0), *h1 = peer_smem(buf, 1);
    for (int x = r * (ML / 2) + threadIdx.x; x < (r + 1) * (ML / 2); x += P::THREADS) {
      const double2 u = h0[pad16(x)];
      const double2 t = cmul(h1[pad16(x)], __ldg(a.fft_tw + x));
      emit(x, cadd(u, t));
      emit(x + ML, csubd(u, t));
    }
    cluster_sync_all();
  }
}

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

template <int LOGM>
__global__ void __launch_bounds__(256, (LOGM <= 13 ? 2 : 1)) encode_real_kernel(EncodeArgs a) {
  constexpr int M = 1 << LOGM, LH = LOGM - 1, H = 1 << LH;
  constexpr int THREADS = 256, PER = M / THREADS;
  using P = FftPlan<LH>;
  static_assert(P::THREADS == THREADS, "plan");
  extern __shared__ __align__(16) double2 buf[];  // FFT buffer [H + H/16], then twiddles [H/2]
  double2 *stw = buf + H + H / 16;
  double *bufd = reinterpret_cast<double *>(buf);
  __shared__ __align__(8) uint64_t mbar;
  const size_t b = blockIdx.x;
  const int tid = threadIdx.x;
  if (tid == 0) mbar_init(&mbar, 1);
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(&mbar, (uint32_t)(M * sizeof(double) + (H / 2) * sizeof(double2)));
    bulk_g2s(buf, a.slots + b * M, M * sizeof(double), &mbar);  // raw slots into the buffer prefix
    bulk_g2s(stw, a.fft_tw_h, (H / 2) * sizeof(double2), &mbar);
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
  fft_pass<LH, 0, P::K1, THREADS, true, false, 1, true>(stw, lds, sts);
  __syncthreads();
  fft_pass<LH, P::K1, P::K2, THREADS, true, false, 1, true>(stw, lds, sts);
  __syncthreads();
  fft_pass<LH, P::K1 + P::K2, P::K3, THREADS, true, false, 1, true>(stw, lds, sts);
  __syncthreads();
  int64_t *m = a.m_out + b * (2 * M);
  const double scale = a.scale;  // Delta / M
  constexpr int V = 4;  // independent post-processing iterations per batch
  static_assert(H % (THREADS * V) == 0, "post tiling");
#pragma unroll 1
  for (int j0 = tid; j0 < H; j0 += THREADS * V) {
    double2 w[V], tw0[V], tw1[V];
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const int j = j0 + u * THREADS;
      w[u] = __ldg(a.fft_tw + j);
      tw0[u] = __ldg(a.twist + j);
      tw1[u] = __ldg(a.twist + j + H);
    }
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const int j = j0 + u * THREADS;
      const double2 xj = buf[pad16(j)], xr = conj2(buf[pad16((H - j) & (H - 1))]);
      const double2 e = make_double2(0.5 * (xj.x + xr.x), 0.5 * (xj.y + xr.y));
      const double2 d = make_double2(0.5 * (xj.x - xr.x), 0.5 * (xj.y - xr.y));
      const double2 o = make_double2(d.y, -d.x);  // -i d
      const double2 t = cmul(o, w[u]);
      const double2 y0 = cmul(cadd(e, t), tw0[u]), y1 = cmul(csubd(e, t), tw1[u]);
      m[j] = llround(y0.x * scale);  // plain stores: the path kernel re-reads m from L2
      m[j + M] = llround(y0.y * scale);
      m[j + H] = llround(y1.x * scale);
      m[j + H + M] = llround(y1.y * scale);
    }
  }
}

// ============================================================ decode (C-10)
// Mirror image of encode.  Split at M = 2^14: the first DIF stage (pairs j,
// j + M/2) is computed by each CTA for its half straight from the global
// coefficients; the remaining stages are an independent M/2-point transform
// whose bit-reversed outputs are positions [r M/2, (r+1) M/2).
template <int LOGM>
__global__ void __launch_bounds__(FftPlan<(LOGM > 13 ? LOGM - 1 : LOGM)>::THREADS) decode_kernel(DecodeArgs a) {
  constexpr bool SPLIT = LOGM > 13;
  constexpr int LL = SPLIT ? LOGM - 1 : LOGM;
  constexpr int M = 1 << LOGM, ML = 1 << LL;
  constexpr int TWS = SPLIT ? 2 : 1;
  using P = FftPlan<LL>;
  extern __shared__ __align__(16) double2 buf[];
  const size_t b = blockIdx.x / (SPLIT ? 2 : 1);
  const int r = SPLIT ? (int)cluster_rank() : 0;
  const int64_t *x = a.coeff + b * (2 * M);
  auto lds = [&](int i) { return buf[pad16(i)]; };
  auto sts = [&](int i, double2 v) { buf[pad16(i)] = v; };
  auto twisted = [&](int j) {
    const double2 v = make_double2((double)x[j], (double)x[j + M]);
    return cmul(v, conj2(__ldg(a.twist + j)));
  };
  if constexpr (!SPLIT) {
    fft_pass<LL, P::K1 + P::K2, P::K3, P::THREADS, false, true>(a.fft_tw, twisted, sts);
  } else {
    for (int j = threadIdx.x; j < ML; j += P::THREADS) {
      const double2 u = twisted(j), v = twisted(j + ML);
      buf[pad16(j)] = r == 0 ? cadd(u, v) : cmul(csubd(u, v), conj2(__ldg(a.fft_tw + j)));
    }
    __syncthreads();
    fft_pass<LL, P::K1 + P::K2, P::K3, P::THREADS, false, true, TWS>(a.fft_tw, lds, sts);
  }
  __syncthreads();
  fft_pass<LL, P::K1, P::K2, P::THREADS, false, true, TWS>(a.fft_tw, lds, sts);
  __syncthreads();
  fft_pass<LL, 0, P::K1, P::THREADS, false, true, TWS>(a.fft_tw, lds, sts);
  __syncthreads();
  double2 *out = reinterpret_cast<double2 *>(a.slots_out) + b * M;
  for (int k = threadIdx.x; k < M; k += P::THREADS) {
    const int pos = a.perm[k] - r * ML;
    if (SPLIT && (unsigned)pos >= (unsigned)ML) continue;
    const double2 v = buf[pad16(pos)];
    out[k] = make_double2(v.x * a.inv_scale, v.y * a.inv_scale);
  }
}

template <int LOGM> static size_t fft_smem() {
  constexpr int LL = LOGM > 13 ? LOGM - 1 : LOGM;
  return ((1 << LL) + ((1 << LL) >> 4)) * sizeof(double2);
}
template <int LOGM>
static cudaError_t launch_encode_t(const EncodeArgs &a, size_t batch, cudaStream_t s) {
  if (!a.complex_slots) {
    constexpr int H = 1 << (LOGM - 1);
    return launch_ex(encode_real_kernel<LOGM>, dim3((unsigned)batch), 256,
                     (H + H / 16 + H / 2) * sizeof(double2), 1, s, a);
  }
  constexpr int C = LOGM > 13 ? 2 : 1;
  return launch_ex(encode_kernel<LOGM>, dim3((unsigned)(batch * C)), FftPlan<(LOGM > 13 ? LOGM - 1 : LOGM)>::THREADS,
                   fft_smem<LOGM>(), C, s, a);
}
cudaError_t launch_encode(int log_n, const EncodeArgs &a, size_t batch, cudaStream_t s) {
#define CALL(K) launch_encode_t<K - 1>(a, batch, s)
  ZINC_LOGN_SWITCH(log_n, CALL)
#undef CALL
}

template <int LOGM>
static cudaError_t launch_decode_t(const DecodeArgs &a, size_t batch, cudaStream_t s) {
  constexpr int C = LOGM > 13 ? 2 : 1;
  return launch_ex(decode_kernel<LOGM>, dim3((unsigned)(batch * C)), FftPlan<(LOGM > 13 ? LOGM - 1 : LOGM)>::THREADS,
                   fft_smem<LOGM>(), C, s, a);
}
cudaError_t launch_decode(int log_n, const DecodeArgs &a, size_t batch, cudaStream_t s) {
#define CALL(K) launch_decode_t<K - 1>(a, batch, s)
  ZINC_LOGN_SWITCH(log_n, CALL)
#undef CALL
}


}  // namespace zinc
