// k_fft.cu -- CKKS encode (C-6) and decode (C-10): FP64 FFT kernels.
#include "encode_real.cuh"

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
  // Slot k lands at bit-reversed position brv(h_k), h_k = (5^k mod 2N - 1) / 4.  h_k's lowest
  // bit is k's parity (5^k = 1 or 5 mod 8), so half r of the split takes exactly the slots
  // k = 2i + r.  The order g = 5^k mod 2N is generated in registers (2N = 4M is a power of
  // two) and U independent slot loads are kept in flight per thread.
  constexpr int KS = SPLIT ? 2 : 1, CNT = M / KS, U = 8;
  static_assert(CNT % (P::THREADS * U) == 0, "scatter tiling");
  constexpr uint32_t MASK = 4u * M - 1u;
  const uint32_t gstep = pow5_mod_pow2((uint32_t)(KS * P::THREADS), MASK);
  uint32_t g = pow5_mod_pow2((uint32_t)(KS * threadIdx.x + r), MASK);
#pragma unroll 1
  for (int i0 = threadIdx.x; i0 < CNT; i0 += P::THREADS * U) {
    double2 zv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t k = (size_t)KS * (i0 + u * P::THREADS) + r;
      zv[u] = a.complex_slots ? __ldcs(reinterpret_cast<const double2 *>(a.slots) + b * M + k)
                              : make_double2(__ldcs(a.slots + b * M + k), 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t h = g >> 2;
      const int pos = (int)(__brev(h) >> (32 - LOGM)) - r * ML;
      buf[pad16(pos)] = zv[u];
      g = (g * gstep) & MASK;
    }
  }
  // split: the sub-transform's twiddles W_M^(2e) = W_{M/2}^e (e < M/4, 64 KiB at M = 2^14) come
  // into shared memory by one TMA bulk copy, issued before the scatter, beside the FFT buffer
  double2 *stw = buf + ML + ML / 16;
  __shared__ __align__(8) uint64_t tw_mbar;
  if constexpr (SPLIT) {
    if (threadIdx.x == 0) {
      mbar_init(&tw_mbar, 1);
      mbar_expect_tx(&tw_mbar, (uint32_t)(fft_twpad_size(M / 4) * sizeof(double2)));
      bulk_g2s(stw, a.fft_tw_hp, (uint32_t)(fft_twpad_size(M / 4) * sizeof(double2)), &tw_mbar);
    }
  }
  __syncthreads();
  if constexpr (SPLIT) mbar_wait(&tw_mbar, 0);
  auto lds = [&](int i) { return buf[pad16(i)]; };
  auto sts = [&](int i, double2 v) { buf[pad16(i)] = v; };
  if constexpr (SPLIT) {
    fft_pass<LL, 0, P::K1, P::THREADS, true, false, 1, 2>(stw, lds, sts);
    __syncthreads();
    fft_pass<LL, P::K1, P::K2, P::THREADS, true, false, 1, 2>(stw, lds, sts);
  } else {
    fft_pass<LL, 0, P::K1, P::THREADS, true, false, TWS>(a.fft_tw, lds, sts);
    __syncthreads();
    fft_pass<LL, P::K1, P::K2, P::THREADS, true, false, TWS>(a.fft_tw, lds, sts);
  }
  __syncthreads();
  // Under a programmatic dependent launch the previous Zinc kernel may still read the scratch
  // this encode overwrites: the loads and the first passes overlapped it, the stores wait.
  pdl_trigger();
  if (a.wait_mode == 0) pdl_wait();
  int64_t *m = a.m_out + b * a.m_stride;
  const double scale = a.scale;  // Delta / M, a power of two
  // twist zeta^-j from two small L1-resident tables instead of 16 B of L2 table per output
  const double2 *tA = a.twist_split, *tB = a.twist_split + M / 64;
  auto emit = [&](int j, double2 v) {
    const double2 w = cmul(v, cmul(__ldg(tA + (j >> 6)), __ldg(tB + (j & 63))));
    if (a.wide) {
      store_i128(m + 2 * j, w.x * scale);
      store_i128(m + 2 * (j + M), w.y * scale);
    } else {
      m[deint_idx(j, a.deint_log, LOGM + 1)] = llround(w.x * scale);
      m[deint_idx(j + M, a.deint_log, LOGM + 1)] = llround(w.y * scale);
    }
  };
  if constexpr (!SPLIT) {
    fft_pass<LL, P::K1 + P::K2, P::K3, P::THREADS, true, false>(a.fft_tw, lds, emit);
  } else {
    fft_pass<LL, P::K1 + P::K2, P::K3, P::THREADS, true, false, 1, 2>(stw, lds, sts);
    cluster_sync_all();
    const double2 *h0 = peer_smem(buf, 0), *h1 = peer_smem(buf, 1);
    // U independent iterations: their DSMEM, twiddle and twist loads are all in flight
    // before the first multiply (one at a time, each iteration exposed ~3 load latencies)
    constexpr int U = 4;
    static_assert((ML / 2) % (P::THREADS * U) == 0, "exchange tiling");
#pragma unroll 1
    for (int x0 = r * (ML / 2) + threadIdx.x; x0 < (r + 1) * (ML / 2); x0 += P::THREADS * U) {
      double2 u[U], h[U], w[U], t0a[U], t0b[U], t1a[U], t1b[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int x = x0 + k * P::THREADS;
        u[k] = h0[pad16(x)];
        h[k] = h1[pad16(x)];
        w[k] = __ldg(a.fft_tw + x);
        t0a[k] = __ldg(tA + (x >> 6));
        t0b[k] = __ldg(tB + (x & 63));
        t1a[k] = __ldg(tA + ((x + ML) >> 6));
        t1b[k] = __ldg(tB + ((x + ML) & 63));
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int x = x0 + k * P::THREADS;
        const double2 t = cmul(h[k], w[k]);
        const double2 y0 = cmul(cadd(u[k], t), cmul(t0a[k], t0b[k]));
        const double2 y1 = cmul(csubd(u[k], t), cmul(t1a[k], t1b[k]));
        if (a.wide) {
          store_i128(m + 2 * x, y0.x * scale);
          store_i128(m + 2 * (x + M), y0.y * scale);
          store_i128(m + 2 * (x + ML), y1.x * scale);
          store_i128(m + 2 * (x + ML + M), y1.y * scale);
        } else {
          const int d = a.deint_log;
          m[deint_idx(x, d, LOGM + 1)] = llround(y0.x * scale);
          m[deint_idx(x + M, d, LOGM + 1)] = llround(y0.y * scale);
          m[deint_idx(x + ML, d, LOGM + 1)] = llround(y1.x * scale);
          m[deint_idx(x + ML + M, d, LOGM + 1)] = llround(y1.y * scale);
        }
      }
    }
    cluster_sync_all();
  }
  if (a.wait_mode == 1) pdl_wait();  // completion still implies the previous kernel's (stream order)
}

// ============================================================ encode, real slots
// (body in encode_real.cuh)
template <int LOGM, bool WIDE>
__global__ void __launch_bounds__(256, (LOGM <= 13 ? 2 : 1)) encode_real_kernel(EncodeArgs a) {
  extern __shared__ __align__(16) double2 buf[];
  encode_real_body<LOGM, WIDE>(a, blockIdx.x, buf);
}
// Latency variants for small batches (fewer messages than SMs): the same encode with more
// threads on one message: F = 1: 512 threads, radix-8 passes; F = 2: 1024 threads, radix-4
// passes (N >= 2^14).
template <int LOGM, int F> struct FastEnc {
  static constexpr int THREADS = (F == 2 && LOGM >= 13) ? 1024 : 512, NPASS = THREADS == 1024 ? 6 : 4;
};
template <int LOGM, bool WIDE, int F>
__global__ void __launch_bounds__(FastEnc<LOGM, F>::THREADS, 1) encode_real_fast_kernel(EncodeArgs a) {
  extern __shared__ __align__(16) double2 buf[];
  encode_real_body<LOGM, WIDE, FastEnc<LOGM, F>::THREADS, FastEnc<LOGM, F>::NPASS>(a, blockIdx.x, buf);
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
  const int64_t *x = a.coeff + b * (2 * M) * (a.wide ? 2 : 1);
  auto lds = [&](int i) { return buf[pad16(i)]; };
  auto sts = [&](int i, double2 v) { buf[pad16(i)] = v; };
  auto twisted = [&](int j) {
    const double2 v = a.wide ? make_double2(load_i128(x + 2 * j), load_i128(x + 2 * (j + M)))
                             : make_double2((double)x[j], (double)x[j + M]);
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
// complex-slot encode: split CTAs also hold the sub-transform's twiddle table (M/4 entries)
template <int LOGM> static size_t encode_smem() {
  return fft_smem<LOGM>() + (LOGM > 13 ? (size_t)fft_twpad_size((1 << LOGM) / 4) * sizeof(double2) : 0);
}
template <int LOGM>
static cudaError_t launch_encode_t(const EncodeArgs &a, size_t batch, cudaStream_t s) {
  if (!a.complex_slots) {
    if constexpr (LOGM >= 12) {
      if (a.fast == 1) {
        constexpr int T = FastEnc<LOGM, 1>::THREADS;
        if (a.wide) return launch_ex(encode_real_fast_kernel<LOGM, true, 1>, dim3((unsigned)batch), T, encode_real_smem<LOGM>(), 1, s, a);
        return launch_ex(encode_real_fast_kernel<LOGM, false, 1>, dim3((unsigned)batch), T, encode_real_smem<LOGM>(), 1, s, a);
      }
      if (a.fast == 2) {
        constexpr int T = FastEnc<LOGM, 2>::THREADS;
        if (a.wide) return launch_ex(encode_real_fast_kernel<LOGM, true, 2>, dim3((unsigned)batch), T, encode_real_smem<LOGM>(), 1, s, a);
        return launch_ex(encode_real_fast_kernel<LOGM, false, 2>, dim3((unsigned)batch), T, encode_real_smem<LOGM>(), 1, s, a);
      }
    }
    if (a.wide) return launch_ex(encode_real_kernel<LOGM, true>, dim3((unsigned)batch), 256, encode_real_smem<LOGM>(), 1, s, a);
    return launch_ex(encode_real_kernel<LOGM, false>, dim3((unsigned)batch), 256, encode_real_smem<LOGM>(), 1, s, a);
  }
  constexpr int C = LOGM > 13 ? 2 : 1;
  return launch_ex(encode_kernel<LOGM>, dim3((unsigned)(batch * C)), FftPlan<(LOGM > 13 ? LOGM - 1 : LOGM)>::THREADS,
                   encode_smem<LOGM>(), C, s, a);
}
// Messages one full wave of the (throughput) encode kernel covers: resident CTAs per SM (the
// occupancy calculator, with the kernel's dynamic shared memory) x SMs / CTAs per message.
template <int LOGM>
static size_t encode_wave_msgs_t(bool complex_slots, int num_sms) {
  int per_sm = 0;
  if (!complex_slots) {
    if (set_smem(encode_real_kernel<LOGM, false>, encode_real_smem<LOGM>()) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, encode_real_kernel<LOGM, false>, 256,
                                                      encode_real_smem<LOGM>()) != cudaSuccess)
      return 0;
    return (size_t)per_sm * num_sms;
  }
  constexpr int C = LOGM > 13 ? 2 : 1;
  if (set_smem(encode_kernel<LOGM>, encode_smem<LOGM>()) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, encode_kernel<LOGM>,
                                                    FftPlan<(LOGM > 13 ? LOGM - 1 : LOGM)>::THREADS,
                                                    encode_smem<LOGM>()) != cudaSuccess)
    return 0;
  return (size_t)per_sm * num_sms / C;
}
size_t encode_wave_msgs(int log_n, bool complex_slots, int num_sms) {
  switch (log_n) {
    case 12: return encode_wave_msgs_t<11>(complex_slots, num_sms);
    case 13: return encode_wave_msgs_t<12>(complex_slots, num_sms);
    case 14: return encode_wave_msgs_t<13>(complex_slots, num_sms);
    case 15: return encode_wave_msgs_t<14>(complex_slots, num_sms);
  }
  return 0;
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
