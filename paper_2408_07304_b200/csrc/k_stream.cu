// k_stream.cu -- Zinc add/inject (COEFF form), the debug sampler and the integer-peak microkernel.
#include <algorithm>

#include "zinc_coeff.cuh"

namespace zinc {

// ============================================================ Zinc, COEFF form
template <int LC>
__global__ void __launch_bounds__(256, 3) zinc_coeff_kernel(ZincCoeffArgs a) {
  extern __shared__ __align__(16) uint64_t tile[];
  zinc_coeff_body<LC>(a, blockIdx.x, blockIdx.y, tile);
}

// ============================================================ Eq. 2: batched (+) and aggregation
// out = [a + b]_q word by word over [count][2][L][N] (either form: the NTT is
// linear).  16-byte loads/stores; the limb of word w is (w / N) mod L.
__global__ void __launch_bounds__(256) ct_add_kernel(CtAddArgs a) {
  const size_t pairs = a.words / 2;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < pairs; p += (size_t)gridDim.x * blockDim.x) {
    const size_t w = 2 * p;
    const uint64_t q = __ldg(&a.limbs[(w >> a.log_n) % a.L].q);
    const ulonglong2 x = ld2_nc(a.a + w), y = ld2_nc(a.b + w);
    st2_cs(a.out + w, add_mod(x.x, y.x, q), add_mod(x.y, y.y, q));
  }
}
// out = [sum_b ct_b]_q: one thread per word pair of the [2][L][N] result, walking
// the batch with U independent 16-byte loads in flight (HBM-bound read of the
// whole batch, one write).
__global__ void __launch_bounds__(256) ct_sum_kernel(CtSumArgs a) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t words = (size_t)2 * a.L << a.log_n;
  if (2 * p >= words) return;
  const size_t w = 2 * p;
  const uint64_t q = __ldg(&a.limbs[(w >> a.log_n) % a.L].q);
  uint64_t s0 = 0, s1 = 0;
  constexpr int U = 8;
  size_t b = 0;
  for (; b + U <= a.batch; b += U) {
    ulonglong2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld2_nc(a.ct + (b + u) * words + w);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      s0 = add_mod(s0, v[u].x, q);
      s1 = add_mod(s1, v[u].y, q);
    }
  }
  for (; b < a.batch; ++b) {
    const ulonglong2 v = ld2_nc(a.ct + b * words + w);
    s0 = add_mod(s0, v.x, q);
    s1 = add_mod(s1, v.y, q);
  }
  st2(a.out + w, s0, s1);
}

cudaError_t launch_ct_add(const CtAddArgs &a, cudaStream_t s) {
  const size_t pairs = a.words / 2;
  const unsigned blocks = (unsigned)std::min<size_t>((pairs + 255) / 256, 148 * 16);
  ct_add_kernel<<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_ct_sum(const CtSumArgs &a, cudaStream_t s) {
  const size_t pairs = ((size_t)2 * a.L << a.log_n) / 2;
  ct_sum_kernel<<<(unsigned)((pairs + 255) / 256), 256, 0, s>>>(a);
  return cudaGetLastError();
}

// ============================================================ wide plaintexts (f3)
// res[b][i][j] = (hi 2^64 + lo) mod q_i for 128-bit coefficients (the paper's own
// parameters put |Delta z| above 2^63).
__global__ void __launch_bounds__(256) lift_kernel(LiftArgs a) {
  const size_t total = a.batch * (size_t)a.n;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t b = idx / a.n, j = idx % a.n;
    const int64_t lo = a.m[2 * idx], hi = a.m[2 * idx + 1];
    for (int i = 0; i < a.L; ++i) a.res[(b * a.L + i) * a.n + j] = reduce_i128(hi, (uint64_t)lo, a.limbs[i]);
  }
}
// Eq. 4 on a ciphertext of m = 0: c1 += m (residues in the ciphertext's form).
__global__ void __launch_bounds__(256) pt_add_kernel(PtAddArgs a) {
  const size_t ln = (size_t)a.L * a.n, pairs = a.batch * ln / 2;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < pairs; p += (size_t)gridDim.x * blockDim.x) {
    const size_t w = 2 * p, b = w / ln, r = w % ln;
    const uint64_t q = __ldg(&a.limbs[r / a.n].q);
    uint64_t *c1 = a.ct + b * 2 * ln + r;
    const ulonglong2 x = ld2_nc(a.res + w);
    uint64_t c0, c1v;
    ld2(c1, c0, c1v);
    st2(c1, add_mod(c0, x.x, q), add_mod(c1v, x.y, q));
  }
}
cudaError_t launch_lift(const LiftArgs &a, cudaStream_t s) {
  const size_t total = a.batch * (size_t)a.n;
  lift_kernel<<<(unsigned)std::min<size_t>((total + 255) / 256, 148 * 16), 256, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_pt_add(const PtAddArgs &a, cudaStream_t s) {
  const size_t pairs = a.batch * (size_t)a.L * a.n / 2;
  pt_add_kernel<<<(unsigned)std::min<size_t>((pairs + 255) / 256, 148 * 16), 256, 0, s>>>(a);
  return cudaGetLastError();
}

// ============================================================ Shoup companions of a key
// w' = floor(w 2^64 / q) for canonical words w of a key [rows][L][N] (limb (idx >> log N) mod L),
// so the per-message pointwise products pk u^ (vanilla) and c2 s (decryption) are Shoup
// products (mul_shoup_lazy) instead of Barrett products of two variables.  The estimate
// x floor(2^128 / q) / 2^64 is at most 2 short; the remainder x 2^64 - w' q (< 3q, exact in
// 64 bits) corrects it.
__global__ void __launch_bounds__(256) shoup_prep_kernel(const LimbConst *limbs, const uint64_t *w, uint64_t *wp,
                                                          size_t words, int log_n, int L) {
  pdl_trigger();  // in a PDL chain: the next kernel may launch; this one reads only the key
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < words; idx += (size_t)gridDim.x * blockDim.x) {
    const LimbConst &c = limbs[(idx >> log_n) % L];
    const uint64_t x = w[idx];
    uint64_t est = x * c.qinv_hi + __umul64hi(x, c.qinv_lo);
    uint64_t r = (uint64_t)0 - est * c.q;
    while (r >= c.q) {
      r -= c.q;
      ++est;
    }
    wp[idx] = est;
  }
  pdl_wait();  // complete only after the kernel before it (the chain's order stays transitive)
}
cudaError_t launch_shoup_prep(const LimbConst *limbs, const uint64_t *w, uint64_t *wp, size_t words, int log_n, int L,
                              cudaStream_t s) {
  const unsigned blocks = (unsigned)std::min<size_t>((words + 255) / 256, 148 * 8);
  shoup_prep_kernel<<<blocks, 256, 0, s>>>(limbs, w, wp, words, log_n, L);
  return cudaGetLastError();
}

// ============================================================ vanilla combine (small batches)
// After a transform-split vanilla NTT-form launch: c1 = NTT(m + e1) + pk1 u^, c2 = NTT(e2) +
// pk2 u^ (Eq. 8) word by word, u^ from a.u_hat.  16-byte accesses.
__global__ void __launch_bounds__(256) vanilla_combine_kernel(VanillaArgs a, size_t batch, int n) {
  pdl_trigger();
  pdl_wait();  // the transforms' outputs
  const size_t ln = (size_t)a.L * n, pairs = batch * ln / 2;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < pairs; p += (size_t)gridDim.x * blockDim.x) {
    const size_t w = 2 * p, b = w / ln, r = w % ln;
    const int limb = (int)(r / n);
    const uint64_t q = __ldg(&a.limbs[limb].q);
    uint64_t *c0 = a.ct + b * 2 * ln + r, *c1 = c0 + ln;
    const LimbConst &c = a.limbs[limb];
    const ulonglong2 u = ld2_nc(a.u_hat + w), p1 = ld2_nc(a.pk + r), p2 = ld2_nc(a.pk + ln + r);
    uint64_t a0, a1, b0, b1;
    ld2(c0, a0, a1);
    ld2(c1, b0, b1);
    // u^ is canonical; Barrett products (no Shoup companions on this small-batch path)
    st2_cs(c0, add_mod(a0, mul_mod(p1.x, u.x, c), q), add_mod(a1, mul_mod(p1.y, u.y, c), q));
    st2_cs(c1, add_mod(b0, mul_mod(p2.x, u.x, c), q), add_mod(b1, mul_mod(p2.y, u.y, c), q));
  }
}
cudaError_t launch_vanilla_combine(const VanillaArgs &a, size_t batch, int n, cudaStream_t s) {
  const size_t pairs = batch * (size_t)a.L * n / 2;
  return launch_ex(vanilla_combine_kernel, dim3((unsigned)std::min<size_t>((pairs + 255) / 256, 148 * 8)), 256, 0, 1, s,
                   a, batch, n);
}

// ============================================================ samplers (debug)
__global__ void sample_kernel(SampleArgs a) {
  size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.n) return;
  if (a.tag == TAG_SK || a.tag == TAG_ENC_U) {
    uint4 w = stream_block(a.seed, a.msg, a.tag, 0, (uint32_t)(c / 4));
    uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    reinterpret_cast<int64_t *>(a.out)[c] = tern(ws[c % 4]);
  } else if (a.tag == TAG_PK_A) {
    uint4 w = stream_block(a.seed, a.msg, a.tag, a.limb, (uint32_t)c);
    reinterpret_cast<uint64_t *>(a.out)[c] = uniform_mod(w, a.q);
  } else {
    uint4 w = stream_block(a.seed, a.msg, a.tag, 0, (uint32_t)(c / 2));
    reinterpret_cast<int64_t *>(a.out)[c] = (c & 1) ? cbd_hi(w) : cbd_lo(w);
  }
}

// ============================================================ integer peak (K11)
// 8 independent register-resident butterflies per thread per iteration, no memory
// traffic: the measured integer peak the transform kernels are held to.  VARIANT
// selects the butterfly the kernels actually run (common.cuh):
//  0 ct_bfly     lazy Harvey forward butterfly, exact Shoup quotient (4 partial products)
//  1 ct_bfly_nr  lazy-free forward butterfly (q < 2^58: every CKKS forward transform here)
//  2 ct_bfly_a   forward butterfly with one conditional subtraction (q up to 2^60)
//  3 gs_bfly     inverse Gentleman-Sande butterfly (every inverse transform)
template <int VARIANT>
__global__ void __launch_bounds__(256) int_peak_kernel(IntPeakArgs a) {
  const uint64_t q = a.q, two_q = 2 * a.q;
  uint64_t v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = (threadIdx.x * 16 + r + blockIdx.x) % q;
  uint64_t w = a.w, wp = a.wp;
  for (int it = 0; it < a.iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if constexpr (VARIANT == 0) ct_bfly(v[r], v[r + 8], w, wp, q, two_q);
      else if constexpr (VARIANT == 1) ct_bfly_nr(v[r], v[r + 8], w, wp, q, two_q);
      else if constexpr (VARIANT == 2) ct_bfly_a(v[r], v[r + 8], w, wp, q, 2 * two_q);
      else gs_bfly(v[r], v[r + 8], w, wp, q, 2 * two_q);
    }
    w += (v[0] & 1);  // keep w loop-variant so the compiler cannot hoist
  }
  uint64_t acc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc ^= v[r];
  if (acc == 0x1234567890ABCDEFull) a.sink[0] = acc;
}

size_t zinc_coeff_smem(int L, int threads) { return ((size_t)2 * L * 2 * threads + 8 * L) * sizeof(uint64_t); }

cudaError_t launch_zinc_coeff(const ZincCoeffArgs &a, int threads, int grid_y, size_t smem_pad, cudaStream_t s) {
  dim3 grid(a.n / (2 * threads), grid_y);
  const size_t smem = std::min<size_t>(zinc_coeff_smem(a.L, threads) + smem_pad, 227 * 1024);
  switch (a.L) {
    case 3: return launch_ex(zinc_coeff_kernel<3>, grid, threads, smem, 1, s, a);
    case 4: return launch_ex(zinc_coeff_kernel<4>, grid, threads, smem, 1, s, a);
    case 8: return launch_ex(zinc_coeff_kernel<8>, grid, threads, smem, 1, s, a);
    case 16: return launch_ex(zinc_coeff_kernel<16>, grid, threads, smem, 1, s, a);
  }
  return launch_ex(zinc_coeff_kernel<0>, grid, threads, smem, 1, s, a);
}

cudaError_t launch_sample(const SampleArgs &a, cudaStream_t s) {
  unsigned blocks = (unsigned)((a.n + 255) / 256);
  sample_kernel<<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_int_peak(const IntPeakArgs &a, int variant, int blocks, cudaStream_t s) {
  switch (variant) {
    case 0: int_peak_kernel<0><<<blocks, 256, 0, s>>>(a); break;
    case 1: int_peak_kernel<1><<<blocks, 256, 0, s>>>(a); break;
    case 2: int_peak_kernel<2><<<blocks, 256, 0, s>>>(a); break;
    default: int_peak_kernel<3><<<blocks, 256, 0, s>>>(a); break;
  }
  return cudaGetLastError();
}


}  // namespace zinc
