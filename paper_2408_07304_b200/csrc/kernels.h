// kernels.h -- argument blocks and launchers of the kernels in k_*.cu
// (internal to libzinc.so; the public ABI is include/zinc.h).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "common.cuh"

namespace zinc {

using Tw = ulonglong2;  // {w, floor(w 2^64 / q)}

// Programmatic dependent launch for the launches made while a PdlScope is alive on this
// thread: the next kernel in the stream may start once every CTA of the previous one has
// started (griddepcontrol.launch_dependents) and must griddepcontrol.wait before touching
// the previous kernel's outputs.  Used by the encode -> Zinc chunk pipeline.
// L2 prefetch request handed from the chunk pipeline to the next Zinc COEFF launch
struct L2Prefetch {
  const void *p = nullptr;
  size_t bytes = 0;
};
inline thread_local L2Prefetch g_l2_prefetch;
inline thread_local bool g_launch_pdl = false;
struct PdlScope {
  bool old;
  explicit PdlScope(bool on) : old(g_launch_pdl) { g_launch_pdl = on; }
  ~PdlScope() { g_launch_pdl = old; }
};

struct ZincCoeffArgs {
  const LimbConst *limbs;
  const uint64_t *cache;  // [2][L][N]
  const int64_t *m;       // [batch][N] or null (m = 0)
  uint64_t *ct;           // [batch][2][L][N]
  size_t batch, msgs_per_cta;
  uint64_t seed, msg_base;
  uint64_t qmin;          // min_i q_i (fast-path bound)
  int n, L;
  int discard_m;          // m is library scratch: discard its L2 lines after reading
  const int64_t *m128;    // CKKS 128-bit plaintexts (int64 pairs [batch][N][2]); overrides m
  const char *prefetch;   // the next chunk's slots: warmed into L2 while this chunk streams
  size_t prefetch_bytes;  // (16-byte multiple; 0: none)
  int wide_hb;            // 128-bit plaintexts: 63 - bits(q_max), the "tiny high word" bound (zinc_coeff.cuh)
  size_t m_stride;        // int64 words between messages' plaintexts in m (N, or 2 L N when the
                          // plaintexts sit in the ciphertexts' last c2 limb, see encrypt_any)
};
struct VanillaArgs {
  const LimbConst *limbs;
  const Tw *tw, *itw;
  const uint64_t *pk;     // [2][L][N] NTT form
  const uint64_t *pk_sh;  // [2][L][N] Shoup companions floor(pk 2^64 / q_i) (shoup_prep_kernel)
  const int64_t *m;       // [batch][N] or null
  uint64_t *ct;
  uint64_t *u_hat;        // small batches, NTT form: the u transform's output [batch][L][N] (else null)
  uint64_t seed, msg_base;
  int L, limbs_per_cta;
  int m_deint;            // log2 of the de-interleave of m (EncodeArgs::deint_log); 0: natural order
};
struct ZincNttArgs {
  const LimbConst *limbs;
  const Tw *tw;
  const uint64_t *cache;  // NTT form
  const int64_t *m;
  uint64_t *ct;
  uint64_t seed, msg_base;
  int L, limbs_per_cta;
  int t_split;            // small batches: the two transforms on separate CTAs (gridDim.z = 2)
  int m_deint;            // log2 of the de-interleave of m (EncodeArgs::deint_log); 0: natural order
};
struct KeygenArgs {
  const LimbConst *limbs;
  const Tw *tw;
  uint64_t *pk, *sk_ntt;
  int8_t *sk_coeff;
  uint64_t seed;
  int L;
};
struct DecryptArgs {
  const LimbConst *limbs;
  const Tw *tw, *itw;
  const uint64_t *sk_ntt, *ct;
  const uint64_t *sk_sh;  // [L][N] Shoup companions of sk_ntt
  int64_t *coeff_out;
  int32_t *status_out;
  uint64_t *xl_out;       // BFV: residues [B][L][N] for bfv_scale_kernel
  int64_t *x128_out;      // wide CKKS: x from limbs 0 and 1 (two-limb CRT), int64 pairs [B][N][2]
  uint64_t q0inv_q1;      // q_0^-1 mod q_1
  int L;
  int plain_ckks;         // CKKS, 64-bit coefficients: the kernels compile out BFV / BGV / wide
};
struct LiftArgs {           // 128-bit plaintexts -> RNS residues (f3)
  const LimbConst *limbs;
  const int64_t *m;         // int64 pairs [B][N][2]
  uint64_t *res;            // [B][L][N]
  size_t batch;
  int n, L;
};
struct PtAddArgs {          // c1 += plaintext residues (Eq. 4 on a ciphertext of m = 0)
  const LimbConst *limbs;
  const uint64_t *res;      // [B][L][N] (in the ciphertext's form)
  uint64_t *ct;             // [B][2][L][N]
  size_t batch;
  int n, L;
};
struct BfvScaleArgs {
  const LimbConst *limbs;
  const uint64_t *xl;     // [B][L][N]
  int64_t *m_out;         // [B][N], m in [0, t)
  size_t batch;
  int n, L;
};
struct EncodeArgs {
  const double *slots;
  int complex_slots;
  const int *perm;
  const double2 *fft_tw, *twist;
  const double2 *fft_tw_h;  // W_{M/2}^e, e < M/4 (real-slot path)
  const double2 *fft_tw_hp; // the same table padded for shared memory (fft_twpad), TMA-staged by the encodes
  const double2 *post_tw;   // real-slot split step: [A | B | A5 | B5] (encode_real_post)
  const double2 *twist_split;  // complex-slot twist zeta^-j = A'[j >> 6] B[j & 63], j < M: [A' | B]
  int wide;                 // m_out holds 128-bit coefficients (int64 pairs)
  int fast;                 // real slots, batch below the SM count: the latency variant (more threads)
  double scale;
  int64_t *m_out;
  size_t m_stride;          // int64 words between messages' plaintexts in m_out (N; 2N when wide)
  int wait_mode;            // PDL: 0 wait for the previous kernel before the plaintext stores,
                            // 1 after them (the stores go to a region no earlier kernel touches)
  int deint_log;            // d > 0: coefficient x is stored at (x mod 2^d) N / 2^d + (x >> d), the order
                            // in which the CTAs of a 2^d-CTA cluster transform read their subsequences
                            // x = 2^d i + r (contiguous instead of stride 2^d); 64-bit plaintexts only
};
struct DecodeArgs {
  const int64_t *coeff;     // int64 [B][N], or int64 pairs [B][N][2] when wide
  int wide;
  const int *perm;
  const double2 *fft_tw, *twist;
  double inv_scale;
  double *slots_out;
};
struct NttArgs {
  const LimbConst *limbs;
  const Tw *tw, *itw;
  uint64_t *data;
  int L;
};
struct CtAddArgs {
  const LimbConst *limbs;
  const uint64_t *a, *b;
  uint64_t *out;
  size_t words;           // count * 2 * L * N
  int log_n, L;
};
struct CtSumArgs {
  const LimbConst *limbs;
  const uint64_t *ct;     // [batch][2][L][N]
  uint64_t *out;          // [2][L][N]
  size_t batch;
  int log_n, L;
};
struct SampleArgs {
  uint32_t tag, limb;
  uint64_t seed, msg, q;
  size_t n;
  void *out;
};
struct IntPeakArgs {
  uint64_t q, w, wp;
  int iters;
  uint64_t *sink;
};

size_t zinc_coeff_smem(int L, int threads);
cudaError_t launch_zinc_coeff(const ZincCoeffArgs &a, int threads, int grid_y, size_t smem_pad, cudaStream_t s);
cudaError_t launch_vanilla(int log_n, const VanillaArgs &a, int form, int mode, size_t batch, int groups,
                           cudaStream_t s);
cudaError_t launch_zinc_ntt(int log_n, const ZincNttArgs &a, int mode, size_t batch, int groups, cudaStream_t s);
// S-CTA cluster kernels for N = 2^14, 2^15 (k_split.cu)
cudaError_t launch_zinc_ntt_split(int log_n, const ZincNttArgs &a, int mode, size_t batch, int groups, cudaStream_t s);
cudaError_t launch_vanilla_split(int log_n, const VanillaArgs &a, int form, int mode, size_t batch, int groups,
                                 cudaStream_t s);
cudaError_t launch_decrypt_split(int log_n, const DecryptArgs &a, int form, bool nr, size_t batch, cudaStream_t s);
cudaError_t launch_keygen(int log_n, const KeygenArgs &a, cudaStream_t s);
cudaError_t launch_decrypt(int log_n, const DecryptArgs &a, int form, size_t batch, cudaStream_t s);
cudaError_t launch_bfv_scale(const BfvScaleArgs &a, cudaStream_t s);
cudaError_t launch_lift(const LiftArgs &a, cudaStream_t s);
cudaError_t launch_pt_add(const PtAddArgs &a, cudaStream_t s);
cudaError_t launch_encode(int log_n, const EncodeArgs &a, size_t batch, cudaStream_t s);
// messages per full wave of the encode kernel (0 if unknown)
size_t encode_wave_msgs(int log_n, bool complex_slots, int num_sms);
cudaError_t launch_decode(int log_n, const DecodeArgs &a, size_t batch, cudaStream_t s);
// small-batch latency path (k_small.cu): real-slot encode of one message per C-CTA cluster
// (C = small_cluster_ctas()), alone (plaintexts to a.m_out) or fused with the COEFF-form Zinc
// add/inject (R cluster replicas per message, PP ciphertext polynomials per replica)
int small_cluster_ctas();
cudaError_t launch_encode_cluster(int log_n, const EncodeArgs &a, size_t batch, cudaStream_t s);
cudaError_t launch_zinc_coeff_small(int log_n, const EncodeArgs &e, const ZincCoeffArgs &z, size_t batch, int R,
                                    int PP, cudaStream_t s);
cudaError_t launch_ntt(int log_n, const NttArgs &a, int inv, size_t polys, cudaStream_t s);
cudaError_t launch_sample(const SampleArgs &a, cudaStream_t s);
cudaError_t launch_ct_add(const CtAddArgs &a, cudaStream_t s);
cudaError_t launch_ct_sum(const CtSumArgs &a, cudaStream_t s);
// w' = floor(w 2^64 / q_i) for the `words` words of keys [rows][L][N] (pk, sk)
// ct0 += pk1 u^, ct1 += pk2 u^ after a transform-split vanilla NTT-form launch (a.u_hat)
cudaError_t launch_vanilla_combine(const VanillaArgs &a, size_t batch, int n, cudaStream_t s);
cudaError_t launch_shoup_prep(const LimbConst *limbs, const uint64_t *w, uint64_t *wp, size_t words, int log_n, int L,
                              cudaStream_t s);
cudaError_t launch_int_peak(const IntPeakArgs &a, int variant, int blocks, cudaStream_t s);

}  // namespace zinc
