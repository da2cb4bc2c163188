/*
 * zinc.h -- C ABI of libzinc.so, the B200 (sm_100a) hot path of arXiv 2408.07304
 * ("Zinc"): batched CKKS/RLWE public-key encryption over RNS polynomials, in the
 * vanilla form (Eq. 8) and the Zinc form (PAPER.md:214-223,
 * Algorithm 1), plus the supporting keygen (Eq. 7), cache precompute
 * (PAPER.md:164-166), encode and decrypt/decode (Eq. 10) calls.
 *
 * The calls follow the paper's problem statement Pi~ = (Gen, Enc_z, Dec)
 * extending Pi = (Gen, Enc, Dec, +, x).  Numeric contract
 * (primes, psi, NTT order, Philox layout, encoding): docs/CONVENTIONS.md
 * (C-1..C-10).
 *
 * Conventions for every call below
 *  - Buffers are DEVICE pointers owned by the caller (e.g. torch tensors) on the
 *    context's device unless a parameter says "host".  They must be 16-byte
 *    aligned.  The library never keeps a pointer after a call returns.
 *  - Layouts are C order:  RNS polynomial uint64[L][N]; ciphertext, public key
 *    and cache uint64[2][L][N] with component 0 = the paper's c1 (carries m,
 *    PAPER.md:185) and 1 = c2; a batch is uint64[B][2][L][N].  Every stored word
 *    is the canonical residue in [0, q_i).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Device calls are asynchronous on it and never synchronise the host; faults
 *    surface at the caller's next synchronisation.
 *  - Every call returns a zinc_status; on failure zinc_last_error() returns a
 *    thread-local message.  Arguments are validated before any launch:
 *    NULL pointers, bad enums, misaligned pointers -> ZINC_EINVAL.  batch == 0
 *    is a no-op returning ZINC_OK.
 *  - Randomness: a (seed, message index) pair is a nonce; the caller must never
 *    reuse one.  Message b of a batch uses msg = msg_base + b, so a batch split
 *    across GPUs with msg_base = global offset gives bit-identical output.
 *  - There is no CPU fallback: every compute step runs in this library's CUDA
 *    kernels.
 */
#ifndef ZINC_H
#define ZINC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct zinc_ctx zinc_ctx; /* opaque: params + device tables, bound to one device */
typedef void *zinc_stream_t;      /* a cudaStream_t */

typedef enum {
  ZINC_OK = 0,
  ZINC_EINVAL = -1,       /* bad argument */
  ZINC_EUNSUPPORTED = -2, /* valid but not implemented (e.g. a kind at this N) */
  ZINC_ECUDA = -3,        /* a CUDA runtime call or launch failed */
  ZINC_ENOMEM = -4,       /* device or host allocation failed */
  ZINC_EPARAMS = -5       /* no parameter set exists (no prime found, ...) */
} zinc_status;

/* Ciphertext / cache representation (reading A4).  NTT: both
 * components stored as NTT(c) in the order of C-3; COEFF: coefficient vectors.
 * NTT(COEFF-form ct) == NTT-form ct bit for bit. */
typedef enum { ZINC_FORM_NTT = 0, ZINC_FORM_COEFF = 1 } zinc_form;

/* Plaintext input kinds.  COEFF_I64: int64[B][N] integer plaintext polynomial
 * (the bit-exact contract); SLOTS_F64: double[B][N/2] real slots;
 * SLOTS_C128: double[B][N/2][2] complex slots (re, im).  Slots are encoded per
 * C-6 (canonical embedding, scale 2^log_scale) inside the library. */
typedef enum {
  ZINC_PT_COEFF_I64 = 0,
  ZINC_PT_SLOTS_F64 = 1,
  ZINC_PT_SLOTS_C128 = 2,
  ZINC_PT_COEFF_I128 = 3 /* int64[B][N][2]: coefficient j = hi 2^64 + lo with (lo, hi) at [j][0], [j][1] */
} zinc_pt_kind;

/* ---- context ------------------------------------------------------------ */

/* Create a context on CUDA device `device`: ring degree N = 2^log_n
 * (12 <= log_n <= 15), L = num_limbs RNS primes (1 <= L <= 32) of the listed
 * bit sizes (20 <= bits <= 60; the lazy butterfly needs q < 2^62), chosen per
 * C-1 (largest primes q < 2^b, q = 1 mod 2N); psi per C-2; scale
 * Delta = 2^log_scale (1 <= log_scale <= 60).  Builds the twiddle and FFT tables
 * on the host and uploads them (synchronous; not a hot call).  *out receives
 * the context; free it with zinc_ctx_destroy.  Limb 0 must be the largest prime
 * (decryption's CRT check, C-10) or ZINC_EPARAMS is returned. */
zinc_status zinc_ctx_create(int log_n, int num_limbs, const int *limb_bits, int log_scale,
                            int device, zinc_ctx **out);
zinc_status zinc_ctx_destroy(zinc_ctx *ctx);

/* Scheme of a context (section 4.2). */
typedef enum { ZINC_SCHEME_CKKS = 0, ZINC_SCHEME_BFV = 1, ZINC_SCHEME_BGV = 2 } zinc_scheme;

/* zinc_ctx_create for a scheme.  CKKS: as zinc_ctx_create (plain_modulus ignored).
 * BFV (Eq. 12): c1 = [pk1.u + e1 + Delta.m]_Q, Delta = floor(Q/t), Q = prod q_i; Zinc
 *   unchanged.  BGV (Eq. 13): c1 = [pk1.u + t.e1 + m]_Q, c2 = [pk2.u + t.e2]_Q;
 *   keygen uses the t-scaled key error pk1 = [-a.sk + t.e]_Q (reading A17) and Zinc injects
 *   t.e1', t.e2'.  plain_modulus t: 2 <= t < 2^32 and t < every q_i, else
 *   ZINC_EINVAL / ZINC_EPARAMS; log_scale is ignored for BFV / BGV.  Plaintexts of BFV / BGV
 *   contexts are int64 coefficients (kind ZINC_PT_COEFF_I64 only); the library uses each
 *   coefficient's residue m mod t in [0, t) (reading A18).  ckks_decrypt_batch on such a
 *   context writes m in [0, t) to coeff_out (BGV: from limb 0 with the CRT status as for
 *   CKKS; BFV: round(t.x/Q) mod t from every limb, status 0) and needs slots_out == NULL. */
zinc_status zinc_ctx_create_scheme(int log_n, int num_limbs, const int *limb_bits, int scheme,
                                   uint64_t plain_modulus, int log_scale, int device,
                                   zinc_ctx **out);
/* Scheme and plaintext modulus of a context (host pointers, each may be NULL). */
zinc_status zinc_ctx_scheme(const zinc_ctx *ctx, int *scheme, uint64_t *plain_modulus);

/* Host copies of the moduli q_i and roots psi_i (arrays of L, host pointers). */
zinc_status zinc_ctx_moduli(const zinc_ctx *ctx, uint64_t *q_out, uint64_t *psi_out);
/* N, L, log_scale of the context (host pointers, each may be NULL). */
zinc_status zinc_ctx_info(const zinc_ctx *ctx, int *log_n, int *num_limbs, int *log_scale);

/* ---- Gen: Eq. 7, C-5 ----------------------------------- */

/* sk <- R_2, a <- R_q, e <- chi (CBD eta=21, reading A3);
 * pk1 = [-a.sk + e]_q, pk2 = a.  Outputs (device): sk_ntt uint64[L][N] (NTT
 * form), sk_coeff int8[N] in {-1,0,1} (may be NULL), pk_ntt uint64[2][L][N]
 * (NTT form). */
zinc_status zinc_keygen(const zinc_ctx *ctx, uint64_t seed, uint64_t *sk_ntt, int8_t *sk_coeff,
                        uint64_t *pk_ntt, zinc_stream_t stream);

/* ---- Zinc precomputation: PAPER.md:164-166 ("caches a single Enc(0)"), C-8 - */

/* cache = vanilla Enc(0) under pk_ntt with message index 2^64-1 and seed
 * `seed`, stored in `form`.  cache: uint64[2][L][N]. */
zinc_status zinc_precompute_cache(const zinc_ctx *ctx, const uint64_t *pk_ntt, uint64_t seed,
                                  zinc_form form, uint64_t *cache, zinc_stream_t stream);

/* ---- Enc_z: Algorithm 1, Eq. 4 + Eq. 9, C-9 ------------ */

/* For b in [0, batch): c = zero + m_b (m added to c1 only, reading A2);
 * e1', e2' <- chi (Philox stream (seed, msg_base + b), tags 7/8);
 * ct_b = ([c1 + e1']_q, [c2 + e2']_q), in the cache's form (the caller passes the
 * form the cache was built in).  In NTT form the added polynomials are
 * transformed (NTT(m + e1'), NTT(e2')).  pt: see zinc_pt_kind.
 * ct: uint64[batch][2][L][N]. */
zinc_status zinc_encrypt_batch(const zinc_ctx *ctx, const uint64_t *cache, zinc_form form,
                               zinc_pt_kind kind, const void *pt, size_t batch, uint64_t seed,
                               uint64_t msg_base, uint64_t *ct, zinc_stream_t stream);

/* ---- Enc: Eq. 8 with c2 = [pk2.u + e2]_q (reading A1), C-7 */

/* For b in [0, batch): u <- R_2, e1, e2 <- chi (tags 4/5/6);
 * c1 = [pk1.u + e1 + m_b]_q, c2 = [pk2.u + e2]_q, stored in `form`.
 * pk_ntt: uint64[2][L][N] NTT form.  ct: uint64[batch][2][L][N]. */
zinc_status ckks_encrypt_batch(const zinc_ctx *ctx, const uint64_t *pk_ntt, zinc_form form,
                               zinc_pt_kind kind, const void *pt, size_t batch, uint64_t seed,
                               uint64_t msg_base, uint64_t *ct, zinc_stream_t stream);

/* ---- Dec: Eq. 10, C-10 --------------------------------- */

/* x = [c1 + c2.sk]_q per limb; coeff_out[b] (int64[N], may be NULL) = x
 * centred mod q_0; status_out[b] (int32, may be NULL) = 0 if x_0 mod q_i ==
 * x^(i) on every limb (CRT consistency), else 1; slots_out[b] (double[N/2][2],
 * may be NULL) = decode(x) = (1/Delta) sum_j x_j zeta^(g_k j).  ct in `form`. */
zinc_status ckks_decrypt_batch(const zinc_ctx *ctx, const uint64_t *sk_ntt, zinc_form form,
                               const uint64_t *ct, size_t batch, double *slots_out,
                               int64_t *coeff_out, int32_t *status_out, zinc_stream_t stream);

/* ---- Eq. 2: batched (+) and aggregation -------------------- */

/* out_b = [x_b + y_b]_q componentwise for b < batch; ciphertexts uint64[batch][2][L][N]
 * in one form (either: the NTT is linear); out may alias x or y.  Dec(out_b) = m_x + m_y
 * (+ noise) in every scheme. */
zinc_status zinc_ct_add_batch(const zinc_ctx *ctx, const uint64_t *x, const uint64_t *y,
                              size_t batch, uint64_t *out, zinc_stream_t stream);
/* Aggregation: out = [sum_b ct_b]_q, one ciphertext uint64[2][L][N] (batch 0 -> zero). */
zinc_status zinc_ct_sum_batch(const zinc_ctx *ctx, const uint64_t *ct, size_t batch,
                              uint64_t *out, zinc_stream_t stream);

/* Wide decryption (f3): x = [c1 + c2.sk]_Q recovered in (-q0 q1 / 2, q0 q1 / 2] from limbs 0
 * and 1 by CRT, CRT-checked on every other limb (status 1 on a mismatch); coeff128_out
 * (int64[B][N][2], may be NULL) receives x, slots_out (may be NULL) its decoding.  Needs
 * L >= 2 and |m + v| < q0 q1 / 2. */
zinc_status ckks_decrypt_batch_wide(const zinc_ctx *ctx, const uint64_t *sk_ntt, zinc_form form,
                                    const uint64_t *ct, size_t batch, double *slots_out,
                                    int64_t *coeff128_out, int32_t *status_out,
                                    zinc_stream_t stream);

/* ---- support / test exports ---------------------------------------------- */

/* Encode slots (kind SLOTS_F64 or SLOTS_C128) to int64[batch][N] per C-6. */
zinc_status ckks_encode_batch_wide(const zinc_ctx *ctx, zinc_pt_kind kind, const void *slots,
                                   size_t batch, int64_t *m_out /* [batch][N][2] */,
                                   zinc_stream_t stream);
/* (ckks_encode_batch_wide: the same, into 128-bit coefficients; ckks_encode_batch below.) */
zinc_status ckks_encode_batch(const zinc_ctx *ctx, zinc_pt_kind kind, const void *slots,
                              size_t batch, int64_t *m_out, zinc_stream_t stream);

/* In-place forward (C-3) / inverse NTT of `count` RNS polynomials uint64[count][L][N]
 * (inputs must be canonical residues). */
zinc_status zinc_ntt_forward(const zinc_ctx *ctx, uint64_t *data, size_t count, zinc_stream_t stream);
zinc_status zinc_ntt_inverse(const zinc_ctx *ctx, uint64_t *data, size_t count, zinc_stream_t stream);

/* Draw n coefficients of the Philox stream (seed, msg, tag, limb) per C-4.
 * tag 1..8.  Ternary tags (1, 4) and CBD tags (2, 5, 6, 7, 8) write int64 values
 * (limb ignored); the uniform tag 3 writes uint64 residues mod q_limb. */
zinc_status zinc_debug_sample(const zinc_ctx *ctx, int tag, uint64_t seed, uint64_t msg,
                              int limb, size_t n, void *out, zinc_stream_t stream);

/* Integer-peak microkernel: `iters` rounds of 8 independent
 * register-resident butterflies per thread with limb 0's modulus, grid = blocks x
 * 256 threads; writes a checksum to sink[0] (device uint64).  `variant` is the
 * butterfly the transform kernels run (PAPER.md:308-317 prices a transform in
 * butterflies): 0 lazy Harvey forward (exact Shoup quotient), 1 lazy-free forward
 * (the CKKS forward transforms when every q < 2^58; needs q_0 < 2^58), 2 forward
 * with one conditional subtraction (q up to 2^60), 3 inverse Gentleman-Sande.
 * *butterflies (host) receives the number of butterflies launched. */
zinc_status zinc_int_peak(const zinc_ctx *ctx, int variant, int blocks, int iters, uint64_t *sink,
                          double *butterflies, zinc_stream_t stream);

/* Host-buffer encryption (end-to-end API): the same result as
 * zinc_encrypt_batch / ckks_encrypt_batch (path 0 = Zinc with `key` = cache,
 * path 1 = vanilla with `key` = pk_ntt, both device pointers) but pt and ct are
 * HOST pointers.  The batch is pipelined in chunks of `chunk` messages (0: 256)
 * over two streams the call creates and destroys: H2D of the plaintexts, the
 * kernels, D2H of the ciphertexts, overlapped.  Device staging buffers come from
 * the device's stream-ordered pool and are released before the call returns.
 * Ordering: the first copy waits for the work already queued on `stream` (e.g.
 * the zinc_precompute_cache / zinc_keygen that produced `key`).  Host buffers
 * should be pinned (cudaHostAlloc / torch pin_memory) for full bandwidth.
 * Blocks the calling thread until the last ciphertext has reached the host; on
 * any error both internal streams are drained before returning, so no copy
 * still references the caller's buffers. */
zinc_status zinc_encrypt_batch_host(const zinc_ctx *ctx, int path, const uint64_t *key,
                                    zinc_form form, zinc_pt_kind kind, const void *pt_host,
                                    size_t batch, uint64_t seed, uint64_t msg_base,
                                    uint64_t *ct_host, size_t chunk, zinc_stream_t stream);

/* Kernel tracing.  Ids of the library's kernels: */
enum {
  ZINC_K_ZINC_COEFF = 0, /* Zinc add/inject, COEFF form          */
  ZINC_K_ZINC_NTT = 1,   /* Zinc, NTT form                        */
  ZINC_K_VANILLA = 2,    /* vanilla encryption (both forms)       */
  ZINC_K_KEYGEN = 3,
  ZINC_K_ENCODE = 4,
  ZINC_K_DECRYPT = 5,
  ZINC_K_DECODE = 6,
  ZINC_K_NTT = 7,
  ZINC_K_SAMPLE = 8,
  ZINC_K_INT_PEAK = 9,
  ZINC_K_BFV_SCALE = 10, /* BFV decryption: round(t.x/Q) mod t from the RNS residues */
  ZINC_K_CT_ADD = 11,    /* batched ciphertext addition (Eq. 2) */
  ZINC_K_CT_SUM = 12,    /* aggregation of a batch */
  ZINC_K_LIFT = 13,      /* 128-bit plaintexts -> RNS residues */
  ZINC_K_PT_ADD = 14,    /* c1 += plaintext residues */
  ZINC_K_SHOUP_PREP = 15, /* Shoup companions of pk / sk for the pointwise key products */
  ZINC_K_COUNT = 16
};
/* on != 0: clear the trace and bracket every following kernel launch with CUDA
 * events recorded on the launch's own stream; on == 0: stop recording. */
zinc_status zinc_profile_enable(int on);
/* Wait for the recorded events and return, per kernel id, the summed device
 * time in ms and the launch count (host arrays of ZINC_K_COUNT). */
zinc_status zinc_profile_read(double *ms, uint64_t *launches);
/* Name of kernel id (static string, "?" if out of range). */
const char *zinc_kernel_name(int id);

/* Number of kernel launches this library issued since the last reset (all
 * threads); used by bench.py's gpu_launches claim. */
uint64_t zinc_launch_count(void);
void zinc_launch_count_reset(void);

/* Process-wide tuning knobs (launch geometry only; results never change):
 *  ZINC_TUNE_COEFF_MSGS_PER_CTA   messages per CTA of the COEFF-form Zinc kernel (0, default: 8 when
 *                                 L <= 4, else 2)
 *  ZINC_TUNE_ENCODE_CHUNK_BYTES   bytes of int64 plaintexts encoded per chunk when the input is slots
 *                                 and the path is Zinc COEFF form (default 32 MiB: the chunk stays
 *                                 resident in the 126 MB L2 between the encode and the add/inject)
 *  ZINC_TUNE_PDL                  1 (default): the serial encode -> path chunk pipeline chains its
 *                                 launches with programmatic dependent launch; 0: plain stream order
 *  ZINC_TUNE_L2_PREFETCH          1 (default): in the Zinc COEFF chunk pipeline, each add/inject
 *                                 launch prefetches the next chunk's slots into L2 for its encode
 *  ZINC_TUNE_NTT_CHUNK_MSGS       messages per chunk when slots feed a transform path (Zinc NTT form,
 *                                 vanilla): 0 (default) = 16 waves of the path kernel's CTAs
 *  ZINC_TUNE_SPLIT                transform kernels at N >= 2^14: 1 (default) the faster family per path
 *                                 (S = N / 2^12 CTA clusters of 2^12 words per CTA for Zinc NTT form,
 *                                 vanilla COEFF form and decryption; 2-CTA kernels for vanilla NTT
 *                                 form); 2: S-CTA clusters everywhere; 0: 2-CTA kernels everywhere
 *  ZINC_TUNE_SMALL_ENCODE         real-slot encode of fewer messages than SMs: 0 (default) the throughput
 *                                 kernel (256 threads, radix-16: 15 us per message at N = 2^14, measured
 *                                 fastest), 1 512 threads radix-8 (18 us), 2 1024 threads radix-4 (21 us)
 *  ZINC_TUNE_PT_IN_CT             Zinc COEFF form from slots: stage each encoded plaintext in its own
 *                                 ciphertext's last c2 limb (no scratch; encodes need not wait for the
 *                                 previous add/inject) instead of double-buffered scratch: 2 always,
 *                                 1 (default) for a single chunk and for L <= 4, 0 never
 *  ZINC_TUNE_SMALL_CLUSTER        real slots, at most (SMs / 8) messages: 1 (default) each message's
 *                                 encode runs on an 8-CTA cluster, and Zinc COEFF form fuses the
 *                                 add/inject into the same launch (k_small.cu); 0: the throughput
 *                                 kernels (one CTA per message's encode, then the path kernel)
 *  ZINC_TUNE_M_DEINT             slots feeding an NTT-form transform path at N >= 2^14: 1 (default) the
 *                                 encode writes its scratch plaintexts de-interleaved by the cluster
 *                                 size of the path kernel, so every CTA reads its subsequence
 *                                 x = S i + r contiguously; 0: natural order (strided reads)
 * Sets knob to value (>= 0); *old_value (host, may be NULL) receives the previous value. */
enum { ZINC_TUNE_COEFF_MSGS_PER_CTA = 0, ZINC_TUNE_ENCODE_CHUNK_BYTES = 1, ZINC_TUNE_PDL = 2,
       ZINC_TUNE_L2_PREFETCH = 3, ZINC_TUNE_NTT_CHUNK_MSGS = 4, ZINC_TUNE_SPLIT = 5, ZINC_TUNE_SMALL_ENCODE = 6,
       ZINC_TUNE_PT_IN_CT = 7, ZINC_TUNE_SMALL_CLUSTER = 8, ZINC_TUNE_M_DEINT = 9,
       ZINC_TUNE_COUNT = 10 };
zinc_status zinc_tune(int knob, long long value, long long *old_value);

/* Thread-local message for the last non-OK status of this thread. */
const char *zinc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* ZINC_H */
