// api.cu -- the C ABI of libzinc.so (include/zinc.h): validation, parameter
// generation (C-1, C-2, twiddle / FFT tables), and kernel dispatch.
//
// Parameter generation here is written independently of oracle/ (different
// Miller-Rabin base set, table-driven twiddles); tests check both against the
// SURVEY Appendix A values.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/zinc.h"
#include "kernels.h"

using namespace zinc;
typedef unsigned __int128 u128;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};

static zinc_status fail(zinc_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}
#define CUDA_TRY(expr)                                                               \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return fail(ZINC_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));      \
  } while (0)
// ------------------------------------------------------------------ tracing
// When enabled, every launch is bracketed by two CUDA events on its stream.
struct TraceRec { int id; cudaEvent_t a, b; };
static std::mutex g_trace_mu;
static std::atomic<int> g_trace_on{0};
static std::vector<TraceRec> g_trace;
static std::vector<cudaEvent_t> g_event_pool;
static double g_trace_ms[ZINC_K_COUNT];
static uint64_t g_trace_n[ZINC_K_COUNT];
static const char *kKernelNames[ZINC_K_COUNT] = {"zinc_coeff_kernel", "zinc_ntt_kernel", "vanilla_kernel",
                                                 "keygen_kernel", "encode_kernel", "decrypt_kernel",
                                                 "decode_kernel", "ntt_kernel", "sample_kernel", "int_peak_kernel",
                                                 "bfv_scale_kernel", "ct_add_kernel", "ct_sum_kernel",
                                                 "lift_kernel", "pt_add_kernel", "shoup_prep_kernel"};
static cudaEvent_t pool_event() {
  cudaEvent_t e = nullptr;
  if (!g_event_pool.empty()) {
    e = g_event_pool.back();
    g_event_pool.pop_back();
  } else {
    cudaEventCreate(&e);
  }
  return e;
}
struct TraceScope {
  int id;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  TraceScope(int id_, cudaStream_t s_) : id(id_), s(s_) {
    if (g_trace_on.load(std::memory_order_relaxed)) {
      std::lock_guard<std::mutex> l(g_trace_mu);
      a = pool_event();
      cudaEventRecord(a, s);
    }
  }
  ~TraceScope() {
    if (a) {
      std::lock_guard<std::mutex> l(g_trace_mu);
      cudaEvent_t b = pool_event();
      cudaEventRecord(b, s);
      g_trace.push_back({id, a, b});
    }
  }
};
#define LAUNCH(id, stream, expr)                                                     \
  do {                                                                               \
    cudaError_t _e;                                                                  \
    {                                                                                \
      TraceScope _ts((id), (stream));                                                \
      _e = (expr);                                                                   \
    }                                                                                \
    g_launches.fetch_add(1, std::memory_order_relaxed);                              \
    if (_e != cudaSuccess)                                                           \
      return fail(ZINC_ECUDA, "launch %s failed: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

// NVTX range around every ABI call (tracing); a no-op unless a tool
// (nsys / ncu --nvtx) injects the NVTX library.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

// CKKS scales from 2^48 up encode slots into 128-bit coefficients (f3).
static const int kWideLogScale = 48;

// ------------------------------------------------------------------ tuning
static std::atomic<long long> g_tune[ZINC_TUNE_COUNT] = {{0}, {32ll << 20}, {1}, {1}, {0}, {1}, {0}, {1}, {1}, {1}};

// ------------------------------------------------------------------ context
struct zinc_ctx {
  int device, log_n, n, L, log_scale;
  int num_sms = 0;
  size_t encode_wave_msgs[2] = {0, 0};  // messages per full encode wave: real, complex slots
  int scheme = ZINC_SCHEME_CKKS;
  uint64_t t = 0;  // plaintext modulus (BFV, BGV)
  bool wide = false;  // CKKS with log_scale >= 48: slot plaintexts take the 128-bit path
  std::vector<uint64_t> q, psi;
  std::vector<LimbConst> h_limbs;
  LimbConst *d_limbs = nullptr;
  Tw *d_tw = nullptr, *d_itw = nullptr;
  double2 *d_fft_tw = nullptr, *d_twist = nullptr, *d_fft_tw_h = nullptr, *d_fft_tw_hp = nullptr, *d_post_tw = nullptr;
  double2 *d_twist_split = nullptr;
  int *d_perm = nullptr;
  uint64_t qmin = 0;
  // Immutable after zinc_ctx_create: calls only read the context, so calls on
  // different streams (or threads) may overlap.
};

// ------------------------------------------------------------------ number theory (host)
static uint64_t mulm(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((u128)a * b % m); }
static uint64_t powm(uint64_t a, uint64_t e, uint64_t m) {
  uint64_t r = 1;
  a %= m;
  for (; e; e >>= 1, a = mulm(a, a, m))
    if (e & 1) r = mulm(r, a, m);
  return r;
}
// Deterministic Miller-Rabin for 64-bit n (7-base set of Jim Sinclair).
static bool prime64(uint64_t n) {
  if (n < 4) return n >= 2;
  if (n % 2 == 0 || n % 3 == 0) return false;
  uint64_t d = n - 1;
  int s = __builtin_ctzll(d);
  d >>= s;
  static const uint64_t A[7] = {2, 325, 9375, 28178, 450775, 9780504, 1795265022};
  for (uint64_t a : A) {
    uint64_t x = a % n;
    if (x == 0) continue;
    x = powm(x, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s && comp; ++r) {
      x = mulm(x, x, n);
      if (x == n - 1) comp = false;
    }
    if (comp) return false;
  }
  return true;
}
static uint32_t brv(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; ++i, x >>= 1) r = (r << 1) | (x & 1u);
  return r;
}
static uint64_t shoup(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }

// C-1: for each listed size, the largest unused prime < 2^b that is 1 mod 2N.
static bool gen_primes(int log_n, int L, const int *bits, std::vector<uint64_t> &q) {
  const uint64_t step = 2ull << log_n;
  q.assign(L, 0);
  for (int i = 0; i < L; ++i) {
    uint64_t top = 1ull << bits[i];
    for (int j = 0; j < i; ++j)
      if (bits[j] == bits[i]) top = std::min(top, q[j]);
    uint64_t c = ((top - 2) / step) * step + 1;  // largest 1 mod step below top
    while (c >= top) c -= step;
    while (c > step && !prime64(c)) c -= step;
    if (c <= step) return false;
    q[i] = c;
  }
  return true;
}
// C-2: smallest primitive 2N-th root of unity.
static uint64_t gen_psi(uint64_t q, int log_n) {
  const uint64_t n = 1ull << log_n;
  uint64_t g = 0;
  for (uint64_t x = 2; !g; ++x) {
    uint64_t c = powm(x, (q - 1) >> (log_n + 1), q);
    if (powm(c, n, q) == q - 1) g = c;
  }
  uint64_t best = g, g2 = mulm(g, g, q), p = g;
  for (uint64_t k = 0; k < n; ++k, p = mulm(p, g2, q)) best = std::min(best, p);
  return best;
}

template <class T>
static zinc_status upload(T **dst, const std::vector<T> &src) {
  CUDA_TRY(cudaMalloc((void **)dst, src.size() * sizeof(T)));
  CUDA_TRY(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return ZINC_OK;
}

static bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

// Stream-ordered scratch, released (cudaFreeAsync on its stream) on every exit path.
// cudaSetDevice only when the device is not already current (it is on every call of a
// one-GPU process; the runtime call itself costs host time on the small-batch path).
static cudaError_t use_device(int d) {
  int cur = -1;
  if (cudaGetDevice(&cur) == cudaSuccess && cur == d) return cudaSuccess;
  return cudaSetDevice(d);
}

struct ScratchBuf {
  void *p = nullptr;
  cudaStream_t s;
  explicit ScratchBuf(cudaStream_t s_) : s(s_) {}
  ScratchBuf(const ScratchBuf &) = delete;
  ScratchBuf &operator=(const ScratchBuf &) = delete;
  ~ScratchBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
  }
  cudaError_t alloc(size_t bytes) {
    release();
    return cudaMallocAsync(&p, bytes, s);
  }
  template <class T> T *as() const { return static_cast<T *>(p); }
};

extern "C" {

const char *zinc_last_error(void) { return g_err.c_str(); }

const char *zinc_kernel_name(int id) { return (id >= 0 && id < ZINC_K_COUNT) ? kKernelNames[id] : "?"; }

zinc_status zinc_profile_enable(int on) {
  std::lock_guard<std::mutex> l(g_trace_mu);
  if (on) {
    for (auto &r : g_trace) { g_event_pool.push_back(r.a); g_event_pool.push_back(r.b); }
    g_trace.clear();
    for (int i = 0; i < ZINC_K_COUNT; ++i) { g_trace_ms[i] = 0; g_trace_n[i] = 0; }
  }
  g_trace_on.store(on ? 1 : 0);
  return ZINC_OK;
}

zinc_status zinc_profile_read(double *ms, uint64_t *launches) {
  std::lock_guard<std::mutex> l(g_trace_mu);
  for (auto &r : g_trace) {
    float t = 0;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess)
      return fail(ZINC_ECUDA, "trace event query failed");
    g_trace_ms[r.id] += t;
    g_trace_n[r.id] += 1;
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  g_trace.clear();
  for (int i = 0; i < ZINC_K_COUNT; ++i) {
    if (ms) ms[i] = g_trace_ms[i];
    if (launches) launches[i] = g_trace_n[i];
  }
  return ZINC_OK;
}
uint64_t zinc_launch_count(void) { return g_launches.load(); }

zinc_status zinc_tune(int knob, long long value, long long *old_value) {
  if (knob < 0 || knob >= ZINC_TUNE_COUNT) return fail(ZINC_EINVAL, "bad tuning knob %d", knob);
  if (value < 0) return fail(ZINC_EINVAL, "tuning value must be >= 0");
  const long long prev = g_tune[knob].exchange(value);
  if (old_value) *old_value = prev;
  return ZINC_OK;
}
void zinc_launch_count_reset(void) { g_launches.store(0); }

zinc_status zinc_ctx_destroy(zinc_ctx *ctx) {
  if (!ctx) return ZINC_OK;
  cudaSetDevice(ctx->device);
  cudaFree(ctx->d_limbs);
  cudaFree(ctx->d_tw);
  cudaFree(ctx->d_itw);
  cudaFree(ctx->d_fft_tw);
  cudaFree(ctx->d_twist);
  cudaFree(ctx->d_post_tw);
  cudaFree(ctx->d_twist_split);
  cudaFree(ctx->d_fft_tw_h);
  cudaFree(ctx->d_fft_tw_hp);
  cudaFree(ctx->d_perm);
  delete ctx;
  return ZINC_OK;
}

zinc_status zinc_ctx_create(int log_n, int L, const int *limb_bits, int log_scale, int device,
                            zinc_ctx **out) {
  return zinc_ctx_create_scheme(log_n, L, limb_bits, ZINC_SCHEME_CKKS, 0, log_scale, device, out);
}

zinc_status zinc_ctx_create_scheme(int log_n, int L, const int *limb_bits, int scheme, uint64_t plain_modulus,
                                   int log_scale, int device, zinc_ctx **out) {
  if (!out || !limb_bits) return fail(ZINC_EINVAL, "null argument");
  if (scheme != ZINC_SCHEME_CKKS && scheme != ZINC_SCHEME_BFV && scheme != ZINC_SCHEME_BGV)
    return fail(ZINC_EINVAL, "bad scheme %d", scheme);
  if (scheme != ZINC_SCHEME_CKKS && (plain_modulus < 2 || plain_modulus >= (1ull << 32)))
    return fail(ZINC_EINVAL, "plain modulus %llu outside [2, 2^32)", (unsigned long long)plain_modulus);
  *out = nullptr;
  if (log_n < 12 || log_n > 15) return fail(ZINC_EINVAL, "log_n %d outside [12, 15]", log_n);
  if (L < 1 || L > 32) return fail(ZINC_EINVAL, "num_limbs %d outside [1, 32]", L);
  if (scheme != ZINC_SCHEME_CKKS) log_scale = 1;  // unused by BFV / BGV
  if (log_scale < 1 || log_scale > 60) return fail(ZINC_EINVAL, "log_scale %d outside [1, 60]", log_scale);
  for (int i = 0; i < L; ++i)
    if (limb_bits[i] < 20 || limb_bits[i] > 60)
      return fail(ZINC_EINVAL, "limb %d: %d bits outside [20, 60]", i, limb_bits[i]);
  zinc_ctx *c = new zinc_ctx();
  c->device = device;
  c->scheme = scheme;
  c->t = scheme == ZINC_SCHEME_CKKS ? 0 : plain_modulus;
  c->wide = scheme == ZINC_SCHEME_CKKS && log_scale >= kWideLogScale;
  c->log_n = log_n;
  c->n = 1 << log_n;
  c->L = L;
  c->log_scale = log_scale;
  if (!gen_primes(log_n, L, limb_bits, c->q)) { delete c; return fail(ZINC_EPARAMS, "no prime found"); }
  for (int i = 1; i < L; ++i)
    if (c->q[i] > c->q[0]) { delete c; return fail(ZINC_EPARAMS, "limb 0 must hold the largest prime (C-10)"); }
  for (int i = 0; i < L; ++i)
    if (c->t && c->t >= c->q[i]) { delete c; return fail(ZINC_EPARAMS, "plain modulus must be below every q_i"); }
  const int n = c->n;
  std::vector<Tw> tw((size_t)L * n), itw((size_t)L * n);
  c->psi.resize(L);
  c->h_limbs.resize(L);
  for (int i = 0; i < L; ++i) {
    const uint64_t q = c->q[i];
    const uint64_t psi = gen_psi(q, log_n), ipsi = powm(psi, q - 2, q);
    c->psi[i] = psi;
    std::vector<uint64_t> pw(n), ipw(n);
    pw[0] = ipw[0] = 1;
    for (int e = 1; e < n; ++e) { pw[e] = mulm(pw[e - 1], psi, q); ipw[e] = mulm(ipw[e - 1], ipsi, q); }
    for (int k = 0; k < n; ++k) {
      uint64_t w = pw[brv(k, log_n)], iw = ipw[brv(k, log_n)];
      tw[(size_t)i * n + k] = make_ulonglong2(w, shoup(w, q));
      itw[(size_t)i * n + k] = make_ulonglong2(iw, shoup(iw, q));
    }
    LimbConst &lc = c->h_limbs[i];
    memset(&lc, 0, sizeof(lc));
    lc.q = q;
    lc.two_q = 2 * q;
    lc.mu64 = (uint64_t)(((u128)1 << 64) / q);
    lc.b = 64 - __builtin_clzll(q);
    lc.bmu = (uint64_t)(((u128)1 << (2 * lc.b)) / q);
    lc.ninv = powm((uint64_t)n % q, q - 2, q);
    lc.ninv_sh = shoup(lc.ninv, q);
    lc.ninv_w = mulm(lc.ninv, itw[(size_t)i * n + 1].x, q);
    lc.ninv_w_sh = shoup(lc.ninv_w, q);
    lc.r64 = (uint64_t)(((u128)1 << 64) % q);
    lc.r64_sh = shoup(lc.r64, q);
    // reduce_fold: q = 2^b - c; one fold maps x < 2^64 below 2^b + (2^(64-b) - 1) c + (2^b - 1)
    {
      const uint64_t fc = (1ull << lc.b) - q;
      lc.fold_mask = (lc.b >= 64) ? ~0ull : (1ull << lc.b) - 1;
      lc.fold_c = (uint32_t)fc;
      lc.fold_n = 0;
      if (lc.b >= 33 && lc.b <= 63 && fc < (1ull << 32)) {
        const u128 two_q = (u128)2 * q;
        const u128 b1 = (u128)lc.fold_mask + (u128)(~0ull >> lc.b) * fc;  // bound after one fold
        const u128 b2 = (u128)lc.fold_mask + (u128)(b1 >> lc.b) * fc;    // after two
        if (b1 < two_q) lc.fold_n = 1;
        else if ((b1 >> lc.b) < (1ull << 32) && b2 < two_q) lc.fold_n = 2;
      }
      lc.fold_sh = lc.b > 32 ? lc.b - 32 : 0;
      lc.fold_mhi = lc.b > 32 ? (uint32_t)((1ull << (lc.b - 32)) - 1) : 0;
      const u128 qinv = ~(u128)0 / q;  // floor((2^128 - 1) / q) = floor(2^128 / q) for q not a power of 2
      lc.qinv_hi = (uint64_t)(qinv >> 64);
      lc.qinv_lo = (uint64_t)qinv;
    }
    // scheme constants (section 4.2)
    lc.scheme = (uint32_t)scheme;
    if (c->t) {
      const uint64_t t = c->t;
      lc.t = t;
      lc.t_mu = (uint64_t)(((u128)1 << 64) / t);
      // Delta = floor(Q/t) mod q_i = -(Q mod t) t^-1 mod q_i  (Q = Delta t + (Q mod t), q_i | Q)
      uint64_t qmod_t = 1 % t;
      for (int k = 0; k < L; ++k) qmod_t = (uint64_t)((u128)qmod_t * (c->q[k] % t) % t);
      const uint64_t tinv = powm(t, q - 2, q);
      lc.delta = mulm((q - qmod_t % q) % q, tinv, q);
      lc.delta_sh = shoup(lc.delta, q);
      // BFV decryption: t Q~_i / q_i = I_i + F_i with Q~_i = (Q/q_i)^-1 mod q_i
      uint64_t qt = 1;
      for (int k = 0; k < L; ++k)
        if (k != i) qt = mulm(qt, c->q[k] % q, q);
      const uint64_t qtilde = powm(qt, q - 2, q);
      const u128 num = (u128)t * qtilde;
      uint64_t ip = (uint64_t)(num / q);
      const u128 rem = num % q;
      u128 f = ((rem << 64) + q / 2) / q;  // round(F_i 2^64)
      if (f >> 64) { f = 0; ip += 1; }
      lc.dec_i = ip % t;
      lc.dec_f = (uint64_t)f;
    }
  }
  // FFT tables for encode / decode (C-6): M = N/2
  const int M = n / 2, log_m = log_n - 1;
  std::vector<double2> ftw(M / 2), twist(M), ftw_h(M / 4);
  std::vector<int> perm(M);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int e = 0; e < M / 2; ++e) {
    long double ang = -2.0L * pi * (long double)e / (long double)M;
    ftw[e] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  for (int e = 0; e < M / 4; ++e) {  // W_{M/2}^e: the real-slot encode's half-length FFT
    long double ang = -2.0L * pi * (long double)e / (long double)(M / 2);
    ftw_h[e] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  for (int j = 0; j < M; ++j) {
    long double ang = -pi * (long double)j / (long double)n;
    twist[j] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  // complex-slot encode twist zeta^-j = A'[j / 64] B[j % 64], j < M = N/2
  std::vector<double2> twist_split;
  for (int x = 0; x < M / 64; ++x) {
    long double ang = -pi * 64.0L * (long double)x / (long double)n;
    twist_split.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
  }
  for (int x = 0; x < 64; ++x) {
    long double ang = -pi * (long double)x / (long double)n;
    twist_split.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
  }
  // split tables of the real-slot encode's post step: t_j = e^{-i pi j/N} = A[j/64] B[j%64],
  // p_j = e^{-5 i pi j/N} = A5[j/64] B5[j%64], j < N/4
  const int na = (n / 4) / 64;
  std::vector<double2> post_tw;
  for (int k : {1, 5}) {
    for (int x = 0; x < na; ++x) {
      long double ang = -pi * (long double)k * 64.0L * (long double)x / (long double)n;
      post_tw.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
    }
    for (int x = 0; x < 64; ++x) {
      long double ang = -pi * (long double)k * (long double)x / (long double)n;
      post_tw.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
    }
  }
  uint64_t g = 1;
  for (int k = 0; k < M; ++k) {
    perm[k] = (int)brv((uint32_t)((g - 1) / 4), log_m);
    g = g * 5 % (2ull * n);
  }
  // the padded copy the encode kernels stage in shared memory (fft.cuh fft_twpad)
  std::vector<double2> ftw_hp((size_t)fft_twpad_size(M / 4), make_double2(0.0, 0.0));
  for (int e = 0; e < M / 4; ++e) ftw_hp[(size_t)fft_twpad(e)] = ftw_h[e];
  zinc_status st;
  if (cudaSetDevice(device) != cudaSuccess) { delete c; return fail(ZINC_ECUDA, "cudaSetDevice(%d) failed", device); }
  if ((st = upload(&c->d_fft_tw_hp, ftw_hp)) || (st = upload(&c->d_limbs, c->h_limbs)) || (st = upload(&c->d_tw, tw)) || (st = upload(&c->d_itw, itw)) ||
      (st = upload(&c->d_fft_tw, ftw)) || (st = upload(&c->d_twist, twist)) || (st = upload(&c->d_perm, perm)) ||
      (st = upload(&c->d_fft_tw_h, ftw_h)) || (st = upload(&c->d_post_tw, post_tw)) ||
      (st = upload(&c->d_twist_split, twist_split))) {
    zinc_ctx_destroy(c);
    return st;
  }
  c->qmin = *std::min_element(c->q.begin(), c->q.end());
  if (cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    zinc_ctx_destroy(c);
    return fail(ZINC_ECUDA, "device attribute query failed");
  }
  for (int cx = 0; cx < 2; ++cx) c->encode_wave_msgs[cx] = encode_wave_msgs(log_n, cx == 1, c->num_sms);
  cudaGetLastError();  // an occupancy query failure only disables the wave rounding
  // stream-ordered scratch (slot encodes) comes from the default pool: keep it
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = c;
  return ZINC_OK;
}

zinc_status zinc_ctx_moduli(const zinc_ctx *ctx, uint64_t *q_out, uint64_t *psi_out) {
  if (!ctx) return fail(ZINC_EINVAL, "null ctx");
  for (int i = 0; i < ctx->L; ++i) {
    if (q_out) q_out[i] = ctx->q[i];
    if (psi_out) psi_out[i] = ctx->psi[i];
  }
  return ZINC_OK;
}

zinc_status zinc_ctx_scheme(const zinc_ctx *ctx, int *scheme, uint64_t *plain_modulus) {
  if (!ctx) return fail(ZINC_EINVAL, "null ctx");
  if (scheme) *scheme = ctx->scheme;
  if (plain_modulus) *plain_modulus = ctx->t;
  return ZINC_OK;
}

zinc_status zinc_ctx_info(const zinc_ctx *ctx, int *log_n, int *num_limbs, int *log_scale) {
  if (!ctx) return fail(ZINC_EINVAL, "null ctx");
  if (log_n) *log_n = ctx->log_n;
  if (num_limbs) *num_limbs = ctx->L;
  if (log_scale) *log_scale = ctx->log_scale;
  return ZINC_OK;
}

// ------------------------------------------------------------------ helpers
static zinc_status check_ptrs(std::initializer_list<const void *> ps) {
  for (const void *p : ps) {
    if (!p) return fail(ZINC_EINVAL, "null pointer argument");
    if (!aligned16(p)) return fail(ZINC_EINVAL, "pointer %p not 16-byte aligned", p);
  }
  return ZINC_OK;
}
static zinc_status check_form(int form) {
  return (form == ZINC_FORM_NTT || form == ZINC_FORM_COEFF) ? ZINC_OK : fail(ZINC_EINVAL, "bad form %d", form);
}
static zinc_status check_kind(int kind) {
  return (kind >= ZINC_PT_COEFF_I64 && kind <= ZINC_PT_COEFF_I128) ? ZINC_OK : fail(ZINC_EINVAL, "bad kind %d", kind);
}
static size_t pt_stride_bytes(const zinc_ctx *c, int kind) {
  return kind == ZINC_PT_COEFF_I64 ? (size_t)c->n * 8 : kind == ZINC_PT_SLOTS_F64 ? (size_t)c->n / 2 * 8
       : kind == ZINC_PT_COEFF_I128 ? (size_t)c->n * 16 : (size_t)c->n * 8;
}

static EncodeArgs encode_args(const zinc_ctx *c, int kind, const void *slots, int64_t *m) {
  EncodeArgs a{};
  a.slots = (const double *)slots;
  a.complex_slots = kind == ZINC_PT_SLOTS_C128;
  a.perm = c->d_perm;
  a.fft_tw = c->d_fft_tw;
  a.twist = c->d_twist;
  a.fft_tw_h = c->d_fft_tw_h;
  a.fft_tw_hp = c->d_fft_tw_hp;
  a.post_tw = c->d_post_tw;
  a.twist_split = c->d_twist_split;
  a.scale = ldexp(1.0, c->log_scale - (c->log_n - 1));
  a.m_out = m;
  return a;
}

// The small-batch latency path (k_small.cu): real slots, few enough messages that one 8-CTA
// cluster per message still leaves SMs over (knob ZINC_TUNE_SMALL_CLUSTER).
static bool small_cluster(const zinc_ctx *c, int kind, size_t batch) {
  return kind == ZINC_PT_SLOTS_F64 && g_tune[ZINC_TUNE_SMALL_CLUSTER].load() != 0 &&
         batch * (size_t)small_cluster_ctas() <= (size_t)c->num_sms;
}

static zinc_status encode_into(const zinc_ctx *c, int kind, const void *slots, size_t batch, int64_t *m,
                               cudaStream_t s, bool wide = false, size_t m_stride = 0, int wait_mode = 0,
                               int deint_log = 0) {
  EncodeArgs a = encode_args(c, kind, slots, m);
  a.deint_log = deint_log;
  a.wide = wide ? 1 : 0;
  a.m_stride = m_stride ? m_stride : (size_t)c->n * (wide ? 2 : 1);
  a.wait_mode = wait_mode;
  // few messages: a latency variant with more threads per message (knob ZINC_TUNE_SMALL_ENCODE)
  a.fast = batch < (size_t)c->num_sms ? (int)g_tune[ZINC_TUNE_SMALL_ENCODE].load() : 0;
  if (small_cluster(c, kind, batch) && !wide)
    LAUNCH(ZINC_K_ENCODE, s, launch_encode_cluster(c->log_n, a, batch, s));
  else
    LAUNCH(ZINC_K_ENCODE, s, launch_encode(c->log_n, a, batch, s));
  return ZINC_OK;
}

// One encryption path over messages whose int64 plaintexts are at m (or none).
enum Path { PATH_ZINC = 0, PATH_VANILLA = 1 };
// Instantiation of the NTT-path kernels: 0 CKKS with lazy-free forward transforms (all
// q < 2^58, so (3 + 4 log2 N) q < 2^64, see ct_bfly_nr), 1 CKKS with conditional
// subtractions, 2 BFV / BGV.
static int kernel_mode(const zinc_ctx *c) {
  if (c->scheme != ZINC_SCHEME_CKKS) return 2;
  for (uint64_t q : c->q)
    if (q >= (1ull << 58)) return 1;
  return 0;
}
static ZincCoeffArgs zinc_coeff_args(const zinc_ctx *c, const uint64_t *cache, const int64_t *m, size_t batch,
                                     uint64_t seed, uint64_t msg_base, uint64_t *ct) {
  ZincCoeffArgs a{};
  a.limbs = c->d_limbs;
  a.cache = cache;
  a.m = m;
  a.ct = ct;
  a.batch = batch;
  a.seed = seed;
  a.msg_base = msg_base;
  a.n = c->n;
  a.L = c->L;
  a.qmin = c->qmin;
  {
    const uint64_t qmax = *std::max_element(c->q.begin(), c->q.end());
    int bits = 0;
    while (bits < 64 && (qmax >> bits)) ++bits;
    a.wide_hb = std::max(0, std::min(31, 63 - bits));
  }
  a.m_stride = (size_t)c->n;
  // messages per CTA (tuning knob): grid = coefficient tiles x message groups
  // 0 (default): 8 messages per CTA when the cache tile is small (L <= 4: amortises the tile
  // staging over more stores; C2 +7 %), else 2 (measured, profiles/r02_zinc_coeff_sweep.txt)
  const long long mpc = g_tune[ZINC_TUNE_COEFF_MSGS_PER_CTA].load();
  a.msgs_per_cta = (size_t)(mpc > 0 ? mpc : (c->L <= 4 ? 8 : 2));
  return a;
}
// The S-CTA cluster transform kernels (k_split.cu) serve N = 2^14 and 2^15.  Knob 1 (auto):
// the faster kernel family per path as measured on B200 (profiles/r02_sweep_*.jsonl): split
// for Zinc NTT form, vanilla COEFF form and decryption; the 2-CTA parity-split kernel for
// vanilla NTT form.  2: split everywhere; 0: 2-CTA kernels everywhere.
enum SplitUse { SPLIT_ZINC_NTT, SPLIT_VANILLA_NTT, SPLIT_VANILLA_COEFF, SPLIT_DECRYPT };
static bool use_split(const zinc_ctx *c, SplitUse what) {
  const long long k = g_tune[ZINC_TUNE_SPLIT].load();
  if (c->log_n < 14 || k == 0) return false;
  return k == 2 || what != SPLIT_VANILLA_NTT;
}
static int limbs_per_cta(const zinc_ctx *c, size_t batch) {
  size_t want = 2 * (size_t)c->num_sms;
  if (batch >= want) return c->L;
  int groups = (int)std::min<size_t>((size_t)c->L, (want + batch - 1) / batch);
  return (c->L + groups - 1) / groups;
}
// The vanilla NTT form's transform-split small-batch launch (its three transforms on separate
// CTAs, u^ through scratch, then vanilla_combine_kernel): when a handful of messages would leave
// SMs idle.
static bool vanilla_t_split(const zinc_ctx *c, int form, size_t batch) {
  const int lpc = limbs_per_cta(c, batch);
  const int groups = (c->L + lpc - 1) / lpc;
  return c->log_n >= 14 && g_tune[ZINC_TUNE_SPLIT].load() != 0 && form == ZINC_FORM_NTT &&
         batch * (size_t)groups * 3 * ((size_t)c->n >> 12) <= 2 * (size_t)c->num_sms;
}
// uhat_scratch: room for batch x L x N words the caller allocated with its own scratch (one pool
// allocation per call on the small-batch path instead of two); null: allocate here.
static zinc_status run_path(const zinc_ctx *c, int path, const uint64_t *key, int form, const int64_t *m,
                            size_t batch, uint64_t seed, uint64_t msg_base, uint64_t *ct, cudaStream_t s,
                            bool m_is_scratch = false, size_t m_stride = 0, uint64_t *uhat_scratch = nullptr,
                            int m_deint = 0) {
  if (path == PATH_ZINC && form == ZINC_FORM_COEFF) {
    ZincCoeffArgs a = zinc_coeff_args(c, key, m, batch, seed, msg_base, ct);
    a.discard_m = m_is_scratch ? 1 : 0;
    if (m_stride) a.m_stride = m_stride;
    a.prefetch = (const char *)g_l2_prefetch.p;
    a.prefetch_bytes = g_l2_prefetch.bytes & ~(size_t)15;
    int threads = 256;
    while (threads > 32 && zinc_coeff_smem(c->L, threads) > 72 * 1024) threads /= 2;
    const size_t gy = (batch + a.msgs_per_cta - 1) / a.msgs_per_cta;
    // small batches: smaller coefficient tiles, so the grid still covers every SM
    while (threads > 32 && (size_t)(c->n / (2 * threads)) * gy < (size_t)c->num_sms) threads /= 2;
    LAUNCH(ZINC_K_ZINC_COEFF, s, launch_zinc_coeff(a, threads, (int)gy, 0, s));
    return ZINC_OK;
  }
  const int lpc = limbs_per_cta(c, batch);
  const int groups = (c->L + lpc - 1) / lpc;
  if (path == PATH_ZINC) {
    ZincNttArgs a{};
    a.limbs = c->d_limbs;
    a.tw = c->d_tw;
    a.cache = key;
    a.m = m;
    a.ct = ct;
    a.seed = seed;
    a.msg_base = msg_base;
    a.L = c->L;
    a.limbs_per_cta = lpc;
    a.m_deint = m_deint;
    // a handful of messages: the two transforms on separate CTAs as well
    a.t_split = batch * (size_t)groups * 2 * ((size_t)c->n >> 12) <= 2 * (size_t)c->num_sms ? 1 : 0;
    if (use_split(c, SPLIT_ZINC_NTT))
      LAUNCH(ZINC_K_ZINC_NTT, s, launch_zinc_ntt_split(c->log_n, a, kernel_mode(c), batch, groups, s));
    else
      LAUNCH(ZINC_K_ZINC_NTT, s, launch_zinc_ntt(c->log_n, a, kernel_mode(c), batch, groups, s));
    return ZINC_OK;
  }
  VanillaArgs a{};
  a.limbs = c->d_limbs;
  a.tw = c->d_tw;
  a.itw = c->d_itw;
  a.pk = key;
  a.m = m;
  a.ct = ct;
  a.seed = seed;
  a.msg_base = msg_base;
  a.L = c->L;
  a.limbs_per_cta = lpc;
  a.m_deint = m_deint;
  // a handful of messages (NTT form): the three transforms on separate CTAs, then a combine
  const bool t_split = vanilla_t_split(c, form, batch);
  ScratchBuf uhat(s), pk_sh(s);
  if (t_split) {
    if (!uhat_scratch) CUDA_TRY(uhat.alloc(batch * (size_t)c->L * c->n * 8));
    a.u_hat = uhat_scratch ? uhat_scratch : uhat.as<uint64_t>();
  } else {
    // Shoup companions of pk: the per-message pointwise products pk u^ become Shoup products
    // (the transform-split launch's combine kernel uses Barrett products instead)
    const size_t key_words = (size_t)2 * c->L * c->n;
    CUDA_TRY(pk_sh.alloc(key_words * 8));
    LAUNCH(ZINC_K_SHOUP_PREP, s, launch_shoup_prep(c->d_limbs, key, pk_sh.as<uint64_t>(), key_words, c->log_n, c->L, s));
    a.pk_sh = pk_sh.as<uint64_t>();
  }
  if (t_split || use_split(c, form == ZINC_FORM_NTT ? SPLIT_VANILLA_NTT : SPLIT_VANILLA_COEFF))
    LAUNCH(ZINC_K_VANILLA, s, launch_vanilla_split(c->log_n, a, form, kernel_mode(c), batch, groups, s));
  else
    LAUNCH(ZINC_K_VANILLA, s, launch_vanilla(c->log_n, a, form, kernel_mode(c), batch, groups, s));
  if (t_split) LAUNCH(ZINC_K_VANILLA, s, launch_vanilla_combine(a, batch, c->n, s));
  return ZINC_OK;
}

// 128-bit plaintexts (f3: the paper's Delta = 2^55 puts |m_j| past 2^63).  Eq. 4
// taken literally: per chunk, [encode slots to 128-bit coefficients ->] lift them
// to RNS residues (-> NTT in NTT form), run the path with m = 0 and add the
// residues into c1.  Same ciphertext bits as adding m inside the path kernels
// (all arithmetic is exact); costs one more pass over c1.
static zinc_status encrypt_wide(const zinc_ctx *c, int path, const uint64_t *key, int form, int kind, const void *pt,
                                size_t batch, uint64_t seed, uint64_t msg_base, uint64_t *ct, cudaStream_t s) {
  const bool slots = kind != ZINC_PT_COEFF_I128;
  const bool direct = path == PATH_ZINC && form == ZINC_FORM_COEFF;  // kernel reads 128-bit m itself
  const size_t n = c->n, L = c->L;
  const size_t per_msg = (slots ? n * 16 : 0) + (direct ? 0 : L * n * 8);
  // direct (Zinc COEFF from slots): double-buffered chunks of 4x the 64-bit chain's bytes (the
  // wide encode needs a few hundred messages per launch to fill the GPU) chained with
  // programmatic dependent launches, as encrypt_any's chain; otherwise 256 MiB chunks
  const bool chain = direct && slots && g_tune[ZINC_TUNE_PDL].load() != 0;
  const size_t budget = chain ? (size_t)std::max<long long>(per_msg, 4 * g_tune[ZINC_TUNE_ENCODE_CHUNK_BYTES].load())
                              : (size_t)(256ull << 20);
  const size_t chunk = per_msg ? std::max<size_t>(1, std::min(batch, budget / per_msg)) : batch;
  const int nb = chain && batch > chunk ? 2 : 1;
  ScratchBuf m128b(s), resb(s);
  if (slots) CUDA_TRY(m128b.alloc(nb * chunk * n * 16));
  if (!direct) CUDA_TRY(resb.alloc(chunk * L * n * 8));
  int64_t *m128 = m128b.as<int64_t>();
  uint64_t *res = resb.as<uint64_t>();
  const size_t in_stride = pt_stride_bytes(c, kind), ct_stride = 2 * L * n;
  zinc_status st = ZINC_OK;
  size_t k = 0;
  for (size_t off = 0; off < batch && st == ZINC_OK; off += chunk, ++k) {
    const size_t cnt = std::min(chunk, batch - off);
    int64_t *mk = m128 + (k % nb) * chunk * n * 2;
    const int64_t *mw = slots ? mk : (const int64_t *)((const char *)pt + off * in_stride);
    {
      PdlScope pdl_scope(chain && k > 0);
      if (slots && (st = encode_into(c, kind, (const char *)pt + off * in_stride, cnt, mk, s, true))) break;
    }
    PdlScope pdl_scope(chain);
    if (direct) {  // the add/inject kernel reads 128-bit plaintexts itself
      ZincCoeffArgs za = zinc_coeff_args(c, key, nullptr, cnt, seed, msg_base + off, ct + off * ct_stride);
      za.m128 = mw;
      int threads = 256;
      while (threads > 32 && zinc_coeff_smem(c->L, threads) > 72 * 1024) threads /= 2;
      const size_t gy = (cnt + za.msgs_per_cta - 1) / za.msgs_per_cta;
      LAUNCH(ZINC_K_ZINC_COEFF, s, launch_zinc_coeff(za, threads, (int)gy, 0, s));
      continue;
    }
    LiftArgs la{c->d_limbs, mw, res, cnt, (int)n, (int)L};
    LAUNCH(ZINC_K_LIFT, s, launch_lift(la, s));
    if (form == ZINC_FORM_NTT) {
      NttArgs na{};
      na.limbs = c->d_limbs;
      na.tw = c->d_tw;
      na.itw = c->d_itw;
      na.data = res;
      na.L = (int)L;
      LAUNCH(ZINC_K_NTT, s, launch_ntt(c->log_n, na, 0, cnt * L, s));
    }
    if ((st = run_path(c, path, key, form, nullptr, cnt, seed, msg_base + off, ct + off * ct_stride, s))) break;
    PtAddArgs pa{c->d_limbs, res, ct + off * ct_stride, cnt, (int)n, (int)L};
    LAUNCH(ZINC_K_PT_ADD, s, launch_pt_add(pa, s));
  }
  return st;
}

// Encryption with any plaintext kind: int64 plaintexts go straight to the path
// kernel; slots are encoded chunk by chunk into stream-ordered scratch
// (double-buffered) on the caller's stream, and the launches of the chain
// (encode 0, path 0, encode 1, path 1, ...) are programmatic dependent launches:
// each kernel's prologue (TMA staging, sampling, the encode's FFT) overlaps the
// tail of the kernel before it, and only its reads of the previous kernel's
// output (and the encode's scratch stores) wait (griddepcontrol.wait).
//  - Zinc COEFF form (HBM-bound): 32 MiB chunks, so the encoded plaintexts are
//    still in L2 when the add/inject kernel reads them; each add/inject launch
//    also warms the next chunk's slots into L2.
//  - transform paths (Zinc NTT form, vanilla; integer-bound): chunks of whole
//    waves of the path kernel, large enough that its last partial wave is a
//    small fraction of the chunk.
static zinc_status encrypt_any(const zinc_ctx *c, int path, const uint64_t *key, int form, int kind,
                               const void *pt, size_t batch, uint64_t seed, uint64_t msg_base, uint64_t *ct,
                               cudaStream_t s) {
  if (kind == ZINC_PT_COEFF_I64) return run_path(c, path, key, form, (const int64_t *)pt, batch, seed, msg_base, ct, s);
  if (kind == ZINC_PT_COEFF_I128 || c->wide) return encrypt_wide(c, path, key, form, kind, pt, batch, seed, msg_base, ct, s);
  const size_t per_msg = (size_t)c->n * 8;
  const bool coeff_zinc = path == PATH_ZINC && form == ZINC_FORM_COEFF;
  if (coeff_zinc && c->scheme == ZINC_SCHEME_CKKS && small_cluster(c, kind, batch)) {
    // a handful of messages: encode and add/inject in one launch; R cluster replicas per
    // message (each encodes, then streams PP of the 2L ciphertext polynomials) fill the SMs
    const int polys = 2 * c->L;
    int R = (int)std::max<size_t>(1, 2 * (size_t)c->num_sms / (batch * (size_t)small_cluster_ctas()));
    R = std::min(R, polys);
    const int PP = (polys + R - 1) / R;
    R = (polys + PP - 1) / PP;
    const EncodeArgs e = encode_args(c, kind, pt, nullptr);
    const ZincCoeffArgs z = zinc_coeff_args(c, key, nullptr, batch, seed, msg_base, ct);
    LAUNCH(ZINC_K_ZINC_COEFF, s, launch_zinc_coeff_small(c->log_n, e, z, batch, R, PP, s));
    return ZINC_OK;
  }
  size_t chunk;
  if (coeff_zinc) {
    const size_t chunk_bytes = (size_t)std::max<long long>(per_msg, g_tune[ZINC_TUNE_ENCODE_CHUNK_BYTES].load());
    chunk = chunk_bytes / per_msg;
    // whole waves of the encode: its last wave would otherwise run part-empty once per chunk
    // (C4: 128 messages = 1.73 waves of 74 -> 148; C3: 256 of 296 -> 296), within 1.25x the bytes
    const size_t w = c->encode_wave_msgs[kind == ZINC_PT_SLOTS_C128];
    if (w > 0) {
      const size_t r = std::max<size_t>(1, (chunk + w / 2) / w) * w;
      if (r * 4 <= chunk * 5) chunk = r;
    }
  } else {
    const long long knob = g_tune[ZINC_TUNE_NTT_CHUNK_MSGS].load();
    // 16 waves of two message-CTA groups per SM (the transform kernels' residency)
    chunk = knob > 0 ? (size_t)knob : (size_t)16 * 2 * c->num_sms;
  }
  chunk = std::max<size_t>(1, std::min(batch, chunk));
  const bool pdl = g_tune[ZINC_TUNE_PDL].load() != 0;
  const int nb = batch > chunk ? 2 : 1;
  const size_t in_stride = pt_stride_bytes(c, kind);
  const size_t ct_stride = (size_t)2 * c->L * c->n;
  // Zinc COEFF form: each message's encoded plaintext goes into its own ciphertext's last c2
  // limb (N words of the 2 L N it will write).  The add/inject thread that owns coefficients
  // j, j + 1 reads m[j], m[j + 1] there before it overwrites those words, and no other kernel
  // touches the slab in between: no scratch allocation, no buffer reuse between chunks, so an
  // encode's plaintext stores need not wait for the previous add/inject (wait_mode 1), and the
  // overwritten lines are written back once, as ciphertext.
  // Knob 1 (auto) takes it for a single chunk (the small-batch latency path: no scratch
  // allocation, 2.3 us of host time) and at L <= 4 (C2: +1.8 %); measured even at C4 and 0.5 %
  // behind the scratch chain at C3 (profiles/r02b_pt_in_ct_ab.txt).
  const long long pic = g_tune[ZINC_TUNE_PT_IN_CT].load();
  const bool in_ct = coeff_zinc && (pic == 2 || (pic == 1 && (batch <= chunk || c->L <= 4)));
  ScratchBuf mbuf(s);
  // a single-chunk vanilla NTT call on the transform-split path gets its u^ scratch here too
  const bool uh = !coeff_zinc && path == PATH_VANILLA && batch <= chunk && vanilla_t_split(c, form, batch);
  const size_t uh_words = uh ? batch * (size_t)c->L * c->n : 0;
  if (!in_ct) CUDA_TRY(mbuf.alloc(nb * chunk * per_msg + uh_words * 8));
  int64_t *m = mbuf.as<int64_t>();
  uint64_t *uhat_scratch = uh ? reinterpret_cast<uint64_t *>(m + nb * chunk * c->n) : nullptr;
  zinc_status st = ZINC_OK;
  size_t k = 0;
  for (size_t off = 0, cnt = 0; off < batch && st == ZINC_OK; off += cnt, ++k) {
    cnt = std::min(chunk, batch - off);
    int64_t *mb = in_ct ? (int64_t *)(ct + off * ct_stride + (ct_stride - c->n)) : m + (size_t)(k % nb) * chunk * c->n;
    const size_t mstride = in_ct ? ct_stride : (size_t)c->n;
    // NTT-form transform paths at N >= 2^14: the CTAs of a cluster read the subsequences
    // x = S i + r of m (S = 2 for the parity-split vanilla kernel, N / 2^12 for the S-CTA
    // kernels), so the encode writes the scratch de-interleaved by S and every CTA's read is
    // contiguous (whole 32-byte sectors instead of 8 bytes of each)
    int deint = 0;
    if (!coeff_zinc && form == ZINC_FORM_NTT && c->log_n >= 14 && g_tune[ZINC_TUNE_M_DEINT].load() != 0 &&
        !small_cluster(c, kind, cnt)) {
      if (path == PATH_ZINC) deint = use_split(c, SPLIT_ZINC_NTT) ? c->log_n - 12 : 0;
      else deint = (vanilla_t_split(c, form, cnt) || use_split(c, SPLIT_VANILLA_NTT)) ? c->log_n - 12 : 1;
    }
    {
      // the first launch keeps a full dependency on whatever produced the inputs (its
      // loads precede its griddepcontrol.wait); later ones chain on this pipeline's kernels
      PdlScope pdl_scope(pdl && k > 0);
      st = encode_into(c, kind, (const char *)pt + off * in_stride, cnt, mb, s, false, mstride, in_ct ? 1 : 0, deint);
    }
    PdlScope pdl_scope(pdl);
    // the Zinc COEFF kernel of this chunk warms the next chunk's slots into L2 for its encode
    const size_t nxt = std::min(chunk, batch - (off + cnt));
    const bool pf = coeff_zinc && g_tune[ZINC_TUNE_L2_PREFETCH].load() != 0 && nxt > 0 && aligned16(pt) &&
                    in_stride % 16 == 0;
    g_l2_prefetch = pf ? L2Prefetch{(const char *)pt + (off + cnt) * in_stride, nxt * in_stride} : L2Prefetch{};
    if (st == ZINC_OK)
      st = run_path(c, path, key, form, mb, cnt, seed, msg_base + off, ct + off * ct_stride, s, !in_ct, mstride,
                    uhat_scratch, deint);
    g_l2_prefetch = L2Prefetch{};
  }
  return st;
}

static zinc_status check_encrypt(const zinc_ctx *c, const uint64_t *key, int form, int kind, const void *pt,
                                 uint64_t *ct) {
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  zinc_status st;
  if ((st = check_form(form)) || (st = check_kind(kind)) || (st = check_ptrs({key, pt, ct}))) return st;
  if (c->scheme != ZINC_SCHEME_CKKS && kind != ZINC_PT_COEFF_I64)
    return fail(ZINC_EINVAL, "BFV / BGV contexts take integer plaintext coefficients (ZINC_PT_COEFF_I64)");
  if (use_device(c->device) != cudaSuccess) return fail(ZINC_ECUDA, "cudaSetDevice failed");
  return ZINC_OK;
}

// ------------------------------------------------------------------ ABI calls
zinc_status zinc_keygen(const zinc_ctx *c, uint64_t seed, uint64_t *sk_ntt, int8_t *sk_coeff, uint64_t *pk_ntt,
                        zinc_stream_t stream) {
  NvtxRange nr("zinc_keygen");
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  zinc_status st;
  if ((st = check_ptrs({sk_ntt, pk_ntt}))) return st;
  CUDA_TRY(use_device(c->device));
  KeygenArgs a{};
  a.limbs = c->d_limbs;
  a.tw = c->d_tw;
  a.pk = pk_ntt;
  a.sk_ntt = sk_ntt;
  a.sk_coeff = sk_coeff;
  a.seed = seed;
  a.L = c->L;
  LAUNCH(ZINC_K_KEYGEN, (cudaStream_t)stream, launch_keygen(c->log_n, a, (cudaStream_t)stream));
  return ZINC_OK;
}

zinc_status zinc_precompute_cache(const zinc_ctx *c, const uint64_t *pk_ntt, uint64_t seed, zinc_form form,
                                  uint64_t *cache, zinc_stream_t stream) {
  NvtxRange nr("zinc_precompute_cache");
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  zinc_status st;
  if ((st = check_form(form)) || (st = check_ptrs({pk_ntt, cache}))) return st;
  CUDA_TRY(use_device(c->device));
  // C-8: vanilla Enc(0), message index 2^64 - 1
  return run_path(c, PATH_VANILLA, pk_ntt, form, nullptr, 1, seed, UINT64_MAX, cache, (cudaStream_t)stream);
}

zinc_status zinc_encrypt_batch(const zinc_ctx *c, const uint64_t *cache, zinc_form form, zinc_pt_kind kind,
                               const void *pt, size_t batch, uint64_t seed, uint64_t msg_base, uint64_t *ct,
                               zinc_stream_t stream) {
  NvtxRange nr("zinc_encrypt_batch");
  if (batch == 0) return ZINC_OK;
  zinc_status st = check_encrypt(c, cache, form, kind, pt, ct);
  if (st) return st;
  return encrypt_any(c, PATH_ZINC, cache, form, kind, pt, batch, seed, msg_base, ct, (cudaStream_t)stream);
}

zinc_status ckks_encrypt_batch(const zinc_ctx *c, const uint64_t *pk_ntt, zinc_form form, zinc_pt_kind kind,
                               const void *pt, size_t batch, uint64_t seed, uint64_t msg_base, uint64_t *ct,
                               zinc_stream_t stream) {
  NvtxRange nr("ckks_encrypt_batch");
  if (batch == 0) return ZINC_OK;
  zinc_status st = check_encrypt(c, pk_ntt, form, kind, pt, ct);
  if (st) return st;
  return encrypt_any(c, PATH_VANILLA, pk_ntt, form, kind, pt, batch, seed, msg_base, ct, (cudaStream_t)stream);
}

static zinc_status decrypt_impl(const zinc_ctx *c, const uint64_t *sk_ntt, int form, const uint64_t *ct,
                                size_t batch, double *slots_out, int64_t *coeff_out, int64_t *coeff128_out,
                                int32_t *status_out, bool wide, cudaStream_t s);

zinc_status ckks_decrypt_batch(const zinc_ctx *c, const uint64_t *sk_ntt, zinc_form form, const uint64_t *ct,
                               size_t batch, double *slots_out, int64_t *coeff_out, int32_t *status_out,
                               zinc_stream_t stream) {
  NvtxRange nr("ckks_decrypt_batch");
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  if (c->wide && coeff_out)
    return fail(ZINC_EINVAL, "log_scale >= 48: coefficients are 128-bit, use ckks_decrypt_batch_wide");
  return decrypt_impl(c, sk_ntt, form, ct, batch, slots_out, coeff_out, nullptr, status_out, c->wide,
                      (cudaStream_t)stream);
}

zinc_status ckks_decrypt_batch_wide(const zinc_ctx *c, const uint64_t *sk_ntt, zinc_form form, const uint64_t *ct,
                                    size_t batch, double *slots_out, int64_t *coeff128_out, int32_t *status_out,
                                    zinc_stream_t stream) {
  NvtxRange nr("ckks_decrypt_batch_wide");
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  if (c->scheme != ZINC_SCHEME_CKKS) return fail(ZINC_EINVAL, "wide decryption is for CKKS contexts");
  if (c->L < 2) return fail(ZINC_EINVAL, "wide decryption needs at least two limbs");
  return decrypt_impl(c, sk_ntt, form, ct, batch, slots_out, nullptr, coeff128_out, status_out, true,
                      (cudaStream_t)stream);
}

static zinc_status decrypt_impl(const zinc_ctx *c, const uint64_t *sk_ntt, int form, const uint64_t *ct,
                                size_t batch, double *slots_out, int64_t *coeff_out, int64_t *coeff128_out,
                                int32_t *status_out, bool wide, cudaStream_t s) {
  if (batch == 0) return ZINC_OK;
  zinc_status st;
  if ((st = check_form(form)) || (st = check_ptrs({sk_ntt, ct}))) return st;
  for (const void *p : {(const void *)slots_out, (const void *)coeff_out, (const void *)status_out})
    if (p && ((uintptr_t)p & 7u)) return fail(ZINC_EINVAL, "output pointer misaligned");
  if (coeff128_out && ((uintptr_t)coeff128_out & 15u)) return fail(ZINC_EINVAL, "output pointer misaligned");
  if (c->scheme != ZINC_SCHEME_CKKS && slots_out)
    return fail(ZINC_EINVAL, "BFV / BGV decryption has no slot decoding (slots_out must be NULL)");
  CUDA_TRY(use_device(c->device));
  ScratchBuf xb(s), xwb(s), xlb(s), skb(s);
  CUDA_TRY(skb.alloc((size_t)c->L * c->n * 8));
  LAUNCH(ZINC_K_SHOUP_PREP, s, launch_shoup_prep(c->d_limbs, sk_ntt, skb.as<uint64_t>(), (size_t)c->L * c->n, c->log_n, c->L, s));
  if (!coeff_out) CUDA_TRY(xb.alloc(batch * (size_t)c->n * 8));
  if (wide && !coeff128_out) CUDA_TRY(xwb.alloc(batch * (size_t)c->n * 16));
  int64_t *x = coeff_out ? coeff_out : xb.as<int64_t>();
  int64_t *xw = coeff128_out ? coeff128_out : xwb.as<int64_t>();
  DecryptArgs a{};
  a.limbs = c->d_limbs;
  a.tw = c->d_tw;
  a.itw = c->d_itw;
  a.sk_ntt = sk_ntt;
  a.sk_sh = skb.as<uint64_t>();
  a.ct = ct;
  a.coeff_out = x;
  a.status_out = status_out;
  a.L = c->L;
  a.plain_ckks = c->scheme == ZINC_SCHEME_CKKS && !wide;
  if (wide) {
    a.x128_out = xw;
    a.q0inv_q1 = powm(c->q[0] % c->q[1], c->q[1] - 2, c->q[1]);
  }
  if (c->scheme == ZINC_SCHEME_BFV) {
    CUDA_TRY(xlb.alloc(batch * (size_t)c->L * c->n * 8));
    a.xl_out = xlb.as<uint64_t>();
  }
  st = ZINC_OK;
  {
    cudaError_t e;
    {
      TraceScope ts(ZINC_K_DECRYPT, s);
      e = use_split(c, SPLIT_DECRYPT) ? launch_decrypt_split(c->log_n, a, form, kernel_mode(c) == 0, batch, s)
                       : launch_decrypt(c->log_n, a, form, batch, s);
    }
    g_launches.fetch_add(1);
    if (e != cudaSuccess) st = fail(ZINC_ECUDA, "decrypt launch: %s", cudaGetErrorString(e));
  }
  if (st == ZINC_OK && c->scheme == ZINC_SCHEME_BFV) {
    BfvScaleArgs f{};
    f.limbs = c->d_limbs;
    f.xl = xlb.as<uint64_t>();
    f.m_out = x;
    f.batch = batch;
    f.n = c->n;
    f.L = c->L;
    LAUNCH(ZINC_K_BFV_SCALE, s, launch_bfv_scale(f, s));
    if (status_out) CUDA_TRY(cudaMemsetAsync(status_out, 0, batch * sizeof(int32_t), s));
  }
  xlb.release();
  if (st == ZINC_OK && slots_out) {
    DecodeArgs d{};
    d.coeff = wide ? xw : x;
    d.wide = wide ? 1 : 0;
    d.perm = c->d_perm;
    d.fft_tw = c->d_fft_tw;
    d.twist = c->d_twist;
    d.inv_scale = ldexp(1.0, -c->log_scale);
    d.slots_out = slots_out;
    cudaError_t e;
    {
      TraceScope ts(ZINC_K_DECODE, s);
      e = launch_decode(c->log_n, d, batch, s);
    }
    g_launches.fetch_add(1);
    if (e != cudaSuccess) st = fail(ZINC_ECUDA, "decode launch: %s", cudaGetErrorString(e));
  }
  return st;
}

zinc_status zinc_ct_add_batch(const zinc_ctx *c, const uint64_t *x, const uint64_t *y, size_t batch, uint64_t *out,
                              zinc_stream_t stream) {
  NvtxRange nr("zinc_ct_add_batch");
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  if (batch == 0) return ZINC_OK;
  zinc_status st;
  if ((st = check_ptrs({x, y, out}))) return st;
  CUDA_TRY(use_device(c->device));
  CtAddArgs a{};
  a.limbs = c->d_limbs;
  a.a = x;
  a.b = y;
  a.out = out;
  a.words = batch * 2 * (size_t)c->L * c->n;
  a.log_n = c->log_n;
  a.L = c->L;
  LAUNCH(ZINC_K_CT_ADD, (cudaStream_t)stream, launch_ct_add(a, (cudaStream_t)stream));
  return ZINC_OK;
}

zinc_status zinc_ct_sum_batch(const zinc_ctx *c, const uint64_t *ct, size_t batch, uint64_t *out,
                              zinc_stream_t stream) {
  NvtxRange nr("zinc_ct_sum_batch");
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  zinc_status st;
  if ((st = check_ptrs({out})) || (batch && (st = check_ptrs({ct})))) return st;
  CUDA_TRY(use_device(c->device));
  CtSumArgs a{};
  a.limbs = c->d_limbs;
  a.ct = ct;
  a.out = out;
  a.batch = batch;  // batch 0 writes the zero ciphertext
  a.log_n = c->log_n;
  a.L = c->L;
  LAUNCH(ZINC_K_CT_SUM, (cudaStream_t)stream, launch_ct_sum(a, (cudaStream_t)stream));
  return ZINC_OK;
}

zinc_status ckks_encode_batch_wide(const zinc_ctx *c, zinc_pt_kind kind, const void *slots, size_t batch,
                                   int64_t *m_out, zinc_stream_t stream) {
  NvtxRange nr("ckks_encode_batch_wide");
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  if (batch == 0) return ZINC_OK;
  if (kind != ZINC_PT_SLOTS_F64 && kind != ZINC_PT_SLOTS_C128) return fail(ZINC_EINVAL, "encode needs a slot kind");
  zinc_status st;
  if ((st = check_ptrs({slots, m_out}))) return st;
  CUDA_TRY(use_device(c->device));
  return encode_into(c, kind, slots, batch, m_out, (cudaStream_t)stream, true);
}

zinc_status ckks_encode_batch(const zinc_ctx *c, zinc_pt_kind kind, const void *slots, size_t batch, int64_t *m_out,
                              zinc_stream_t stream) {
  NvtxRange nr("ckks_encode_batch");
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  if (batch == 0) return ZINC_OK;
  if (kind != ZINC_PT_SLOTS_F64 && kind != ZINC_PT_SLOTS_C128) return fail(ZINC_EINVAL, "encode needs a slot kind");
  zinc_status st;
  if ((st = check_ptrs({slots, m_out}))) return st;
  CUDA_TRY(use_device(c->device));
  return encode_into(c, kind, slots, batch, m_out, (cudaStream_t)stream);
}

static zinc_status ntt_dir(const zinc_ctx *c, uint64_t *data, size_t count, int inv, zinc_stream_t stream) {
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  if (count == 0) return ZINC_OK;
  zinc_status st;
  if ((st = check_ptrs({data}))) return st;
  CUDA_TRY(use_device(c->device));
  NttArgs a{};
  a.limbs = c->d_limbs;
  a.tw = c->d_tw;
  a.itw = c->d_itw;
  a.data = data;
  a.L = c->L;
  LAUNCH(ZINC_K_NTT, (cudaStream_t)stream, launch_ntt(c->log_n, a, inv, count * c->L, (cudaStream_t)stream));
  return ZINC_OK;
}
zinc_status zinc_ntt_forward(const zinc_ctx *c, uint64_t *data, size_t count, zinc_stream_t stream) {
  NvtxRange nr("zinc_ntt_forward");
  return ntt_dir(c, data, count, 0, stream);
}
zinc_status zinc_ntt_inverse(const zinc_ctx *c, uint64_t *data, size_t count, zinc_stream_t stream) {
  NvtxRange nr("zinc_ntt_inverse");
  return ntt_dir(c, data, count, 1, stream);
}

zinc_status zinc_debug_sample(const zinc_ctx *c, int tag, uint64_t seed, uint64_t msg, int limb, size_t n, void *out,
                              zinc_stream_t stream) {
  NvtxRange nr("zinc_debug_sample");
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  if (tag < 1 || tag > 8) return fail(ZINC_EINVAL, "bad tag %d", tag);
  if (limb < 0 || limb >= c->L) return fail(ZINC_EINVAL, "bad limb %d", limb);
  if (n == 0) return ZINC_OK;
  zinc_status st;
  if ((st = check_ptrs({out}))) return st;
  CUDA_TRY(use_device(c->device));
  SampleArgs a{};
  a.tag = (uint32_t)tag;
  a.limb = (uint32_t)limb;
  a.seed = seed;
  a.msg = msg;
  a.q = c->q[limb];
  a.n = n;
  a.out = out;
  LAUNCH(ZINC_K_SAMPLE, (cudaStream_t)stream, launch_sample(a, (cudaStream_t)stream));
  return ZINC_OK;
}

zinc_status zinc_int_peak(const zinc_ctx *c, int variant, int blocks, int iters, uint64_t *sink,
                          double *butterflies, zinc_stream_t stream) {
  NvtxRange nr("zinc_int_peak");
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  if (blocks < 1 || iters < 1) return fail(ZINC_EINVAL, "blocks and iters must be positive");
  if (variant < 0 || variant > 3) return fail(ZINC_EINVAL, "bad butterfly variant %d", variant);
  if (variant == 1 && c->q[0] >= (1ull << 58)) return fail(ZINC_EINVAL, "lazy-free butterflies need q < 2^58");
  zinc_status st;
  if ((st = check_ptrs({sink}))) return st;
  CUDA_TRY(use_device(c->device));
  IntPeakArgs a{};
  a.q = c->q[0];
  a.w = c->psi[0];
  a.wp = shoup(c->psi[0], c->q[0]);
  a.iters = iters;
  a.sink = sink;
  LAUNCH(ZINC_K_INT_PEAK, (cudaStream_t)stream, launch_int_peak(a, variant, blocks, (cudaStream_t)stream));
  if (butterflies) *butterflies = (double)blocks * 256.0 * 8.0 * (double)iters;
  return ZINC_OK;
}

zinc_status zinc_encrypt_batch_host(const zinc_ctx *c, int path, const uint64_t *key, zinc_form form,
                                    zinc_pt_kind kind, const void *pt_host, size_t batch, uint64_t seed,
                                    uint64_t msg_base, uint64_t *ct_host, size_t chunk, zinc_stream_t stream) {
  NvtxRange nr("zinc_encrypt_batch_host");
  if (!c) return fail(ZINC_EINVAL, "null ctx");
  if (batch == 0) return ZINC_OK;
  if (path != PATH_ZINC && path != PATH_VANILLA) return fail(ZINC_EINVAL, "bad path %d", path);
  zinc_status st;
  if ((st = check_form(form)) || (st = check_kind(kind)) || (st = check_ptrs({key, pt_host, ct_host}))) return st;
  if (c->scheme != ZINC_SCHEME_CKKS && kind != ZINC_PT_COEFF_I64)
    return fail(ZINC_EINVAL, "BFV / BGV contexts take integer plaintext coefficients (ZINC_PT_COEFF_I64)");
  if (chunk == 0) chunk = 256;
  chunk = std::min(chunk, batch);
  CUDA_TRY(use_device(c->device));
  const size_t in_stride = pt_stride_bytes(c, kind);
  const size_t ct_words = (size_t)2 * c->L * c->n;
  // Per-call resources (the context stays immutable): two streams, an event ordering them
  // after the caller's stream, and pool-allocated staging buffers on each stream.
  struct Res {
    cudaStream_t h[2] = {nullptr, nullptr};
    cudaEvent_t ready = nullptr;
    void *pt[2] = {nullptr, nullptr};
    uint64_t *ct[2] = {nullptr, nullptr};
    ~Res() {
      for (int k = 0; k < 2; ++k) {
        if (h[k]) {
          if (pt[k]) cudaFreeAsync(pt[k], h[k]);
          if (ct[k]) cudaFreeAsync(ct[k], h[k]);
          cudaStreamSynchronize(h[k]);
          cudaStreamDestroy(h[k]);
        }
      }
      if (ready) cudaEventDestroy(ready);
    }
  } R;
  CUDA_TRY(cudaEventCreateWithFlags(&R.ready, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(R.ready, (cudaStream_t)stream));
  for (int k = 0; k < 2; ++k) {
    CUDA_TRY(cudaStreamCreateWithFlags(&R.h[k], cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamWaitEvent(R.h[k], R.ready, 0));
    if (cudaMallocAsync(&R.pt[k], chunk * in_stride, R.h[k]) != cudaSuccess ||
        cudaMallocAsync((void **)&R.ct[k], chunk * ct_words * 8, R.h[k]) != cudaSuccess)
      return fail(ZINC_ENOMEM, "host pipeline buffers (%zu messages)", chunk);
  }
  // the two streams alternate chunks: H2D, kernels, D2H
  size_t idx = 0;
  cudaError_t ce = cudaSuccess;
  for (size_t off = 0; off < batch; off += chunk, ++idx) {
    const int k = (int)(idx & 1);
    cudaStream_t s = R.h[k];
    const size_t cnt = std::min(chunk, batch - off);
    ce = cudaMemcpyAsync(R.pt[k], (const char *)pt_host + off * in_stride, cnt * in_stride, cudaMemcpyHostToDevice, s);
    if (ce != cudaSuccess) break;
    if ((st = encrypt_any(c, path, key, form, kind, R.pt[k], cnt, seed, msg_base + off, R.ct[k], s))) break;
    ce = cudaMemcpyAsync(ct_host + off * ct_words, R.ct[k], cnt * ct_words * 8, cudaMemcpyDeviceToHost, s);
    if (ce != cudaSuccess) break;
  }
  for (int k = 0; k < 2; ++k) {
    const cudaError_t e = cudaStreamSynchronize(R.h[k]);
    if (ce == cudaSuccess) ce = e;
  }
  if (st == ZINC_OK && ce != cudaSuccess) st = fail(ZINC_ECUDA, "host pipeline: %s", cudaGetErrorString(ce));
  return st;
}

}  // extern "C"
