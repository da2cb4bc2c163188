// kcommon.cuh -- helpers shared by the kernel translation units of libzinc.so:
// the small-sample samplers (C-4), 16-byte global loads/stores, and the
// cluster-capable launcher.  (Internal; the public ABI is include/zinc.h.)
#pragma once
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.h"
#include "ntt.cuh"

namespace zinc {


// ============================================================ sampling helpers
// Fill int8 smem arrays with the limb-independent small samples of one message
// (C-4: ternary / CBD draws use limb 0 and are reduced into every limb).
template <int THREADS>
ZINC_DEV void sample_ternary_smem(int8_t *dst, int n, uint64_t seed, uint64_t msg, uint32_t tag) {
  for (int blk = threadIdx.x; blk < n / 4; blk += THREADS) {
    uint4 w = stream_block(seed, msg, tag, 0, blk);
    char4 t = make_char4(tern(w.x), tern(w.y), tern(w.z), tern(w.w));
    reinterpret_cast<char4 *>(dst)[blk] = t;
  }
}
// Ternary packed 2 bits per coefficient (t + 1 in {0, 1, 2}): N/4 bytes.
template <int THREADS>
ZINC_DEV void sample_ternary_packed(uint8_t *dst, int n, uint64_t seed, uint64_t msg, uint32_t tag) {
  for (int blk = threadIdx.x; blk < n / 4; blk += THREADS) {
    uint4 w = stream_block(seed, msg, tag, 0, blk);
    dst[blk] = (uint8_t)((tern(w.x) + 1) | ((tern(w.y) + 1) << 2) | ((tern(w.z) + 1) << 4) | ((tern(w.w) + 1) << 6));
  }
}
ZINC_DEV int tern_at(const uint8_t *p, int x) { return (int)((p[x >> 2] >> ((x & 3) * 2)) & 3u) - 1; }
// Parity-split samplers (the even/odd cluster transform): coefficients 2i + r only, stored at i.
template <int THREADS>
ZINC_DEV void sample_cbd_parity(int8_t *dst, int n, uint64_t seed, uint64_t msg, uint32_t tag, int r) {
  for (int blk = threadIdx.x; blk < n / 2; blk += THREADS) {
    const uint4 w = stream_block(seed, msg, tag, 0, blk);  // coefficients 2 blk, 2 blk + 1
    dst[blk] = (int8_t)(r ? cbd_hi(w) : cbd_lo(w));
  }
}
template <int THREADS>
ZINC_DEV void sample_ternary_parity(uint8_t *dst, int n, uint64_t seed, uint64_t msg, uint32_t tag, int r) {
  // block b: coefficients 4b..4b+3; parity r keeps 4b + r (local 2b) and 4b + 2 + r (local 2b + 1)
  for (int blk2 = threadIdx.x; blk2 < n / 8; blk2 += THREADS) {
    uint32_t packed = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint4 w = stream_block(seed, msg, tag, 0, 2 * blk2 + h);
      packed |= (uint32_t)(tern(r ? w.y : w.x) + 1) << (4 * h);  // selects, not a local array
      packed |= (uint32_t)(tern(r ? w.w : w.z) + 1) << (4 * h + 2);
    }
    dst[blk2] = (uint8_t)packed;
  }
}
// The parity samplers for the CTA pair together: both parities are the halves of the same Philox
// blocks, so each CTA draws half of the blocks and hands the partner's samples over distributed
// shared memory (32-bit stores of four CBD samples / sixteen packed ternary samples).  A cluster
// barrier must precede (the partner is running) and follow (its stores have landed).
template <int THREADS>
ZINC_DEV void sample_cbd_parity_pair(int8_t *dst, int n, uint64_t seed, uint64_t msg, uint32_t tag, int r) {
  const uint32_t peer = dsmem_addr(dst, (uint32_t)(r ^ 1));
  const int quarter = n / 4;  // blocks per CTA
  for (int b4 = threadIdx.x; b4 < quarter / 4; b4 += THREADS) {
    const int b0 = r * quarter + 4 * b4;
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 w = stream_block(seed, msg, tag, 0, (uint32_t)(b0 + j));  // coefficients 2 blk, 2 blk + 1
      lo |= ((uint32_t)cbd_lo(w) & 0xFFu) << (8 * j);
      hi |= ((uint32_t)cbd_hi(w) & 0xFFu) << (8 * j);
    }
    *reinterpret_cast<uint32_t *>(dst + b0) = r ? hi : lo;
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(peer + (uint32_t)b0), "r"(r ? lo : hi) : "memory");
  }
}
template <int THREADS>
ZINC_DEV void sample_ternary_parity_pair(uint8_t *dst, int n, uint64_t seed, uint64_t msg, uint32_t tag, int r) {
  // block b: coefficients 4b..4b+3; parity p keeps 4b + p (local 2b) and 4b + 2 + p (local 2b + 1);
  // byte blk2 of a parity's buffer packs blocks 2 blk2, 2 blk2 + 1
  const uint32_t peer = dsmem_addr(dst, (uint32_t)(r ^ 1));
  const int per_cta = n / 16;  // bytes per CTA
  for (int w4 = threadIdx.x; w4 < per_cta / 4; w4 += THREADS) {
    const int byte0 = r * per_cta + 4 * w4;
    uint32_t even = 0, odd = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 w = stream_block(seed, msg, tag, 0, (uint32_t)(2 * (byte0 + j) + h));
        even |= ((uint32_t)(tern(w.x) + 1) | ((uint32_t)(tern(w.z) + 1) << 2)) << (8 * j + 4 * h);
        odd |= ((uint32_t)(tern(w.y) + 1) | ((uint32_t)(tern(w.w) + 1) << 2)) << (8 * j + 4 * h);
      }
    *reinterpret_cast<uint32_t *>(dst + byte0) = r ? odd : even;
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(peer + (uint32_t)byte0), "r"(r ? even : odd) : "memory");
  }
}
template <int THREADS>
ZINC_DEV void sample_cbd_smem(int8_t *dst, int n, uint64_t seed, uint64_t msg, uint32_t tag) {
  for (int blk = threadIdx.x; blk < n / 2; blk += THREADS) {
    uint4 w = stream_block(seed, msg, tag, 0, blk);
    reinterpret_cast<char2 *>(dst)[blk] = make_char2(cbd_lo(w), cbd_hi(w));
  }
}

ZINC_DEV void ld2(const uint64_t *p, uint64_t &a, uint64_t &b) {
  ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(p);
  a = v.x; b = v.y;
}
ZINC_DEV void st2(uint64_t *p, uint64_t a, uint64_t b) {
  *reinterpret_cast<ulonglong2 *>(p) = make_ulonglong2(a, b);
}
// streaming (evict-first) 128-bit store: ciphertexts are written once
ZINC_DEV void st2_cs(uint64_t *p, uint64_t a, uint64_t b) {
  asm volatile("st.global.cs.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
// 256-bit (four-word, 32-byte aligned) forms: sm_100's LDG / STG .256.  A thread that moves four
// consecutive words with two 128-bit accesses touches its 32-byte sector twice; the L1 data pipe
// counts sector accesses.  ZINC_LDST256 = 0 falls back to two 128-bit accesses.
#ifndef ZINC_LDST256
#define ZINC_LDST256 1
#endif
struct U64x4 {
  uint64_t v[4];
};
ZINC_DEV U64x4 ld4_nc(const uint64_t *p) {  // read-only data, no L1 allocation
  U64x4 r;
#if ZINC_LDST256
  asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(r.v[0]), "=l"(r.v[1]), "=l"(r.v[2]), "=l"(r.v[3]) : "l"(p));
#else
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(r.v[0]), "=l"(r.v[1]) : "l"(p));
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(r.v[2]), "=l"(r.v[3]) : "l"(p + 2));
#endif
  return r;
}
ZINC_DEV U64x4 ld4(const uint64_t *p) {  // coherent: words this kernel wrote earlier
  U64x4 r;
#if ZINC_LDST256
  asm volatile("ld.global.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(r.v[0]), "=l"(r.v[1]), "=l"(r.v[2]), "=l"(r.v[3]) : "l"(p) : "memory");
#else
  ld2(p, r.v[0], r.v[1]);
  ld2(p + 2, r.v[2], r.v[3]);
#endif
  return r;
}
ZINC_DEV void st4(uint64_t *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
#if ZINC_LDST256
  asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
#else
  st2(p, a, b);
  st2(p + 2, c, d);
#endif
}
ZINC_DEV void st4_cs(uint64_t *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {  // streaming (evict-first)
#if ZINC_LDST256
  asm volatile("st.global.cs.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
#else
  st2_cs(p, a, b);
  st2_cs(p + 2, c, d);
#endif
}
ZINC_DEV ulonglong2 ld2_nc(const void *p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}

// CKKS plaintext words of a CTA's subsequence x = 2^log_s i + r (i < nl) all below q_min / 2 in
// absolute value (q_min over the CTA's limbs): then every lift of m + e is branch-free
// (lift_small) for every limb, decided once per message instead of per word, limb and transform.
// ms: the CTA's subsequence of m (m_sub).
template <int THREADS>
ZINC_DEV bool plaintext_small_sub(MSub ms, int nl, const LimbConst *limbs, int lo, int hi) {
  if (!ms.p) return true;
  uint64_t qmin = ~0ull;
  for (int i = lo; i < hi; ++i) qmin = min(qmin, limbs[i].q);
  const uint64_t half = qmin >> 1;
  int big = 0;
#pragma unroll 4
  for (int i = threadIdx.x; i < nl; i += THREADS) big |= (uint64_t)ldm(ms.p + i * ms.stride) + half >= qmin;
  return !__syncthreads_or(big);
}

// The three inputs of a vanilla NTT-form limb as one two-phase load (t = 0: m + e1, 1: e2, 2: u),
// so the three transforms run through one copy of the transform code.  Samples sit at x >> SHIFT.
template <bool INTS, int SHIFT>
struct VanTLoad {
  const int64_t *m;
  const int8_t *se1, *se2;
  const uint8_t *su;
  const LimbConst &c;
  int t;
  int ms;  // m is the CTA's subsequence (m_sub): word x sits at m[(x >> SHIFT) ms]
  ZINC_DEV int64_t fetch(int x) const { return (t == 0 && m) ? ldm(m + (x >> SHIFT) * ms) : 0; }
  ZINC_DEV uint64_t lift(int64_t raw, int x) const {
    const int i = x >> SHIFT;
    return t == 0 ? pt_plus_e<INTS>(raw, se1[i], c) : t == 1 ? err_term<INTS>(se2[i], c)
                                                             : reduce_small(tern_at(su, i), c.q);
  }
  bool all_small;  // CTA-uniform (plaintext_small, or t > 0: no plaintext term)
  ZINC_DEV uint64_t operator()(int x) const { return lift(fetch(x), x); }
  // CKKS: |m| < q/2 makes |m + e| < q, and the residue is branch-free (t = 1, 2: raw = 0)
  ZINC_DEV bool uniform_small() const { return !INTS && all_small; }
  ZINC_DEV uint64_t lift_small(int64_t raw, int x) const {
    const int i = x >> SHIFT;
    const int64_t v = raw + (t == 0 ? se1[i] : t == 1 ? se2[i] : tern_at(su, i));
    return (uint64_t)v + (c.q & (uint64_t)(v >> 63));
  }
};

// ============================================================ smem epilogues
// Transform outputs go back into the CTA's own shared-memory buffer (final-pass
// groups are disjoint and each is read before it is written, so this is safe in
// place); after a barrier a streaming epilogue walks the buffer in coalesced
// word pairs.  Decoupling the epilogue's global loads (cache, pk, ct) from the
// butterflies lets U iterations of 16-byte loads be in flight per thread
// instead of exposing one L2 round trip per 16-word group.
template <int LOGN, int LM = 14>
ZINC_DEV auto to_smem(uint64_t *sm) {
  const int loff = local_off<LOGN, LM>();
  return [sm, loff](int base, uint64_t (&v)[16]) {
#pragma unroll
    for (int r = 0; r < 16; ++r) sm[pad16(base - loff + r)] = v[r];
  };
}
// f(xg, v0, v1): words xg, xg + 1 (global, xg even) of this CTA's share.
template <int LOGN, int U = 4, int LM = 14, class F>
ZINC_DEV void stream_pairs(const uint64_t *sm, F f) {
  constexpr int NL = Geo<LOGN, LM>::NL, THREADS = Geo<LOGN, LM>::THREADS;
  static_assert(NL % (2 * THREADS * U) == 0, "epilogue tiling");
  const int loff = local_off<LOGN, LM>();
#pragma unroll 1
  for (int x0 = 2 * threadIdx.x; x0 < NL; x0 += 2 * THREADS * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int x = x0 + u * 2 * THREADS;
      f(x + loff, sm[pad16(x)], sm[pad16(x + 1)]);
    }
  }
}
// Coalesced prologue: the CTA's share of a global limb into the smem buffer.
template <int LOGN, int U = 4, int LM = 14>
ZINC_DEV void load_share(uint64_t *sm, const uint64_t *src) {
  constexpr int NL = Geo<LOGN, LM>::NL, THREADS = Geo<LOGN, LM>::THREADS;
  const int loff = local_off<LOGN, LM>();
#pragma unroll 1
  for (int x0 = 2 * threadIdx.x; x0 < NL; x0 += 2 * THREADS * U) {
    ulonglong2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = *reinterpret_cast<const ulonglong2 *>(src + loff + x0 + u * 2 * THREADS);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int x = x0 + u * 2 * THREADS;
      sm[pad16(x)] = v[u].x;
      sm[pad16(x + 1)] = v[u].y;
    }
  }
}

// ============================================================ TMA bulk copies
// 1-D bulk async copies global -> shared (cp.async.bulk, the non-tensor TMA
// path) completing on an mbarrier transaction count.
ZINC_DEV uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
ZINC_DEV void mbar_init(uint64_t *mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
ZINC_DEV void mbar_expect_tx(uint64_t *mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
}
ZINC_DEV void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mbar)) : "memory");
}
ZINC_DEV void mbar_wait(uint64_t *mbar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(mbar)), "r"(parity) : "memory");
  }
}

// Twiddle-table entries [0, kSmemTw) of one limb, staged into shared memory by
// one TMA bulk copy on a dedicated mbarrier (one phase per staged limb).
struct TwStager {
  uint64_t *mbar;
  uint32_t phase;
  ZINC_DEV void init() {
    if (threadIdx.x == 0) mbar_init(mbar, 1);
    phase = 0;
  }
  // caller: every thread of the CTA has finished reading dst (a barrier precedes)
  ZINC_DEV void issue(Tw *dst, const Tw *src) {
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(mbar, (uint32_t)(kSmemTw * sizeof(Tw)));
      bulk_g2s(dst, src, (uint32_t)(kSmemTw * sizeof(Tw)), mbar);
    }
  }
  // the first `count` entries only (count * 16 bytes)
  ZINC_DEV void issue_n(Tw *dst, const Tw *src, int count) {
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(mbar, (uint32_t)(count * sizeof(Tw)));
      bulk_g2s(dst, src, (uint32_t)(count * sizeof(Tw)), mbar);
    }
  }
  ZINC_DEV void wait() {
    mbar_wait(mbar, phase);
    phase ^= 1u;
  }
};

// ============================================================ launchers
// The dynamic shared-memory opt-in of a kernel, set once per (kernel, device, size): a
// cudaFuncSetAttribute per launch cost ~1 us of host time on every small-batch call.
template <class K>
inline cudaError_t set_smem(K kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;  // below the default limit: no opt-in needed
  static std::mutex mu;
  static std::vector<std::tuple<const void *, int, size_t>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const void *k = reinterpret_cast<const void *>(kernel);
  {
    std::lock_guard<std::mutex> l(mu);
    for (const auto &d : done)
      if (std::get<0>(d) == k && std::get<1>(d) == dev && std::get<2>(d) >= bytes) return cudaSuccess;
  }
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> l(mu);
    done.emplace_back(k, dev, bytes);
  }
  return e;
}

// Programmatic dependent launch (PdlScope in kernels.h): kernels trigger their dependents
// early and wait for their prerequisite grid before touching its outputs.
ZINC_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
ZINC_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// Launch with an optional thread-block cluster along x (2 for the N = 2^15 split).
template <class... KArgs, class... Args>
inline cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, int threads, size_t smem, int cluster,
                             cudaStream_t s, Args... args) {
  cudaError_t e = set_smem(kernel, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (g_launch_pdl) {  // programmatic dependent launch (see PdlScope)
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  e = cudaLaunchKernelEx(&cfg, kernel, args...);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int LOGN, int LM = 14> static size_t ntt_smem_bytes() {
  return SmemWords<Geo<LOGN, LM>::LOGL>::value * sizeof(uint64_t);
}
template <int LOGN, int LM = 14> static dim3 msg_grid(size_t count, int groups = 1) {
  return dim3((unsigned)(count * Geo<LOGN, LM>::CLUSTER), groups);
}

#define ZINC_LOGN_SWITCH(log_n, CALL) \
  switch (log_n) {                    \
    case 12: return CALL(12);         \
    case 13: return CALL(13);         \
    case 14: return CALL(14);         \
    case 15: return CALL(15);         \
  }                                   \
  return cudaErrorInvalidValue;


}  // namespace zinc
