// k_pipe.cu -- the slots -> Zinc COEFF-form path as ONE persistent producer /
// consumer kernel (S3 + S4 S5 S8; C-6, C-9; Algorithm 1).
// Opt-in: zinc_tune(ZINC_TUNE_OVERLAP, 3).
//
// Chunked launches (encode chunk k, add/inject chunk k, ...) serialise the
// latency-bound FP64 encode with the HBM-bound stream: every chunk boundary is a
// grid-wide barrier, so the encode time is exposed (~15 % of the C3 step even
// with programmatic dependent launch).  Here every CTA of one co-resident grid
// (cooperative launch: the grid never exceeds what fits on the GPU at once)
// takes one of two roles for the whole batch, assigned per SM so that every SM
// carries the same mix:
//   encoder  (enc_per_sm per SM): claims messages in order (atomic counter),
//            encodes one into a ring of R int64 plaintext slots kept in L2, and
//            publishes it (st.release of the slot's lap count);
//   streamer (the rest, a multiple of the tile count): owns one coefficient tile
//            of 512, staged into shared memory by TMA once; the streamers of a
//            tile claim its message groups in order from a per-tile counter,
//            wait until the group's messages are published, stream their 2L
//            ciphertext rows and return the slot share (red.release).
// An encoder reuses a ring slot only after every tile of the message that
// last occupied it was consumed.  Claims are in message order and R >= mpc,
// so the lowest unfinished message can always progress (no deadlock); every
// wait is additionally bounded by a 2 s timeout that sets a flag instead of
// hanging the device.  Polls are relaxed loads followed by one acquire (an
// acquire per poll invalidates the SM's L1 each time).  Plaintext loads use
// ld.global.cg (L2, coherent within the launch; L1 may hold a ring slot's
// previous lap) and the consumed lines are dropped with discard.global.L2.
// Results are bit-identical to the chunked path (same Philox counters, same
// encode arithmetic; tested).
//
// Measured at C3: on par with the PDL-chained chunks (6.5 ms
// per 16384 messages), not better.  An encoder CTA needs ~20 us per message
// (latency-bound FFT with 8 warps, its loads competing with the saturated HBM),
// so ~70 CTAs must encode at all times, and the streamers that remain, paying a
// flag poll and an exposed plaintext load per group, do not reach the copy rate
// the standalone add/inject kernel reaches.
#include "encode_real.cuh"
#include "zinc_coeff.cuh"

namespace zinc {

namespace {

constexpr int kTile = 512;  // coefficients per work item (2 per thread)

}  // namespace

template <int LC, int LOGM, int MINB, int NPASS>
__global__ void __launch_bounds__(256, MINB) zinc_pipe_kernel(PipeArgs p) {
  extern __shared__ __align__(16) uint64_t smem[];
  __shared__ uint32_t s_claim;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x;
  const ZincCoeffArgs &a = p.z;
  uint32_t *claim = p.sync, *flag = p.sync + 2, *ready = p.sync + 4, *consumed = ready + p.ring;
  uint32_t *tile_next = consumed + p.ring;  // [tiles]: next message group of each coefficient tile
  uint32_t *sm_count = tile_next + p.tiles;  // [256]: CTAs that arrived on each SM
  const uint32_t R = (uint32_t)p.ring;
  const uint32_t batch = (uint32_t)a.batch;

  // Roles by SM, not by block index: the first enc_per_sm CTAs to arrive on an SM encode,
  // the others take streamer indices in arrival order (any beyond p.streamers encode too),
  // so every SM carries the same mix and no coefficient tile's streamers sit on busier SMs.
  __shared__ uint32_t s_role;
  constexpr uint32_t kEncoder = 0xffffffffu;
  if (tid == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    uint32_t role = kEncoder;
    if (atomicAdd(&sm_count[smid & 255u], 1u) >= (uint32_t)p.enc_per_sm) {
      const uint32_t k = atomicAdd(&claim[1], 1u);
      if (k < (uint32_t)p.streamers) role = k;
    }
    s_role = role;
  }
  __syncthreads();
  const uint32_t role = s_role;

  if (role == kEncoder) {
    // ---------------------------------------------------------------- encoder
    double2 *buf = reinterpret_cast<double2 *>(smem);
    for (;;) {
      if (tid == 0) s_claim = atomicAdd(&claim[0], 1u);
      __syncthreads();
      const uint32_t b = s_claim;
      __syncthreads();
      if (b >= batch) break;
      const uint32_t slot = b % R, lap = b / R;
      encode_real_lite_body<LOGM, NPASS>(p.e, b, slot, buf, [&] {
        if (tid == 0 && lap > 0) wait_geq(&consumed[slot], lap * (uint32_t)p.tiles, flag);
        __syncthreads();
      });
      __syncthreads();
      if (tid == 0) st_release(&ready[slot], lap + 1);  // cumulative over the CTA's stores (bar.sync above)
    }
    return;
  }

  // ------------------------------------------------------------------ streamer
  // streamer k owns coefficient tile k % tiles (staged into shared memory once for the
  // whole launch); the G streamers of a tile claim its message groups in order from a
  // per-tile counter (the next claim is in flight while the current group streams)
  constexpr int L = LC;
  static_assert(LC > 0, "pipe kernel needs a compile-time limb count");
  uint64_t *tile = smem;
  uint64_t *sq = tile + (size_t)2 * L * kTile;
  if (tid < L) sq[tid] = a.limbs[tid].q;
  const int tix = (int)(role % (uint32_t)p.tiles), j0 = tix * kTile;
  if (tid == 0) {
    mbar_init(&mbar, 1);
    mbar_expect_tx(&mbar, (uint32_t)(2 * L * kTile * sizeof(uint64_t)));
    for (int r = 0; r < 2 * L; ++r)
      bulk_g2s(tile + (size_t)r * kTile, a.cache + (size_t)r * a.n + j0, kTile * sizeof(uint64_t), &mbar);
    s_claim = atomicAdd(&tile_next[tix], 1u);
  }
  __syncthreads();
  uint32_t grp = s_claim;
  __syncthreads();  // every thread has read the first claim
  mbar_wait(&mbar, 0);
  const size_t lnn = (size_t)L * a.n;
  const uint64_t qmin = a.qmin;
  const uint32_t mpc = (uint32_t)a.msgs_per_cta;
  const int jl = 2 * tid, j = j0 + jl;
  for (;;) {
    const uint32_t b_begin = grp * mpc;
    if (b_begin >= batch) break;
    const uint32_t b_end = min(b_begin + mpc, batch);
    if (tid == 0) {
      const uint32_t nxt = atomicAdd(&tile_next[tix], 1u);  // in flight while polling
      for (uint32_t b = b_begin; b < b_end; ++b) wait_geq(&ready[b % R], b / R + 1, flag);
      s_claim = nxt;
    }
    __syncthreads();
    const uint32_t grp_next = s_claim;  // rewritten only after the barrier that ends this item
    ulonglong2 mv = ld2_cg(a.m + (size_t)(b_begin % R) * a.n + j);
    for (uint32_t b = b_begin; b < b_end; ++b) {
      const uint64_t msg = a.msg_base + b;
      const int64_t m0 = (int64_t)mv.x, m1 = (int64_t)mv.y;
      const int64_t *mrow = a.m + (size_t)(b % R) * a.n + j;
      if (b + 1 < b_end) mv = ld2_cg(a.m + (size_t)((b + 1) % R) * a.n + j);
      const uint4 w1 = stream_block(a.seed, msg, TAG_ZINC_E1, 0, (uint32_t)(j >> 1));
      const uint4 w2 = stream_block(a.seed, msg, TAG_ZINC_E2, 0, (uint32_t)(j >> 1));
      const int e0 = cbd_lo(w1), e1 = cbd_hi(w1), f0 = cbd_lo(w2), f1 = cbd_hi(w2);
      const int64_t v0 = m0 + e0, v1 = m1 + e1;
      const uint64_t a0 = v0 < 0 ? (uint64_t)0 - (uint64_t)v0 : (uint64_t)v0;
      const uint64_t a1 = v1 < 0 ? (uint64_t)0 - (uint64_t)v1 : (uint64_t)v1;
      const bool in_range = (m0 > -(1ll << 62)) && (m0 < (1ll << 62)) && (m1 > -(1ll << 62)) && (m1 < (1ll << 62));
      const bool small = in_range && a0 < qmin && a1 < qmin;
      uint64_t *out = a.ct + (size_t)b * 2 * lnn + j;
      if (__all_sync(0xffffffffu, small)) {
#pragma unroll
        for (int i = 0; i < L; ++i) {
          const uint64_t q = sq[i];
          uint64_t z10, z11, z20, z21;
          ld2(tile + (size_t)i * kTile + jl, z10, z11);
          ld2(tile + (size_t)(L + i) * kTile + jl, z20, z21);
          st2_cs(out + (size_t)i * a.n, mod_add_signed(z10, v0, q), mod_add_signed(z11, v1, q));
          st2_cs(out + lnn + (size_t)i * a.n, mod_add_signed(z20, f0, q), mod_add_signed(z21, f1, q));
        }
      } else {
#pragma unroll 1
        for (int i = 0; i < L; ++i) {
          const LimbConst &c = a.limbs[i];
          const uint64_t q = c.q;
          uint64_t z10, z11, z20, z21;
          ld2(tile + (size_t)i * kTile + jl, z10, z11);
          ld2(tile + (size_t)(L + i) * kTile + jl, z20, z21);
          st2_cs(out + (size_t)i * a.n, add_mod(z10, pt_plus_e(m0, e0, c), q), add_mod(z11, pt_plus_e(m1, e1, c), q));
          st2_cs(out + lnn + (size_t)i * a.n, add_mod(z20, err_term(f0, c), q), add_mod(z21, err_term(f1, c), q));
        }
      }
      // this ring slot's lines are dead once read: drop them without a write-back
      if ((tid & 7) == 0) asm volatile("discard.global.L2 [%0], 128;" ::"l"(mrow) : "memory");
    }
    __syncthreads();  // every thread's plaintext loads of this item have completed
    if (tid == 0)
      for (uint32_t b = b_begin; b < b_end; ++b) red_release_add(&consumed[b % R], 1u);
    grp = grp_next;
  }
}

template <int LC, int LOGM, int MINB, int NPASS>
static cudaError_t launch_pipe_t(const PipeArgs &p, int num_sms, cudaStream_t s) {
  const size_t smem = std::max(encode_real_lite_smem<LOGM>(), (size_t)2 * LC * kTile * 8 + LC * 8);
  cudaError_t e = set_smem(zinc_pipe_kernel<LC, LOGM, MINB, NPASS>, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, zinc_pipe_kernel<LC, LOGM, MINB, NPASS>, 256, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  PipeArgs q = p;
  const int grid = per_sm * num_sms;
  // enc_per_sm encoders on every SM; the streamers are the largest multiple of the tile
  // count that fits in the rest, leaving at least one encoder
  q.enc_per_sm = std::max(0, std::min(p.enc_per_sm, per_sm - 1));
  const int G = std::min(grid - q.enc_per_sm * num_sms, grid - 1) / p.tiles;
  if (G < 1) return cudaErrorInvalidConfiguration;
  q.streamers = G * p.tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (the roles wait on each other)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, zinc_pipe_kernel<LC, LOGM, MINB, NPASS>, q);
  return e != cudaSuccess ? e : cudaGetLastError();
}

bool pipe_supported(int log_n, int L) {
  return (log_n == 12 && L == 3) || (log_n == 13 && L == 4) || (log_n == 14 && L == 8);
}

size_t pipe_sync_words(int ring, int tiles) { return 4 + 2 * (size_t)ring + (size_t)tiles + 256; }

// variant: 0 = 3 CTAs/SM with radix-8 encode passes, 1 = 3 CTAs/SM radix-16, 2 = 2 CTAs/SM radix-16
template <int LC, int LOGM>
static cudaError_t launch_pipe_v(const PipeArgs &p, int variant, int num_sms, cudaStream_t s) {
  switch (variant) {
    case 1: return launch_pipe_t<LC, LOGM, 3, 3>(p, num_sms, s);
    case 2: return launch_pipe_t<LC, LOGM, 2, 3>(p, num_sms, s);
  }
  return launch_pipe_t<LC, LOGM, 3, 4>(p, num_sms, s);
}

cudaError_t launch_zinc_pipe(int log_n, const PipeArgs &p, int variant, int num_sms, cudaStream_t s) {
  switch (log_n) {
    case 12: return p.z.L == 3 ? launch_pipe_v<3, 11>(p, variant, num_sms, s) : cudaErrorInvalidValue;
    case 13: return p.z.L == 4 ? launch_pipe_v<4, 12>(p, variant, num_sms, s) : cudaErrorInvalidValue;
    case 14: return p.z.L == 8 ? launch_pipe_v<8, 13>(p, variant, num_sms, s) : cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}

}  // namespace zinc
