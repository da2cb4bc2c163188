#include <stdint.h>
#include <cuda_runtime.h>
#define DEV __device__ __forceinline__
DEV uint64_t umulhi_approx(uint64_t a, uint64_t b) {
  const uint32_t al = (uint32_t)a, ah = (uint32_t)(a >> 32), bl = (uint32_t)b, bh = (uint32_t)(b >> 32);
  return (uint64_t)ah * bh + __umulhi(al, bh) + __umulhi(ah, bl);
}
// V0: current
DEV void bf0(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wp, uint64_t q, uint64_t two_q) {
  const uint64_t t = w * Y - umulhi_approx(wp, Y) * q;
  Y = X - t + 2 * two_q;
  X = X + t;
}
// V1: PTX with explicit 32-bit pieces
DEV void bf1(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wp, uint64_t q, uint64_t four_q) {
  uint64_t t;
  asm("{\n\t.reg .u32 yl, yh, wl, wh, pl, ph, ql, qh, h1, h2, Ql, Qh, tl, th, ul, uh;\n\t"
      "mov.b64 {yl, yh}, %1;\n\tmov.b64 {wl, wh}, %2;\n\tmov.b64 {pl, ph}, %3;\n\tmov.b64 {ql, qh}, %4;\n\t"
      // Q = ph*yh + hi(pl*yh) + hi(ph*yl)
      "mul.hi.u32 h1, pl, yh;\n\t"
      "mul.hi.u32 h2, ph, yl;\n\t"
      "mad.lo.cc.u32 Ql, ph, yh, h1;\n\t"
      "madc.hi.u32 Qh, ph, yh, 0;\n\t"
      "add.cc.u32 Ql, Ql, h2;\n\t"
      "addc.u32 Qh, Qh, 0;\n\t"
      // wY low: wl*yl (wide) + (wl*yh + wh*yl) << 32
      "mul.lo.u32 tl, wl, yl;\n\t"
      "mul.hi.u32 th, wl, yl;\n\t"
      "mad.lo.u32 th, wl, yh, th;\n\t"
      "mad.lo.u32 th, wh, yl, th;\n\t"
      // Qq low
      "mul.lo.u32 ul, Ql, ql;\n\t"
      "mul.hi.u32 uh, Ql, ql;\n\t"
      "mad.lo.u32 uh, Ql, qh, uh;\n\t"
      "mad.lo.u32 uh, Qh, ql, uh;\n\t"
      "sub.cc.u32 tl, tl, ul;\n\t"
      "subc.u32 th, th, uh;\n\t"
      "mov.b64 %0, {tl, th};\n\t}"
      : "=l"(t) : "l"(Y), "l"(w), "l"(wp), "l"(q));
  Y = X - t + four_q;
  X = X + t;
}
// V2: C with 64-bit mul of wide pieces, letting compiler choose
DEV void bf2(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wp, uint64_t q, uint64_t four_q) {
  const uint32_t yl = (uint32_t)Y, yh = (uint32_t)(Y >> 32);
  const uint32_t pl = (uint32_t)wp, ph = (uint32_t)(wp >> 32);
  const uint64_t Q = (uint64_t)ph * yh + (uint64_t)(__umulhi(pl, yh)) + __umulhi(ph, yl);
  const uint64_t t = w * Y - Q * q;
  Y = X + (four_q - t);
  X = X + t;
}

// V3: Q via mul.wide + 3-input adds; wY and Qq via wide + two 32-bit mads
DEV void bf3(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wp, uint64_t q, uint64_t four_q) {
  uint64_t t;
  asm("{\n\t.reg .u32 yl, yh, wl, wh, pl, ph, ql, qh, h1, h2, Ql, Qh, tl, th, ul, uh;\n\t.reg .u64 Q, T, U;\n\t"
      "mov.b64 {yl, yh}, %1;\n\tmov.b64 {wl, wh}, %2;\n\tmov.b64 {pl, ph}, %3;\n\tmov.b64 {ql, qh}, %4;\n\t"
      "mul.hi.u32 h1, pl, yh;\n\t"
      "mul.hi.u32 h2, ph, yl;\n\t"
      "mul.wide.u32 Q, ph, yh;\n\t"
      "mov.b64 {Ql, Qh}, Q;\n\t"
      "add.cc.u32 Ql, Ql, h1;\n\t"
      "addc.u32 Qh, Qh, 0;\n\t"
      "add.cc.u32 Ql, Ql, h2;\n\t"
      "addc.u32 Qh, Qh, 0;\n\t"
      "mul.wide.u32 T, wl, yl;\n\t"
      "mov.b64 {tl, th}, T;\n\t"
      "mad.lo.u32 th, wl, yh, th;\n\t"
      "mad.lo.u32 th, wh, yl, th;\n\t"
      "mul.wide.u32 U, Ql, ql;\n\t"
      "mov.b64 {ul, uh}, U;\n\t"
      "mad.lo.u32 uh, Ql, qh, uh;\n\t"
      "mad.lo.u32 uh, Qh, ql, uh;\n\t"
      "sub.cc.u32 tl, tl, ul;\n\t"
      "subc.u32 th, th, uh;\n\t"
      "mov.b64 %0, {tl, th};\n\t}"
      : "=l"(t) : "l"(Y), "l"(w), "l"(wp), "l"(q));
  Y = X - t + four_q;
  X = X + t;
}
// V4: C formulation of V3 (32-bit pieces, 64-bit adds of 32-bit values)
DEV void bf4(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wp, uint64_t q, uint64_t four_q) {
  const uint32_t yl = (uint32_t)Y, yh = (uint32_t)(Y >> 32), wl = (uint32_t)w, wh = (uint32_t)(w >> 32);
  const uint32_t pl = (uint32_t)wp, ph = (uint32_t)(wp >> 32), ql = (uint32_t)q, qh = (uint32_t)(q >> 32);
  const uint64_t Q = (uint64_t)ph * yh + ((uint64_t)__umulhi(pl, yh) + __umulhi(ph, yl));
  const uint32_t Ql = (uint32_t)Q, Qh = (uint32_t)(Q >> 32);
  const uint64_t T = (uint64_t)wl * yl + ((uint64_t)(wl * yh + wh * yl) << 32);
  const uint64_t U = (uint64_t)Ql * ql + ((uint64_t)(Ql * qh + Qh * ql) << 32);
  const uint64_t t = T - U;
  Y = X - t + four_q;
  X = X + t;
}

// V5: s = hi(pl yh) + hi(ph yl) first (33 bits), then one wide multiply-add
DEV void bf5(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wp, uint64_t q, uint64_t four_q) {
  const uint32_t yl = (uint32_t)Y, yh = (uint32_t)(Y >> 32), wl = (uint32_t)w, wh = (uint32_t)(w >> 32);
  const uint32_t pl = (uint32_t)wp, ph = (uint32_t)(wp >> 32), ql = (uint32_t)q, qh = (uint32_t)(q >> 32);
  const uint64_t s = (uint64_t)__umulhi(pl, yh) + __umulhi(ph, yl);
  const uint64_t Q = (uint64_t)ph * yh + s;
  const uint32_t Ql = (uint32_t)Q, Qh = (uint32_t)(Q >> 32);
  const uint64_t T = (uint64_t)wl * yl + ((uint64_t)(wl * yh + wh * yl) << 32);
  const uint64_t U = (uint64_t)Ql * ql + ((uint64_t)(Ql * qh + Qh * ql) << 32);
  const uint64_t t = T - U;
  Y = X - t + four_q;
  X = X + t;
}
// V6: PTX: s via add.cc/addc of the two highs, then mad.wide
DEV void bf6(uint64_t &X, uint64_t &Y, uint64_t w, uint64_t wp, uint64_t q, uint64_t four_q) {
  uint64_t t;
  asm("{\n\t.reg .u32 yl, yh, wl, wh, pl, ph, ql, qh, h1, h2, sl, sh, Ql, Qh, tl, th, ul, uh;\n\t.reg .u64 Q, T, U, S;\n\t"
      "mov.b64 {yl, yh}, %1;\n\tmov.b64 {wl, wh}, %2;\n\tmov.b64 {pl, ph}, %3;\n\tmov.b64 {ql, qh}, %4;\n\t"
      "mul.hi.u32 h1, pl, yh;\n\t"
      "mul.hi.u32 h2, ph, yl;\n\t"
      "add.cc.u32 sl, h1, h2;\n\t"
      "addc.u32 sh, 0, 0;\n\t"
      "mov.b64 S, {sl, sh};\n\t"
      "mad.wide.u32 Q, ph, yh, S;\n\t"
      "mov.b64 {Ql, Qh}, Q;\n\t"
      "mul.wide.u32 T, wl, yl;\n\t"
      "mov.b64 {tl, th}, T;\n\t"
      "mad.lo.u32 th, wl, yh, th;\n\t"
      "mad.lo.u32 th, wh, yl, th;\n\t"
      "mul.wide.u32 U, Ql, ql;\n\t"
      "mov.b64 {ul, uh}, U;\n\t"
      "mad.lo.u32 uh, Ql, qh, uh;\n\t"
      "mad.lo.u32 uh, Qh, ql, uh;\n\t"
      "sub.cc.u32 tl, tl, ul;\n\t"
      "subc.u32 th, th, uh;\n\t"
      "mov.b64 %0, {tl, th};\n\t}"
      : "=l"(t) : "l"(Y), "l"(w), "l"(wp), "l"(q));
  Y = X - t + four_q;
  X = X + t;
}
template <int V>
__global__ void __launch_bounds__(256) kreg(uint64_t q, uint64_t w0, uint64_t wp0, int iters, uint64_t *sink) {
  uint64_t v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = (threadIdx.x * 16 + r + blockIdx.x) % q;
  uint64_t w = w0, wp = wp0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (V == 0) bf0(v[r], v[r + 8], w, wp, q, 2 * q);
      else if (V == 3) bf3(v[r], v[r + 8], w, wp, q, 4 * q);
      else bf6(v[r], v[r + 8], w, wp, q, 4 * q);
    }
    w += (v[0] & 1);
  }
  uint64_t acc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc ^= v[r];
  if (acc == 0x1234567890ABCDEFull) sink[0] = acc;
}
template <int V>
__global__ void __launch_bounds__(256) kpeak(const uint64_t *tw, uint64_t q, int iters, uint64_t *sink) {
  uint64_t v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = (threadIdx.x * 16 + r + blockIdx.x) % q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const uint64_t w = tw[2 * (it * 8 + r)], wp = tw[2 * (it * 8 + r) + 1];  // distinct twiddles
      if (V == 0) bf0(v[r], v[r + 8], w, wp, q, 2 * q);
      else if (V == 1) bf1(v[r], v[r + 8], w, wp, q, 4 * q);
      else if (V == 2) bf2(v[r], v[r + 8], w, wp, q, 4 * q);
      else if (V == 3) bf3(v[r], v[r + 8], w, wp, q, 4 * q);
      else if (V == 4) bf4(v[r], v[r + 8], w, wp, q, 4 * q);
      else if (V == 5) bf5(v[r], v[r + 8], w, wp, q, 4 * q);
      else bf6(v[r], v[r + 8], w, wp, q, 4 * q);
    }
  }
  uint64_t acc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc ^= v[r];
  if (acc == 0x1234567890ABCDEFull) sink[0] = acc;
}
template __global__ void kpeak<0>(const uint64_t *, uint64_t, int, uint64_t *);
template __global__ void kpeak<1>(const uint64_t *, uint64_t, int, uint64_t *);
template __global__ void kpeak<2>(const uint64_t *, uint64_t, int, uint64_t *);
template __global__ void kpeak<3>(const uint64_t *, uint64_t, int, uint64_t *);
template __global__ void kpeak<4>(const uint64_t *, uint64_t, int, uint64_t *);
template __global__ void kpeak<5>(const uint64_t *, uint64_t, int, uint64_t *);
template __global__ void kpeak<6>(const uint64_t *, uint64_t, int, uint64_t *);

#include <cstdio>
int main() {
  uint64_t q = (1ull << 54) - 33 * (1ull << 15) + 1;  // any odd 54-bit modulus (throughput only)
  uint64_t w = 123456789012345ull % q;
  unsigned __int128 wpx = ((unsigned __int128)w << 64) / q;
  uint64_t wp = (uint64_t)wpx, *sink;
  cudaMalloc(&sink, 8);
  const int blocks = 148 * 8, iters = 2000;
  for (int rep = 0; rep < 3; ++rep)
  for (int V : {0, 3, 6}) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int k = 0; k < 2; ++k) {
      cudaEventRecord(a);
      if (V == 0) kreg<0><<<blocks, 256>>>(q, w, wp, iters, sink);
      else if (V == 3) kreg<3><<<blocks, 256>>>(q, w, wp, iters, sink);
      else kreg<6><<<blocks, 256>>>(q, w, wp, iters, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bf = (double)blocks * 256 * iters * 8;
    printf("V%d %.3f ms  %.1f G bfly/s\n", V, ms, bf / ms / 1e6);
  }
  return 0;
}
