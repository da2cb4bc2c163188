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
// 8 independent register-resident lazy Shoup butterflies per iteration, the
// same instruction mix as the NTT passes, no memory traffic.
__global__ void __launch_bounds__(256) int_peak_kernel(IntPeakArgs a) {
  const uint64_t q = a.q, two_q = 2 * a.q;
  uint64_t v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = (threadIdx.x * 16 + r + blockIdx.x) % q;
  uint64_t w = a.w, wp = a.wp;
  for (int it = 0; it < a.iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) ct_bfly(v[r], v[r + 8], w, wp, q, two_q);
    w += (v[0] & 1);  // keep w loop-variant so the compiler cannot hoist
  }
  uint64_t acc = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc ^= v[r];
  if (acc == 0x1234567890ABCDEFull) a.sink[0] = acc;
}

size_t zinc_coeff_smem(int L, int threads) { return ((size_t)2 * L * 2 * threads + 4 * L) * sizeof(uint64_t); }

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

cudaError_t launch_int_peak(const IntPeakArgs &a, int blocks, cudaStream_t s) {
  int_peak_kernel<<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}


}  // namespace zinc
