// k_fused.cu -- horizontally fused "encode chunk k+1 | Zinc-add chunk k" kernel.
//
// With slot input the COEFF-form Zinc path is encode (FP64 FFT, latency-bound
// per CTA) followed by the HBM-bound add/inject.  Launched back to back they
// serialise; on two streams the block scheduler still drains the streaming
// kernel's backlog first.  Here ONE grid carries both roles: every P-th CTA
// (P = grid / enc_ctas) encodes one of the next chunk's messages into one half
// of a double-buffered L2-resident int64 scratch, the others stream the current
// chunk's ciphertexts from the other half.  Blocks dispatch roughly in index
// order, so the two roles stay interleaved on every SM for the whole launch
// (FP64 FFT work beside HBM-bound stores); they share nothing inside the launch
// (chunk k's plaintexts were written by the previous launch).
#include "encode_real.cuh"
#include "zinc_coeff.cuh"

namespace zinc {

template <int LC, int LOGM>
__global__ void __launch_bounds__(256, 2) zinc_coeff_encode_kernel(ZincCoeffArgs za, EncodeArgs ea, int enc_ctas,
                                                                   int gx) {
  extern __shared__ __align__(16) uint64_t smem[];
  const int bid = blockIdx.x;
  const int P = enc_ctas > 0 ? max(1, (int)gridDim.x / enc_ctas) : 1 << 30;
  const int e = bid / P;
  if (bid % P == 0 && e < enc_ctas) {
    encode_real_body<LOGM, false>(ea, (size_t)e, reinterpret_cast<double2 *>(smem));
  } else {
    const int z = bid - min(enc_ctas, e + 1);
    zinc_coeff_body<LC>(za, z % gx, z / gx, smem);
  }
}

template <int LC, int LOGM>
static cudaError_t launch_fused_t(const ZincCoeffArgs &za, int gy, const EncodeArgs &ea, int enc_ctas,
                                  cudaStream_t s) {
  const int gx = za.n / 512;
  const size_t smem = std::max(zinc_coeff_smem(za.L, 256), encode_real_smem<LOGM>());
  const unsigned grid = (unsigned)(enc_ctas + gx * gy);
  if (grid == 0) return cudaSuccess;
  return launch_ex(zinc_coeff_encode_kernel<LC, LOGM>, dim3(grid), 256, smem, 1, s, za, ea, enc_ctas, gx);
}

bool fused_supported(int log_n, int L) { return log_n >= 12 && log_n <= 14 && L <= 8; }

cudaError_t launch_zinc_coeff_encode(int log_n, const ZincCoeffArgs &za, int gy, const EncodeArgs &ea, int enc_ctas,
                                     cudaStream_t s) {
  switch (log_n) {
    case 12: return za.L == 3 ? launch_fused_t<3, 11>(za, gy, ea, enc_ctas, s) : launch_fused_t<0, 11>(za, gy, ea, enc_ctas, s);
    case 13: return za.L == 4 ? launch_fused_t<4, 12>(za, gy, ea, enc_ctas, s) : launch_fused_t<0, 12>(za, gy, ea, enc_ctas, s);
    case 14: return za.L == 8 ? launch_fused_t<8, 13>(za, gy, ea, enc_ctas, s) : launch_fused_t<0, 13>(za, gy, ea, enc_ctas, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace zinc
