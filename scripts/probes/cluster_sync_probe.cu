// Stress test of cluster rendezvous variants for the split transforms' DSMEM exchanges.
// Each round every CTA writes `round` into all of its smem words, rendezvous, reads one word
// of every peer (checks == round), rendezvous again (WAR), repeat.  Counts mismatches.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 cluster_sync_probe.cu -o probe && ./probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t cta_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t maddr(const void *p, uint32_t rank) {
  uint32_t ra; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank)); return ra;
}
__device__ __forceinline__ uint64_t ldc(uint32_t a) { uint64_t v; asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory"); return v; }

template <int MODE, int S>
__device__ __forceinline__ void rendezvous(uint64_t *mb, uint32_t &k) {
  if (MODE == 0) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    return;
  }
  __syncthreads();
  if (threadIdx.x < S) {
    uint32_t ra = maddr(mb + (k & 1), threadIdx.x);
    if (MODE == 1) asm volatile("mbarrier.arrive.release.cta.shared::cluster.b64 _, [%0];" :: "r"(ra) : "memory");
    else if (MODE == 2) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(ra) : "memory");
    else { asm volatile("fence.acq_rel.cta;" ::: "memory"); asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" :: "r"(ra) : "memory"); }
  }
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mb + (k & 1)), par = (k >> 1) & 1u;
  uint32_t done = 0;
  while (!done) {
    if (MODE == 2)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(a), "r"(par) : "memory");
    else
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(a), "r"(par) : "memory");
  }
  ++k;
}

template <int MODE, int S>
__global__ void __launch_bounds__(256) probe(int rounds, unsigned long long *errs) {
  extern __shared__ uint64_t buf[];  // 4096 words
  __shared__ __align__(8) uint64_t mb[2];
  if (threadIdx.x == 0) {
    for (int j = 0; j < 2; ++j) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(mb + j)), "r"(S));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  uint32_t k = 0;
  const uint32_t r = cta_rank();
  unsigned long long e = 0;
  for (int round = 1; round <= rounds; ++round) {
    for (int i = threadIdx.x; i < 4096; i += 256) buf[i] = ((uint64_t)round << 32) | (r << 16) | i;
    rendezvous<MODE, S>(mb, k);
    for (int i = threadIdx.x; i < 4096; i += 256) {
      const uint32_t c = (i + r) % S;
      const uint64_t v = ldc(maddr(buf + i, c));
      if (v != (((uint64_t)round << 32) | (c << 16) | i)) ++e;
    }
    rendezvous<MODE, S>(mb, k);
  }
  if (e) atomicAdd(errs, e);
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MODE, int S>
void run(const char *name) {
  unsigned long long *d, h = 0;
  cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  cudaFuncSetAttribute(probe<MODE, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 8);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148 * 3 / S * S * 4); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 4096 * 8;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = S; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaError_t err = cudaLaunchKernelEx(&cfg, probe<MODE, S>, 2000, d);
  cudaEventRecord(b);
  cudaError_t e2 = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-40s S=%d launch=%s sync=%s errors=%llu ms=%.2f\n", name, S, cudaGetErrorString(err), cudaGetErrorString(e2), h, ms);
  cudaFree(d);
}

int main() {
  run<0, 4>("barrier.cluster release/acquire");
  run<1, 4>("mbarrier release.cta / acquire.cta");
  run<2, 4>("mbarrier release.cluster / acquire.cluster");
  run<3, 4>("fence.acq_rel.cta + relaxed.cluster");
  run<0, 8>("barrier.cluster release/acquire");
  run<1, 8>("mbarrier release.cta / acquire.cta");
  run<2, 8>("mbarrier release.cluster / acquire.cluster");
  run<3, 8>("fence.acq_rel.cta + relaxed.cluster");
  return 0;
}
