// Minimal reproducer for the one racecheck report on the CTA-pair GEMM kernels
// (profiles/round2/racecheck_pair_banded.txt: "Write access at <kernel>+0xfff...fe80 and Read
// access at the tcgen05.alloc.cta_group::2 line").  This kernel does ONLY what the GEMM's
// warp 2 does with TMEM in a 2-CTA cluster: alloc (cta_group::2) into a shared-memory slot,
// relinquish, cluster barrier, read the slot, cluster barrier, dealloc.  No other shared
// memory access exists, so any racecheck hazard here is the sanitizer's view of the 2-CTA
// allocation instruction itself (it writes the TMEM address into both CTAs' slots).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o tools/tmem_alloc_race tools/tmem_alloc_race.cu
//   compute-sanitizer --tool racecheck ./tools/tmem_alloc_race
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) tmem_pair_alloc_kernel(unsigned* out) {
  __shared__ unsigned slot;
  const unsigned warp = threadIdx.x / 32;
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned base = slot;
  if (threadIdx.x == 0) out[blockIdx.x] = base;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(base) : "memory");
  }
}

int main() {
  unsigned* d;
  cudaMalloc(&d, 2 * 148 * sizeof(unsigned));
  tmem_pair_alloc_kernel<<<148, 256>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned h[4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("tmem_pair_alloc_kernel: %s, TMEM base of CTAs 0..3: %u %u %u %u\n", cudaGetErrorString(e), h[0], h[1], h[2], h[3]);
  return e == cudaSuccess ? 0 : 1;
}
