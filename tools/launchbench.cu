// launchbench.cu — fixed per-launch cost of a persistent 1-CTA/SM kernel on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launchbench tools/launchbench.cu && ./launchbench
// Event-timed (like bench.py) launch of an EMPTY kernel after an L2 flush, varying
// dynamic shared memory (carveout switch vs the flush kernel), TMEM alloc/dealloc,
// cluster dims and PDL; plus back-to-back launches of the same kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e = (x);                                                                 \
    if (e != cudaSuccess) {                                                              \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);    \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)

__global__ void flush_kernel(float4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_float4(0, 0, 0, 0);
}

template <bool TMEM>
__global__ void __launch_bounds__(256, 1) empty_kernel(int* sink) {
  extern __shared__ uint8_t smem[];
  __shared__ uint32_t slot;
  if (TMEM) {
    if (threadIdx.x / 32 == 2) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&slot)),
                   "n"(256)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x / 32 == 2)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "n"(256));
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 100000) sink[0] = smem[0];
}

struct Variant {
  const char* name;
  int smem;
  bool tmem;
  int cluster;
  bool pdl;
};

int main() {
  const size_t flush_vec = (256ull << 20) / 16;
  float4* buf;
  int* sink;
  CK(cudaMalloc(&buf, flush_vec * 16));
  CK(cudaMalloc(&sink, 16));
  CK(cudaFuncSetAttribute(empty_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - 1024));
  CK(cudaFuncSetAttribute(empty_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - 1024));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const Variant vars[] = {
      {"smem 0", 0, false, 1, false},
      {"smem 48K", 48 << 10, false, 1, false},
      {"smem 100K", 100 << 10, false, 1, false},
      {"smem 200K", 200 << 10, false, 1, false},
      {"smem 226K", 226 << 10, false, 1, false},
      {"smem 226K +tmem", 226 << 10, true, 1, false},
      {"smem 226K +tmem +pdl", 226 << 10, true, 1, true},
      {"smem 226K +tmem cluster2", 226 << 10, true, 2, false},
  };
  for (const Variant& v : vars) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = v.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    cfg.attrs = attr;
    cfg.numAttrs = 0;
    if (v.pdl) {
      attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
      ++cfg.numAttrs;
    }
    if (v.cluster > 1) {
      attr[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
      attr[cfg.numAttrs].val.clusterDim.x = v.cluster;
      attr[cfg.numAttrs].val.clusterDim.y = 1;
      attr[cfg.numAttrs].val.clusterDim.z = 1;
      ++cfg.numAttrs;
    }
    auto launch = [&]() {
      return v.tmem ? cudaLaunchKernelEx(&cfg, empty_kernel<true>, sink)
                    : cudaLaunchKernelEx(&cfg, empty_kernel<false>, sink);
    };
    for (int i = 0; i < 5; ++i) CK(launch());
    CK(cudaStreamSynchronize(st));
    // (1) after a flush, one launch between events
    std::vector<float> t;
    for (int i = 0; i < 30; ++i) {
      flush_kernel<<<148 * 8, 256, 0, st>>>(buf, flush_vec);
      CK(cudaEventRecord(e0, st));
      CK(launch());
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    // (2) 200 back-to-back launches
    CK(cudaEventRecord(e0, st));
    for (int i = 0; i < 200; ++i) CK(launch());
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    // (3) empty event pair after a flush (event overhead)
    std::vector<float> te;
    for (int i = 0; i < 30; ++i) {
      flush_kernel<<<148 * 8, 256, 0, st>>>(buf, flush_vec);
      CK(cudaEventRecord(e0, st));
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float m2;
      CK(cudaEventElapsedTime(&m2, e0, e1));
      te.push_back(m2 * 1e3f);
    }
    std::sort(te.begin(), te.end());
    printf("%-28s after-flush median %6.2f us (min %6.2f)  back-to-back %6.2f us/launch  empty-events %5.2f us\n",
           v.name, t[t.size() / 2], t[0], ms * 1e3f / 200, te[te.size() / 2]);
  }
  return 0;
}
