// membench.cu — B200 memory-system constants that bound the Stream-K++ kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench tools/membench.cu && ./membench
// Measures (CUDA events, best of 5): coalesced LDG/STG float4 bandwidth and 1-D
// bulk-copy (cp.async.bulk global->shared) bandwidth, for L2-resident (32 MiB) and
// DRAM-resident (2 GiB) buffers, with all SMs and with a single CTA.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e = (x);                                                                 \
    if (e != cudaSuccess) {                                                              \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);    \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)

template <int U>
__global__ void ldg_kernel(const float4* __restrict__ src, size_t n_vec, int reps, float4* sink) {
  float4 acc = make_float4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (int r = 0; r < reps; ++r) {
    for (size_t base = ((size_t)blockIdx.x * blockDim.x + threadIdx.x); base < n_vec; base += stride) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t i = base + (size_t)u * gridDim.x * blockDim.x;
        v[u] = i < n_vec ? __ldcg(src + i) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
      }
    }
  }
  if (acc.x == 12345.f) sink[0] = acc;
}

template <int U>
__global__ void stg_kernel(float4* dst, size_t n_vec, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  const float4 v = make_float4(threadIdx.x, 1, 2, 3);
  for (int r = 0; r < reps; ++r)
    for (size_t base = ((size_t)blockIdx.x * blockDim.x + threadIdx.x); base < n_vec; base += stride) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t i = base + (size_t)u * gridDim.x * blockDim.x;
        if (i < n_vec) dst[i] = v;
      }
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Each CTA streams its contiguous share with `inflight` bulk copies of `chunk` bytes in flight.
__global__ void bulk_kernel(const char* src, size_t bytes_per_cta, uint32_t chunk, uint32_t inflight,
                            int reps) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t bars[16];
  if (threadIdx.x != 0) return;
  for (uint32_t i = 0; i < inflight; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const char* base = src + (size_t)blockIdx.x * bytes_per_cta;
  const size_t n_chunks = bytes_per_cta / chunk;
  uint32_t phase[16] = {0};
  for (int r = 0; r < reps; ++r) {
    for (size_t c = 0; c < n_chunks; ++c) {
      const uint32_t slot = c % inflight;
      if (c >= inflight || r > 0) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile(
              "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
              "selp.u32 %0, 1, 0, p;\n\t}"
              : "=r"(ok)
              : "r"(smem_u32(&bars[slot])), "r"(phase[slot]));
        phase[slot] ^= 1;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[slot])),
                   "r"(chunk)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sm + slot * chunk)),
          "l"(base + c * chunk), "r"(chunk), "r"(smem_u32(&bars[slot]))
          : "memory");
    }
  }
  for (uint32_t i = 0; i < inflight; ++i) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bars[i])), "r"(phase[i]));
  }
}

// Each CTA writes its contiguous share from shared memory with bulk S2G copies of
// `chunk` bytes, `inflight` bulk groups outstanding.
__global__ void bulk_store_kernel(char* dst, size_t bytes_per_cta, uint32_t chunk, uint32_t inflight,
                                  int reps) {
  extern __shared__ __align__(1024) char sm[];
  if (threadIdx.x != 0) return;
  char* base = dst + (size_t)blockIdx.x * bytes_per_cta;
  const size_t n_chunks = bytes_per_cta / chunk;
  for (int r = 0; r < reps; ++r) {
    for (size_t c = 0; c < n_chunks; ++c) {
      const uint32_t slot = c % inflight;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + c * chunk),
                   "r"(smem_u32(sm + slot * chunk)), "r"(chunk)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (inflight == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      else if (inflight == 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename F>
static float best_ms(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int i = 0; i < 6; ++i) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = 2ull << 30, small = 32ull << 20;
  char* buf;
  float4* sink;
  CK(cudaMalloc(&buf, big));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(buf, 1, big));
  printf("SMs %d\n", sms);
  for (size_t sz : {small, big}) {
    const int reps = sz == small ? 20 : 1;
    const size_t nv = sz / 16;
    for (int grid : {sms, 2 * sms, 1}) {
      const int r = grid == 1 ? 1 : reps;
      const size_t n = grid == 1 ? std::min(nv, (size_t)(8 << 20) / 16) : nv;
      float ms = best_ms([&] { ldg_kernel<8><<<grid, 512>>>((const float4*)buf, n, r, sink); });
      printf("ldg  %5s grid %4d: %8.1f GB/s (%.1f GB/s per CTA)\n", sz == small ? "L2" : "DRAM", grid,
             n * 16.0 * r / ms / 1e6, n * 16.0 * r / ms / 1e6 / grid);
      ms = best_ms([&] { stg_kernel<4><<<grid, 512>>>((float4*)buf, n, r); });
      printf("stg  %5s grid %4d: %8.1f GB/s (%.1f GB/s per CTA)\n", sz == small ? "L2" : "DRAM", grid,
             n * 16.0 * r / ms / 1e6, n * 16.0 * r / ms / 1e6 / grid);
    }
  }
  CK(cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (size_t sz : {small, big}) {
    for (uint32_t chunk : {2048u, 8192u, 32768u}) {
      for (uint32_t inflight : {2u, 6u, 12u}) {
        if ((size_t)chunk * inflight > 196608) continue;
        for (int grid : {sms, 1}) {
          const size_t per_cta = grid == 1 ? (size_t)(8 << 20) : (sz / sms) / chunk * chunk;
          const int reps = (sz == small && grid != 1) ? 10 : 1;
          float ms = best_ms([&] {
            bulk_kernel<<<grid, 32, chunk * inflight>>>(buf, per_cta, chunk, inflight, reps);
          });
          printf("bulk %5s chunk %6u inflight %2u grid %4d: %8.1f GB/s (%.1f per CTA)\n",
                 sz == small ? "L2" : "DRAM", chunk, inflight, grid, per_cta * grid * reps / ms / 1e6,
                 per_cta * reps / ms / 1e6);
        }
      }
    }
  }
  CK(cudaFuncSetAttribute(bulk_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (size_t sz : {small, big}) {
    for (uint32_t chunk : {4096u, 16384u, 32768u}) {
      for (uint32_t inflight : {2u, 4u, 8u}) {
        if ((size_t)chunk * inflight > 196608) continue;
        for (int grid : {sms, 1}) {
          const size_t per_cta = grid == 1 ? (size_t)(8 << 20) : (sz / sms) / chunk * chunk;
          const int reps = (sz == small && grid != 1) ? 10 : 1;
          float ms = best_ms([&] {
            bulk_store_kernel<<<grid, 32, chunk * inflight>>>(buf, per_cta, chunk, inflight, reps);
          });
          printf("bulkst %5s chunk %6u inflight %2u grid %4d: %8.1f GB/s (%.1f per CTA)\n",
                 sz == small ? "L2" : "DRAM", chunk, inflight, grid, per_cta * grid * reps / ms / 1e6,
                 per_cta * reps / ms / 1e6);
        }
      }
    }
  }
  for (int grid : {sms, 1}) {
    const size_t n = grid == 1 ? (size_t)(8 << 20) / 16 : small / 16;
    const int r = grid == 1 ? 1 : 20;
    float ms = best_ms([&] { stg_kernel<8><<<grid, 1024>>>((float4*)buf, n, r); });
    printf("stg1024 L2 grid %4d: %8.1f GB/s (%.1f GB/s per CTA)\n", grid, n * 16.0 * r / ms / 1e6,
           n * 16.0 * r / ms / 1e6 / grid);
  }
  CK(cudaGetLastError());
  return 0;
}
