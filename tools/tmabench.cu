// tmabench.cu — per-SM TMA tensor-load throughput vs operations per stage.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmabench tools/tmabench.cu && ./tmabench
// A ring of S stages of 32 KiB; each stage is filled by OPS tensor loads (3-D box
// {64 bf16, 64 rows, 4/OPS chunks}) from an L2-resident 64 MiB tensor; a consumer
// thread releases stages as they land.  Reports GB/s per CTA for 1 and 148 CTAs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(ph));
}

template <int OPS>
__global__ void ring_kernel(const __grid_constant__ CUtensorMap tm, int iters, int stages, int rows) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t full[16];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  constexpr int CH = 4 / OPS;  // chunks per op
  uint32_t phase[16] = {0};
  const int rows_total = rows;
  for (int it = 0; it < iters + stages; ++it) {
    const int s = it % stages;
    if (it >= stages) {
      wait_bar(&full[s], phase[s]);
      phase[s] ^= 1;
    }
    if (it < iters) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(32768)
                   : "memory");
      const int row = ((blockIdx.x * 37 + it) * 64) % rows_total;
      for (int o = 0; o < OPS; ++o) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(sm + s * 32768 + o * (32768 / OPS))),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(row), "r"(((blockIdx.x + it) % 4) * 4 + o * CH),
            "r"(smem_u32(&full[s]))
            : "memory");
      }
    }
  }
}

int main() {
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  // tensor: [chunks=16][rows=4096][64 bf16] (128 B rows) = 8 MiB, x8 copies region = L2 resident
  void* buf;
  cudaMalloc(&buf, 64ull << 20);
  cudaMemset(buf, 0, 64ull << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int row_stride : {128, 1024, 8192, 32768})
  for (int ops : {1, 2, 4}) {
    if (row_stride != 128 && ops != 2) continue;
    CUtensorMap tm;
    const int ch = 4 / ops;
    // rows of 128 B at `row_stride`; 16 "chunks" of 64 columns side by side in a row
    // when row_stride >= 2 KiB, else stacked (contiguous case)
    const int rows = row_stride >= 2048 ? (int)((64ull << 20) / row_stride) : 4096;
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, 16};
    cuuint64_t strides[2] = {(cuuint64_t)row_stride, row_stride >= 2048 ? 128ull : 128ull * 4096};
    cuuint32_t box[3] = {64, 64, (cuuint32_t)ch};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d\n", (int)r);
      return 1;
    }
    for (int stages : {4, 6}) {
      for (int grid : {1, sms}) {
        const int iters = 2000;
        const size_t smem = 32768 * stages;
        void (*k)(CUtensorMap, int, int, int) = ops == 1 ? ring_kernel<1> : ops == 2 ? ring_kernel<2> : ring_kernel<4>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
          cudaEventRecord(a);
          k<<<grid, 32, smem>>>(tm, iters, stages, rows - 64);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep && ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        printf("row_stride %6d ops/stage %d (box %5d B) stages %d grid %3d: %7.1f GB/s per CTA, %8.1f GB/s total  %s\n", ops,
               row_stride, 32768 / ops, stages, grid, 32768.0 * iters / best / 1e6, 32768.0 * iters * grid / best / 1e6,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
