// tmabench.cu — per-SM TMA tensor-load throughput vs bytes per op and ops per stage.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmabench tools/tmabench.cu && ./tmabench
// One thread per CTA keeps a ring of S stages in flight; each stage of STAGE bytes
// is filled by OPS tensor loads of 3-D boxes {64 bf16, 64 rows, chunks} (8 KiB per
// chunk, SWIZZLE_128B) from an L2-resident 64 MiB tensor and released as it lands.
// Reports GB/s per CTA and ns per stage for 1 and 148 CTAs: if the time per stage
// stays flat as STAGE grows, the TMA op (not bytes) is the per-SM limit.
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

__global__ void ring_kernel(const __grid_constant__ CUtensorMap tm, int iters, int stages, int stage_bytes,
                            int ops, int rows) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t full[16];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int op_bytes = stage_bytes / ops;
  const int ch = op_bytes / 8192;  // chunks per op
  uint32_t phase[16] = {0};
  for (int it = 0; it < iters + stages; ++it) {
    const int s = it % stages;
    if (it >= stages) {
      wait_bar(&full[s], phase[s]);
      phase[s] ^= 1;
    }
    if (it < iters) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                   "r"(stage_bytes)
                   : "memory");
      const int row = ((blockIdx.x * 37 + it) * 64) % rows;
      for (int o = 0; o < ops; ++o) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(sm + s * stage_bytes + o * op_bytes)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(row), "r"(o * ch),
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
  // tensor [16 chunks][rows][64 bf16]: rows of 128 B, chunk stride = rows*128 (64 MiB, L2 resident)
  void* buf;
  cudaMalloc(&buf, 64ull << 20);
  cudaMemset(buf, 0, 64ull << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int rows = 32768;  // 16 chunks x 32768 rows x 128 B = 64 MiB
  for (int stage_bytes : {16384, 32768, 65536}) {
    for (int ops : {1, 2, 4}) {
      const int ch = stage_bytes / ops / 8192;
      if (ch < 1) continue;
      CUtensorMap tm;
      cuuint64_t dims[3] = {64, (cuuint64_t)rows, 16};
      cuuint64_t strides[2] = {128, 128ull * rows};
      cuuint32_t box[3] = {64, 64, (cuuint32_t)ch};
      cuuint32_t es[3] = {1, 1, 1};
      CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        return 1;
      }
      for (int stages : {3, 6}) {
        if (stages * stage_bytes > 200 * 1024) continue;
        for (int grid : {1, sms}) {
          const int iters = 3000;
          const size_t smem = (size_t)stage_bytes * stages;
          cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          float best = 1e30f;
          for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(a);
            ring_kernel<<<grid, 32, smem>>>(tm, iters, stages, stage_bytes, ops, rows - 64);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep && ms < best) best = ms;
          }
          cudaError_t e = cudaGetLastError();
          printf("stage %6d B ops %d (op %6d B) stages %d grid %3d: %7.1f GB/s per CTA %8.1f GB/s total  %6.1f ns/stage %s\n",
                 stage_bytes, ops, stage_bytes / ops, stages, grid, (double)stage_bytes * iters / best / 1e6,
                 (double)stage_bytes * iters * grid / best / 1e6, best * 1e6 / iters,
                 e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
      }
    }
  }
  return 0;
}
