// skpp_gemm.cu — persistent Stream-K++ GEMM for sm_100a (B200).
//
// Replaces the reference's schedule executor (gemmsched executor.py:51-124):
// there every WorkItem runs `c[r0:r1,c0:c1] += a[r0:r1,k0:k1] @ b[k0:k1,c0:c1]`
// on the host in float64, with the `+=` standing for the atomic fixup of
// Algorithm 1.  Here one launch runs a whole schedule:
//
//   grid    = g CTAs (one per SM, co-resident), CTA x == workgroup x;
//   warp 0  = TMA producer: walks x's items (skpp_sched.h) and streams the
//             A (K-major, swizzled) and B (N-major, SW128) k-blocks of each
//             item's [kb, ke) range through an S-stage shared-memory ring;
//   warp 1  = MMA issuer: one thread issues tcgen05.mma kind::f16
//             (M=128, N=BN, K=16) into an fp32 TMEM accumulator, double
//             buffered across items; accumulate is reset at each item's kb;
//   warp 2  = TMEM allocator;
//   warps 4-7 = epilogue: tcgen05.ld rows of the accumulator and, by role,
//             FULL  -> convert and store C,
//             PEER  -> write the fp32 partial to workspace slot x, release flag[x],
//             OWNER -> acquire flags of peers x+1..peer_hi, add their partials
//                      in increasing CTA order (fixed => deterministic), store C.
// Flags are self-cleaning (the owner zeroes each flag it consumed), so the
// kernel is CUDA-graph replay safe without an epoch parameter.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>

#include "../../include/skpp.h"
#include "skpp_sched.h"

namespace skpp {

void set_error(const std::string& msg);  // skpp_host.cpp

constexpr int kBM = 128;
constexpr int kThreads = 256;
constexpr int kEpiWarp0 = 4;
constexpr uint32_t kSmemBudget = 196608;  // operand ring budget (192 KiB)

#ifndef SKPP_WATCHDOG_CYCLES
#define SKPP_WATCHDOG_CYCLES (1ull << 35)  // ~17 s at 1.9 GHz: trap instead of hanging
#endif

// ---------------------------------------------------------------- PTX glue --

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void watchdog(long long start, int where) {
  if (clock64() - start > (long long)SKPP_WATCHDOG_CYCLES) {
    printf("skpp watchdog: CTA %d thread %d stuck at %d\n", blockIdx.x, threadIdx.x, where);
    __trap();
  }
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, int where) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, parity)) watchdog(t0, where);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 consecutive fp32 columns: thread (lane) gets its row's 32 values.
__device__ __forceinline__ void tmem_ld_32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void epi_bar_sync() {
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float4 ld_cg_f4(const float4* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// UMMA shared-memory matrix descriptor (sm_100 format, version 1).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

// ------------------------------------------------------------ kernel config --

template <int BN, int BK>
struct Cfg {
  static constexpr uint32_t A_BYTES = kBM * BK * 2;
  static constexpr uint32_t B_BYTES = BK * BN * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t STAGES_RAW = kSmemBudget / STAGE_BYTES;
  static constexpr uint32_t STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr uint32_t TMEM_COLS = 2 * BN <= 32    ? 32
                                        : 2 * BN <= 64  ? 64
                                        : 2 * BN <= 128 ? 128
                                        : 2 * BN <= 256 ? 256
                                                        : 512;
  static constexpr uint32_t BAR_BYTES = 256;
  static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + BAR_BYTES + 1024;
  // A: K-major, one swizzle atom along K (BK*2 bytes = 32/64/128 B)
  static constexpr uint32_t A_LAYOUT = BK == 64 ? 2u : (BK == 32 ? 4u : 6u);
  static constexpr uint32_t A_SBO = 8 * BK * 2;  // 8 rows of one atom
  // B: N-major SW128, 64-column chunks of BK rows x 128 B
  static constexpr uint32_t B_LAYOUT = 2u;
  static constexpr uint32_t B_LBO = BK * 128;  // next 64-wide N chunk
  static constexpr uint32_t B_SBO = 1024;      // next 8 K-rows
  static_assert(BN % 64 == 0 && BN <= 256, "BN");
  static_assert(BK == 16 || BK == 32 || BK == 64, "BK");
  static_assert(STAGES >= 2, "stages");
};

struct GemmParams {
  Sched s;
  uint32_t M, N;
  uint32_t idesc;
  int32_t out_dtype;
  void* C;
  uint64_t ldc;
  uint32_t c_vec_ok;
  float* ws;
  uint32_t* flags;
  int64_t* trace;
  uint64_t trace_cap;
  int64_t* trace_counts;
};

__device__ __forceinline__ void record_item(const GemmParams& p, uint32_t x, uint64_t idx,
                                            const Item& it) {
  if (p.trace == nullptr || idx >= p.trace_cap) return;
  int64_t* r = p.trace + ((uint64_t)x * p.trace_cap + idx) * SKPP_TRACE_FIELDS;
  r[0] = (int64_t)it.tile;
  r[1] = (int64_t)it.kb;
  r[2] = (int64_t)it.ke;
  r[3] = it.role == ROLE_FULL ? 0 : 1;
  r[4] = (int64_t)it.phase;
  r[5] = (int64_t)it.role;
}

// Convert and store 32 consecutive columns of one output row.
__device__ __forceinline__ void store_row_chunk(const GemmParams& p, uint64_t row, uint64_t col0,
                                                const float* v) {
  if (row >= p.M || col0 >= p.N) return;
  const bool full = p.c_vec_ok && col0 + 32 <= p.N;
  if (p.out_dtype == SKPP_F32) {
    float* c = reinterpret_cast<float*>(p.C) + row * p.ldc + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        reinterpret_cast<float4*>(c)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    } else {
      for (int j = 0; j < 32 && col0 + j < p.N; ++j) c[j] = v[j];
    }
  } else if (p.out_dtype == SKPP_BF16) {
    __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(p.C) + row * p.ldc + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 w;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v[8 * j + 0], v[8 * j + 1]);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(v[8 * j + 2], v[8 * j + 3]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * j + 4], v[8 * j + 5]);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(v[8 * j + 6], v[8 * j + 7]);
        memcpy(&w.x, &h0, 4);
        memcpy(&w.y, &h1, 4);
        memcpy(&w.z, &h2, 4);
        memcpy(&w.w, &h3, 4);
        reinterpret_cast<uint4*>(c)[j] = w;
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < p.N; ++j) c[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    __half* c = reinterpret_cast<__half*>(p.C) + row * p.ldc + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 w;
        __half2 h0 = __floats2half2_rn(v[8 * j + 0], v[8 * j + 1]);
        __half2 h1 = __floats2half2_rn(v[8 * j + 2], v[8 * j + 3]);
        __half2 h2 = __floats2half2_rn(v[8 * j + 4], v[8 * j + 5]);
        __half2 h3 = __floats2half2_rn(v[8 * j + 6], v[8 * j + 7]);
        memcpy(&w.x, &h0, 4);
        memcpy(&w.y, &h1, 4);
        memcpy(&w.z, &h2, 4);
        memcpy(&w.w, &h3, 4);
        reinterpret_cast<uint4*>(c)[j] = w;
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < p.N; ++j) c[j] = __float2half_rn(v[j]);
    }
  }
}

template <int BN, int BK>
__global__ void __launch_bounds__(kThreads, 1)
    streamk_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, const GemmParams p) {
  using C = Cfg<BN, BK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t x = blockIdx.x;
  const Sched& s = p.s;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (uint32_t i = 0; i < C::STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (1 lane)
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      Cursor cur;
      cursor_init(cur, s, x);
      Item it;
      while (cursor_next(cur, s, x, it)) {
        const int32_t m0 = (int32_t)(it.tile / s.n_tiles) * kBM;
        const int32_t n0 = (int32_t)(it.tile % s.n_tiles) * BN;
        for (uint64_t kk = it.kb; kk < it.ke; ++kk) {
          mbar_wait(&empty_bar[stage], phase ^ 1, 1);
          mbar_arrive_expect_tx(&full_bar[stage], C::STAGE_BYTES);
          const int32_t k0 = (int32_t)(kk * BK);
          tma_load_2d(sA + stage * C::A_BYTES, &tmA, k0, m0, &full_bar[stage]);
#pragma unroll
          for (int j = 0; j < BN / 64; ++j)
            tma_load_2d(sB + stage * C::B_BYTES + j * (BK * 128), &tmB, n0 + 64 * j, k0,
                        &full_bar[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (1 lane)
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, local = 0;
      Cursor cur;
      cursor_init(cur, s, x);
      Item it;
      while (cursor_next(cur, s, x, it)) {
        const uint32_t as = local & 1, aph = (local >> 1) & 1;
        mbar_wait(&tempty_bar[as], aph ^ 1, 2);
        tc_fence_after();
        const uint32_t dtm = tmem_base + as * BN;
        for (uint64_t kk = it.kb; kk < it.ke; ++kk) {
          mbar_wait(&full_bar[stage], phase, 3);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = umma_desc(a_addr + k * 32, 0, C::A_SBO, C::A_LAYOUT);
            const uint64_t bd = umma_desc(b_addr + k * 2048, C::B_LBO, C::B_SBO, C::B_LAYOUT);
            umma_f16(dtm, ad, bd, p.idesc, (kk > it.kb || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull_bar[as]);
        ++local;
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------ epilogue (4 warps)
    const uint32_t ew = warp - kEpiWarp0;  // TMEM lane quarter of this warp
    const uint32_t row = ew * 32 + lane;    // tile row owned by this thread
    const bool leader = (row == 0);
    uint32_t local = 0;
    Cursor cur;
    cursor_init(cur, s, x);
    Item it;
    while (cursor_next(cur, s, x, it)) {
      const uint32_t as = local & 1, aph = (local >> 1) & 1;
      if (leader) record_item(p, x, local, it);
      mbar_wait(&tfull_bar[as], aph, 4);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((ew * 32) << 16) + as * BN;
      const uint64_t grow = (it.tile / s.n_tiles) * kBM + row;
      const uint64_t gcol = (it.tile % s.n_tiles) * BN;
      float v[32];
      if (it.role == ROLE_PEER) {
        float4* slot = reinterpret_cast<float4*>(p.ws + (uint64_t)x * kBM * BN);
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          tmem_ld_32(taddr + c * 32, v);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            slot[(c * 8 + j) * kBM + row] =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[as]);
        __threadfence();
        epi_bar_sync();
        if (leader) st_release_gpu(p.flags + x, 1u);
      } else {
        if (it.role == ROLE_OWNER) {
          if (leader) {
            for (uint64_t q = x + 1; q <= it.peer_hi; ++q) {
              if (ld_acquire_gpu(p.flags + q) != 1u) {
                const long long t0 = clock64();
                while (ld_acquire_gpu(p.flags + q) != 1u) {
                  __nanosleep(64);
                  watchdog(t0, 5);
                }
              }
              p.flags[q] = 0u;  // consumed: self-cleaning for the next launch
            }
          }
          epi_bar_sync();
        }
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          tmem_ld_32(taddr + c * 32, v);
          if (it.role == ROLE_OWNER) {
            for (uint64_t q = x + 1; q <= it.peer_hi; ++q) {
              const float4* src = reinterpret_cast<const float4*>(p.ws + q * kBM * BN);
              float4 t[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) t[j] = ld_cg_f4(src + (c * 8 + j) * kBM + row);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                v[4 * j] += t[j].x;
                v[4 * j + 1] += t[j].y;
                v[4 * j + 2] += t[j].z;
                v[4 * j + 3] += t[j].w;
              }
            }
          }
          store_row_chunk(p, grow, gcol + c * 32, v);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[as]);
      }
      ++local;
    }
    if (leader && p.trace_counts != nullptr) p.trace_counts[x] = (int64_t)local;
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(C::TMEM_COLS)
                 : "memory");
  }
}

// Decode-only: every CTA walks its items with the same cursor and records them.
__global__ void schedule_trace_kernel(const Sched s, int64_t* trace, uint64_t cap,
                                      int64_t* counts) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= s.g) return;
  Cursor cur;
  cursor_init(cur, s, x);
  Item it;
  uint64_t n = 0;
  while (cursor_next(cur, s, x, it)) {
    if (n < cap) {
      int64_t* r = trace + ((uint64_t)x * cap + n) * SKPP_TRACE_FIELDS;
      r[0] = (int64_t)it.tile;
      r[1] = (int64_t)it.kb;
      r[2] = (int64_t)it.ke;
      r[3] = it.role == ROLE_FULL ? 0 : 1;
      r[4] = (int64_t)it.phase;
      r[5] = (int64_t)it.role;
    }
    ++n;
  }
  counts[x] = (int64_t)n;
}

// ------------------------------------------------------------------- host --

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

static int make_map(CUtensorMap* map, const void* base, int dtype, uint64_t inner,
                    uint64_t outer, uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer,
                    CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return SKPP_ELAUNCH;
  }
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld_elems * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dtype == SKPP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                          : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                  2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
    return SKPP_ELAUNCH;
  }
  return SKPP_OK;
}

static bool sched_from_c(const skpp_sched_t& c, Sched& s) {
  s.dp_tiles = c.dp_tiles;
  s.sk_tiles = c.sk_tiles;
  s.ipt = c.iters_per_tile;
  s.ipw = c.ipw;
  s.sk_iters = c.sk_iters;
  s.n_tiles = c.n_tiles;
  s.g = c.g;
  s.sk_first = c.sk_first;
  return true;
}

template <int BN, int BK>
static int max_coresident_impl(int* ctas) {
  using C = Cfg<BN, BK>;
  constexpr int kMaxDev = 64;
  static int cache[kMaxDev] = {0};  // 0 = not yet queried
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur >= 0 && cur < kMaxDev && cache[cur] > 0) {
    *ctas = cache[cur];
    return SKPP_OK;
  }
  auto kern = streamk_gemm_kernel<BN, BK>;
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (e != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    return SKPP_ELAUNCH;
  }
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, C::SMEM);
  if (e != cudaSuccess) {
    set_error(std::string("occupancy query: ") + cudaGetErrorString(e));
    return SKPP_ELAUNCH;
  }
  *ctas = per_sm * sms;
  if (cur >= 0 && cur < kMaxDev) cache[cur] = *ctas;
  return SKPP_OK;
}

template <int BN, int BK>
static int launch_impl(const skpp_sched_t& cs, uint64_t M, uint64_t N, uint64_t K,
                       const skpp_operands_t& ops, void* ws, int64_t* trace, uint64_t trace_cap,
                       int64_t* trace_counts, cudaStream_t stream) {
  using C = Cfg<BN, BK>;
  static std::once_flag attr_once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once, [] {
    attr_err = cudaFuncSetAttribute(streamk_gemm_kernel<BN, BK>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  });
  if (attr_err != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
    return SKPP_ELAUNCH;
  }
  CUtensorMap ma, mb;
  const CUtensorMapSwizzle aswz = BK == 64   ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : BK == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                             : CU_TENSOR_MAP_SWIZZLE_32B;
  int rc = make_map(&ma, ops.a, ops.in_dtype, K, M, (uint64_t)ops.lda, BK, kBM, aswz);
  if (rc) return rc;
  rc = make_map(&mb, ops.b, ops.in_dtype, N, K, (uint64_t)ops.ldb, 64, BK,
                CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;

  GemmParams p;
  memset(&p, 0, sizeof(p));
  sched_from_c(cs, p.s);
  p.M = (uint32_t)M;
  p.N = (uint32_t)N;
  const uint32_t ab = ops.in_dtype == SKPP_BF16 ? 1u : 0u;
  p.idesc = (1u << 4) | (ab << 7) | (ab << 10) | (0u << 15) | (1u << 16) |
            ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
  p.out_dtype = ops.out_dtype;
  p.C = ops.c;
  p.ldc = (uint64_t)ops.ldc;
  const uint64_t esz = ops.out_dtype == SKPP_F32 ? 4 : 2;
  p.c_vec_ok = ((reinterpret_cast<uintptr_t>(ops.c) % 16) == 0 && (p.ldc * esz) % 16 == 0) ? 1 : 0;
  p.ws = reinterpret_cast<float*>(ws);
  p.flags = ws ? reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(ws) +
                                             (uint64_t)cs.g * kBM * BN * 4)
               : nullptr;
  p.trace = trace;
  p.trace_cap = trace_cap;
  p.trace_counts = trace_counts;

  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(cs.g);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  int nattr = 0;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cap);
  if (cs.sk_tiles > 0 && cap == cudaStreamCaptureStatusNone) {
    // Stream-K owners spin on peers: every CTA must be resident at once.
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    nattr = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = nattr;
  cudaError_t e = cudaLaunchKernelEx(&cfg, streamk_gemm_kernel<BN, BK>, ma, mb, p);
  if (e != cudaSuccess) {
    set_error(std::string("GEMM launch failed: ") + cudaGetErrorString(e));
    return SKPP_ELAUNCH;
  }
  return SKPP_OK;
}

// Calls f(integral_constant<BN>, integral_constant<BK>) for the instantiated tile shapes.
template <typename F>
static int dispatch_tile(const skpp_tile_t* t, F&& f) {
  using I64 = std::integral_constant<int, 64>;
  using I128 = std::integral_constant<int, 128>;
  using I256 = std::integral_constant<int, 256>;
  using I32 = std::integral_constant<int, 32>;
  using I16 = std::integral_constant<int, 16>;
  if (t->blk_m != (uint32_t)kBM) return SKPP_ETILE;
  if (t->blk_k == 64) {
    if (t->blk_n == 64) return f(I64{}, I64{});
    if (t->blk_n == 128) return f(I128{}, I64{});
    if (t->blk_n == 256) return f(I256{}, I64{});
  } else if (t->blk_k == 32) {
    if (t->blk_n == 64) return f(I64{}, I32{});
    if (t->blk_n == 128) return f(I128{}, I32{});
    if (t->blk_n == 256) return f(I256{}, I32{});
  } else if (t->blk_k == 16) {
    if (t->blk_n == 64) return f(I64{}, I16{});
    if (t->blk_n == 128) return f(I128{}, I16{});
    if (t->blk_n == 256) return f(I256{}, I16{});
  }
  return SKPP_ETILE;
}

}  // namespace skpp

using namespace skpp;

extern "C" int skpp_tile_supported(const skpp_tile_t* t) {
  if (!t) return 0;
  if (t->blk_m != (uint32_t)kBM) return 0;
  if (t->blk_n != 64 && t->blk_n != 128 && t->blk_n != 256) return 0;
  if (t->blk_k != 16 && t->blk_k != 32 && t->blk_k != 64) return 0;
  return 1;
}

extern "C" uint64_t skpp_workspace_bytes(const skpp_problem_t* p, const skpp_tile_t* t,
                                         uint32_t g) {
  (void)p;
  if (!t) return 0;
  const uint64_t part = (uint64_t)g * t->blk_m * t->blk_n * 4;
  const uint64_t flags = (((uint64_t)g * 4) + 255) / 256 * 256;
  return part + flags;
}

extern "C" int skpp_set_device(int device) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    set_error(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    return SKPP_ELAUNCH;
  }
  return SKPP_OK;
}

extern "C" int skpp_device_info(int device, int32_t* sm_count, int32_t* cc_major,
                                int32_t* cc_minor) {
  int v = 0;
  cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    set_error(std::string("cudaDeviceGetAttribute: ") + cudaGetErrorString(e));
    return SKPP_ELAUNCH;
  }
  if (sm_count) *sm_count = v;
  cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, device);
  if (cc_major) *cc_major = v;
  cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, device);
  if (cc_minor) *cc_minor = v;
  return SKPP_OK;
}

static int max_coresident_dispatch(const skpp_tile_t* t, int* ctas) {
  return dispatch_tile(t, [&](auto bn, auto bk) {
    return max_coresident_impl<decltype(bn)::value, decltype(bk)::value>(ctas);
  });
}

extern "C" int skpp_max_coresident(const skpp_tile_t* t, int32_t* ctas) {
  if (!skpp_tile_supported(t)) {
    set_error("tile shape not implemented by the sm_100a kernel");
    return SKPP_ETILE;
  }
  int c = 0;
  int rc = max_coresident_dispatch(t, &c);
  if (rc == SKPP_OK && ctas) *ctas = c;
  return rc;
}

static int check_device() {
  int dev = 0, major = 0, minor = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    set_error(std::string("no CUDA device: ") + cudaGetErrorString(e));
    return SKPP_EARCH;
  }
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) {
    set_error("libskpp kernels are built for sm_100a (B200); device is sm_" +
              std::to_string(major) + std::to_string(minor));
    return SKPP_EARCH;
  }
  return SKPP_OK;
}

extern "C" int skpp_gemm_launch(const skpp_problem_t* p, const skpp_tile_t* t,
                                const skpp_policy_t* pol, uint32_t g, const skpp_operands_t* ops,
                                void* workspace, uint64_t workspace_bytes, int64_t* trace,
                                uint64_t trace_cap, int64_t* trace_counts, void* stream) {
  if (!p || !t || !pol || !ops) {
    set_error("null argument");
    return SKPP_EINVAL;
  }
  if (!skpp_tile_supported(t)) {
    set_error("tile shape " + std::to_string(t->blk_m) + "x" + std::to_string(t->blk_n) + "x" +
              std::to_string(t->blk_k) +
              " is not implemented by the sm_100a kernel (blk_m=128, blk_n in {64,128,256}, "
              "blk_k in {16,32,64})");
    return SKPP_ETILE;
  }
  if (ops->in_dtype != SKPP_F16 && ops->in_dtype != SKPP_BF16) {
    set_error("in_dtype must be fp16 or bf16");
    return SKPP_EINVAL;
  }
  if (ops->out_dtype != SKPP_F32 && ops->out_dtype != SKPP_F16 && ops->out_dtype != SKPP_BF16) {
    set_error("out_dtype must be fp32, fp16 or bf16");
    return SKPP_EINVAL;
  }
  if (p->m < 1 || p->n < 1 || p->k < 1 || p->m >= (1ull << 31) || p->n >= (1ull << 31) ||
      p->k >= (1ull << 31)) {
    set_error("problem dimensions must be in [1, 2^31) for the device kernel");
    return SKPP_EINVAL;
  }
  if (!ops->a || !ops->b || !ops->c) {
    set_error("null operand pointer");
    return SKPP_EINVAL;
  }
  if ((reinterpret_cast<uintptr_t>(ops->a) % 16) || (reinterpret_cast<uintptr_t>(ops->b) % 16) ||
      (ops->lda * 2) % 16 || (ops->ldb * 2) % 16 || ops->lda < (int64_t)p->k ||
      ops->ldb < (int64_t)p->n || ops->ldc < (int64_t)p->n) {
    set_error("TMA needs 16-byte aligned A/B bases and row strides (lda, ldb multiples of 8) "
              "with lda >= k, ldb >= n, ldc >= n");
    return SKPP_EALIGN;
  }
  if (g < 1) {
    set_error("g must be >= 1");
    return SKPP_EINVAL;
  }
  int rc = check_device();
  if (rc) return rc;
  skpp_sched_t cs;
  rc = skpp_sched_make(p, t, g, pol, &cs);
  if (rc) return rc;
  if (cs.sk_tiles > 0) {
    if (workspace_bytes < skpp_workspace_bytes(p, t, g) || workspace == nullptr) {
      set_error("workspace too small: need " + std::to_string(skpp_workspace_bytes(p, t, g)) +
                " bytes");
      return SKPP_EWORKSPACE;
    }
    int co = 0;
    rc = max_coresident_dispatch(t, &co);
    if (rc) return rc;
    if ((int64_t)g > co) {
      set_error("g=" + std::to_string(g) + " exceeds the " + std::to_string(co) +
                " co-resident CTAs the Stream-K fixup needs");
      return SKPP_EGRID;
    }
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return dispatch_tile(t, [&](auto bn, auto bk) {
    return launch_impl<decltype(bn)::value, decltype(bk)::value>(
        cs, p->m, p->n, p->k, *ops, workspace, trace, trace_cap, trace_counts, st);
  });
}

extern "C" int skpp_schedule_trace_device(const skpp_problem_t* p, const skpp_tile_t* t,
                                          const skpp_policy_t* pol, uint32_t g, int64_t* trace,
                                          uint64_t trace_cap, int64_t* trace_counts,
                                          void* stream) {
  if (!trace || !trace_counts) {
    set_error("null trace buffer");
    return SKPP_EINVAL;
  }
  skpp_sched_t cs;
  int rc = skpp_sched_make(p, t, g, pol, &cs);
  if (rc) return rc;
  Sched s;
  sched_from_c(cs, s);
  const uint32_t threads = 128;
  schedule_trace_kernel<<<(g + threads - 1) / threads, threads, 0,
                          reinterpret_cast<cudaStream_t>(stream)>>>(s, trace, trace_cap,
                                                                     trace_counts);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("trace launch failed: ") + cudaGetErrorString(e));
    return SKPP_ELAUNCH;
  }
  return SKPP_OK;
}
