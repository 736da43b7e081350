// skpp_gemm.cu — persistent Stream-K++ GEMM for sm_100a (B200).
//
// Replaces the reference's schedule executor (gemmsched executor.py:51-124):
// there every WorkItem runs `c[r0:r1,c0:c1] += a[r0:r1,k0:k1] @ b[k0:k1,c0:c1]`
// on the host in float64, with the `+=` standing for the atomic fixup of
// Algorithm 1.  Here one launch runs a whole schedule:
//
//   grid      = g CTAs (one per SM, co-resident), CTA x == workgroup x;
//   warp 0    = TMA producer: walks x's items (skpp_sched.h) and streams the
//               A (K-major, swizzled) and B (N-major, SW128) k-blocks of each
//               item's [kb, ke) range through an S-stage shared-memory ring;
//   warp 1    = MMA issuer: one thread issues tcgen05.mma kind::f16
//               (M=128, N=BN, K=16) into an fp32 TMEM accumulator, double
//               buffered across items; accumulate is reset at each item's kb;
//   warp 2    = TMEM allocator;
//   warps 4-7 = epilogue, two phases:
//     phase 1, per item in order: tcgen05.ld the accumulator rows; a FULL
//       item is packed into swizzled shared-memory staging (two 4 KiB buffers
//       per warp) and TMA-stored to C; a partial item is written with
//       coalesced stores to this CTA's workspace slot, whose flag is then
//       released.  No CTA waits on another in phase 1.
//     phase 2, after all items (all 8 warps): a CTA reduces at most one
//       split tile, a band of its rows over ALL contributors' slots, summed in
//       a fixed order (peers in increasing CTA order, then the owner) so the
//       result is deterministic, staged in shared memory and stored to C with
//       coalesced row stores.
//   Every CTA produces all its partials before it waits, so the wait graph
//   is acyclic; flags carry an epoch kept in the workspace header, so the
//   kernel is CUDA-graph replay safe.
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
constexpr uint32_t kRingBudget = 196608;   // operand ring (192 KiB)
constexpr uint32_t kStageBuf = 4096;       // one epilogue staging buffer: 32 rows x 128 B
constexpr uint32_t kStagingBytes = 4 * 2 * kStageBuf;
// Workspace: a fixed 32 KiB control block, then 2 slots of BM x BN fp32 per CTA.
//   [0, 256)          header: [0] epoch of the last completed Stream-K launch, [1] arrivals,
//                     [8 + par] CTAs started, [16 + par] abandoned bands (phase 2, par = epoch & 1)
//   [1 KiB, 9 KiB)    slot flags, 2 per CTA (== epoch when the slot holds this launch's partial)
//   [9 KiB, 17 KiB)   band states [2 parities][kMaxCtas] per reducing CTA: 0 none,
//                     1 abandoned, 2 claimed by the last-starting CTA, 3 taken back
// Fixed offsets: plans of any grid size share one workspace without their control words
// ever overlapping another plan's partial slots.  Launch e uses the parity e & 1 words and
// resets the other parity's for launch e + 1 (which starts only after this grid completed).
constexpr uint32_t kMaxCtas = 1024;
// Slot-flag value (epoch | kOwnerDone) of an owner item whose tile the owner finished itself in
// phase 1 (owner reduction, see the epilogue): no partial in the slot, nothing left to reduce.
// Epochs stay below 2^31 (one per Stream-K launch on a workspace).
constexpr uint32_t kOwnerDone = 0x80000000u;
// Bound of the owner's phase-1 wait for the other contributor's partial (~4 us): the liveness
// protocol needs every wait in phase 1 to be bounded; on timeout the owner publishes its partial.
constexpr long long kOwnerWaitCycles = 8000;
constexpr uint64_t kWsFlagsOff = 1024;
constexpr uint64_t kWsStatesOff = kWsFlagsOff + 2ull * kMaxCtas * 4;
constexpr uint64_t kWsCtlBytes = 32768;
static_assert(kWsStatesOff + 2ull * kMaxCtas * 4 <= kWsCtlBytes, "workspace control block");

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
// 3-D box: (n within a 64-column chunk, k, chunk) -> smem [chunk][k][64]
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            int32_t c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, int32_t c0,
                                                 int32_t c1, int32_t c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0,
                                             int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(src))
      : "memory");
}
// L2 cache-policy variants (createpolicy): B k-slices are re-read by the next wave
// (evict_last); C tiles are written once (evict_first).
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                                 int32_t c2, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair_hint(void* dst, const CUtensorMap* map, int32_t c0,
                                                      int32_t c1, int32_t c2, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar) & 0xFEFFFFFFu),
      "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, const void* src, int32_t c0,
                                                  int32_t c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(src)), "l"(pol)
      : "memory");
}

// L2 prefetch of a tensor box (no shared memory, no barrier).  Safe before
// griddepcontrol.wait: L2 is the point of coherence, so a line the previous kernel
// still writes is updated in place; the prefetch can only be wasted, never stale.
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// ---- CTA-pair (cta_group::2) helpers
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Both CTAs of the pair load their own smem but complete on the LEADER's barrier
// (clearing the peer bit of the shared::cluster address selects CTA rank 0).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int32_t c0,
                                                 int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// Arrive on the barrier at this smem offset in BOTH CTAs of the pair once the
// pair MMAs issued so far complete.
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_rank(uint64_t* bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
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

// 32 lanes x 32 consecutive fp32 columns: each thread gets its row's 32 values.
__device__ __forceinline__ void tmem_ld_32(uint32_t taddr, uint32_t* r) {
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
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void epi_bar_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void phase2_bar_sync() { asm volatile("bar.sync 2, 256;" ::: "memory"); }

__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t atom_cas_acq_rel_gpu(uint32_t* p, uint32_t cmp, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "l"(p), "r"(cmp), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ float4 ld_cg_f4(const float4* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

// UMMA shared-memory matrix descriptor (sm_100 format, version 1).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

__device__ __forceinline__ uint32_t pack2(float a, float b, int out_dtype) {
  if (out_dtype == SKPP_BF16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ------------------------------------------------------------ kernel config --

// BN = N of the MMA (= tile width); CG = CTAs per MMA (1, or 2 for a
// cta_group::2 pair whose tile is 256 rows: each CTA holds 128 rows of A and
// BN/2 columns of B, and 128 accumulator lanes x BN columns of TMEM).
template <int BN, int BK, int CG>
struct Cfg {
  static constexpr int BNC = BN / CG;  // B columns loaded by each CTA
  static constexpr uint32_t A_BYTES = kBM * BK * 2;
  static constexpr uint32_t B_BYTES = BK * BNC * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t STAGES_RAW = kRingBudget / STAGE_BYTES;
  static constexpr uint32_t STAGES = STAGES_RAW > 32 ? 32 : STAGES_RAW;
  static constexpr uint32_t RING_BYTES = STAGES * STAGE_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BN <= 32    ? 32
                                        : 2 * BN <= 64  ? 64
                                        : 2 * BN <= 128 ? 128
                                        : 2 * BN <= 256 ? 256
                                                        : 512;
  static constexpr uint32_t BAR_BYTES = ((2 * STAGES + 5) * 8 + 32 + 16 * 4 + 1023) / 1024 * 1024;
  static constexpr uint32_t SMEM = RING_BYTES + kStagingBytes + BAR_BYTES + 1024;
  // A: K-major, one swizzle atom along K (BK*2 bytes = 32/64/128 B)
  // BK = 128: two SW128 sub-tiles of [128 rows][64 k] (one TMA box each, 16 KiB apart)
  static constexpr uint32_t A_LAYOUT = BK >= 64 ? 2u : (BK == 32 ? 4u : 6u);
  static constexpr uint32_t A_SBO = BK >= 64 ? 1024u : 8 * BK * 2;  // 8 rows of one atom
  static constexpr uint32_t A_OPS = BK > 64 ? BK / 64 : 1;          // TMA boxes per stage
  static constexpr uint32_t A_SUB = A_BYTES / A_OPS;                // bytes per A sub-tile
  // B: N-major SW128, 64-column chunks of BK rows x 128 B
  static constexpr uint32_t B_LAYOUT = 2u;
  static constexpr uint32_t B_LBO = BK * 128;  // next 64-wide N chunk
  static constexpr uint32_t B_SBO = 1024;      // next 8 K-rows
  static_assert(BN % 64 == 0 && BN <= 256 && BNC % 64 == 0, "BN");
  static_assert(CG == 1 || CG == 2, "CG");
  static_assert(BK == 16 || BK == 32 || BK == 64 || BK == 128, "BK");
  static_assert(STAGES >= 2, "stages");
  static_assert(SMEM <= 232448, "shared memory");
};

struct GemmParams {
  Sched s;
  uint32_t M, N;
  uint32_t idesc;
  int32_t out_dtype;
  void* C;
  uint64_t ldc;
  uint32_t c_vec_ok;   // C base and row stride 16-byte aligned
  uint32_t c_tma;      // C tensor map valid: phase-1 FULL tiles use TMA stores
  float* ws;           // 2g partial slots of BM x BN fp32, row-major
  uint32_t* flags;     // 2g slot flags (== epoch when the slot holds this launch's partial)
  uint32_t* hdr;       // [0] epoch of the last completed launch, [1] CTAs of this launch that read [0]
  uint32_t* bstate;    // [2][kMaxCtas] band states of the reducing CTAs (parity = epoch & 1)
  uint32_t abandon_cycles;  // phase-2 flag wait before a reducer checks whether every CTA started
  int64_t* trace;
  uint64_t trace_cap;
  int64_t* trace_counts;
  uint64_t* timeline;  // debug: TL_EVENTS %globaltimer stamps per CTA, or null
  uint32_t b3d;         // tmB is the 3-D (n64, k, chunk) map: one B load per stage
  uint32_t a3d;         // tmA is the 3-D (k64, row, chunk) map: one A load per BK=128 stage
  uint32_t a_tx;        // A bytes per stage per CTA (the A box covers round_up(M, 8) rows when M < 128)
  uint32_t l2_prefetch; // k-blocks of the first item prefetched to L2 before griddepcontrol.wait
  uint32_t l2_hints;    // B loads evict_last, C stores evict_first (skpp_set_l2_hints)
  uint32_t debug;       // skpp_set_debug: bit 0 = always take the two-pass (owner-late) fixup path,
                        // bit 1 = abandon at once (every band whose flags are not already up goes
                        // through the abandon / last-arriver path)
  uint32_t raster;      // tile order: 0 = row-major (reference), G = bands of G tile rows (tile_rc)
  uint32_t ragged;      // last row / column tile at most half full: partials and bands skip rows >= M, cols >= N
};

// Debug timeline (skpp_debug_timeline): per-CTA %globaltimer stamps.
enum : int {
  TL_START = 0,       // all warps past setup (barriers + TMEM)
  TL_FIRST_TMA = 1,   // producer issued its first load
  TL_FIRST_FULL = 2,  // MMA saw its first stage land
  TL_MMA_DONE = 3,    // MMA issued its last commit
  TL_PHASE1 = 4,      // epilogue finished all items (stores / partials)
  TL_WAITED = 5,      // epilogue finished waiting for the first split tile's flags
  TL_PHASE2 = 6,      // epilogue finished the reductions
  TL_END = 7,         // every warp done (the last starter's cleanup included)
  TL_EPI_FIRST = 8,   // epilogue saw its first accumulator
  TL_PART_ISSUED = 9, // first partial: all TMA stores issued
  TL_PART_FLAG = 10,  // first partial: flag released
  TL_SUM1 = 11,       // phase 2: first summation pass done (thread 128)
  TL_SUM2 = 12,       // phase 2: owner pass done (only when the owner was late)
  TL_BS0 = 13,        // band_sum (first pass, thread 128): clock64 at entry,
  TL_BS1 = 14,        //   after its first batch of partial loads returned,
  TL_BS2 = 15,        //   and at exit (SM cycles, not ns)
  TL_P2_STORED = 16,  // phase 2, thread 0: first band stored to C
  TL_ENTRY = 21,      // thread 0 at kernel entry (before barrier init and griddepcontrol.wait)
  TL_C_TMA = 22,      // SM cycles from griddepcontrol.wait returning to the first A load (thread 0)
  TL_CP_INIT = 25,    // prologue, SM cycles since entry (thread 0): barriers initialised,
  TL_CP_TMEM = 26,    //   TMEM allocated and the CTA (pair) synchronised,
  TL_CP_PREF = 27,    //   first item decoded and its L2 prefetches issued (just before the wait)
  TL_CP_DEC = 28,     //   first item decoded (before its L2 prefetches)
  TL_CLK_ENTRY = 24,  // clock64 at TL_ENTRY and at TL_END (thread 0): the SM clock rate over the
  TL_CLK_END = 31,    //   kernel against %globaltimer
  TL_EVENTS = 32
};
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Per-k-block stamps of CTA 0 (issue by the producer, arrival seen by the MMA
// warp) in SM clock cycles (clock64; %globaltimer reads are too slow here),
// after the per-CTA table: timeline[gridDim.x*TL_EVENTS + 2*k + {0,1}].
constexpr int TL_KSTAMPS = 256;
#define SKPP_KSTAMP(p, k, which)                                                          \
  do {                                                                                    \
    if ((p).timeline && blockIdx.x == 0 && (k) < TL_KSTAMPS)                              \
      (p).timeline[(uint64_t)gridDim.x * TL_EVENTS + 2 * (k) + (which)] = clock64();      \
  } while (0)
#define SKPP_STAMP(p, ev) \
  do { if ((p).timeline) (p).timeline[(uint64_t)blockIdx.x * TL_EVENTS + (ev)] = gtimer(); } while (0)

// One trace row: the item (tile, kb, ke, write mode, phase, role) and the C tile it wrote.
__device__ __forceinline__ void write_trace_row(int64_t* r, const Item& it, uint64_t tm, uint64_t tn) {
  r[0] = (int64_t)it.tile;
  r[1] = (int64_t)it.kb;
  r[2] = (int64_t)it.ke;
  r[3] = it.role == ROLE_FULL ? 0 : 1;
  r[4] = (int64_t)it.phase;
  r[5] = (int64_t)it.role;
  r[6] = (int64_t)tm;
  r[7] = (int64_t)tn;
}
__device__ __forceinline__ void record_item(const GemmParams& p, uint32_t x, uint64_t idx, const Item& it,
                                            uint64_t tm, uint64_t tn) {
  if (p.trace == nullptr || idx >= p.trace_cap) return;
  write_trace_row(p.trace + ((uint64_t)x * p.trace_cap + idx) * SKPP_TRACE_FIELDS, it, tm, tn);
}

// Direct (non-TMA) store of one packed 128-byte row segment; used only when C
// is not 16-byte aligned.  `w` holds 32 fp32 or 64 16-bit values.
__device__ __forceinline__ void store_row_direct(const GemmParams& p, uint64_t row, uint64_t col0,
                                                 const uint32_t* w) {
  if (row >= p.M) return;
  if (p.out_dtype == SKPP_F32) {
    float* c = reinterpret_cast<float*>(p.C) + row * p.ldc;
    for (int j = 0; j < 32 && col0 + j < p.N; ++j) c[col0 + j] = __uint_as_float(w[j]);
  } else {
    uint16_t* c = reinterpret_cast<uint16_t*>(p.C) + row * p.ldc;
    for (int j = 0; j < 64 && col0 + j < p.N; ++j)
      c[col0 + j] = (uint16_t)(w[j >> 1] >> (16 * (j & 1)));
  }
}

// Convert and store 4 consecutive columns of one output row (phase-2 reduction).
__device__ __forceinline__ void store_vec4(const GemmParams& p, uint64_t row, uint64_t col,
                                           float4 a) {
  if (row >= p.M || col >= p.N) return;
  const bool full = p.c_vec_ok && col + 4 <= p.N;
  if (p.out_dtype == SKPP_F32) {
    float* c = reinterpret_cast<float*>(p.C) + row * p.ldc + col;
    if (full) {
      *reinterpret_cast<float4*>(c) = a;
    } else {
      const float v[4] = {a.x, a.y, a.z, a.w};
      for (int j = 0; j < 4 && col + j < p.N; ++j) c[j] = v[j];
    }
  } else {
    uint16_t* c = reinterpret_cast<uint16_t*>(p.C) + row * p.ldc + col;
    const uint32_t lo = pack2(a.x, a.y, p.out_dtype), hi = pack2(a.z, a.w, p.out_dtype);
    if (full) {
      *reinterpret_cast<uint2*>(c) = make_uint2(lo, hi);
    } else {
      const uint32_t w[2] = {lo, hi};
      for (int j = 0; j < 4 && col + j < p.N; ++j) c[j] = (uint16_t)(w[j >> 1] >> (16 * (j & 1)));
    }
  }
}

// Tile index -> C tile (skpp_sched.h tile_coords).  RASTER is a template parameter so
// that the reference-order instantiations (tile_order == 0, the parity mode) compile to the
// plain row-major division; a runtime branch here measured 0.5-1% slower on cfg2 and
// decode shapes.
template <bool RASTER>
__device__ __forceinline__ void tile_rc(const Sched& s, uint32_t raster, uint64_t t, uint64_t& tm, uint64_t& tn) {
  tile_coords(s, RASTER ? raster : 0u, t, tm, tn);
}

struct ReduceArgs {
  const float4* wsv;   // workspace slots as float4[2g_cta][BN/4][128]
  uint64_t slot_v;     // float4 per slot
  uint64_t slot0;      // slot of contributor x0 (first or last item)
  uint64_t x0;         // first contributing workgroup
  uint32_t rank;       // row half (CTA rank in the pair)
  uint32_t nc;         // contributors
  uint64_t* tl;        // debug timeline row of this CTA, or null
};

__device__ __forceinline__ void wait_flag(const uint32_t* flag, uint32_t epoch) {
  if (ld_acquire_gpu(flag) == epoch) return;
  const long long t0 = clock64();
  while (ld_acquire_gpu(flag) != epoch) {
    __nanosleep(32);
    watchdog(t0, 5);
  }
}

// Bounded flag wait of phase 2: true when the flag shows this launch's epoch before
// `cycles` SM cycles have passed since t0.
__device__ __forceinline__ bool wait_flag_until(const uint32_t* flag, uint32_t epoch, long long t0,
                                                uint32_t cycles) {
  while (ld_acquire_gpu(flag) != epoch) {
    if (clock64() - t0 > (long long)cycles) return false;
    __nanosleep(32);
  }
  return true;
}

// Owner flag of a split tile in phase 2: 1 = the owner's partial is published, 2 = the owner
// finished the tile itself in phase 1 (epoch | kOwnerDone), 0 = neither within `cycles`.
__device__ __forceinline__ uint32_t wait_owner_flag(const uint32_t* flag, uint32_t epoch, long long t0,
                                                   uint32_t cycles) {
  while (true) {
    const uint32_t v = ld_acquire_gpu(flag);
    if (v == epoch) return 1u;
    if (v == (epoch | kOwnerDone)) return 2u;
    if (clock64() - t0 > (long long)cycles) return 0u;
    __nanosleep(32);
  }
}

// Header words of the liveness protocol (phase 2), per parity of the launch epoch.
constexpr uint32_t kHdrStarted = 8;   // hdr[8 + par]: CTAs of the launch that have started
constexpr uint32_t kHdrAbandon = 16;  // hdr[16 + par]: some band of the launch was abandoned

// A phase-2 flag wait timed out (thread 0).  Returns 1 to keep waiting, 0 when the band was
// handed to the launch's last-starting CTA.  If every CTA has started, every partial will
// be published: keep waiting.  Otherwise mark the band abandoned (state 1) and flag the
// launch, then look again: if the last CTA started meanwhile it may have missed the mark,
// so take the band back (CAS 1 -> 3; the last starter claims with CAS 1 -> 2, exactly one
// succeeds).  The RMW reads of the counter order the marks before any later start.
__device__ __noinline__ uint32_t abandon_or_wait(uint32_t* hdr, uint32_t par, uint32_t* bst) {
  if (atom_add_acq_rel_gpu(hdr + kHdrStarted + par, 0u) >= gridDim.x) return 1u;
  atom_cas_acq_rel_gpu(bst, 0u, 1u);
  atom_add_acq_rel_gpu(hdr + kHdrAbandon + par, 1u);
  if (atom_add_acq_rel_gpu(hdr + kHdrStarted + par, 0u) >= gridDim.x && atom_cas_acq_rel_gpu(bst, 1u, 3u) == 1u)
    return 1u;
  return 0u;
}

// Phase 2 works on a BAND of rows of the split tile: reducer idx of nr owns rows
// [R0, R0 + nrows) of its row half and every column.  Element e of the band is
// column group j = e / nrows, band row ro = e % nrows, i.e. float4 (j*128 + R0 + ro)
// of every slot, so consecutive threads read consecutive rows of one column group
// (coalesced; slots are column-group major).  Terms are added in the fixed order
// peer x0+1, ..., peer x0+nc-1, owner x0 (term index i < nc-1 is peer x0+1+i,
// term nc-1 is x0), starting from +0, so the bits never depend on timing or on
// whether the owner term was added in the same pass.  The band is accumulated
// in shared memory (stage[ro][j], row stride V+1 float4) and stored to C row by
// row (coalesced) by band_store.
__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void st_shared_f4(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// Scalars passed by value: a noinline callee keeps them in registers.
template <int G, int KB>
__device__ __noinline__ void band_sum(const float4* __restrict__ wsv, uint64_t slot_v, uint64_t peer_slot0,
                                      uint32_t peer_slot_step, uint64_t owner_slot, uint32_t nc,
                                      uint32_t R0, uint32_t nrows, uint32_t V, uint32_t sstride,
                                      uint32_t term_begin, uint32_t term_end, uint32_t accumulate,
                                      uint32_t stage, uint32_t ft, uint64_t* tl) {
  const bool stamp = tl != nullptr && ft == kEpiWarp0 * 32 && term_begin == 0;
  if (stamp) tl[TL_BS0] = clock64();
  bool first = true;
  const uint32_t total = nrows * V;
  for (uint32_t e0 = ft; e0 < total; e0 += G * kThreads) {
    float4 acc[G];
    uint32_t off[G];
    uint32_t saddr[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t e = e0 + g * kThreads;
      const uint32_t j = e / nrows, ro = e - j * nrows;
      off[g] = j * kBM + R0 + ro;
      saddr[g] = stage + (ro * sstride + j) * 16;
      acc[g] = (accumulate && e < total) ? ld_shared_f4(saddr[g]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (uint32_t t0 = term_begin; t0 < term_end; t0 += KB) {
      float4 q[G][KB];
#pragma unroll
      for (int b = 0; b < KB; ++b) {
        if (t0 + b < term_end) {
          const uint64_t slot = (t0 + b < nc - 1) ? peer_slot0 + (uint64_t)(t0 + b) * peer_slot_step : owner_slot;
          const float4* src = wsv + slot * slot_v;
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (e0 + g * kThreads < total) q[g][b] = ld_cg_f4(src + off[g]);
        }
      }
#pragma unroll
      for (int b = 0; b < KB; ++b) {
        if (t0 + b < term_end) {
#pragma unroll
          for (int g = 0; g < G; ++g) {
            if (stamp && first && b == 0 && g == 0) {
              tl[TL_BS1] = clock64() + (q[0][0].x == 12345.f ? 1 : 0);  // after the first load returned
              first = false;
            }
            acc[g].x += q[g][b].x;
            acc[g].y += q[g][b].y;
            acc[g].z += q[g][b].z;
            acc[g].w += q[g][b].w;
          }
        }
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (e0 + g * kThreads < total) st_shared_f4(saddr[g], acc[g]);
  }
  if (stamp) tl[TL_BS2] = clock64();
}

// Store the reduced band: consecutive threads take consecutive column groups of
// one row, so a warp writes 512 contiguous bytes of C (fp32) per instruction.
template <uint32_t V>
__device__ __forceinline__ void band_store(const GemmParams& p, uint32_t stage, uint32_t nrows,
                                           uint32_t Vv, uint64_t row0, uint64_t col0, uint32_t ft) {
  const uint32_t total = nrows * V;
  for (uint32_t e = ft; e < total; e += kThreads) {
    const uint32_t ro = e / V, j = e - ro * V;
    if (j < Vv) store_vec4(p, row0 + ro, col0 + 4 * j, ld_shared_f4(stage + (ro * (V + 1) + j) * 16));
  }
}

// Term i < nc-1 is peer x0+1+i (its first Stream-K item: slot 2*cta, cta =
// (x0+1+i)*CG + rank); term nc-1 is the owner x0 (slot0).  Register-staged
// loads, <= 24 float4 in flight per thread: larger variants spill, and a
// cp.async variant (all terms' bands in flight through the idle ring) measured
// 3-20% slower on every fixup-heavy shape tried (tools/ab_reduce.py).
// V = column groups to reduce (<= BN/4 for a ragged last column tile); the stage
// row stride is the tile's BN/4 + 1 (SV) for every tile.
template <int CG, uint32_t SV>
__device__ __forceinline__ void band_reduce(const ReduceArgs& ra, uint32_t R0, uint32_t nrows, uint32_t V,
                                            uint32_t term_begin, uint32_t term_end, bool accumulate,
                                            uint32_t stage, uint32_t ft) {
  const uint64_t peer0 = 2 * ((ra.x0 + 1) * CG + ra.rank);
  if (ra.nc <= 4)
    band_sum<4, 4>(ra.wsv, ra.slot_v, peer0, 2 * CG, ra.slot0, ra.nc, R0, nrows, V, SV + 1, term_begin, term_end,
                   accumulate, stage, ft, ra.tl);
  else
    band_sum<2, 12>(ra.wsv, ra.slot_v, peer0, 2 * CG, ra.slot0, ra.nc, R0, nrows, V, SV + 1, term_begin, term_end,
                    accumulate, stage, ft, ra.tl);
}

// Hand an accumulator stage back to the MMA issuer (the rank-0 CTA's barrier).
template <int CG>
__device__ __forceinline__ void release_acc_t(uint64_t* bar) {
  if constexpr (CG == 1)
    mbar_arrive(bar);
  else
    mbar_arrive_rank(bar, 0);
}
#define release_acc(bar) release_acc_t<CG>(bar)

template <int BN, int BK, int CG, bool RASTER = false>
__global__ void __launch_bounds__(kThreads, 1)
    streamk_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmC, const __grid_constant__ GemmParams p) {
  using C = Cfg<BN, BK, CG>;
  constexpr uint32_t TILE_M = kBM * CG;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* stg = smem + C::RING_BYTES;  // epilogue staging, 1024-aligned
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg + kStagingBytes);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* red_bar = tempty_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_bar + 1);
  uint64_t* split_smem = red_bar + 2;                       // phase-2 work list (2 tiles)
  uint32_t* nsplit_smem = reinterpret_cast<uint32_t*>(red_bar + 4);

  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;  // row half of the pair tile

  const uint32_t x = blockIdx.x / CG;                      // workgroup (pair) id
  const Sched& s = p.s;

  const long long c_entry = clock64();
  if (threadIdx.x == 0 && p.timeline) {
    SKPP_STAMP(p, TL_ENTRY);
    p.timeline[(uint64_t)blockIdx.x * TL_EVENTS + TL_CLK_ENTRY] = c_entry;
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (uint32_t i = 0; i < C::STAGES; ++i) {
      mbar_init(&full_bar[i], 2);  // the A and the B producer
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 4 * CG);  // every epilogue warp of the pair
    }
    mbar_init(red_bar, 1);
    nsplit_smem[4] = 0u;  // last-starter cleanup (set by the epilogue leader)
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_shared();
    if (p.timeline) p.timeline[(uint64_t)blockIdx.x * TL_EVENTS + TL_CP_INIT] = clock64() - c_entry;
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) {
    cluster_sync();  // peer barriers initialised and TMEM allocated on both CTAs
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0 && p.timeline) p.timeline[(uint64_t)blockIdx.x * TL_EVENTS + TL_CP_TMEM] = clock64() - c_entry;
  // The producers decode their first item here, before griddepcontrol.wait (it depends only on
  // the kernel parameters), so the first loads issue right after the wait.  While the previous
  // kernel drains, they also pull the first `p.l2_prefetch` k-blocks of it into L2 (A by warp 0,
  // B by warp 3), so the first stages land from L2.
  Cursor pcur;
  Item pit;
  uint64_t ptm = 0, ptn = 0;
  bool pmore = false;
  if ((warp == 0 || warp == 3) && lane == 0) {
    cursor_init(pcur, s, x);
    pmore = cursor_next(pcur, s, x, pit);
    if (pmore) tile_rc<RASTER>(s, p.raster, pit.tile, ptm, ptn);
    if (threadIdx.x == 0 && p.timeline) p.timeline[(uint64_t)blockIdx.x * TL_EVENTS + TL_CP_DEC] = clock64() - c_entry;
    if (pmore && p.l2_prefetch) {
      const int32_t m0 = (int32_t)(ptm * TILE_M + rank * kBM);
      const int32_t n0 = (int32_t)(ptn * BN + rank * C::BNC);
      const uint64_t kend = pit.kb + p.l2_prefetch < pit.ke ? pit.kb + p.l2_prefetch : pit.ke;
      for (uint64_t kk = pit.kb; kk < kend; ++kk) {
        const int32_t k0 = (int32_t)(kk * BK);
        if (warp == 0) {
          if (C::A_OPS > 1 && p.a3d)
            tma_prefetch_3d(&tmA, 0, m0, k0 / 64);
          else
            for (uint32_t j = 0; j < C::A_OPS; ++j) tma_prefetch_2d(&tmA, k0 + 64 * j, m0);
        } else if (p.b3d) {
          tma_prefetch_3d(&tmB, 0, k0, n0 / 64);
        } else {
          for (int j = 0; j < C::BNC / 64; ++j) tma_prefetch_2d(&tmB, n0 + 64 * j, k0);
        }
      }
    }
  }
  // Programmatic dependent launch: everything above (barrier init, TMEM
  // allocation, descriptor and L2 prefetch) overlaps the previous kernel's tail;
  // no global memory written by earlier work is read before this wait.
  if (threadIdx.x == 0 && p.timeline) p.timeline[(uint64_t)blockIdx.x * TL_EVENTS + TL_CP_PREF] = clock64() - c_entry;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const long long c_wait = clock64();
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) SKPP_STAMP(p, TL_START);

  if ((warp == 0 || warp == 3) && lane == 0) {
    // ------------------------------------------------ TMA producers
    // Two issuing threads — warp 0 loads A, warp 3 loads B — because a single
    // thread's wait + expect_tx + TMA issue sequence (~250 ns per stage) is a
    // throughput limit of its own; each arrives once per stage on the full
    // barrier with its own byte count.
    const bool load_a = warp == 0;
    uint32_t stage = 0, phase = 0, kcount = 0, n_full = 0;
    bool first_load = true;
    const uint64_t pol_b = l2_policy_evict_last();
    for (; pmore; pmore = cursor_next(pcur, s, x, pit) && (tile_rc<RASTER>(s, p.raster, pit.tile, ptm, ptn), true)) {
      const Item& it = pit;
      const uint64_t tm_ = ptm, tn_ = ptn;
      const int32_t m0 = (int32_t)(tm_ * TILE_M + rank * kBM);
      const int32_t n0 = (int32_t)(tn_ * BN + rank * C::BNC);
      // Serpentine K: every other FULL item of this workgroup walks K backwards.  A
      // workgroup's consecutive FULL items run in consecutive waves, and every
      // workgroup of a wave streams (nearly) all of B; walking the next wave's K in
      // the opposite direction starts it on the k-slices the previous wave touched
      // last, which are still in L2.  Only the order of the fp32 accumulation inside
      // a tile changes (fixed per tile => deterministic); the MMA warp only counts stages.
      const bool reverse = it.role == ROLE_FULL && (n_full++ & 1u);
      for (uint64_t i = 0; i < it.ke - it.kb; ++i) {
        const uint64_t kk = reverse ? it.ke - 1 - i : it.kb + i;
        mbar_wait(&empty_bar[stage], phase ^ 1, 1);
        if (load_a) {
          SKPP_KSTAMP(p, kcount, 0);
          ++kcount;
          if (first_load) {
            SKPP_STAMP(p, TL_FIRST_TMA);
            if (p.timeline) p.timeline[(uint64_t)blockIdx.x * TL_EVENTS + TL_C_TMA] = clock64() - c_wait;
            first_load = false;
          }
        }
        // the MMA-issuing (rank-0) CTA's barrier expects the bytes of the whole pair
        if (rank == 0)
          mbar_arrive_expect_tx(&full_bar[stage], CG * (load_a ? p.a_tx : C::B_BYTES));
        const int32_t k0 = (int32_t)(kk * BK);
        if constexpr (CG == 1) {
          if (load_a) {
            if (C::A_OPS > 1 && p.a3d) {  // both 64-deep sub-tiles in one 3-D box
              tma_load_3d(sA + stage * C::A_BYTES, &tmA, 0, m0, k0 / 64, &full_bar[stage]);
            } else {
#pragma unroll
              for (uint32_t j = 0; j < C::A_OPS; ++j)
                tma_load_2d(sA + stage * C::A_BYTES + j * C::A_SUB, &tmA, k0 + 64 * j, m0, &full_bar[stage]);
            }
          } else if (p.b3d) {  // all of the stage's B columns in one 3-D box
            if (p.l2_hints)
              tma_load_3d_hint(sB + stage * C::B_BYTES, &tmB, 0, k0, n0 / 64, &full_bar[stage], pol_b);
            else
              tma_load_3d(sB + stage * C::B_BYTES, &tmB, 0, k0, n0 / 64, &full_bar[stage]);
          } else {
#pragma unroll
            for (int j = 0; j < C::BNC / 64; ++j)
              tma_load_2d(sB + stage * C::B_BYTES + j * (BK * 128), &tmB, n0 + 64 * j, k0,
                          &full_bar[stage]);
          }
        } else {
          if (load_a) {
            if (C::A_OPS > 1 && p.a3d) {
              tma_load_3d_pair(sA + stage * C::A_BYTES, &tmA, 0, m0, k0 / 64, &full_bar[stage]);
            } else {
#pragma unroll
              for (uint32_t j = 0; j < C::A_OPS; ++j)
                tma_load_2d_pair(sA + stage * C::A_BYTES + j * C::A_SUB, &tmA, k0 + 64 * j, m0, &full_bar[stage]);
            }
          } else if (p.b3d) {
            if (p.l2_hints)
              tma_load_3d_pair_hint(sB + stage * C::B_BYTES, &tmB, 0, k0, n0 / 64, &full_bar[stage], pol_b);
            else
              tma_load_3d_pair(sB + stage * C::B_BYTES, &tmB, 0, k0, n0 / 64, &full_bar[stage]);
          } else {
#pragma unroll
            for (int j = 0; j < C::BNC / 64; ++j)
              tma_load_2d_pair(sB + stage * C::B_BYTES + j * (BK * 128), &tmB, n0 + 64 * j, k0,
                               &full_bar[stage]);
          }
        }
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (1 lane of the rank-0 CTA)
    if (lane == 0 && rank == 0) {
      uint32_t stage = 0, phase = 0, local = 0, kcount = 0;
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
          SKPP_KSTAMP(p, kcount, 1);
          ++kcount;
          if (local == 0 && kk == it.kb) SKPP_STAMP(p, TL_FIRST_FULL);
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // k-step k covers elements [16k, 16k+16): sub-tile 16k/64, 32 B per step inside it
            const uint64_t ad = umma_desc(a_addr + (k * 16 / 64) * C::A_SUB + (k * 16 % 64) * 2, 0,
                                          C::A_SBO, C::A_LAYOUT);
            const uint64_t bd = umma_desc(b_addr + k * 2048, C::B_LBO, C::B_SBO, C::B_LAYOUT);
            if constexpr (CG == 1)
              umma_f16(dtm, ad, bd, p.idesc, (kk > it.kb || k > 0) ? 1u : 0u);
            else
              umma_f16_pair(dtm, ad, bd, p.idesc, (kk > it.kb || k > 0) ? 1u : 0u);
          }
          if constexpr (CG == 1)
            umma_commit(&empty_bar[stage]);
          else
            umma_commit_pair(&empty_bar[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CG == 1)
          umma_commit(&tfull_bar[as]);
        else
          umma_commit_pair(&tfull_bar[as]);
        ++local;
      }
      SKPP_STAMP(p, TL_MMA_DONE);
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------ epilogue (4 warps)
    const uint32_t ew = warp - kEpiWarp0;    // TMEM lane quarter / staging owner
    const uint32_t row = ew * 32 + lane;      // tile row held by this thread
    const uint32_t et = threadIdx.x - kEpiWarp0 * 32;  // 0..127
    const bool leader = (et == 0);
    const uint32_t cta = blockIdx.x;  // workspace slots are per CTA (per row half)
    const bool out16 = p.out_dtype != SKPP_F32;
    // Launch epoch (Stream-K launches only): every CTA reads the epoch of the last
    // completed launch and arrives on a counter; the LAST arrival — after every
    // CTA has read it — advances the header for the next launch and resets the
    // counter.  All of it happens here, at the start, hidden behind the mainloop;
    // the next launch reads the header only after griddepcontrol.wait, i.e. after
    // this grid completed.  The leader alone publishes flags; phase 2 gets the
    // epoch through shared memory.
    uint32_t epoch = 0;
    if (s.sk_tiles && leader) {
      epoch = ld_relaxed_gpu(p.hdr) + 1u;
      asm volatile("fence.acq_rel.gpu;" ::: "memory");  // the read above precedes the arrival
      if (atomicAdd(p.hdr + 1, 1u) == gridDim.x - 1) {
        p.hdr[1] = 0u;
        p.hdr[0] = epoch;
      }
      // liveness protocol (phase 2): count this CTA as started; the last one to start
      // learns here whether any band was abandoned before it started (none can be after)
      const uint32_t par = epoch & 1u, np = par ^ 1u;
      uint32_t cleanup = 0;
      if (atom_add_acq_rel_gpu(p.hdr + kHdrStarted + par, 1u) == gridDim.x - 1)
        cleanup = ld_acquire_gpu(p.hdr + kHdrAbandon + par) != 0u ? 1u : 0u;
      nsplit_smem[4] = cleanup;
      // reset the other parity's words for the next Stream-K launch on this workspace
      // (it touches them only after this grid has completed)
      for (uint32_t i = blockIdx.x; i < kMaxCtas; i += gridDim.x) p.bstate[np * kMaxCtas + i] = 0u;
      if (blockIdx.x == 0) {
        p.hdr[kHdrStarted + np] = 0u;
        p.hdr[kHdrAbandon + np] = 0u;
      }
    }
    const uint32_t stg_base = smem_u32(stg) + ew * 2 * kStageBuf;
    uint32_t sbuf = 0;  // staging buffer toggle of this warp
    const uint64_t pol_c = l2_policy_evict_first();
    uint64_t split_tiles[1];
    uint32_t n_split = 0, sk_seen = 0, local = 0;
    Cursor cur;
    cursor_init(cur, s, x);
    Item it;
    while (cursor_next(cur, s, x, it)) {
      const uint32_t as = local & 1, aph = (local >> 1) & 1;
      mbar_wait(&tfull_bar[as], aph, 4);
      tc_fence_after();
      if (leader && local == 0) SKPP_STAMP(p, TL_EPI_FIRST);
      const uint32_t taddr = tmem_base + ((ew * 32) << 16) + as * BN;
      const bool partial = it.role != ROLE_FULL;
      const uint64_t slot = 2ull * cta + (sk_seen == 0 ? 0 : 1);
      uint64_t tm_, tn_;
      tile_rc<RASTER>(s, p.raster, it.tile, tm_, tn_);
      if (leader && rank == 0) record_item(p, x, local, it, tm_, tn_);
      const uint64_t tile_row0 = tm_ * TILE_M + rank * kBM;
      const uint64_t tile_col0 = tn_ * BN;
      // Owner reduction.  A split tile with exactly two contributors whose owner item is
      // this workgroup's LAST Stream-K item (its range began in an earlier tile) is finished
      // here instead of at the end of the launch: the other contributor x+1 holds the rest of the
      // tile as its FIRST Stream-K item, published long before this item completes, so the
      // epilogue adds that partial to its accumulator and stores C — (0 + p[x+1]) + p[x], the
      // phase-2 order, so the bits are identical — while the MMA moves on to the next item.  No
      // partial of this item is written, and x+1 skips the tile in phase 2 (the slot flag says
      // epoch | kOwnerDone).  The wait for x+1 is bounded (liveness); on timeout this item
      // publishes its partial as usual.
      bool reduce_peer = false;
      if (partial && it.role == ROLE_OWNER && it.peer_hi == (uint64_t)x + 1 && sk_seen >= 1 && !(p.debug & 16u)) {
        if (leader) {
          const uint32_t* pf = p.flags + 2ull * ((uint64_t)(x + 1) * CG + rank);
          uint32_t ok = 0;
          const long long t0 = clock64();
          while (true) {
            if (ld_acquire_gpu(pf) == epoch) {
              ok = 1;
              break;
            }
            if (clock64() - t0 > kOwnerWaitCycles) break;
            __nanosleep(32);
          }
          nsplit_smem[9] = ok;  // one owner item per workgroup at most: the word is written once
        }
        epi_bar_sync();  // the decision, and the peer partial (acquired by the leader), for all
        reduce_peer = nsplit_smem[9] != 0u;
      }
      if (partial && !reduce_peer) {
        // Partial slot layout: float4[BN/4][BM] ("column-group major"): a warp's
        // store of one column group is 32 consecutive rows = 512 contiguous bytes,
        // and a contributor's share of columns is one contiguous range.
        float4* dst = reinterpret_cast<float4*>(p.ws + slot * (uint64_t)(kBM * BN)) + row;
        // Only rows < M and columns < N are ever reduced (phase 2 bounds its bands the same
        // way: exact rows, 32-column chunks), so the partial of a ragged or skinny tile
        // (decode-like M = 1..127) costs only its valid rows and chunks on the SM's store
        // port.  A warp skips its TMEM reads when all its 32 rows are past M; threads skip
        // the stores of rows past M; every warp skips the 32-column chunks past N.
        const bool warp_rows_ok = tile_row0 + ew * 32 < p.M;
        const bool warp_rows_all = tile_row0 + ew * 32 + 32 <= p.M;
        const bool row_ok = tile_row0 + row < p.M;
        const uint64_t cols_left = p.N - tile_col0;
        const int chunks_ok = cols_left >= (uint64_t)BN ? BN / 32 : (int)((cols_left + 31) / 32);
        if (!p.ragged || (warp_rows_all && chunks_ok == BN / 32)) {  // full tile: every row and column chunk
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t w[32];
            tmem_ld_32(taddr + c * 32, w);
            tmem_ld_wait();
            if (c == BN / 32 - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) release_acc(&tempty_bar[as]);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
              dst[(c * 8 + j) * kBM] = make_float4(__uint_as_float(w[4 * j]), __uint_as_float(w[4 * j + 1]),
                                                   __uint_as_float(w[4 * j + 2]), __uint_as_float(w[4 * j + 3]));
          }
        } else {
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            if (warp_rows_ok && c < chunks_ok) {
              uint32_t w[32];
              tmem_ld_32(taddr + c * 32, w);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (row_ok)
                  dst[(c * 8 + j) * kBM] = make_float4(__uint_as_float(w[4 * j]), __uint_as_float(w[4 * j + 1]),
                                                     __uint_as_float(w[4 * j + 2]), __uint_as_float(w[4 * j + 3]));
            }
            if (c == BN / 32 - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) release_acc(&tempty_bar[as]);
            }
          }
        }
        if (leader && n_split == 0) SKPP_STAMP(p, TL_PART_ISSUED);
        // publish: every thread's stores happen-before the barrier; the leader's
        // gpu-scope release then covers them (release is cumulative — CUTLASS's stream-K
        // barrier publishes the same way).  st.release.gpu already emits the MEMBAR.GPU; an
        // explicit fence.acq_rel.gpu before it doubled the membar and cost 2-5% per launch on
        // fixup-bound shapes (decode 16x4096x4096 -4.5%, cfg1 -5%, cfg2 -2.5%, same-box A/B).
        epi_bar_sync();
        if (leader) st_release_gpu(p.flags + slot, epoch);
        if (leader && n_split == 0) SKPP_STAMP(p, TL_PART_FLAG);
        // the CTA reduces (phase 2) only the tile of its FIRST Stream-K item
        if (sk_seen == 0) split_tiles[n_split++] = it.tile - s.dp_tiles;
      } else {
        // One chunk = 128 bytes of a row: 32 fp32 columns or 64 16-bit columns.
        const int ccols = out16 ? 64 : 32;
#pragma unroll 1
        for (int c = 0; c < BN / ccols; ++c) {
          uint32_t w[32];
          if (out16) {
            uint32_t r0[32], r1[32];
            tmem_ld_32(taddr + c * 64, r0);
            tmem_ld_32(taddr + c * 64 + 32, r1);
            tmem_ld_wait();
            if (reduce_peer) {  // owner reduction: add the other contributor's 64 columns, 32 at a time
              const float4* src = reinterpret_cast<const float4*>(p.ws) +
                                  (2ull * ((uint64_t)(x + 1) * CG + rank)) * (uint64_t)(kBM * (BN / 4)) +
                                  (uint64_t)(c * 16) * kBM + row;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                uint32_t* r = h ? r1 : r0;
                float4 q[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) q[j] = ld_cg_f4(src + (uint64_t)(h * 8 + j) * kBM);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  r[4 * j] = __float_as_uint((0.f + q[j].x) + __uint_as_float(r[4 * j]));
                  r[4 * j + 1] = __float_as_uint((0.f + q[j].y) + __uint_as_float(r[4 * j + 1]));
                  r[4 * j + 2] = __float_as_uint((0.f + q[j].z) + __uint_as_float(r[4 * j + 2]));
                  r[4 * j + 3] = __float_as_uint((0.f + q[j].w) + __uint_as_float(r[4 * j + 3]));
                }
              }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              w[j] = pack2(__uint_as_float(r0[2 * j]), __uint_as_float(r0[2 * j + 1]), p.out_dtype);
              w[16 + j] = pack2(__uint_as_float(r1[2 * j]), __uint_as_float(r1[2 * j + 1]), p.out_dtype);
            }
          } else if (reduce_peer) {
            // the other contributor's 32 columns of this row (column groups c*8 .. c*8+7 of its
            // slot, float4[BN/4][128]), loaded before the TMEM read so the L2 latency overlaps
            const float4* src = reinterpret_cast<const float4*>(p.ws) +
                                (2ull * ((uint64_t)(x + 1) * CG + rank)) * (uint64_t)(kBM * (BN / 4)) +
                                (uint64_t)(c * 8) * kBM + row;
            float4 q[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) q[j] = ld_cg_f4(src + (uint64_t)j * kBM);
            tmem_ld_32(taddr + c * 32, w);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              w[4 * j] = __float_as_uint((0.f + q[j].x) + __uint_as_float(w[4 * j]));
              w[4 * j + 1] = __float_as_uint((0.f + q[j].y) + __uint_as_float(w[4 * j + 1]));
              w[4 * j + 2] = __float_as_uint((0.f + q[j].z) + __uint_as_float(w[4 * j + 2]));
              w[4 * j + 3] = __float_as_uint((0.f + q[j].w) + __uint_as_float(w[4 * j + 3]));
            }
          } else {
            tmem_ld_32(taddr + c * 32, w);
            tmem_ld_wait();
          }
          if (c == BN / ccols - 1) {
            // all TMEM reads of this item complete: hand the accumulator stage back
            tc_fence_before();
            __syncwarp();
            if (lane == 0) release_acc(&tempty_bar[as]);
          }
          if (p.c_tma) {
            const uint32_t buf = stg_base + sbuf * kStageBuf;
            if (lane == 0) bulk_wait_read<1>();  // the store that used `buf` has read it
            __syncwarp();
            const uint32_t rbase = buf + lane * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              st_shared_v4(rbase + ((j ^ (lane & 7)) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2],
                           w[4 * j + 3]);
            fence_async_shared();
            __syncwarp();
            if (lane == 0) {
              if (p.l2_hints)
                tma_store_2d_hint(&tmC, stg + (buf - smem_u32(stg)), (int32_t)(tile_col0 + c * ccols),
                                  (int32_t)(tile_row0 + ew * 32), pol_c);
              else
                tma_store_2d(&tmC, stg + (buf - smem_u32(stg)), (int32_t)(tile_col0 + c * ccols),
                             (int32_t)(tile_row0 + ew * 32));
              bulk_commit();
            }
            sbuf ^= 1;
          } else {
            store_row_direct(p, tile_row0 + row, tile_col0 + c * ccols, w);
          }
        }
        if (reduce_peer && leader) st_release_gpu(p.flags + slot, epoch | kOwnerDone);
      }
      if (it.phase == PHASE_SK) ++sk_seen;
      ++local;
    }
    if (leader && rank == 0 && p.trace_counts != nullptr) p.trace_counts[x] = (int64_t)local;
    if (leader) SKPP_STAMP(p, TL_PHASE1);

    // hand the split tiles to the whole CTA for phase 2
    if (leader) {
      split_smem[0] = split_tiles[0];
      nsplit_smem[0] = n_split;
      nsplit_smem[3] = epoch;
    }
    if (lane == 0) bulk_wait<0>();  // staging must outlive the in-flight TMA stores
  }

  // ---- phase 2 (all 8 warps): cooperative fixed-order reduction of the split
  // tile of this CTA's first Stream-K item.  The reducers of tile u are the
  // contributors whose first Stream-K item lies in u: x0 (only if its range
  // starts exactly at the tile) .. x1, so every CTA reduces at most one tile
  // and every split tile has at least one reducer (x1).  Reducer idx of nr
  // owns the row band [idx*128/nr, (idx+1)*128/nr) of its row half and sums it
  // over ALL nc contributors' slots in a fixed order (band_sum).  One pass
  // when the owner x0 has published by the time the peers have (every
  // contributor ends its mainloop together); otherwise the peers are summed
  // first and x0 — whose item may be its LAST — is added when it lands.
  //
  // Liveness without co-residency.  Phase 1 never waits on another CTA, so once every
  // CTA of the launch has STARTED, every partial will be published and the flag waits
  // below terminate.  Each CTA counts itself on started[par] at kernel start (hidden
  // behind the mainloop).  A reducer whose flag wait exceeds p.abandon_cycles reads that
  // counter: if every CTA has started it simply keeps waiting; otherwise (some CTA is
  // not resident — another grid holds its SM) it marks its band abandoned and exits,
  // freeing its SM.  The LAST CTA to start (it sees every abandonment made before it
  // started, and none can be made after) reduces the abandoned bands at its end.  A race
  // between a reducer that abandons just as the last CTA starts is settled by one CAS on
  // the band state (1 abandoned -> 2 claimed by the last starter | 3 taken back).
  // Normally nothing times out: the cost is one atomic per CTA at kernel start.
  __syncwarp();          // producer / MMA lanes rejoin their warps
  phase2_bar_sync();     // split tiles published by the epilogue
  if (s.sk_tiles) {
    const uint32_t ft = threadIdx.x;
    const uint32_t n_split = nsplit_smem[0];
    const uint32_t epoch = nsplit_smem[3];  // read by the epilogue leader at kernel start
    const uint32_t par = epoch & 1u;
    constexpr uint32_t V = BN / 4;  // float4 column groups per tile row
    static_assert(C::RING_BYTES >= (uint32_t)kBM * (V + 1) * 16 + 4096, "phase-2 band stage + claim list");
    const float4* wsv = reinterpret_cast<const float4*>(p.ws);
    const uint64_t slot_v = (uint64_t)kBM * V;  // float4 per slot
    volatile uint32_t* peers_seen = nsplit_smem + 2;
    volatile uint32_t* p2w = nsplit_smem + 5;  // [0] a wait timed out, [1] decision, [2] owner ready, [3] claims,
                                               // [5] owner flag of the second pass (= nsplit_smem[10]; [9] is the
                                               // phase-1 owner-reduction decision)
    const uint32_t stage = smem_u32(smem);     // idle operand ring: float4 [row][V+1]
    // Reduce reducer (xr, rk)'s band of split tile u and store it to C.  `bounded`: flag
    // waits may time out and hand the band to the last starter (the CTA's own band);
    // otherwise every CTA has started and the waits are plain.
    auto reduce_band = [&](uint64_t u, uint64_t xr, uint32_t rk, bool bounded, bool stamps) {
      const uint64_t x0 = udiv(u * s.ipt, s.ipw);
      const uint64_t x1 = udiv((u + 1) * s.ipt - 1, s.ipw);
      const uint32_t nc = (uint32_t)(x1 - x0 + 1);
      const bool aligned = x0 * s.ipw == u * s.ipt;  // x0's range starts at tile u
      const uint64_t r_lo = x0 + (aligned ? 0 : 1);
      const uint32_t nr = (uint32_t)(x1 - r_lo + 1);
      const uint32_t idx = (uint32_t)(xr - r_lo);
      // ragged problems only (M or N not a multiple of the tile): bound the band by the
      // rows / column chunks the contributors wrote (phase 1 skips the rest)
      uint32_t rows_ok = kBM, Vv = V;
      uint64_t ttm, ttn;
      tile_rc<RASTER>(s, p.raster, s.dp_tiles + u, ttm, ttn);
      if (p.ragged) {
        const uint64_t tile_rows0 = ttm * TILE_M + rk * kBM;
        if (tile_rows0 >= p.M)
          rows_ok = 0;  // this row half of the tile is entirely past M: empty band below
        else if (p.M - tile_rows0 < (uint64_t)kBM)
          rows_ok = (uint32_t)(p.M - tile_rows0);  // exact: phase 1 wrote rows < M only
        const uint64_t tile_cols0 = ttn * BN;
        if (p.N - tile_cols0 < (uint64_t)BN) Vv = (uint32_t)((p.N - tile_cols0 + 31) / 32 * 32 / 4);
      }
      const uint32_t R0 = (uint32_t)udiv((uint64_t)idx * rows_ok, nr);
      const uint32_t R1 = (uint32_t)udiv((uint64_t)(idx + 1) * rows_ok, nr);
      if (R0 == R1) return;
      // contributor x0+t wrote its first Stream-K item (slot 2*cta), except x0
      // when its range starts inside an earlier tile (tile u is its last item)
      const uint64_t slot0 = 2 * (x0 * CG + rk) + (aligned ? 0 : 1);
      const uint64_t row0 = ttm * TILE_M + rk * kBM + R0;
      const uint64_t gcol0 = ttn * BN;
      const ReduceArgs ra{wsv, slot_v, slot0, x0, rk, nc,
                          (p.timeline && stamps) ? p.timeline + (uint64_t)blockIdx.x * TL_EVENTS : nullptr};
      uint32_t* bst = p.bstate + par * kMaxCtas + xr * CG + rk;
      // Peer flags are awaited by one thread each; thread kThreads-1 polls the
      // owner's flag until either it is up or every peer has been seen.
      uint32_t limit = bounded ? p.abandon_cycles : 0xFFFFFFFFu;
      while (true) {
        if (ft == 0) {
          *peers_seen = 0u;
          p2w[0] = 0u;
        }
        phase2_bar_sync();
        const long long t0 = clock64();
        if (ft < kThreads - 1) {
          for (uint32_t t = 1 + ft; t < nc; t += kThreads - 1) {
            if (!wait_flag_until(p.flags + 2 * ((x0 + t) * CG + rk), epoch, t0, limit)) {
              atomicOr(const_cast<uint32_t*>(p2w), 1u);  // read by the owner poller meanwhile
              break;
            }
            atomicAdd(const_cast<uint32_t*>(peers_seen), 1u);
          }
        }
        if (ft == kThreads - 1) {
          const uint32_t want = nc - 1;
          uint32_t ready = 0;
          while (true) {
            const uint32_t v = ld_acquire_gpu(p.flags + slot0);
            if (v == epoch) { ready = 1; break; }
            if (v == (epoch | kOwnerDone)) { ready = 2; break; }  // finished by the owner
            if (*peers_seen >= want || p2w[0] != 0u) break;
            if (clock64() - t0 > (long long)limit) {
              atomicOr(const_cast<uint32_t*>(p2w), 1u);
              break;
            }
          }
          p2w[2] = ready;
        }
        phase2_bar_sync();
        if (p2w[0] == 0u) break;
        // a wait timed out: keep waiting if every CTA has started, else hand the band off
        if (ft == 0) p2w[1] = limit == 0xFFFFFFFFu ? 1u : abandon_or_wait(p.hdr, par, bst);
        phase2_bar_sync();
        if (p2w[1] == 0u) {
          phase2_bar_sync();  // p2w is rewritten by the next band
          return;             // the last CTA to start reduces this band
        }
        limit = 0xFFFFFFFFu;
      }
      if (stamps) SKPP_STAMP(p, TL_WAITED);
      if (p2w[2] == 2u) {  // the owner reduced the tile in phase 1 (owner reduction): nothing to do
        phase2_bar_sync();
        return;
      }
      const bool owner_ready = p2w[2] != 0u && !(p.debug & 1u);
      const uint32_t nrows = R1 - R0;
      band_reduce<CG, V>(ra, R0, nrows, Vv, 0, owner_ready ? nc : nc - 1, false, stage, ft);
      if (stamps) SKPP_STAMP(p, TL_SUM1);
      if (!owner_ready) {
        if (ft == 0) {
          uint32_t go = 1u;
          uint32_t got = wait_owner_flag(p.flags + slot0, epoch, clock64(), limit);
          if (got == 0u) {
            go = abandon_or_wait(p.hdr, par, bst);
            if (go) got = wait_owner_flag(p.flags + slot0, epoch, clock64(), 0xFFFFFFFFu);
          }
          p2w[1] = go;
          p2w[5] = got;  // not p2w[2]: other threads may still be reading it (owner_ready)
        }
        phase2_bar_sync();  // also orders the stage writes above before the re-reads below
        if (p2w[1] == 0u || p2w[5] == 2u) {
          phase2_bar_sync();
          return;  // handed to the last starter, or finished by the owner (peer sums discarded)
        }
        band_reduce<CG, V>(ra, R0, nrows, Vv, nc - 1, nc, true, stage, ft);
        if (stamps) SKPP_STAMP(p, TL_SUM2);
      }
      phase2_bar_sync();
      band_store<V>(p, stage, nrows, Vv, row0, gcol0, ft);
      if (bounded && ft == 0) SKPP_STAMP(p, TL_P2_STORED);
      phase2_bar_sync();  // stage and p2w are reused by the next band
    };
    for (uint32_t si = 0; si < n_split; ++si)
      reduce_band(split_smem[si], x, rank, true, ft == kEpiWarp0 * 32 && si == 0);
    // The last CTA to start: reduce every band abandoned in this launch.
    if (nsplit_smem[4] != 0u) {
      uint32_t* list = reinterpret_cast<uint32_t*>(smem + C::RING_BYTES - 4096);
      if (ft == 0) p2w[3] = 0u;
      phase2_bar_sync();
      for (uint32_t c = ft; c < gridDim.x; c += kThreads) {
        uint32_t* st = p.bstate + par * kMaxCtas + c;
        if (ld_acquire_gpu(st) == 1u && atom_cas_acq_rel_gpu(st, 1u, 2u) == 1u)
          list[atomicAdd(const_cast<uint32_t*>(p2w + 3), 1u)] = c;
      }
      phase2_bar_sync();
      const uint32_t n_claimed = p2w[3];
      for (uint32_t i = 0; i < n_claimed; ++i) {
        const uint32_t c = list[i];
        const uint64_t xr = c / CG;
        reduce_band(udiv(xr * s.ipw, s.ipt), xr, c % CG, false, false);
      }
    }
    if (ft == kEpiWarp0 * 32) SKPP_STAMP(p, TL_PHASE2);
  }
  if (threadIdx.x == 0 && p.timeline) {
    SKPP_STAMP(p, TL_END);
    p.timeline[(uint64_t)blockIdx.x * TL_EVENTS + TL_CLK_END] = clock64();
  }

  tc_fence_before();
  if constexpr (CG == 2) {
    cluster_sync();  // the peer's MMAs into this CTA's TMEM are complete on both sides
  } else {
    __syncthreads();
  }
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(C::TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(C::TMEM_COLS)
                   : "memory");
  }
}

// Test hook (skpp_test_hold_sms): CTAs that occupy SMs until *release != 0 (or ~35 s).
__global__ void hold_sms_kernel(const volatile uint32_t* release) {
  if (threadIdx.x != 0) return;
  const long long t0 = clock64();
  while (*release == 0u && clock64() - t0 < (1ll << 36)) __nanosleep(2000);
}

// Decode-only: every CTA walks its items with the same cursor and records them.
__global__ void schedule_trace_kernel(const Sched s, uint32_t band, int64_t* trace, uint64_t cap,
                                      int64_t* counts) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= s.g) return;
  Cursor cur;
  cursor_init(cur, s, x);
  Item it;
  uint64_t n = 0;
  while (cursor_next(cur, s, x, it)) {
    if (n < cap) {
      uint64_t tm, tn;
      tile_coords(s, band, it.tile, tm, tn);
      write_trace_row(trace + ((uint64_t)x * cap + n) * SKPP_TRACE_FIELDS, it, tm, tn);
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

static int make_map(CUtensorMap* map, const void* base, CUtensorMapDataType dt, uint32_t esize,
                    uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t box_inner,
                    uint32_t box_outer, CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return SKPP_ELAUNCH;
  }
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld_elems * esize};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
    return SKPP_ELAUNCH;
  }
  return SKPP_OK;
}

static CUtensorMapDataType map_dtype(int d) {
  return d == SKPP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
         : d == SKPP_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                         : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
}

static void sched_from_c(const skpp_sched_t& c, Sched& s) {
  s.dp_tiles = c.dp_tiles;
  s.sk_tiles = c.sk_tiles;
  s.ipt = c.iters_per_tile;
  s.ipw = c.ipw;
  s.sk_iters = c.sk_iters;
  s.n_tiles = c.n_tiles;
  s.g = c.g;
  s.sk_first = c.sk_first;
}

static uint64_t* g_timeline = nullptr;  // skpp_debug_timeline
static int g_pdl = 1;                    // skpp_set_pdl
static int g_coop = 0;                   // skpp_set_cooperative
static int g_b3d = 1;                    // skpp_set_b3d
static int g_a3d = 1;                    // skpp_set_a3d
static int g_l2_prefetch = 2;            // skpp_set_l2_prefetch (k-blocks)
static int g_l2_hints = 1;               // skpp_set_l2_hints
static int g_debug = 0;                  // skpp_set_debug

// A prepared launch: tensor maps, parameters and kernel, built once.
struct Plan {
  const void* func;
  uint32_t smem;
  uint32_t block_n;
  uint32_t cg;      // CTAs per workgroup (2 = cta_group::2 pair)
  CUtensorMap ma, mb, mc;
  GemmParams p;
  skpp_sched_t cs;
  uint64_t ws_bytes;
  void* ws_bound;   // workspace the parameters point into
};

template <int BN, int BK, int CG, bool RASTER = false>
static int kernel_setup(const void** func, uint32_t* smem) {
  using C = Cfg<BN, BK, CG>;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(streamk_gemm_kernel<BN, BK, CG, RASTER>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (err == cudaSuccess && CG == 2)
      err = cudaFuncSetAttribute(streamk_gemm_kernel<BN, BK, CG, RASTER>,
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
  });
  if (err != cudaSuccess) {
    set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(err));
    return SKPP_ELAUNCH;
  }
  *func = reinterpret_cast<const void*>(streamk_gemm_kernel<BN, BK, CG, RASTER>);
  *smem = C::SMEM;
  return SKPP_OK;
}

// Co-resident workgroups (CTAs, or CTA pairs when CG == 2) of one launch.
template <int BN, int BK, int CG>
static int max_coresident_impl(int* groups) {
  constexpr int kMaxDev = 64;
  static int cache[kMaxDev] = {0};  // 0 = not yet queried
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur >= 0 && cur < kMaxDev && cache[cur] > 0) {
    *groups = cache[cur];
    return SKPP_OK;
  }
  const void* func;
  uint32_t smem;
  int rc = kernel_setup<BN, BK, CG>(&func, &smem);
  if (rc) return rc;
  int sms = 0, n = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cur);
  cudaError_t e;
  if constexpr (CG == 1) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, streamk_gemm_kernel<BN, BK, CG>, kThreads, smem);
    n *= sms;
  } else {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaOccupancyMaxActiveClusters(&n, streamk_gemm_kernel<BN, BK, CG>, &cfg);
  }
  if (e != cudaSuccess) {
    set_error(std::string("occupancy query: ") + cudaGetErrorString(e));
    return SKPP_ELAUNCH;
  }
  *groups = n;
  if (cur >= 0 && cur < kMaxDev) cache[cur] = n;
  return SKPP_OK;
}

// Calls f(integral_constant<BN>, integral_constant<BK>, integral_constant<CG>)
// for the instantiated tile shapes: blk_m = 128 (one CTA) or 256 (CTA pair).
template <typename F>
static int dispatch_tile(const skpp_tile_t* t, F&& f) {
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  using I16 = std::integral_constant<int, 16>;
  using I32 = std::integral_constant<int, 32>;
  using I64 = std::integral_constant<int, 64>;
  using I128 = std::integral_constant<int, 128>;
  using I256 = std::integral_constant<int, 256>;
  using I128k = std::integral_constant<int, 128>;
  if (t->blk_m == (uint32_t)kBM) {
    if (t->blk_k == 128) {
      if (t->blk_n == 64) return f(I64{}, I128k{}, I1{});
      if (t->blk_n == 128) return f(I128{}, I128k{}, I1{});
      if (t->blk_n == 256) return f(I256{}, I128k{}, I1{});
    } else if (t->blk_k == 64) {
      if (t->blk_n == 64) return f(I64{}, I64{}, I1{});
      if (t->blk_n == 128) return f(I128{}, I64{}, I1{});
      if (t->blk_n == 256) return f(I256{}, I64{}, I1{});
    } else if (t->blk_k == 32) {
      if (t->blk_n == 64) return f(I64{}, I32{}, I1{});
      if (t->blk_n == 128) return f(I128{}, I32{}, I1{});
      if (t->blk_n == 256) return f(I256{}, I32{}, I1{});
    } else if (t->blk_k == 16) {
      if (t->blk_n == 64) return f(I64{}, I16{}, I1{});
      if (t->blk_n == 128) return f(I128{}, I16{}, I1{});
      if (t->blk_n == 256) return f(I256{}, I16{}, I1{});
    }
  } else if (t->blk_m == 2u * kBM) {
    if (t->blk_k == 128) {
      if (t->blk_n == 128) return f(I128{}, I128k{}, I2{});
      if (t->blk_n == 256) return f(I256{}, I128k{}, I2{});
    } else if (t->blk_k == 64) {
      if (t->blk_n == 128) return f(I128{}, I64{}, I2{});
      if (t->blk_n == 256) return f(I256{}, I64{}, I2{});
    } else if (t->blk_k == 32) {
      if (t->blk_n == 128) return f(I128{}, I32{}, I2{});
      if (t->blk_n == 256) return f(I256{}, I32{}, I2{});
    }
  }
  return SKPP_ETILE;
}

static int check_device() {
  constexpr int kMaxDev = 64;
  static int verified[kMaxDev] = {0};  // 1 = sm_100 checked
  int dev = 0, major = 0, minor = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    set_error(std::string("no CUDA device: ") + cudaGetErrorString(e));
    return SKPP_EARCH;
  }
  if (dev >= 0 && dev < kMaxDev && verified[dev]) return SKPP_OK;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) {
    set_error("libskpp kernels are built for sm_100a (B200); device is sm_" +
              std::to_string(major) + std::to_string(minor));
    return SKPP_EARCH;
  }
  if (dev >= 0 && dev < kMaxDev) verified[dev] = 1;
  return SKPP_OK;
}

}  // namespace skpp

using namespace skpp;

extern "C" int skpp_tile_supported(const skpp_tile_t* t) {
  if (!t) return 0;
  return dispatch_tile(t, [](auto, auto, auto) { return SKPP_OK; }) == SKPP_OK ? 1 : 0;
}

extern "C" uint64_t skpp_workspace_bytes(const skpp_problem_t* p, const skpp_tile_t* t,
                                         uint32_t g) {
  (void)p;
  if (!t) return 0;
  // two partial slots (first / last Stream-K item) of 128 x blk_n fp32 per CTA
  const uint64_t ctas = (uint64_t)g * (t->blk_m > (uint32_t)kBM ? 2 : 1);
  return kWsCtlBytes + 2ull * ctas * kBM * t->blk_n * 4;
}

extern "C" void skpp_debug_timeline(uint64_t* device_buffer) { g_timeline = device_buffer; }
extern "C" void skpp_set_pdl(int enable) { g_pdl = enable ? 1 : 0; }
extern "C" void skpp_set_cooperative(int enable) { g_coop = enable ? 1 : 0; }
extern "C" void skpp_set_b3d(int enable) { g_b3d = enable ? 1 : 0; }
extern "C" void skpp_set_a3d(int enable) { g_a3d = enable ? 1 : 0; }
extern "C" void skpp_set_l2_prefetch(int k_blocks) { g_l2_prefetch = k_blocks > 0 ? k_blocks : 0; }
extern "C" void skpp_set_l2_hints(int enable) { g_l2_hints = enable ? 1 : 0; }
extern "C" void skpp_set_debug(int flags) { g_debug = flags; }

extern "C" int skpp_set_device(int device) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    set_error(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    return SKPP_ELAUNCH;
  }
  return SKPP_OK;
}

extern "C" int skpp_stream_is_capturing(void* stream) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(reinterpret_cast<cudaStream_t>(stream), &st);
  if (e != cudaSuccess) {
    set_error(std::string("cudaStreamIsCapturing: ") + cudaGetErrorString(e));
    return SKPP_ELAUNCH;
  }
  return st == cudaStreamCaptureStatusActive ? 1 : 0;
}

extern "C" int skpp_test_hold_sms(uint32_t ctas, uint32_t smem_bytes, const uint32_t* release, void* stream) {
  if (!release || ctas == 0) {
    set_error("hold_sms: null release flag or no CTAs");
    return SKPP_EINVAL;
  }
  cudaError_t e = cudaFuncSetAttribute(hold_sms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
  if (e == cudaSuccess) {
    hold_sms_kernel<<<ctas, 32, smem_bytes, reinterpret_cast<cudaStream_t>(stream)>>>(release);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    set_error(std::string("hold_sms launch: ") + cudaGetErrorString(e));
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

static int max_coresident_dispatch(const skpp_tile_t* t, int* groups) {
  return dispatch_tile(t, [&](auto bn, auto bk, auto cg) {
    return max_coresident_impl<decltype(bn)::value, decltype(bk)::value, decltype(cg)::value>(groups);
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

extern "C" int skpp_plan_create(const skpp_problem_t* p, const skpp_tile_t* t,
                                const skpp_policy_t* pol, uint32_t g, const skpp_operands_t* ops,
                                int64_t* trace, uint64_t trace_cap, int64_t* trace_counts,
                                void** plan_out) {
  if (!p || !t || !pol || !ops || !plan_out) {
    set_error("null argument");
    return SKPP_EINVAL;
  }
  *plan_out = nullptr;
  if (!skpp_tile_supported(t)) {
    set_error("tile shape " + std::to_string(t->blk_m) + "x" + std::to_string(t->blk_n) + "x" +
              std::to_string(t->blk_k) +
              " is not implemented by the sm_100a kernel (blk_m=128, blk_n in {64,128,256}, "
              "blk_k in {16,32,64,128}; blk_m=256: blk_n in {128,256}, blk_k in {32,64,128})");
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
  Plan* pl = new Plan;
  memset(pl, 0, sizeof(Plan));
  rc = skpp_sched_make(p, t, g, pol, &pl->cs);
  if (rc) {
    delete pl;
    return rc;
  }
  if (pl->cs.sk_tiles > 0) {
    int co = 0;
    rc = max_coresident_dispatch(t, &co);
    if (rc) {
      delete pl;
      return rc;
    }
    // Persistent grid: one wave of workgroups.  (Liveness does not depend on it — see the
    // phase-2 protocol — but a grid of several waves would serialise its fixups.)
    if ((int64_t)g > co || (uint64_t)g * (t->blk_m > (uint32_t)kBM ? 2 : 1) > kMaxCtas) {
      set_error("g=" + std::to_string(g) + " exceeds the " + std::to_string(co) +
                " co-resident workgroups of a persistent Stream-K grid");
      delete pl;
      return SKPP_EGRID;
    }
  }
  rc = dispatch_tile(t, [&](auto bn, auto bk, auto cg) {
    return kernel_setup<decltype(bn)::value, decltype(bk)::value, decltype(cg)::value>(&pl->func, &pl->smem);
  });
  if (rc) {
    delete pl;
    return rc;
  }
  pl->block_n = t->blk_n;
  pl->cg = t->blk_m / kBM;
  const uint32_t BK = t->blk_k;
  const CUtensorMapSwizzle aswz = BK >= 64   ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : BK == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                             : CU_TENSOR_MAP_SWIZZLE_32B;
  const CUtensorMapDataType in_dt = map_dtype(ops->in_dtype);
  // BK = 128 with K % 64 == 0: A as (k in chunk, row, 64-deep chunk) so one 3-D box fills
  // both sub-tiles [chunk][128 rows][64] (the per-SM TMA stage rate falls with fewer ops).
  // Otherwise a chunk could run past a row end, so two 2-D boxes per stage.
  // M < 128: the A box covers only round_up(M, 8) rows (a decode-like M = 1 box would be
  // 99% out of bounds, and TMA's OOB fill is far from free: M = 1 x 14336 x 4096 ran 1.6x
  // slower than M = 128).  The tile's other rows of shared memory keep stale data, so the
  // MMA produces junk there — in accumulator rows >= M, which are never stored or reduced.
  const uint32_t a_rows = p->m < (uint64_t)kBM ? (uint32_t)((p->m + 7) / 8 * 8) : (uint32_t)kBM;
  const bool a3d = g_a3d && BK > 64 && p->k % 64 == 0 && a_rows == (uint32_t)kBM;
  if (a3d) {
    auto fn = encode_fn();
    const cuuint64_t dims[3] = {64, p->m, p->k / 64};
    const cuuint64_t strides[2] = {(cuuint64_t)ops->lda * 2, 128};
    const cuuint32_t box[3] = {64, (cuuint32_t)kBM, BK / 64};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn ? fn(&pl->ma, in_dt, 3, const_cast<void*>(ops->a), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
                    : CUDA_ERROR_NOT_SUPPORTED;
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled (3-D A) failed with CUresult " + std::to_string((int)r));
      rc = SKPP_ELAUNCH;
    }
  } else {
    rc = make_map(&pl->ma, ops->a, in_dt, 2, p->k, p->m, (uint64_t)ops->lda, BK > 64 ? 64 : BK, a_rows, aswz);
  }
  const uint32_t bnc = t->blk_n / (t->blk_m / kBM);  // B columns per CTA
  const bool b3d = g_b3d && p->n % 64 == 0 && bnc > 64;
  if (!rc && b3d) {
    // (n in chunk, k, chunk) view of B: one TMA op per stage fills [chunk][k][64];
    // only when N is a multiple of 64, so no chunk reads past a row.
    auto fn = encode_fn();
    const cuuint64_t dims[3] = {64, p->k, p->n / 64};
    const cuuint64_t strides[2] = {(cuuint64_t)ops->ldb * 2, 128};
    const cuuint32_t box[3] = {64, BK, bnc / 64};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn ? fn(&pl->mb, in_dt, 3, const_cast<void*>(ops->b), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
                    : CUDA_ERROR_NOT_SUPPORTED;
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled (3-D B) failed with CUresult " + std::to_string((int)r));
      rc = SKPP_ELAUNCH;
    }
  } else if (!rc) {
    rc = make_map(&pl->mb, ops->b, in_dt, 2, p->n, p->k, (uint64_t)ops->ldb, 64, BK,
                  CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (rc) {
    delete pl;
    return rc;
  }
  GemmParams& gp = pl->p;
  sched_from_c(pl->cs, gp.s);
  gp.M = (uint32_t)p->m;
  gp.N = (uint32_t)p->n;
  const uint32_t ab = ops->in_dtype == SKPP_BF16 ? 1u : 0u;
  gp.idesc = (1u << 4) | (ab << 7) | (ab << 10) | (0u << 15) | (1u << 16) |
             ((uint32_t)(t->blk_n >> 3) << 17) | ((uint32_t)(t->blk_m >> 4) << 24);
  gp.out_dtype = ops->out_dtype;
  gp.b3d = b3d ? 1 : 0;
  gp.a3d = a3d ? 1 : 0;
  gp.a_tx = a_rows * BK * 2;
  gp.l2_prefetch = (uint32_t)g_l2_prefetch;
  // Tile order: a declared tuning parameter of the tile (skpp_tile_t.tile_order), selected
  // by the sweep like the tile shape; 0 = the reference's row-major order.  Banded orders
  // measured +11% on 4096x14336x4096 and +4% on 8192^3, neutral-to-slower below 4 waves.
  gp.raster = t->tile_order;
  if (gp.raster) {
    rc = dispatch_tile(t, [&](auto bn, auto bk, auto cg) {
      return kernel_setup<decltype(bn)::value, decltype(bk)::value, decltype(cg)::value, true>(&pl->func,
                                                                                            &pl->smem);
    });
    if (rc) {
      delete pl;
      return rc;
    }
  }
  gp.l2_hints = g_l2_hints ? 1 : 0;
  gp.debug = (uint32_t)g_debug;
  // ~20 us at 1.9 GHz: far above any wait of a fully resident grid (flags trail the mainloop
  // by ~1-3 us), short enough that a reducer blocked by a non-resident peer frees its SM soon
  gp.abandon_cycles = (g_debug & 2) ? 0u : 40000u;
  // Skip-invalid-rows/columns mode only where it saves at least half a tile of partial
  // bytes (decode-like M, narrow N): on other shapes the bounds checks cost more than the
  // 32-row / 32-column chunks they would skip.
  {
    const uint64_t mr = p->m % t->blk_m, nr = p->n % t->blk_n;
    gp.ragged = ((mr != 0 && 2 * mr <= t->blk_m) || (nr != 0 && 2 * nr <= t->blk_n)) ? 1u : 0u;
  }
  gp.C = ops->c;
  gp.ldc = (uint64_t)ops->ldc;
  const uint32_t esz = ops->out_dtype == SKPP_F32 ? 4 : 2;
  gp.c_vec_ok = ((reinterpret_cast<uintptr_t>(ops->c) % 16) == 0 && (gp.ldc * esz) % 16 == 0) ? 1 : 0;
  if (gp.c_vec_ok) {
    rc = make_map(&pl->mc, ops->c, map_dtype(ops->out_dtype), esz, p->n, p->m, gp.ldc,
                  128 / esz, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) {
      delete pl;
      return rc;
    }
    gp.c_tma = 1;
  }
  gp.trace = trace;
  gp.trace_cap = trace_cap;
  gp.trace_counts = trace_counts;
  pl->ws_bytes = pl->cs.sk_tiles ? skpp_workspace_bytes(p, t, g) : 0;
  *plan_out = pl;
  return SKPP_OK;
}

extern "C" uint64_t skpp_plan_workspace_bytes(const void* plan) {
  return plan ? static_cast<const Plan*>(plan)->ws_bytes : 0;
}

extern "C" void skpp_plan_destroy(void* plan) { delete static_cast<Plan*>(plan); }

extern "C" int skpp_plan_launch(void* plan, void* workspace, uint64_t workspace_bytes,
                                void* stream) {
  Plan* pl = static_cast<Plan*>(plan);
  if (!pl) {
    set_error("null plan");
    return SKPP_EINVAL;
  }
  GemmParams& gp = pl->p;
  if (pl->cs.sk_tiles > 0) {
    if (workspace == nullptr || workspace_bytes < pl->ws_bytes) {
      set_error("workspace too small: need " + std::to_string(pl->ws_bytes) + " bytes");
      return SKPP_EWORKSPACE;
    }
    if (pl->ws_bound != workspace) {
      uint8_t* base = reinterpret_cast<uint8_t*>(workspace);
      gp.hdr = reinterpret_cast<uint32_t*>(base);
      gp.flags = reinterpret_cast<uint32_t*>(base + kWsFlagsOff);
      gp.bstate = reinterpret_cast<uint32_t*>(base + kWsStatesOff);
      gp.ws = reinterpret_cast<float*>(base + kWsCtlBytes);
      pl->ws_bound = workspace;
    }
  }
  gp.timeline = g_timeline;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(pl->cs.g * pl->cg);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = pl->smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[4];
  cfg.attrs = attr;
  cfg.numAttrs = 0;
  if (g_pdl) {
    attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    ++cfg.numAttrs;
  }
  if (pl->cg == 2) {
    attr[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
    attr[cfg.numAttrs].val.clusterDim.x = 2;
    attr[cfg.numAttrs].val.clusterDim.y = 1;
    attr[cfg.numAttrs].val.clusterDim.z = 1;
    ++cfg.numAttrs;
  }
  // Liveness: phase-2 reducers spin on peer flags, so every CTA of a Stream-K grid
  // must be resident at once.  g never exceeds the co-resident CTAs (checked at plan
  // time), but that alone does not stop another grid (another stream, process or MPS
  // client) from holding SMs while only part of this grid runs.  A cooperative launch
  // makes the hardware gang-schedule the grid (all CTAs or none), so partially resident
  // Stream-K grids — and the cross-grid deadlock they allow — cannot occur.
  // Data-parallel grids have no cross-CTA waits and launch normally.
  if (g_coop && pl->cs.sk_tiles > 0) {
    attr[cfg.numAttrs].id = cudaLaunchAttributeCooperative;
    attr[cfg.numAttrs].val.cooperative = 1;
    ++cfg.numAttrs;
  }
  void* args[4] = {&pl->ma, &pl->mb, &pl->mc, &gp};
  cudaError_t e = cudaLaunchKernelExC(&cfg, pl->func, args);
  if (e != cudaSuccess) {
    set_error(std::string("GEMM launch failed: ") + cudaGetErrorString(e));
    return SKPP_ELAUNCH;
  }
  return SKPP_OK;
}

extern "C" int skpp_gemm_launch(const skpp_problem_t* p, const skpp_tile_t* t,
                                const skpp_policy_t* pol, uint32_t g, const skpp_operands_t* ops,
                                void* workspace, uint64_t workspace_bytes, int64_t* trace,
                                uint64_t trace_cap, int64_t* trace_counts, void* stream) {
  void* plan = nullptr;
  int rc = skpp_plan_create(p, t, pol, g, ops, trace, trace_cap, trace_counts, &plan);
  if (rc) return rc;
  rc = skpp_plan_launch(plan, workspace, workspace_bytes, stream);
  skpp_plan_destroy(plan);
  return rc;
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
                          reinterpret_cast<cudaStream_t>(stream)>>>(s, t->tile_order, trace, trace_cap,
                                                                     trace_counts);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("trace launch failed: ") + cudaGetErrorString(e));
    return SKPP_ELAUNCH;
  }
  return SKPP_OK;
}
