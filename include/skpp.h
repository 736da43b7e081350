/*
 * skpp.h — C ABI of the B200-native Stream-K++ hot path (libskpp.so).
 *
 * Every entry point takes plain pointers, sizes and POD structs with
 * fixed-width integers; no torch or CUDA types cross this boundary (a CUDA
 * stream is passed as `void*`, i.e. a cudaStream_t / CUstream handle).
 * Functions return 0 on success or one of the SKPP_E* codes below; the
 * message of the last failure on the calling thread is `skpp_last_error()`.
 * No C++ exception ever crosses the ABI.
 *
 * Each group cites the reference interface it replaces.  Paths are relative
 * to the reference package `pkg/src/gemmsched/` (arXiv 2408.11417 desk-scale
 * restatement, `gemmsched`).
 */
#ifndef SKPP_H_
#define SKPP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
enum {
  SKPP_OK = 0,
  SKPP_EINVAL = 1,       /* bad argument (shape, dtype, null pointer ...)    */
  SKPP_ETILE = 2,        /* tile shape not implemented by the sm_100a kernel */
  SKPP_EALIGN = 3,       /* TMA alignment (16-B base / 16-B row stride)      */
  SKPP_EARCH = 4,        /* device is not sm_100 (B200)                      */
  SKPP_ELAUNCH = 5,      /* CUDA launch / driver error                       */
  SKPP_EWORKSPACE = 6,   /* workspace smaller than skpp_workspace_bytes()    */
  SKPP_EGRID = 7,        /* g exceeds co-resident CTAs (Stream-K fixup)      */
  SKPP_ECAPACITY = 8,    /* output buffer too small                          */
  /* sieve file format errors, in the reference's validation order
     (sieve.py:338-395 raises these exception classes)                       */
  SKPP_ETRUNCATED = 20,  /* TruncatedError            sieve.py:58-60       */
  SKPP_EBADMAGIC = 21,   /* BadMagicError             sieve.py:46-48       */
  SKPP_EVERSION = 22,    /* UnsupportedVersionError   sieve.py:50-52       */
  SKPP_EFORMAT = 23,     /* SieveFormatError          sieve.py:43-44       */
  SKPP_ECHECKSUM = 24    /* ChecksumError             sieve.py:54-56       */
};

/* element types for skpp_operands_t.in_dtype / out_dtype */
enum { SKPP_F32 = 0, SKPP_F16 = 1, SKPP_BF16 = 2 };

/* policy kinds (types.py:20-25 PolicyKind) */
enum { SKPP_DATA_PARALLEL = 0, SKPP_HYBRID = 1, SKPP_ALL_STREAM_K = 2 };

/* work-item roles recorded in schedule traces */
enum { SKPP_ROLE_FULL = 0, SKPP_ROLE_OWNER = 1, SKPP_ROLE_PEER = 2 };

/* trace record: one int64[8] row per work item, per CTA (workgroup):
   tile, kb, ke, write_mode (0 full, 1 partial), phase (0 sk, 1 dp), role,
   tile_m, tile_n (the C tile the item wrote: scheduler.py:155-165 locate_iter when
   tile_order == 0, the banded map of skpp_tile_t.tile_order otherwise) */
#define SKPP_TRACE_FIELDS 8

typedef struct { uint64_t m, n, k; } skpp_problem_t;           /* types.py:28-45 ProblemSize  */
/* types.py:58-72 TileShape, plus the kernel's tile order (a B200 tuning parameter that is
   not in the reference): 0 = the reference's row-major tile index -> (tile_m, tile_n) map
   (scheduler.py:155-165 locate_iter; the parity mode); G > 0 = bands of G tile rows walked
   column by column (tile t of band b = t / (G*n_tiles), r = t % (G*n_tiles), rows = min(G,
   m_tiles - b*G): tile_m = b*G + r % rows, tile_n = r / rows), so the tiles running
   concurrently share A and B blocks in L2.  The schedule (which workgroup runs which tile
   index and k-range) is the reference's either way; host-only functions ignore the field. */
typedef struct { uint32_t blk_m, blk_n, blk_k, tile_order; } skpp_tile_t;
typedef struct { int32_t kind, sk_batches, sk_first; } skpp_policy_t; /* types.py:95-166 Policy */

/* Closed-form geometry of one (problem, tile, g, policy) schedule:
   scheduler.py:119-128 grid_info, 168-178 hybrid_sk_tiles, 136-152 streamk_ranges. */
typedef struct {
  uint64_t m_tiles, n_tiles, iters_per_tile, total_tiles, total_iters;
  uint64_t dp_tiles;  /* leading data-parallel tiles [0, dp_tiles)            */
  uint64_t sk_tiles;  /* trailing Stream-K tiles [dp_tiles, total_tiles)      */
  uint64_t sk_iters;  /* sk_tiles * iters_per_tile                            */
  uint64_t ipw;       /* ceil(sk_iters / g), iterations per workgroup         */
  uint32_t g, sk_first;
} skpp_sched_t;

/* GEMM operands: row-major A[m,k] (lda), B[k,n] (ldb), C[m,n] (ldc), element strides. */
typedef struct {
  const void* a; int64_t lda;
  const void* b; int64_t ldb;
  void* c; int64_t ldc;
  int32_t in_dtype;   /* SKPP_F16 or SKPP_BF16 */
  int32_t out_dtype;  /* SKPP_F32, SKPP_F16 or SKPP_BF16 */
} skpp_operands_t;

const char* skpp_last_error(void);
const char* skpp_version(void);

/* ---- schedule (replaces scheduler.py:226-254 build_schedule, 257-291 validate_schedule) ---- */

/* Geometry + policy split; SKPP_EINVAL on overflow (scheduler.py:125-126). */
int skpp_sched_make(const skpp_problem_t* p, const skpp_tile_t* t, uint32_t g,
                    const skpp_policy_t* pol, skpp_sched_t* out);
/* Number of work items of the whole schedule and of each workgroup (counts may be NULL). */
int skpp_sched_count(const skpp_sched_t* s, uint64_t* total, uint64_t* counts /*[g]*/);
/* Materialise every workgroup's ordered items, workgroup-major, into rows of
   SKPP_TRACE_FIELDS int64; `offsets` gets g+1 prefix offsets (in items). */
int skpp_sched_items(const skpp_sched_t* s, int64_t* items, uint64_t cap, uint64_t* offsets);
/* The schedule as the reference's per-workgroup item lists (scheduler.py:226-254
   build_schedule): out[(x*max_items + i)*5 + {0..4}] = (tile, local_iter_begin,
   local_iter_end, write_mode 0=full 1=atomic-partial, phase 0=stream-k 1=data-parallel),
   counts[x] = items of workgroup x; SKPP_ECAPACITY if a workgroup has more than max_items. */
int skpp_schedule_trace(const skpp_problem_t* p, const skpp_tile_t* t, uint32_t g,
                        const skpp_policy_t* pol, uint32_t max_items, int32_t* out, int32_t* counts);
/* C tile (tile_m, tile_n) of tile index `tile` under `tile_order` (skpp_tile_t.tile_order;
   0 = scheduler.py:155-165 locate_iter) — the map the GEMM kernel uses. */
int skpp_tile_coords(const skpp_sched_t* s, uint32_t tile_order, uint64_t tile, uint64_t* tile_m,
                     uint64_t* tile_n);
/* Exactly-once audit by interval sweep over items given as flat [start,end) iteration
   intervals (tile*ipt+kb, tile*ipt+ke).  Writes duplicates and gaps. */
int skpp_validate_intervals(const uint64_t* starts, const uint64_t* ends, uint64_t n_items,
                            uint64_t total_iters, uint64_t* duplicates, uint64_t* gaps);

/* ---- GEMM (replaces executor.py:51-124 execute_schedule) ---- */

/* Bytes of fp32 partial workspace + flags that skpp_gemm_launch needs. */
uint64_t skpp_workspace_bytes(const skpp_problem_t* p, const skpp_tile_t* t, uint32_t g);
/* Tile shapes the sm_100a kernel implements: blk_m == 128 with blk_n in {64,128,256}, blk_k in
   {16,32,64,128}; blk_m == 256 (CTA pair) with blk_n in {128,256}, blk_k in {32,64,128}. */
int skpp_tile_supported(const skpp_tile_t* t);
/* Persistent Stream-K++ GEMM C = A @ B on the current device, stream-ordered.
   The workspace must be zero-filled the first time it is used, and the fill must have
   completed (e.g. cudaMemset, or cudaMemsetAsync + a stream sync) before that first launch
   (Stream-K launches use programmatic dependent launch); afterwards the
   kernel keeps it consistent itself (epoch-tagged flags), so one workspace
   serves any number of stream-ordered launches, including CUDA-graph replays.  trace/trace_counts may be
   NULL; otherwise each CTA x writes up to trace_cap items at
   trace[(x*trace_cap + i)*SKPP_TRACE_FIELDS] and its item count at trace_counts[x]. */
int skpp_gemm_launch(const skpp_problem_t* p, const skpp_tile_t* t, const skpp_policy_t* pol,
                     uint32_t g, const skpp_operands_t* ops, void* workspace,
                     uint64_t workspace_bytes, int64_t* trace, uint64_t trace_cap,
                     int64_t* trace_counts, void* stream);
/* Prepared launches (the hot path for repeated GEMMs and CUDA-graph capture):
   skpp_plan_create validates, builds the schedule scalars and TMA descriptors
   once; skpp_plan_launch only binds the workspace and launches on `stream`.
   skpp_gemm_launch == create + launch + destroy. */
int skpp_plan_create(const skpp_problem_t* p, const skpp_tile_t* t, const skpp_policy_t* pol,
                     uint32_t g, const skpp_operands_t* ops, int64_t* trace, uint64_t trace_cap,
                     int64_t* trace_counts, void** plan_out);
uint64_t skpp_plan_workspace_bytes(const void* plan);
int skpp_plan_launch(void* plan, void* workspace, uint64_t workspace_bytes, void* stream);
void skpp_plan_destroy(void* plan);
/* Decode-only kernel: every CTA walks its items with the GEMM's device decoder
   and records them (no math).  Same trace layout as skpp_gemm_launch. */
int skpp_schedule_trace_device(const skpp_problem_t* p, const skpp_tile_t* t,
                               const skpp_policy_t* pol, uint32_t g, int64_t* trace,
                               uint64_t trace_cap, int64_t* trace_counts, void* stream);
/* Make `device` current for this library's CUDA runtime on the calling thread
   (the caller's framework may use a different runtime instance). */
int skpp_set_device(int device);
/* 1 when `stream` is being captured into a CUDA graph, else 0; negative status on error.
   The host glue gives captured launches a workspace of their own (no reference
   counterpart: the reference executor has no graphs). */
int skpp_stream_is_capturing(void* stream);
/* Debug hook: when non-NULL, following launches write 16 %globaltimer stamps per CTA
   (setup done, first load, first stage landed, last MMA, items done, flags seen,
   reductions done, ...) to device_buffer[cta*16 + event].  NULL disables. */
void skpp_debug_timeline(uint64_t* device_buffer);
/* Programmatic dependent launch (default on): a GEMM launched right after another
   kernel runs its prologue (barriers, TMEM, descriptors) under that kernel's tail
   and waits (griddepcontrol.wait) before touching global memory. */
void skpp_set_pdl(int enable);
/* Cooperative launch of Stream-K grids (default off).  Not needed for liveness: a phase-2
   reducer that waits ~20 us for peer flags keeps waiting only if every CTA of the launch has
   started, else it abandons its band to the last CTA to start (skpp_gemm.cu, phase 2), so no
   CTA waits on a CTA that is not resident.  Measured +12-23% per launch on small Stream-K
   shapes (a cooperative grid gets no PDL overlap). */
void skpp_set_cooperative(int enable);
/* Load each stage's B columns with one 3-D TMA box when N % 64 == 0 (default on;
   plans created after the call). */
void skpp_set_b3d(int enable);
/* Load a BK=128 stage's A rows with one 3-D TMA box when K % 64 == 0 (default on; plans
   created after the call). */
void skpp_set_a3d(int enable);
/* k-blocks of each workgroup's first item to prefetch into L2 before the kernel waits on
   the previous grid (PDL); 0 disables (plans created after the call). */
void skpp_set_l2_prefetch(int k_blocks);
/* L2 cache-policy hints on the operand stream (default on; plans created after the call):
   B k-blocks are loaded evict_last (the next wave of tiles re-reads them), C tiles are
   stored evict_first. */
void skpp_set_l2_hints(int enable);
/* Test hooks (plans created after the call): bit 0 forces the two-pass Stream-K fixup
   (peers first, owner added in a second pass) even when the owner is already published;
   bit 1 sets the phase-2 wait bound to 0, so every wait not already satisfied takes the
   timeout decision (keep waiting if every CTA started, else abandon to the last starter);
   bit 4 turns the owner reduction off (two-contributor split tiles whose owner item is the
   owner's last Stream-K item are then reduced in phase 2 like every other split tile);
   results are bit-identical to the normal path by construction (tests check it). */
void skpp_set_debug(int flags);
/* Test hook for the liveness tests: launch `ctas` single-warp CTAs with `smem_bytes` of
   dynamic shared memory each that occupy their SMs until *release != 0 (bounded at ~35 s),
   so a Stream-K grid launched next on another stream is only partially resident. */
int skpp_test_hold_sms(uint32_t ctas, uint32_t smem_bytes, const uint32_t* release, void* stream);
/* SM count, compute capability and the co-resident CTA limit of the GEMM kernel for blk_n. */
int skpp_device_info(int device, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);
int skpp_max_coresident(const skpp_tile_t* t, int32_t* ctas);

/* ---- hashing (replaces hashing.py:41-91 murmur3_x64_128, 129-194 hash24) ---- */

void skpp_murmur3_x64_128(const uint8_t* data, uint64_t len, uint32_t seed, uint64_t out[2]);
void skpp_hash24(uint64_t m, uint64_t n, uint64_t k, uint64_t seed, uint64_t out[2]);

/* ---- Bloom filters (replaces sieve.py:63-104 sizing/probes, 107-166 BloomFilter) ---- */

int skpp_filter_params(uint64_t capacity, double fp_target, uint64_t* m_bits, uint32_t* k_hashes);
uint32_t skpp_filter_seed(uint64_t index);
int skpp_hash_probes(const uint8_t* key24, uint32_t seed, uint64_t m_bits, uint32_t k_hashes,
                     uint64_t* out /*[k_hashes]*/);
int skpp_bloom_insert(uint8_t* bits, uint64_t m_bits, uint32_t k_hashes, uint32_t seed,
                      uint64_t m, uint64_t n, uint64_t k);
int skpp_bloom_contains(const uint8_t* bits, uint64_t m_bits, uint32_t k_hashes, uint32_t seed,
                        uint64_t m, uint64_t n, uint64_t k);
/* All-filters membership (hashing.py:172-189 _query_mask_jit): bit f set iff filter f
   (bits + f*m_bits/8) reports (m,n,k) present.  n_filters <= 64. */
uint64_t skpp_bank_query_mask(const uint8_t* bits, const uint32_t* seeds, uint32_t n_filters,
                              uint64_t m_bits, uint32_t k_hashes, uint64_t m, uint64_t n,
                              uint64_t k);
/* Batched query over `count` sizes (rows of 3 u64) into masks[count]. */
int skpp_bank_query_masks(const uint8_t* bits, const uint32_t* seeds, uint32_t n_filters,
                          uint64_t m_bits, uint32_t k_hashes, const uint64_t* sizes,
                          uint64_t count, uint64_t* masks);
/* Opaque snapshot for the latency-critical single query (sieve.py:283-313 fast path). */
void* skpp_bank_snapshot(const uint8_t* bits, const uint32_t* seeds, uint32_t n_filters,
                         uint64_t m_bits, uint32_t k_hashes);
uint64_t skpp_bank_snapshot_query(const void* snap, uint64_t m, uint64_t n, uint64_t k);
void skpp_bank_snapshot_free(void* snap);

/* ---- sieve file format (replaces sieve.py:315-402 to_bytes / from_bytes) ---- */

typedef struct {
  uint8_t tag, sk_batches, sk_first, reserved;
  uint32_t seed;
  uint64_t m_bits;
  uint32_t k_hashes;
  uint64_t n_inserted;
} skpp_filter_header_t;

uint32_t skpp_crc32(const uint8_t* data, uint64_t len, uint32_t crc);
uint64_t skpp_bank_serialized_bytes(const skpp_filter_header_t* hdrs, uint32_t count);
int skpp_bank_serialize(const skpp_filter_header_t* hdrs, const uint8_t* bits /*concatenated*/,
                        uint32_t count, uint8_t* out, uint64_t cap, uint64_t* written);
/* Validate and parse; on success fills up to `cap` headers and the byte offset of each
   filter's bit array inside `data`.  Error codes follow the reference's check order. */
int skpp_bank_parse(const uint8_t* data, uint64_t len, skpp_filter_header_t* hdrs,
                    uint64_t* bit_offsets, uint32_t cap, uint32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* SKPP_H_ */
