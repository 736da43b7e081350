// skpp_sched.h — closed-form Stream-K++ schedule, shared by the host builder
// and the device decoder of every CTA in the GEMM.
//
// The reference materialises per-workgroup lists of WorkItem objects
// (gemmsched scheduler.py:185-254).  Here a schedule is six scalars
// (dp_tiles, sk_tiles, ipt, ipw, g, sk_first); each workgroup x walks its
// own ordered items with a cursor, so the device never reads a schedule
// from memory.  The walk reproduces, item for item:
//   * data-parallel items  — tiles x, x+g, x+2g, ... < dp_tiles, FULL,
//     phase DATA_PARALLEL (scheduler.py:185-192 _round_robin_items);
//   * Stream-K items       — x's slice [min(x*ipw,I), min((x+1)*ipw,I)) of the
//     region's I = sk_tiles*ipt iterations, cut at tile boundaries, FULL iff
//     [0, ipt), phase STREAM_K (scheduler.py:136-152, 195-223);
//   * order                — SK part first iff policy.sk_first, all-SK and DP
//     have a single part (scheduler.py:244-251).
// Fixup ownership (not in the reference; derived from the same formulas):
// the CTA holding a split tile's iteration 0 owns it and reduces the
// partials of CTAs x0+1 .. floor(((u+1)*ipt-1)/ipw), each of which produces
// that partial as its first Stream-K item.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define SKPP_HD __host__ __device__ __forceinline__
#else
#define SKPP_HD inline
#endif

namespace skpp {

enum : uint32_t { ROLE_FULL = 0, ROLE_OWNER = 1, ROLE_PEER = 2 };
enum : uint32_t { PHASE_SK = 0, PHASE_DP = 1 };

struct Sched {
  uint64_t dp_tiles, sk_tiles, ipt, ipw, sk_iters, n_tiles;
  uint32_t g, sk_first;
};

struct Item {
  uint64_t tile;      // linear row-major tile index (scheduler.py:155-165)
  uint64_t kb, ke;    // local k-iteration range [kb, ke)
  uint32_t role;      // ROLE_*
  uint32_t phase;     // PHASE_*
  uint64_t peer_hi;   // owner only: last contributing CTA (peers are x+1 .. peer_hi)
};

struct Cursor {
  uint32_t part;      // 0, 1 = the two parts in execution order, 2 = exhausted
  uint64_t sk_cur, sk_hi, dp_next;
};

SKPP_HD uint64_t min_u64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// a / b.  On the device a 64-bit division is a ~50-instruction subroutine (I2F.U64, MUFU.RCP,
// F2I.U64 and a correction chain, several hundred cycles of latency); every realistic schedule
// has its dividends and divisors below 2^32, where the 32-bit sequence is a fraction of that.
// The producer decodes its first item right after griddepcontrol.wait, so this is on the
// kernel's critical path.
SKPP_HD uint64_t udiv(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  if (((a | b) >> 32) == 0) return (uint64_t)((uint32_t)a / (uint32_t)b);
#endif
  return a / b;
}

SKPP_HD void cursor_init(Cursor& c, const Sched& s, uint32_t x) {
  c.part = 0;
  c.sk_cur = min_u64((uint64_t)x * s.ipw, s.sk_iters);
  c.sk_hi = min_u64((uint64_t)(x + 1) * s.ipw, s.sk_iters);
  c.dp_next = x;
}

// Advances to the next item of workgroup x; false once the workgroup is done.
SKPP_HD bool cursor_next(Cursor& c, const Sched& s, uint32_t x, Item& it) {
  while (c.part < 2) {
    const bool sk_part = (c.part == 0) == (s.sk_first != 0);
    if (sk_part) {
      if (c.sk_cur < c.sk_hi) {
        const uint64_t u = udiv(c.sk_cur, s.ipt);
        const uint64_t tile_end = (u + 1) * s.ipt;
        const uint64_t e = min_u64(c.sk_hi, tile_end);
        it.tile = s.dp_tiles + u;
        it.kb = c.sk_cur - u * s.ipt;
        it.ke = e - u * s.ipt;
        it.phase = PHASE_SK;
        it.peer_hi = 0;
        if (it.kb == 0 && it.ke == s.ipt) {
          it.role = ROLE_FULL;
        } else if (it.kb == 0) {
          it.role = ROLE_OWNER;
          it.peer_hi = udiv(tile_end - 1, s.ipw);
        } else {
          it.role = ROLE_PEER;
        }
        c.sk_cur = e;
        return true;
      }
    } else if (c.dp_next < s.dp_tiles) {
      it.tile = c.dp_next;
      it.kb = 0;
      it.ke = s.ipt;
      it.role = ROLE_FULL;
      it.phase = PHASE_DP;
      it.peer_hi = 0;
      c.dp_next += s.g;
      return true;
    }
    ++c.part;
  }
  return false;
}

// Item count of workgroup x without walking the Stream-K part item by item.
SKPP_HD uint64_t items_of(const Sched& s, uint32_t x) {
  uint64_t n = 0;
  if (s.dp_tiles > x) n += udiv(s.dp_tiles - x + s.g - 1, s.g);
  const uint64_t lo = min_u64((uint64_t)x * s.ipw, s.sk_iters);
  const uint64_t hi = min_u64((uint64_t)(x + 1) * s.ipw, s.sk_iters);
  if (hi > lo) n += udiv(hi - 1, s.ipt) - udiv(lo, s.ipt) + 1;
  return n;
}

// Tile index -> (tile row, tile column) of C.  band == 0 is the reference's row-major
// order (scheduler.py:155-165 locate_iter: tile_m = t / n_tiles, tile_n = t % n_tiles).
// band == G > 0 (skpp_tile_t.tile_order) walks bands of G tile rows column by column: a
// bijection on [0, T) that keeps the ~g tiles running concurrently inside G rows and
// ~g/G columns, so their A and B blocks stay in L2.  The last band has m_tiles % G rows.
SKPP_HD void tile_coords(const Sched& s, uint32_t band, uint64_t t, uint64_t& tm, uint64_t& tn) {
  if (band == 0) {
    tm = udiv(t, s.n_tiles);
    tn = t - tm * s.n_tiles;
    return;
  }
  const uint64_t m_tiles = udiv(s.dp_tiles + s.sk_tiles, s.n_tiles);
  const uint64_t band_tiles = (uint64_t)band * s.n_tiles;
  const uint64_t b = udiv(t, band_tiles), r = t - b * band_tiles;
  const uint64_t rows = m_tiles - b * band < band ? m_tiles - b * band : band;
  tn = udiv(r, rows);
  tm = b * band + (r - tn * rows);
}

}  // namespace skpp
