"""Oracle restatement of the reference scheduler (gemmsched scheduler.py).

Items are plain tuples ``(tile, kb, ke, write_mode, phase)`` with
write_mode 0 = FULL_STORE / 1 = ATOMIC_PARTIAL and phase 0 = STREAM_K /
1 = DATA_PARALLEL; a schedule is a list (one entry per workgroup) of lists
of items in execution order.  Built by explicit loops over the reference
construction, not by the closed form the product uses.
"""

from __future__ import annotations

FULL, PARTIAL = 0, 1
SK, DP = 0, 1


def cdiv(a: int, b: int) -> int:
    return -(-a // b)


def grid_info(m, n, k, bm, bn, bk):
    """scheduler.py:119-128."""
    mt, nt, ipt = cdiv(m, bm), cdiv(n, bn), cdiv(k, bk)
    return mt, nt, ipt, mt * nt, mt * nt * ipt


def streamk_ranges(total: int, g: int):
    """scheduler.py:136-152: range x = [min(x*ipw, I), min((x+1)*ipw, I))."""
    ipw = cdiv(total, g)
    return [(min(x * ipw, total), min((x + 1) * ipw, total)) for x in range(g)]


def hybrid_sk_tiles(total_tiles: int, g: int, s: int) -> int:
    """scheduler.py:168-178."""
    r = total_tiles % g
    return min(total_tiles, (s - 1) * g + (r if r > 0 else g))


def round_robin(n_tiles: int, g: int, ipt: int):
    """scheduler.py:185-192: tile t -> workgroup t mod g, whole tile, DP phase."""
    wg = [[] for _ in range(g)]
    for t in range(n_tiles):
        wg[t % g].append((t, 0, ipt, FULL, DP))
    return wg


def streamk_region(first_tile: int, n_tiles: int, g: int, ipt: int):
    """scheduler.py:195-223: split the region's iterations evenly, cut at tile edges."""
    wg = []
    for lo, hi in streamk_ranges(n_tiles * ipt, g):
        items = []
        cur = lo
        while cur < hi:
            t = cur // ipt
            end = min(hi, (t + 1) * ipt)
            kb, ke = cur - t * ipt, end - t * ipt
            items.append((first_tile + t, kb, ke, FULL if (kb == 0 and ke == ipt) else PARTIAL, SK))
            cur = end
        wg.append(items)
    return wg


def build_schedule(m, n, k, bm, bn, bk, g, kind, sk_batches=0, sk_first=False):
    """scheduler.py:226-254.  ``kind`` is the PolicyKind value string."""
    _, _, ipt, T, _ = grid_info(m, n, k, bm, bn, bk)
    if kind == "data-parallel":
        return round_robin(T, g, ipt)
    if kind == "all-streamk":
        return streamk_region(0, T, g, ipt)
    sk = hybrid_sk_tiles(T, g, sk_batches)
    dp = T - sk
    dp_part = round_robin(dp, g, ipt)
    sk_part = streamk_region(dp, sk, g, ipt)
    if sk_first:
        return [s + d for s, d in zip(sk_part, dp_part)]
    return [d + s for s, d in zip(sk_part, dp_part)]


def validate(schedule, ipt: int, total: int):
    """scheduler.py:257-291 interval sweep -> (covered_once, duplicates, gaps)."""
    events = []
    for wg in schedule:
        for t, kb, ke, _wm, _ph in wg:
            events.append((t * ipt + kb, 1))
            events.append((t * ipt + ke, -1))
    events.sort()
    covered = dup = depth = prev = 0
    for pos, d in events:
        span = pos - prev
        if span > 0 and depth > 0:
            inside = min(pos, total) - min(prev, total)
            covered += inside
            dup += (depth - 1) * inside + depth * (span - inside)
        prev = pos
        depth += d
    gaps = total - covered
    return dup == 0 and gaps == 0, dup, gaps


def fixup_roles(schedule, ipt: int):
    """Derived (not in the reference): per item 0 full / 1 owner (kb == 0) / 2 peer.

    A split tile's owner is the workgroup holding its iteration 0; every other
    contributor is a peer whose partial the owner reduces.
    """
    out = []
    for wg in schedule:
        roles = []
        for _t, kb, ke, wm, _ph in wg:
            roles.append(0 if wm == FULL else (1 if kb == 0 else 2))
        out.append(roles)
    return out


def locate_tile(t: int, n_tiles: int):
    """scheduler.py:155-165 (locate_iter): tile t is C tile (t // n_tiles, t % n_tiles), row-major."""
    return divmod(t, n_tiles)


def banded_order(m_tiles: int, n_tiles: int, band: int):
    """Not in the reference: the B200 kernel's banded tile order (skpp_tile_t.tile_order,
    include/skpp.h).  Built by enumeration — bands of ``band`` tile rows from the top, each
    walked column by column, rows inside a column top to bottom — so it checks the closed
    form in skpp_sched.h:tile_coords independently.  Returns the list index -> (tile_m, tile_n);
    ``band == 0`` is the reference's row-major order."""
    if band == 0:
        return [locate_tile(t, n_tiles) for t in range(m_tiles * n_tiles)]
    order = []
    for r0 in range(0, m_tiles, band):
        rows = range(r0, min(r0 + band, m_tiles))
        for tn in range(n_tiles):
            for tm in rows:
                order.append((tm, tn))
    return order


def trace_coords(schedule, m_tiles: int, n_tiles: int, band: int = 0):
    """Per workgroup, the (tile_m, tile_n) each item of ``schedule`` writes under tile order
    ``band`` (the last two fields of a device trace row)."""
    order = banded_order(m_tiles, n_tiles, band)
    return [[order[t] for t, _kb, _ke, _wm, _ph in wg] for wg in schedule]
