#!/usr/bin/env python
"""Fixup-workspace traffic from ncu (tools/gpurun_r2_fixup.sh): the Stream-K launch and the
data-parallel launch of the same shape and tile differ only by the partial-tile fixup (same
operand k-blocks, same C), so the per-launch difference of L2 write / read sectors and of DRAM
bytes is the workspace traffic.  Writes -> profiles/round2/ncu_fixup.json (read by bench.py).

    python tools/fixup_traffic.py gpurun_out/fixup
"""

from __future__ import annotations

import csv
import glob
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {"cfg2": (512, 512, 16384, "128x128x128"), "cfg3": (8192, 14336, 4096, "256x256x128b16"),
          "decode16": (16, 4096, 4096, "128x128x128"), "cfg1": (1024, 1024, 1024, "128x128x64")}


def metrics(path: str) -> dict:
    text = open(path).read()
    rows = list(csv.DictReader(io.StringIO(text[text.index('"ID"'):])))
    out = {}
    for r in rows:
        v = r["Metric Value"].replace(",", "")
        try:
            out[r["Metric Name"]] = float(v)
        except ValueError:
            out[r["Metric Name"]] = float("nan")
    return out


def main(src: str = "gpurun_out/fixup") -> None:
    import paper_2408_11417_b200 as sk
    from paper_2408_11417_b200.scheduler import closed_form, count_partials
    from paper_2408_11417_b200.tiles import parse_tile
    from bench import load_peaks

    peaks = load_peaks()
    res = []
    for sk_path in sorted(glob.glob(os.path.join(src, "fixup_*_hybrid1.csv"))):
        wl = os.path.basename(sk_path)[len("fixup_"):-len("_hybrid1.csv")]
        dp_path = sk_path.replace("_hybrid1.csv", "_dp.csv")
        if wl not in SHAPES or not os.path.exists(dp_path):
            continue
        a, b = metrics(sk_path), metrics(dp_path)
        if any(v != v for v in list(a.values()) + list(b.values())):
            continue
        m, n, k, tl = SHAPES[wl]
        tile = parse_tile(tl)
        g = 148 // (tile.blk_m // 128)
        partial, _, _ = count_partials(closed_form(sk.ProblemSize(m, n, k), tile, g, sk.Policy.hybrid(1)))
        # every partial item's valid rows / columns are written once (ragged tiles skip the rest)
        analytic = partial * min(tile.blk_m, m) * min(tile.blk_n, n) * 4
        dur_s = a["gpu__time_duration.sum"] * 1e-9
        wr = (a["lts__t_sectors_op_write.sum"] - b["lts__t_sectors_op_write.sum"]) * 32
        rd = (a["lts__t_sectors_op_read.sum"] - b["lts__t_sectors_op_read.sum"]) * 32
        dram = (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) - (b["dram__bytes_read.sum"] + b["dram__bytes_write.sum"])
        c_bytes = m * n * 4
        c_sectors_dp = b["lts__t_sectors_op_write.sum"] * 32
        res.append({
            "workload": wl, "m": m, "n": n, "k": k, "tile": tl, "policy": "hybrid1 vs data-parallel",
            "sk_duration_us": round(a["gpu__time_duration.sum"] / 1e3, 2),
            "analytic_partial_bytes_written": analytic,
            "l2_write_bytes_delta": int(wr), "l2_read_bytes_delta": int(rd),
            "l2_write_delta_vs_analytic": round(wr / analytic, 3) if analytic else None,
            "dp_l2_write_bytes_vs_c_bytes": round(c_sectors_dp / c_bytes, 3),
            "workspace_dram_bytes": int(dram),
            "workspace_hbm_gbs": round(dram / dur_s / 1e9, 2),
            "workspace_hbm_frac_of_peak": round(dram / dur_s / 1e9 / peaks["hbm_gbs"], 5),
            "workspace_l2_write_gbs": round(wr / dur_s / 1e9, 1),
            "source": f"{os.path.basename(sk_path)} - {os.path.basename(dp_path)} (ncu, one launch each)",
        })
    out = os.path.join(ROOT, "profiles", "round2", "ncu_fixup.json")
    with open(out, "w") as fh:
        json.dump({"method": __doc__.strip().split("\n\n")[0], "peak_hbm_gbs": peaks["hbm_gbs"], "rows": res}, fh,
                  indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
