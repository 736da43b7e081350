#!/usr/bin/env python
"""Summarise an ncu report (or a launch-list CSV) into a small JSON for profiles/.

    python tools/ncu_summary.py rep gpurun_out/prof.ncu-rep  > profiles/x.json
    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/y.json
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "gpc__cycles_elapsed.max": "cycles",
    "gpc__cycles_elapsed.max.per_second": "sm_clock_ghz",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum": "tma_load_bytes",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "launch__grid_size": "grid",
    "sm__cycles_active.avg": "sm_active_cycles_avg",
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1.0, "ms": 1e3, "ns": 1e-3}


def raw(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    header, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[header.index("Kernel Name")]}
        for key, name in KEYS.items():
            if key in header:
                i = header.index(key)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if name in ("dram_read", "dram_write", "tma_load_bytes", "dyn_smem"):
                    v *= SCALE.get(u.split("/")[0], 1.0)
                if name == "duration_us":
                    v *= SCALE.get(u, 1.0)
                d[name] = v
        if "dram_read" in d and "dram_write" in d:
            d["dram_traffic_bytes"] = d["dram_read"] + d["dram_write"]
        res.append(d)
    return res


def launches(path: str) -> dict:
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per: dict[str, list[float]] = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        if "streamk_gemm_kernel<" in name:  # per instantiation <BN, BK, CG, RASTER>
            short = "streamk_gemm_kernel" + name[name.index("<"):name.index(">") + 1]
        else:
            short = name.split("(")[0][-60:]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        per.setdefault(short, []).append(v * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1e-3))
    total = sum(sum(v) for v in per.values())
    return {k: {"launches": len(v), "total_us": round(sum(v), 2), "mean_us": round(sum(v) / len(v), 2),
                "share": round(sum(v) / total, 4)} for k, v in per.items()}


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(json.dumps(raw(path) if mode == "rep" else launches(path), indent=1))
