#!/bin/bash
# DRAM bytes per launch, row-major (SKPP_RASTER=0) vs banded (auto), one ncu capture each.
cd /root/repo
O=gpurun_out/ncur; mkdir -p $O
for r in 0 -1; do
  for s in "4096 14336 4096 hybrid1" "8192 8192 8192 dp"; do
    set -- $s
    SKPP_RASTER=$r timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:streamk_gemm -s 3 -c 1 --csv python tools/profile_gemm.py --m $1 --n $2 --k $3 --policy $4 --tile 256x256x128 --out bf16 --iters 4 > $O/r${r}_$1x$2x$3.csv 2>&1
  done
done
