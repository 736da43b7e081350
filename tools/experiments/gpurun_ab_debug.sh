#!/bin/bash
# Interleaved A/B of a skpp_set_debug bit: AB_BITS (default "0 8") over cfg2 and decode shapes.
cd /root/repo
mkdir -p gpurun_out/ab
BITS=${AB_BITS:-"0 8"}
: > gpurun_out/ab/ab.txt
for r in 1 2 3; do
  for d in $BITS; do
    for cfg in "512 512 16384 hybrid1 128x128x128" "16 4096 4096 hybrid1 128x128x128" "128 4096 4096 hybrid1 128x64x128" "1024 1024 1024 hybrid1 128x128x64" "2048 4096 4096 hybrid1 128x128x64"; do
      set -- $cfg
      SKPP_DEBUG=$d timeout 120 python tools/launch_modes.py $1 $2 $3 $4 $5 2>&1 | grep pdl=1 | sed "s/^/debug=$d /" >> gpurun_out/ab/ab.txt
    done
  done
done
for d in $BITS; do
  SKPP_DEBUG=$d timeout 120 python tools/timeline.py --m 16 --n 4096 --k 4096 --policy hybrid1 --tile 128x128x128 --flush > gpurun_out/ab/tl16_d$d.txt 2>&1
  SKPP_DEBUG=$d timeout 120 python tools/timeline.py --policy hybrid1 --tile 128x128x128 --flush > gpurun_out/ab/tlcfg2_d$d.txt 2>&1
done
