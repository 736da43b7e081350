#!/bin/bash
# Decode-shape (M<=128) breakdown: timelines + launch modes for the candidate tiles.
cd /root/repo
mkdir -p gpurun_out/decode
for m in 16 128; do
  for cfg in "hybrid1 128x128x128" "hybrid1 128x64x128" "ask 128x64x128" "data-parallel 128x64x128" "hybrid1 128x128x64"; do
    set -- $cfg
    timeout 120 python tools/launch_modes.py $m 4096 4096 $1 $2 2>&1 | grep pdl=1 >> gpurun_out/decode/modes.txt
    timeout 120 python tools/timeline.py --m $m --n 4096 --k 4096 --policy $1 --tile $2 --kstamps 12 >> gpurun_out/decode/timeline.txt 2>&1
  done
done
