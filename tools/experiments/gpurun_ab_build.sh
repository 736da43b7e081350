#!/bin/bash
# Interleaved A/B of the in-tree build (A) vs _orig/ (B, SKPP_PKG_ROOT) on a few shapes.
cd /root/repo
mkdir -p gpurun_out/abb
: > gpurun_out/abb/ab.txt
for r in 1 2 3 4; do
  for v in A B; do
    for cfg in "512 512 16384 hybrid1 128x128x128" "512 512 16384 hybrid1 128x128x64" "16 4096 4096 hybrid1 128x128x128"; do
      set -- $cfg
      if [ $v = B ]; then export SKPP_PKG_ROOT=/root/repo/_orig; else unset SKPP_PKG_ROOT; fi
      timeout 120 python tools/launch_modes.py $1 $2 $3 $4 $5 2>&1 | grep pdl=1 | sed "s/^/$v /" >> gpurun_out/abb/ab.txt
    done
  done
done
unset SKPP_PKG_ROOT
