#!/bin/bash
# A (in-tree) vs B (_orig) on decode / ragged shapes, interleaved; then the GPU tests on A.
cd /root/repo
mkdir -p gpurun_out/abd
: > gpurun_out/abd/ab.txt
for r in 1 2 3; do
  for v in A B; do
    for cfg in "16 4096 4096 hybrid1 128x128x128" "48 4096 4096 hybrid1 128x128x128" "100 4096 4096 hybrid1 128x64x128" "16 14336 4096 hybrid1 128x128x128" "512 512 16384 hybrid1 128x128x128"; do
      set -- $cfg
      if [ $v = B ]; then export SKPP_PKG_ROOT=/root/repo/_orig; else unset SKPP_PKG_ROOT; fi
      timeout 120 python tools/launch_modes.py $1 $2 $3 $4 $5 2>&1 | grep pdl=1 | sed "s/^/$v /" >> gpurun_out/abd/ab.txt
    done
  done
done
unset SKPP_PKG_ROOT
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/abd/tests.txt
