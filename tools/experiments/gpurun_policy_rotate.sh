#!/bin/bash
cd /root/repo
mkdir -p gpurun_out/polrot
for s in "4096 14336 4096" "2048 14336 4096" "1024 14336 4096" "4096 4096 4096" "8192 4096 4096"; do
  set -- $s
  timeout 300 python tools/experiments/policy_rotate.py $1 $2 $3 256x256x128 3 >> gpurun_out/polrot/out.txt 2>&1
done
