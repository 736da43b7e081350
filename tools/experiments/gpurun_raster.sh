#!/bin/bash
cd /root/repo
mkdir -p gpurun_out/raster
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/raster/tests.txt
RASTERS="0,-1" timeout 1200 python tools/experiments/raster_ab.py > gpurun_out/raster/ab_auto.txt 2>&1
for w in square8192 cfg2; do
  steps=20000; [ $w = square8192 ] && steps=300
  timeout 600 python bench.py --workload $w --steps $steps > gpurun_out/raster/bench_$w.json 2>gpurun_out/raster/bench_$w.err
done
