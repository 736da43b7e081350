timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
for r in 1 2; do for m in 0 1; do echo "== mc=$m"
for sz in "1024 1024 1024 dp 128x64x128" "1024 1024 1024 dp 128x128x128" "2048 2048 2048 dp 128x128x128" "4096 4096 4096 dp 128x128x128" "2048 4096 4096 dp 128x128x64" "512 512 16384 ask 128x128x128"; do
  SKPP_MC=$m python tools/launch_modes.py $sz 2>&1 | grep "pdl=1\|rror"; done; done; done
