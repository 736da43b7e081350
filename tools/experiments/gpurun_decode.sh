timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gpu_tests.log
for r in 1 2; do for root in _orig ""; do echo "== ${root:-new}"
for sz in "1 14336 4096 dp 128x128x128" "16 4096 4096 hybrid1 128x128x128" "512 512 16384 ask 128x128x128" "1024 1024 1024 dp 128x64x128"; do
  SKPP_PKG_ROOT=$root python tools/launch_modes.py $sz 2>&1 | grep "pdl=1"; done; done; done
