timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests.log
for root in "" _orig; do echo "== ${root:-new}"
for sz in "1 14336 4096 dp 128x128x128" "1 4096 4096 hybrid1 128x128x64" "16 4096 4096 hybrid1 128x128x128" "64 14336 4096 dp 128x128x128" "20 600 4096 hybrid1 256x256x128" "512 512 16384 ask 128x128x128"; do
  SKPP_PKG_ROOT=$root python tools/launch_modes.py $sz | grep "pdl=1"; done; done
