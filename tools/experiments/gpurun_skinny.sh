timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests.log
for m in 16 128; do for t in 128x128x128 128x64x128 128x128x64; do for pol in hybrid1 dp; do python tools/launch_modes.py $m 4096 4096 $pol $t | grep "pdl=1"; done; done; done
python tools/launch_modes.py 512 512 16384 ask 128x128x128 | grep "pdl=1"
