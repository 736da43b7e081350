timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_tests.log
for a in 1 0 1 0; do echo a3d=$a; SKPP_A3D=$a python tools/launch_modes.py 512 512 16384 ask 128x128x128; SKPP_A3D=$a python tools/launch_modes.py 512 512 16384 ask 256x128x128; SKPP_A3D=$a python tools/launch_modes.py 1024 1024 1024 dp 128x128x128; done
