timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests.log
python tools/launch_modes.py 512 512 16384 ask 128x128x128
python tools/launch_modes.py 128 128 1024 ask 128x128x128
python tools/launch_modes.py 1024 1024 1024 hybrid1 128x128x128
python tools/launch_modes.py 512 512 16384 ask 256x256x128
