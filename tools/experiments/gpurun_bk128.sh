timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/gpu_tests.log
for t in 128x128x128 256x256x128 256x128x128 128x256x128 128x128x64; do
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask --tile $t --kstamps 1 2>&1 | grep -E "ask tile|mean arrival|mma_done|phase2"
python tools/timeline.py --m 8192 --n 8192 --k 8192 --policy dp --tile $t --kstamps 1 2>&1 | grep -E "dp tile|mean arrival"
python tools/launch_modes.py 512 512 16384 ask $t
done
python tools/launch_modes.py 8192 8192 8192 dp 256x256x128
