timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gpu_tests.log
for t in 128x128x64 256x256x64; do
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask --tile $t 2>&1 | head -14
done
python tools/timeline.py --m 1024 --n 1024 --k 1024 --policy ask 2>&1 | head -14
