O=gpurun_out/l2h; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 $O/gpu_tests.log
for h in 1 0 1 0; do echo hints=$h; SKPP_L2_HINTS=$h python tools/launch_modes.py 8192 8192 8192 dp 256x256x128; done
for h in 1 0; do echo hints=$h; SKPP_L2_HINTS=$h python tools/launch_modes.py 512 512 16384 ask 128x128x128; SKPP_L2_HINTS=$h python tools/launch_modes.py 4096 4096 4096 dp 256x256x128;  done
for h in 1 0; do
SKPP_L2_HINTS=$h timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:streamk_gemm -s 3 -c 1 python tools/profile_gemm.py --m 8192 --n 8192 --k 8192 --policy dp --tile 256x256x128 --iters 4 > $O/ncu_sq_$h.txt 2>&1
echo hints=$h; grep -E "dram__|duration" $O/ncu_sq_$h.txt
done
