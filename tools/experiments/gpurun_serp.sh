O=gpurun_out/serp; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -2 $O/gpu_tests.log
for t in 256x256x128 256x256x64 128x128x128; do python tools/launch_modes.py 8192 8192 8192 dp $t; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:streamk_gemm -s 3 -c 1 python tools/profile_gemm.py --m 8192 --n 8192 --k 8192 --policy dp --tile 256x256x128 --iters 4 > $O/ncu_sq.txt 2>&1
grep -E "dram__|duration|tensor" $O/ncu_sq.txt
