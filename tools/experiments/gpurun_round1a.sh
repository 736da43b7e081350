set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 300 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench rc=$?
timeout 300 python bench.py --workload square8192 --steps 30 > gpurun_out/bench_sq.json 2> gpurun_out/bench_sq.err; echo rc=$?
timeout 300 python bench.py --workload cfg1 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo rc=$?
timeout 600 python tools/shapes.py > gpurun_out/shapes.jsonl 2> gpurun_out/shapes.err; echo rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/profile_gemm.py --m 512 --n 512 --k 16384 --policy ask --iters 5 --flush; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:streamk_gemm -s 2 -c 1 -o gpurun_out/prof_cfg2_ask python tools/profile_gemm.py --m 512 --n 512 --k 16384 --policy ask --iters 3 --flush > gpurun_out/ncu_cfg2.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:streamk_gemm -s 2 -c 1 -o gpurun_out/prof_sq8192 python tools/profile_gemm.py --m 8192 --n 8192 --k 8192 --policy dp --tile 128x256x64 --iters 3 > gpurun_out/ncu_sq.log 2>&1; echo rc=$?
