# round 2 final profile (session 3 kernel): GPU tests, the driver's default bench command (cfg3 + in-run sweep), the
# reference arm, cfg2 bench, launch list and ncu --set full captures of the selected kernels.
set -x
O=gpurun_out/prof3; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvsmi.txt
nproc > $O/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 $O/gpu_tests.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo bench cfg3 rc=$?
tail -c 400 $O/bench_cfg3.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_reference_cfg3.json 2> $O/bench_reference.err; echo ref rc=$?
timeout 600 python bench.py --workload cfg2 --steps 2000 --sweep-grid none > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo bench cfg2 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv python bench.py --steps 20 --warmup 3 --e2e-steps 2 --cpu-seconds 1 --sweep-grid none > $O/launches_bench.json 2>&1; echo launches rc=$?
cap() {  # name m n k policy tile dtype
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:streamk_gemm -s 3 -c 1 -o $O/$1 \
    python tools/profile_gemm.py --m $2 --n $3 --k $4 --policy $5 --tile $6 --dtype $7 --iters 4 > $O/$1.log 2>&1; echo ncu $1 rc=$?
}
cap cfg3_256x256x128b16_hybrid1 8192 14336 4096 hybrid1 256x256x128b16 bf16
cap cfg2_128x128x128_hybrid1 512 512 16384 hybrid1 128x128x128 bf16
cap decode16_128x128x128_hybrid1 16 4096 4096 hybrid1 128x128x128 bf16
