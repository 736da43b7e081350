# Round profile: bench lines, launch list and ncu captures -> gpurun_out/prof/ (then
# tools/collect_profiles.py copies summaries into profiles/).
set -x
O=gpurun_out/prof; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvsmi.txt
for wl in cfg2 cfg1 square8192; do
  steps=10000; [ $wl = square8192 ] && steps=300
  timeout 600 python bench.py --workload $wl --steps $steps > $O/bench_$wl.json 2> $O/bench_$wl.err; echo bench $wl rc=$?
done
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference_cfg2.json 2> $O/bench_reference.err
# launch list of the default bench command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python bench.py --steps 200 --warmup 3 --e2e-steps 2 --cpu-seconds 1 > $O/launches_bench.json 2>&1; echo launches rc=$?
# full captures of the kernel configurations the bench selects (and the runner-up tile)
cap() {  # name m n k policy tile dtype
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:streamk_gemm -s 3 -c 1 -o $O/$1 \
    python tools/profile_gemm.py --m $2 --n $3 --k $4 --policy $5 --tile $6 --dtype $7 --iters 4 > $O/$1.log 2>&1; echo ncu $1 rc=$?
}
cap cfg2_128x128x128_hybrid1 512 512 16384 hybrid1 128x128x128 bf16
cap cfg2_128x128x64_hybrid1 512 512 16384 hybrid1 128x128x64 bf16
cap cfg1_128x128x128_dp 1024 1024 1024 dp 128x128x128 fp16
cap cfg1_128x64x128_dp 1024 1024 1024 dp 128x64x128 fp16
cap square8192_256x256x64_dp 8192 8192 8192 dp 256x256x64 bf16
cap square8192_256x256x128_dp 8192 8192 8192 dp 256x256x128 bf16
