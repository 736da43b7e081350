# Round profile: benches, launch lists and ncu captures -> gpurun_out/prof/
set -x
O=gpurun_out/prof; mkdir -p $O
for wl in cfg2 cfg1 square8192; do
  steps=200; [ $wl = square8192 ] && steps=30
  timeout 300 python bench.py --workload $wl --steps $steps > $O/bench_$wl.json 2> $O/bench_$wl.err; echo bench $wl rc=$?
done
timeout 300 python bench.py --impl reference --steps 5 > $O/bench_reference_cfg2.json 2> $O/bench_reference.err
# launch list of the default bench command (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python bench.py --steps 20 --warmup 3 --e2e-steps 2 --cpu-seconds 1 > /dev/null 2>&1; echo rc=$?
# full captures of the bench kernels (same tile / policy / dtype as the bench)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:streamk_gemm -s 3 -c 1 -o $O/prof_cfg2 python tools/profile_gemm.py --m 512 --n 512 --k 16384 --policy hybrid1 --iters 4 > $O/ncu_cfg2.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:streamk_gemm -s 3 -c 1 -o $O/prof_cfg1 python tools/profile_gemm.py --m 1024 --n 1024 --k 1024 --policy dp --dtype fp16 --iters 4 > $O/ncu_cfg1.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:streamk_gemm -s 2 -c 1 -o $O/prof_square8192 python tools/profile_gemm.py --m 8192 --n 8192 --k 8192 --policy dp --tile 256x256x64 --iters 3 > $O/ncu_sq.log 2>&1; echo rc=$?
timeout 600 python tools/shapes.py --tiles 128x128x64,256x256x64 > $O/shapes.jsonl 2> $O/shapes.err; echo rc=$?
