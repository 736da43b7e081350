# ncu --set full capture of the (tile, policy) the final bank selects for cfg3, then the default bench
O=gpurun_out/prof4; mkdir -p $O
cap() {  # name m n k policy tile dtype
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:streamk_gemm -s 3 -c 1 -o $O/$1 \
    python tools/profile_gemm.py --m $2 --n $3 --k $4 --policy $5 --tile $6 --dtype $7 --iters 4 > $O/$1.log 2>&1; echo ncu $1 rc=$?
}
cap cfg3_256x256x128b16_hybrid3 8192 14336 4096 hybrid3 256x256x128b16 bf16
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo bench rc=$?
