# round 2: fixup-workspace traffic captures (ncu, Stream-K vs DP), cold-L2 sweep check, the
# CTA-pair TMEM allocation racecheck reproducer, drop-in path host overheads
set -x
O=gpurun_out/fixup; mkdir -p $O
M=gpu__time_duration.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,dram__bytes_read.sum,dram__bytes_write.sum
fx() {  # name m n k policy tile
  timeout 600 ncu --metrics $M --clock-control none -k regex:streamk_gemm -s 3 -c 1 --csv --log-file $O/fixup_$1.csv \
    python tools/profile_gemm.py --m $2 --n $3 --k $4 --policy $5 --tile $6 --iters 4 > $O/fixup_$1.log 2>&1; echo fx $1 rc=$?
}
fx cfg2_hybrid1 512 512 16384 hybrid1 128x128x128
fx cfg2_dp 512 512 16384 dp 128x128x128
fx cfg3_hybrid1 8192 14336 4096 hybrid1 256x256x128b16
fx cfg3_dp 8192 14336 4096 dp 256x256x128b16
fx decode16_hybrid1 16 4096 4096 hybrid1 128x128x128
fx decode16_dp 16 4096 4096 dp 128x128x128
fx cfg1_hybrid1 1024 1024 1024 hybrid1 128x128x64
fx cfg1_dp 1024 1024 1024 dp 128x128x64
tail -3 $O/fixup_cfg3_hybrid1.log
timeout 300 compute-sanitizer --tool racecheck ./tools/tmem_alloc_race > $O/tmem_alloc_racecheck.txt 2>&1; echo tmem rc=$?; cat $O/tmem_alloc_racecheck.txt | cut -c1-250
timeout 300 python tools/e2e_overhead.py > $O/e2e_overhead.jsonl 2>&1; echo e2e rc=$?; cat $O/e2e_overhead.jsonl
timeout 1500 python tools/cold_l2_check.py --max-sets 64 --min-mb 4 --out $O > $O/cold.log 2>&1; echo cold rc=$?; tail -3 $O/cold.log
