# round 2: cooperative-launch check (GPU suite incl. liveness tests, A/B cost) and the
# ncu-measured fixup-workspace traffic (Stream-K policy vs data-parallel, same shape and tile).
set -x
O=gpurun_out/coopfix; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf -x > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 $O/gpu_tests.log
timeout 600 python tools/ab_coop.py > $O/ab_coop.jsonl 2> $O/ab_coop.err; echo ab rc=$?
cat $O/ab_coop.jsonl
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
