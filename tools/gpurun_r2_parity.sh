# round 2: full GPU suite (incl. cfg1/cfg2/cfg3 full-size parity), sanitizers on the banded pair
# kernel <256,128,2,1>, ncu launch list of the cfg3 parity tests, then the 8-tile sweep.
O=gpurun_out/r2parity; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -5 $O/gpu_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:streamk_gemm --csv --log-file $O/launches_cfg3_tests.csv \
  python -m pytest tests/test_gpu_configs.py -q -k "cfg3_selected and 8192x14336" -p no:cacheprovider > $O/ncu_tests.log 2>&1; echo ncu tests rc=$?
grep -o 'streamk_gemm_kernel<[^>]*>' $O/launches_cfg3_tests.csv | sort | uniq -c
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/profile_gemm.py --m 2048 --n 2560 --k 520 --policy hybrid1 --tile 256x256x128b16 --iters 1 > $O/${tool}_pair_banded.txt 2>&1; echo $tool pair banded rc=$?
  tail -n 2 $O/${tool}_pair_banded.txt
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/profile_gemm.py --m 1500 --n 4096 --k 4096 --policy ask --tile 256x256x128b16 --iters 2 > $O/memcheck_pair_banded_ask.txt 2>&1; echo memcheck ask rc=$?
tail -n 2 $O/memcheck_pair_banded_ask.txt
