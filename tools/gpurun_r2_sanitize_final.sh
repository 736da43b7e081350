# sanitizers on the final round-2 kernel (session 3: udiv decode, first item before the wait,
# release-only publish): memcheck / racecheck / synccheck on CG=1 and the banded CTA pair
O=gpurun_out/san3; mkdir -p $O
run() {  # tool name args...
  tool=$1; name=$2; shift 2
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/profile_gemm.py "$@" > $O/${tool}_$name.txt 2>&1
  echo "$tool $name rc=$? :: $(tail -1 $O/${tool}_$name.txt)"
}
run memcheck decode16 --m 16 --n 4096 --k 4096 --policy hybrid1 --tile 128x128x128 --iters 2
run memcheck cfg2 --m 512 --n 512 --k 16384 --policy hybrid1 --tile 128x128x128 --iters 2
run memcheck pair_banded --m 2048 --n 2560 --k 520 --policy hybrid3 --tile 256x256x128b16 --iters 2
run racecheck cfg2ask --m 512 --n 512 --k 2048 --policy ask --tile 128x128x64 --iters 1
run synccheck cfg2h1 --m 512 --n 512 --k 2048 --policy hybrid1 --tile 128x128x64 --iters 1
run synccheck pair_banded --m 2048 --n 2560 --k 520 --policy hybrid1 --tile 256x256x128b16 --iters 1
SKPP_DEBUG=2 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/profile_gemm.py --m 512 --n 512 --k 8192 --policy ask --tile 128x128x64 --iters 2 > $O/memcheck_bound0.txt 2>&1; echo "memcheck bound0 rc=$? :: $(tail -1 $O/memcheck_bound0.txt)"
