# parity (pytest -m gpu, smoke) + compute-sanitizer on the Stream-K fixup paths
set -x
O=gpurun_out/verify; mkdir -p $O
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 $O/gpu_tests.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/profile_gemm.py --m 300 --n 200 --k 520 --policy ask --tile 128x128x128 --iters 2 > $O/memcheck_ask.txt 2>&1; echo memcheck rc=$?
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/profile_gemm.py --m 600 --n 392 --k 1000 --policy hybrid2 --tile 256x256x128 --iters 2 > $O/memcheck_pair.txt 2>&1; echo memcheck pair rc=$?
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/profile_gemm.py --m 512 --n 512 --k 2048 --policy ask --tile 128x128x64 --iters 1 > $O/racecheck.txt 2>&1; echo racecheck rc=$?
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/profile_gemm.py --m 512 --n 512 --k 2048 --policy hybrid1 --tile 128x128x64 --iters 1 > $O/synccheck.txt 2>&1; echo synccheck rc=$?
for f in $O/memcheck_ask.txt $O/memcheck_pair.txt $O/racecheck.txt $O/synccheck.txt; do tail -n 2 $f; done #/memcheck_ask.txt $O/memcheck_pair.txt $O/racecheck.txt $O/synccheck.txt
# skinny / ragged paths (A box of round_up(M,8) rows, partial rows skipped)
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/profile_gemm.py --m 16 --n 600 --k 1000 --policy ask --tile 128x128x128 --iters 2 > $O/memcheck_skinny.txt 2>&1; echo memcheck skinny rc=$?
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/profile_gemm.py --m 20 --n 600 --k 4096 --policy hybrid1 --tile 256x256x128 --iters 1 > $O/racecheck_pair_skinny.txt 2>&1; echo racecheck pair skinny rc=$?
for f in $O/memcheck_skinny.txt $O/racecheck_pair_skinny.txt; do tail -n 2 $f; done
# banded tile order (RASTER instantiation; auto on >= 4 waves): memcheck + racecheck + synccheck
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_gemm.py -m gpu -q -k banded -p no:cacheprovider > $O/memcheck_banded.txt 2>&1; echo memcheck banded rc=$?
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/profile_gemm.py --m 4000 --n 4104 --k 520 --policy hybrid1 --tile 128x128x128b16 --iters 1 > $O/racecheck_banded.txt 2>&1; echo racecheck banded rc=$?
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/profile_gemm.py --m 4000 --n 4104 --k 520 --policy hybrid1 --tile 128x128x128b16 --iters 1 > $O/synccheck_banded.txt 2>&1; echo synccheck banded rc=$?
for f in $O/memcheck_banded.txt $O/racecheck_banded.txt $O/synccheck_banded.txt; do tail -n 2 $f; done
