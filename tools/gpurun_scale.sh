set -x
O=gpurun_out/scale; mkdir -p $O
timeout 2400 python -m paper_2408_11417_b200.sweep --out $O --grid paper+llama --tiles 128x128x64 --emulate-world 1,2,4,8 > $O/log.txt 2>&1; echo rc=$?
tail -c 2000 $O/log.txt
compute-sanitizer --version | head -2
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/profile_gemm.py --m 300 --n 200 --k 520 --policy ask --tile 128x128x64 --iters 2 > $O/memcheck_ask.txt 2>&1; echo memcheck rc=$?
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/profile_gemm.py --m 600 --n 392 --k 1000 --policy hybrid2 --tile 256x256x64 --iters 2 > $O/memcheck_pair.txt 2>&1; echo memcheck pair rc=$?
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/profile_gemm.py --m 512 --n 512 --k 2048 --policy ask --tile 128x128x64 --iters 1 > $O/racecheck.txt 2>&1; echo racecheck rc=$?
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/profile_gemm.py --m 512 --n 512 --k 2048 --policy hybrid1 --tile 128x128x64 --iters 1 > $O/synccheck.txt 2>&1; echo synccheck rc=$?
tail -3 $O/memcheck_ask.txt $O/memcheck_pair.txt $O/racecheck.txt $O/synccheck.txt
