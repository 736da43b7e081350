# round 2: liveness protocol — liveness tests, the full GPU suite, sanitizers on the
# timeout/abandon paths, and a same-box A/B of per-launch time against the pre-protocol build
set -x
O=gpurun_out/live; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_liveness.py -q -rf -x > $O/liveness.log 2>&1; echo liveness rc=$?
tail -3 $O/liveness.log
timeout 300 python tests/_liveness_worker.py partial 2 140 14 . > $O/partial140.txt 2>&1; echo partial rc=$?
cat $O/partial140.txt
timeout 1500 python -m pytest tests -m gpu -q -rf -x > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 $O/gpu_tests.log
SKPP_DEBUG=2 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/profile_gemm.py --m 512 --n 512 --k 8192 --policy ask --tile 128x128x64 --iters 2 > $O/memcheck_bound0.txt 2>&1; echo memcheck rc=$?; tail -1 $O/memcheck_bound0.txt
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tests/_liveness_worker.py partial 1 140 16 . > $O/memcheck_partial.txt 2>&1; echo memcheck partial rc=$?; tail -3 $O/memcheck_partial.txt
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/profile_gemm.py --m 512 --n 512 --k 2048 --policy ask --tile 128x128x64 --iters 1 > $O/racecheck.txt 2>&1; echo racecheck rc=$?; tail -1 $O/racecheck.txt
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/profile_gemm.py --m 512 --n 512 --k 2048 --policy hybrid1 --tile 128x128x64 --iters 1 > $O/synccheck.txt 2>&1; echo synccheck rc=$?; tail -1 $O/synccheck.txt
timeout 1400 python tools/ab_libs.py --libs tools/ab_libs/libskpp_base.so,paper_2408_11417_b200/libskpp.so --rounds 2 > $O/ab.jsonl 2> $O/ab.err; echo ab rc=$?
cat $O/ab.jsonl
