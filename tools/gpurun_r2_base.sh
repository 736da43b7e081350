# round 2 base check at HEAD: smoke, GPU tests, square8192 + cfg2 bench lines
O=gpurun_out/r2base; mkdir -p $O
nproc > $O/nproc.txt; nvidia-smi > $O/smi.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 $O/gpu_tests.log
timeout 600 python bench.py --workload square8192 --steps 200 --warmup 5 > $O/bench_sq.log 2>&1; echo bench rc=$?
tail -c 1500 $O/bench_sq.log
