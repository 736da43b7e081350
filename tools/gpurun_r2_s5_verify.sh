# session 5: HEAD verification on a fresh box — smoke, GPU suite, default bench, reference arm
set -x
O=gpurun_out/s5v; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvsmi.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo bench rc=$?
tail -c 300 $O/bench_default.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo ref rc=$?
