# session 5 final: the committed tree as the driver runs it — smoke, GPU suite, default bench, reference arm
O=gpurun_out/s5final; mkdir -p $O
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_20.json 2> $O/bench_20.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference_20.json 2> $O/bench_reference_20.err; echo "ref rc=$?"
SMOKE_LOOP_SECONDS=600 bash tools/gpurun_s5_smokeloop.sh | tail -2
