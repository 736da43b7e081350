# session 5: after the workspace-fill sync — fresh-process smoke loop, GPU suite, default bench
O=gpurun_out/s5f; mkdir -p $O
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
mkdir -p gpurun_out/s5l; rm -f gpurun_out/s5l/cold.jsonl
SMOKE_LOOP_SECONDS=${LOOP:-1080} bash tools/gpurun_s5_smokeloop.sh | tail -4
