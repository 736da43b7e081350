# session 5: last check of the committed tree after the grid-parameter change
O=gpurun_out/s5last; mkdir -p $O
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_20.json 2> $O/bench_20.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench_20.json'));print(d['value'],d['config']['tile'],d['config']['policy'],d['roofline']['frac'],d['sweep']['pct_within_20pct_of_oracle'])"
