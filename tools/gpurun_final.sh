# round-end style check: build from source, smoke, GPU tests, default bench, reference arm
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final_build.log 2>&1; echo build rc=$?
timeout 300 python __graft_entry__.py smoke; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench rc=$?
timeout 300 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/final_ref.json 2>&1; echo ref rc=$?
python -c "import json;d=json.load(open('gpurun_out/final_bench.json'));print(d['value'],d['ms_per_step'],d['config']['tile'],d['config']['policy'],d['roofline']['frac'],d['e2e']['value'],d['clocks'])"
tail -c 400 gpurun_out/final_ref.json
