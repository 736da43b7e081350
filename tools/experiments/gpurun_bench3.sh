O=gpurun_out/bench3; mkdir -p $O
for wl in cfg2 cfg1 square8192; do
  steps=10000; [ $wl = square8192 ] && steps=300
  timeout 600 python bench.py --workload $wl --steps $steps > $O/bench_$wl.json 2> $O/bench_$wl.err; echo bench $wl rc=$?
  python -c "import json;d=json.load(open('$O/bench_$wl.json'));print(d['value'],d['ms_per_step'],d['config']['tile'],d['config']['policy'],d['roofline']['frac'],d['selection']['selected'],d['selection']['oracle_best'],d['isolated_launch']['us_median'],d['e2e']['value'],d['clocks'])"
done
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref rc=$?
cat $O/bench_reference.json
