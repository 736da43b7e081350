# round 2: cold-L2 sweep (rotating operand sets for every size up to 2.5x L2) vs the shipped warm-swept
# bank, both judged by the in-run cold oracle of tools/llama_bench_table.py on the same box
O=gpurun_out/coldsweep; mkdir -p $O; OS=$O/sweep
timeout 900 python tools/llama_bench_table.py --oracle --md $O/llama_shipped.md > $O/llama_shipped.jsonl 2> $O/llama_shipped.err; echo llama shipped rc=$?; tail -3 $O/llama_shipped.md
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_cfg3_shipped.json 2> $O/bench_shipped.err; echo bench rc=$?
mkdir -p $OS
timeout 2700 python -m paper_2408_11417_b200.sweep --out $OS --grid paper+llama --cold \
  --tiles 128x128x64,128x64x128,128x128x128,256x256x64,256x256x128,128x128x128b16,256x256x128b16 \
  --validate --heldout 300 > $OS/sweep.log 2>&1; echo sweep rc=$?; rm -f $OS/validate.*.csv; head -c 400 $OS/sweep.log
rm -rf paper_2408_11417_b200/banks/b200 && cp -r $OS/tilebank paper_2408_11417_b200/banks/b200
timeout 900 python tools/llama_bench_table.py --oracle --md $O/llama_cold.md > $O/llama_cold.jsonl 2> $O/llama_cold.err; echo llama cold rc=$?; tail -3 $O/llama_cold.md
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_cfg3_cold.json 2> $O/bench_cold.err; echo bench rc=$?
du -sh gpurun_out/coldsweep
