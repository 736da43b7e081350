# session 5: BASELINE cfg3 Llama table (bench protocol, in-run cold oracle) with the shipped 7-tile bank and with the
# 10-tile grid bank, on the same box
O=gpurun_out/s5llama; mkdir -p $O
timeout 900 python tools/llama_bench_table.py --oracle --md $O/llama_shipped.md > $O/llama_shipped.jsonl 2> $O/llama_shipped.err; echo shipped rc=$?; tail -4 $O/llama_shipped.md
timeout 900 python tools/llama_bench_table.py --oracle --bank profiles/round2/session5/tilebank10_grid --md $O/llama_grid.md > $O/llama_grid.jsonl 2> $O/llama_grid.err; echo grid rc=$?; tail -4 $O/llama_grid.md
