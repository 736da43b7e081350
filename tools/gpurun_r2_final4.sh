# round 2 final evidence on the owner-reduction kernel (outputs kept under gpurun's 64 MiB:
# ncu reports stay in /tmp on the box, only their JSON summaries come back): GPU suite + smoke +
# 1000-case fuzz, sanitizers, final 7-tile sweep (-> shipped bank), then with that bank: default
# bench, reference arm, cfg2 bench, ncu of the selected cfg3 / cfg2 / decode16 kernels, launch
# list, Llama cfg3 table
O=gpurun_out/prof6; mkdir -p $O; R=/tmp/ncu6; rm -rf $R; mkdir -p $R
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo tests rc=$?; tail -1 $O/gpu_tests.log
SKPP_FUZZ_CASES=1000 timeout 1500 python -m pytest tests/test_gpu_gemm.py -q -k fuzz > $O/fuzz_1000.txt 2>&1; echo fuzz rc=$?; tail -1 $O/fuzz_1000.txt
bash tools/gpurun_r2_sanitize_final.sh > $O/sanitizers.txt 2>&1; cat $O/sanitizers.txt; mkdir -p $O/san; cp gpurun_out/san3/*.txt $O/san/; rm -rf gpurun_out/san3
OS=gpurun_out/sweep_r2h; mkdir -p $OS
timeout 1500 python -m paper_2408_11417_b200.sweep --out $OS --grid paper+llama \
  --tiles 128x128x64,128x64x128,128x128x128,256x256x64,256x256x128,128x128x128b16,256x256x128b16 \
  --validate --heldout 300 > $OS/sweep.log 2>&1; echo sweep rc=$?; rm -f $OS/validate.*.csv
rm -rf paper_2408_11417_b200/banks/b200 && cp -r $OS/tilebank paper_2408_11417_b200/banks/b200
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference_cfg3.json 2> $O/bench_reference.err; echo ref rc=$?
timeout 600 python bench.py --workload cfg2 --steps 2000 --sweep-grid none > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo cfg2 rc=$?
SEL=$(python -c "import json;d=json.loads(open('$O/bench_cfg3.json').read().strip().splitlines()[-1]);print(d['selection']['selected'])")
echo "cfg3 selected $SEL"
TILE=${SEL%/*}; POL=${SEL#*/}
cap() {  # name m n k policy tile dtype
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:streamk_gemm -s 3 -c 1 -o $R/$1 \
    python tools/profile_gemm.py --m $2 --n $3 --k $4 --policy $5 --tile $6 --dtype $7 --iters 4 > $O/$1.log 2>&1; echo ncu $1 rc=$?
}
cap cfg3_${TILE}_${POL} 8192 14336 4096 $POL $TILE bf16
cap cfg2_128x128x128_hybrid1 512 512 16384 hybrid1 128x128x128 bf16
cap decode16_128x128x128_hybrid1 16 4096 4096 hybrid1 128x128x128 bf16
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $R/launches_cfg3.csv python bench.py --steps 20 --warmup 3 --e2e-steps 2 --cpu-seconds 1 --sweep-grid none > $O/launches_bench.json 2>&1; echo launches rc=$?
python tools/collect_profiles.py $R profiles/round2/final > $O/collect.log 2>&1; echo collect rc=$?
mkdir -p $O/profiles; cp profiles/ncu_bench_*.json $O/profiles/; cp profiles/round2/final/ncu_*.json profiles/round2/final/launches_cfg3.json $O/profiles/ 2>/dev/null
for f in $R/*.ncu-rep; do n=$(basename $f .ncu-rep); timeout 300 ncu -i $f --page source --csv --print-source sass > $R/$n.sass.csv 2>/dev/null; python tools/ncu_hot.py $R/$n.sass.csv 25 > $O/$n.hot_sass.txt 2>&1; done
timeout 1500 python tools/llama_bench_table.py --oracle --md $O/llama_cfg3_table.md > $O/llama_cfg3_table.jsonl 2> $O/llama.err; echo llama rc=$?; tail -3 $O/llama_cfg3_table.md
du -sh gpurun_out
