# round 2, session 3 re-baseline at HEAD: GPU suite, timelines of the shapes furthest below
# roofline (cfg2, decode M=16/128), default bench line
O=gpurun_out/s3base; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 $O/gpu_tests.log
for spec in "512 512 16384 128x128x128 hybrid1" "16 4096 4096 128x128x128 hybrid1" "128 4096 4096 128x128x128 hybrid1" "16 4096 4096 128x128x128 dp" "128 4096 4096 128x64x128 dp"; do
  set -- $spec
  timeout 120 python tools/timeline.py --m $1 --n $2 --k $3 --tile $4 --policy $5 --flush --per-cta 12 >> $O/timeline.txt 2>&1
done
timeout 600 python tools/ab_libs.py --libs tools/ab_libs/libskpp_head.so --rounds 1 > $O/ab_head.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_default.log 2>&1; echo bench rc=$?
tail -c 600 $O/bench_default.log
