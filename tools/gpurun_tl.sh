timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python tools/launch_overhead.py
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask
python tools/timeline.py --m 1024 --n 1024 --k 1024 --policy hybrid1
for t in 128x128x64 256x256x64; do timeout 60 python tools/profile_gemm.py --m 512 --n 512 --k 16384 --policy ask --tile $t --iters 20 --flush; done
timeout 60 python tools/profile_gemm.py --m 1024 --n 1024 --k 1024 --policy hybrid1 --iters 20 --flush
timeout 60 python tools/profile_gemm.py --m 1024 --n 1024 --k 1024 --policy dp --iters 20 --flush
timeout 60 python tools/profile_gemm.py --m 8192 --n 8192 --k 8192 --policy dp --tile 256x256x64 --iters 10
timeout 300 python bench.py > gpurun_out/bench_cfg2.json 2>gpurun_out/bench_cfg2.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg2.json').read().splitlines()[-1]); print('BENCH', d['value'], d['ms_per_step'], d['roofline']['frac'], d['selection']['per_policy_tflops']['hybrid1'], d['e2e']['value'])"
