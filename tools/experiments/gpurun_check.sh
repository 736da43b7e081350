# GPU parity + quick perf check (development loop)
set -x
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -15 gpurun_out/gpu_tests.log
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask --tile 128x256x64
python tools/timeline.py --m 128 --n 128 --k 64 --policy dp
python tools/timeline.py --m 1024 --n 1024 --k 1024 --policy hybrid1
python tools/timeline.py --m 1024 --n 1024 --k 1024 --policy dp
for pol in dp ask; do timeout 60 python tools/profile_gemm.py --m 512 --n 512 --k 16384 --policy $pol --iters 20 --flush; done
timeout 60 python tools/profile_gemm.py --m 128 --n 4096 --k 4096 --policy dp --iters 20
timeout 60 python tools/profile_gemm.py --m 8192 --n 8192 --k 8192 --policy dp --tile 128x256x64 --iters 10
timeout 300 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench rc=$?
tail -2 gpurun_out/bench_cfg2.err
