set -x
mkdir -p gpurun_out/sweep_small
timeout 1500 python -m paper_2408_11417_b200.sweep --out gpurun_out/sweep_small --grid small+llama --tile 128x128x64 > gpurun_out/sweep_small/log.txt 2>&1; echo rc=$?
tail -3 gpurun_out/sweep_small/log.txt
