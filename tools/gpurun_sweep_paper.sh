set -x
mkdir -p gpurun_out/sweep_paper
timeout 3000 python -m paper_2408_11417_b200.sweep --out gpurun_out/sweep_paper --grid paper+llama --tile 128x128x64 > gpurun_out/sweep_paper/log.txt 2>&1; echo rc=$?
tail -3 gpurun_out/sweep_paper/log.txt
