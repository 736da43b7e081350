set -x
O=gpurun_out/scale5; mkdir -p $O
timeout 2700 python -m paper_2408_11417_b200.sweep --out $O --grid paper+llama --tiles 128x128x64,128x64x128,128x128x128,256x256x64,256x256x128 --emulate-world 1,2,4,8 > $O/log.txt 2>&1; echo rc=$?
tail -c 3000 $O/log.txt
