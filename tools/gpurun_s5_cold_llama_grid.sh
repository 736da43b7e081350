# session 5: cold-L2 sweep of the Llama cfg3 shapes over the 7 shipped tiles + 128x128x128g144 (re-measured)
O=gpurun_out/sweep_s5cl; mkdir -p $O
timeout 1200 python -m paper_2408_11417_b200.sweep --out $O --grid llama --cold \
  --tiles 128x128x64,128x64x128,128x128x128,256x256x64,256x256x128,128x128x128b16,256x256x128b16,128x128x128g144 \
  --validate > $O/sweep.log 2>&1; echo sweep rc=$?
tail -c 800 $O/sweep.log
