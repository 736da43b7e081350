# round 2 final production sweep (session-3 kernel): 7 tiles incl. the banded tile orders, paper grid + Llama-3-8B shapes,
# independent re-measurement (validate) and 300 off-grid held-out sizes
O=gpurun_out/sweep_r2f; mkdir -p $O
timeout 1500 python -m paper_2408_11417_b200.sweep --out $O --grid paper+llama \
  --tiles 128x128x64,128x64x128,128x128x128,256x256x64,256x256x128,128x128x128b16,256x256x128b16 \
  --validate --heldout 300 > $O/sweep.log 2>&1; echo sweep rc=$?
tail -c 3000 $O/sweep.log
