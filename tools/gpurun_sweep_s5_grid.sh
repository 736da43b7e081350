# session 5: the production sweep with the persistent grid size as a tile parameter — the 7 shipped tiles plus
# 128x128x128 on 128 / 144 workgroups and 128x64x128 on 128; paper grid + Llama shapes, re-measurement, held-out sizes
O=gpurun_out/sweep_s5g; mkdir -p $O
timeout 1500 python -m paper_2408_11417_b200.sweep --out $O --grid paper+llama \
  --tiles 128x128x64,128x64x128,128x128x128,256x256x64,256x256x128,128x128x128b16,256x256x128b16,128x128x128g128,128x128x128g144,128x64x128g128 \
  --validate --heldout 300 > $O/sweep.log 2>&1; echo sweep rc=$?
tail -c 2500 $O/sweep.log
