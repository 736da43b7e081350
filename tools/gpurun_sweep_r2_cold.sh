# round 2 production sweep, cold-L2 timing for sizes whose operands fit in the L2:
# 7 tiles incl. the banded tile orders, paper grid + Llama-3-8B shapes, independent
# re-measurement (validate) and 300 off-grid held-out sizes
O=gpurun_out/sweep_r2c; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_api.py -q -k cold > $O/test_cold.log 2>&1; echo test rc=$?; tail -2 $O/test_cold.log
timeout 2400 python -m paper_2408_11417_b200.sweep --out $O --grid paper+llama --cold \
  --tiles 128x128x64,128x64x128,128x128x128,256x256x64,256x256x128,128x128x128b16,256x256x128b16 \
  --validate --heldout 300 > $O/sweep.log 2>&1; echo sweep rc=$?
tail -c 1500 $O/sweep.log
