# session 5: smoke() first thing on a fresh box, then compute-sanitizer (memcheck, racecheck, synccheck, initcheck)
# on the smoke sequence (DP, hybrid1, all-streamk at 384x256x1536, tile 128x128x64)
O=gpurun_out/s5z; mkdir -p $O
nvidia-smi --query-gpu=clocks.sm,pstate,power.draw --format=csv,noheader > $O/clocks.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke_first.log 2>&1; echo "smoke first rc=$?"; tail -c 600 $O/smoke_first.log
timeout 120 python tools/smoke_cold.py > $O/cold_first.json 2>&1; cat $O/cold_first.json
for T in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/smoke_cold.py > $O/san_$T.txt 2>&1; echo "$T rc=$?"; tail -3 $O/san_$T.txt
done
