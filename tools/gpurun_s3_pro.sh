O=gpurun_out/s3pro; mkdir -p $O
for dbg in 0 16; do
  SKPP_DEBUG=$dbg timeout 120 python tools/steady_timeline.py --m 16 --n 4096 --k 4096 --tile 128x128x128 --policy hybrid1 > $O/steady_$dbg.txt 2>&1
  grep "us/step\|prologue\|SM cycles" $O/steady_$dbg.txt
done
