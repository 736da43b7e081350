# steady-state (bench protocol) timelines of launches S-1, S for the fixup-bound shapes
O=gpurun_out/s3steady; mkdir -p $O
for spec in "16 4096 4096 128x128x128 hybrid1" "128 4096 4096 128x128x128 hybrid1" "512 512 16384 128x128x128 hybrid1"; do
  set -- $spec
  timeout 120 python tools/steady_timeline.py --m $1 --n $2 --k $3 --tile $4 --policy $5 >> $O/steady.txt 2>&1
done
cat $O/steady.txt
