O=gpurun_out/s3pf; mkdir -p $O
for pf in 0 2 4 8; do
  SKPP_SET=l2_prefetch=$pf timeout 120 python tools/steady_timeline.py --m 16 --n 4096 --k 4096 --tile 128x128x128 --policy hybrid1 > $O/steady_$pf.txt 2>&1
  echo "l2_prefetch=$pf"; grep "us/step\|first_full\|first_tma\|mma_done" $O/steady_$pf.txt | tail -4
done
for pf in 0 2 4 8; do
  SKPP_SET=l2_prefetch=$pf timeout 120 python tools/steady_timeline.py --m 512 --n 512 --k 16384 --tile 128x128x128 --policy hybrid1 > $O/steady_cfg2_$pf.txt 2>&1
  echo "cfg2 l2_prefetch=$pf"; grep "us/step\|first_full\|first_tma\|mma_done" $O/steady_cfg2_$pf.txt | tail -4
done
