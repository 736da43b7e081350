for t in 128x128x128 256x128x128 256x256x128; do
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask --tile $t --kstamps 16 2>&1 | grep -E "ask tile|mean arrival|mma_done|phase1|waited|phase2|k +[0-9]+:"
done
