for t in 128x64x64 128x128x64 128x256x64 256x128x64 256x256x64; do
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask --tile $t --kstamps 1 2>&1 | grep -E "ask tile|mean arrival"
python tools/timeline.py --m 8192 --n 8192 --k 8192 --policy dp --tile $t --kstamps 1 2>&1 | grep -E "dp tile|mean arrival"
done
