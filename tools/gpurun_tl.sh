python tools/timeline.py --m 128 --n 4096 --k 4096 --policy dp --kstamps 20
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask --kstamps 14
python tools/timeline.py --m 8192 --n 8192 --k 8192 --policy dp --tile 256x256x64 --kstamps 14
