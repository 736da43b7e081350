timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask --tile 128x256x64
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask --tile 256x256x64
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask --tile 256x128x64
python tools/timeline.py --m 1024 --n 1024 --k 1024 --policy hybrid1
python tools/timeline.py --m 1 --n 64 --k 65536 --policy ask
for t in 128x128x64 128x256x64 256x256x64 256x128x64; do timeout 60 python tools/profile_gemm.py --m 512 --n 512 --k 16384 --policy ask --tile $t --iters 20 --flush; done
for t in 128x256x64 256x256x64 256x128x64; do timeout 60 python tools/profile_gemm.py --m 8192 --n 8192 --k 8192 --policy dp --tile $t --iters 10; done
