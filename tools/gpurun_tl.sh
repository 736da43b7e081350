timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask
python tools/timeline.py --m 512 --n 512 --k 16384 --policy ask --tile 128x256x64
python tools/timeline.py --m 1024 --n 1024 --k 1024 --policy hybrid1
python tools/timeline.py --m 1 --n 64 --k 65536 --policy ask
for pol in dp ask; do timeout 60 python tools/profile_gemm.py --m 512 --n 512 --k 16384 --policy $pol --iters 20 --flush; done
timeout 60 python tools/profile_gemm.py --m 512 --n 512 --k 16384 --policy ask --tile 128x256x64 --iters 20 --flush
