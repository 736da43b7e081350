mkdir -p gpurun_out/tl
for lib in base prot4; do
 for shape in "--m 512 --n 512 --k 16384 --tile 128x128x128 --policy hybrid1" "--m 16 --n 4096 --k 4096 --tile 128x128x128 --policy hybrid1" "--m 1024 --n 1024 --k 1024 --tile 128x128x64 --policy hybrid1"; do
  SKPP_LIB=tools/ab_libs/libskpp_$lib.so timeout 120 python tools/timeline.py $shape >> gpurun_out/tl/$lib.txt 2>&1
 done
done
cat gpurun_out/tl/base.txt gpurun_out/tl/prot4.txt
