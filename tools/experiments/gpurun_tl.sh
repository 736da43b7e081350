for w in 0 32 256; do
timeout 60 python tools/profile_gemm.py --m 512 --n 512 --k 16384 --policy ask --iters 20 --flush --warm $w
timeout 60 python tools/profile_gemm.py --m 512 --n 512 --k 16384 --policy ask --tile 256x256x64 --iters 20 --flush --warm $w
timeout 60 python tools/profile_gemm.py --m 1024 --n 1024 --k 1024 --policy dp --iters 20 --flush --warm $w --dtype fp16
timeout 60 python tools/profile_gemm.py --m 128 --n 4096 --k 4096 --policy dp --iters 20 --flush --warm $w
timeout 60 python tools/profile_gemm.py --m 128 --n 4096 --k 4096 --policy ask --iters 20 --flush --warm $w
timeout 60 python tools/profile_gemm.py --m 8192 --n 8192 --k 8192 --policy dp --tile 256x256x64 --iters 6 --flush --warm $w
done
