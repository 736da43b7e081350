# same-box A/B of kernel builds (args: lib list for tools/ab_libs.py), output under gpurun_out/s3ab
O=gpurun_out/s3ab; mkdir -p $O
export SKPP_AB_CASES="${SKPP_AB_CASES:-16:4096:4096:128x128x128:hybrid1,128:4096:4096:128x128x128:hybrid1,1:4096:4096:128x128x128:hybrid1,512:512:16384:128x128x128:hybrid1,1024:1024:1024:128x128x64:hybrid1}"
timeout 1200 python tools/ab_libs.py --libs "$1" --rounds ${ROUNDS:-3} > $O/ab_$2.txt 2>&1; echo ab rc=$?; cat $O/ab_$2.txt
