for m in 128 130 136 192 256 260 384; do python tools/launch_modes.py $m 4096 4096 hybrid1 128x128x128 | grep "pdl=1"; done
for m in 1024 1032 1100; do python tools/launch_modes.py $m 4096 4096 dp 128x128x128 | grep "pdl=1"; done
