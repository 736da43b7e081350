for a in 0 3 6 10 0 3 6; do echo ahead=$a
 SKPP_AHEAD=$a python tools/launch_modes.py 512 512 16384 ask 128x128x128 | grep "pdl=1"
 SKPP_AHEAD=$a python tools/launch_modes.py 1 14336 4096 dp 128x128x128 | grep "pdl=1"
 SKPP_AHEAD=$a python tools/launch_modes.py 4096 4096 4096 dp 256x256x128 | grep "pdl=1"
 SKPP_AHEAD=$a python tools/launch_modes.py 256 4096 4096 hybrid1 128x128x128 | grep "pdl=1"
done
