# A/B the working tree against the build in _orig/ (SKPP_PKG_ROOT)
for root in "" _orig; do
  echo "== ${root:-new}"
  SKPP_PKG_ROOT=$root python tools/launch_modes.py 512 512 16384 ask 128x128x128 | grep "pdl=1"
  SKPP_PKG_ROOT=$root python tools/launch_modes.py 1 4096 4096 hybrid1 128x128x128 | grep "pdl=1"
  SKPP_PKG_ROOT=$root python tools/launch_modes.py 64 4096 4096 hybrid1 128x128x128 | grep "pdl=1"
  SKPP_PKG_ROOT=$root python tools/launch_modes.py 256 4096 4096 hybrid1 128x128x128 | grep "pdl=1"
  SKPP_PKG_ROOT=$root python tools/launch_modes.py 1000 1000 1000 hybrid1 128x128x128 | grep "pdl=1"
  SKPP_PKG_ROOT=$root python tools/launch_modes.py 1024 14336 4096 hybrid1 256x256x64 | grep "pdl=1"
  SKPP_PKG_ROOT=$root python tools/launch_modes.py 300 5000 2000 hybrid1 128x128x128 | grep "pdl=1"
done
