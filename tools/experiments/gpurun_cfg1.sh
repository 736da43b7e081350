for t in 128x128x128 128x64x128 128x64x64 128x128x64 256x128x128; do
  for pol in dp hybrid1; do python tools/launch_modes.py 1024 1024 1024 $pol $t | grep "pdl=1"; done
done
