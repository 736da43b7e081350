# session 5: fixup-workspace zero-fill vs the PDL launch right behind it
O=gpurun_out/s5p; mkdir -p $O
for args in "--mode default" "--mode default --stream side" "--mode nopdl" "--mode sync" "--mode default --ws-mib 20 --trials 200" "--mode default --ws-mib 20 --trials 200 --stream side"; do
  timeout 300 python tools/pdl_ws_race.py $args >> $O/race.jsonl 2>> $O/race.err; echo "$args rc=$?"
done
cat $O/race.jsonl; tail -3 $O/race.err
