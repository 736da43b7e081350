# session 5: smoke() failed on a fresh box at HEAD (hybrid1 max |diff| 2196); bisect across kernel builds
O=gpurun_out/s5d; mkdir -p $O
H=$PWD/paper_2408_11417_b200/libskpp.so
for L in $H $PWD/tools/ablibs/libskpp_43840e3.so $PWD/tools/ablibs/libskpp_161c577.so; do
  for i in 1 2 3; do SKPP_LIB=$L timeout 120 python __graft_entry__.py smoke > $O/smoke_$(basename $L)_$i.log 2>&1; echo "$(basename $L) smoke $i rc=$?"; done
  for D in 0 1 16; do SKPP_LIB=$L timeout 300 python tools/smoke_diag.py --reps 200 --debug $D >> $O/diag.jsonl 2>> $O/diag.err; done
  SKPP_LIB=$L timeout 300 python tools/smoke_diag.py --reps 100 --fresh-plan >> $O/diag.jsonl 2>> $O/diag.err
done
tail -5 $O/diag.err
