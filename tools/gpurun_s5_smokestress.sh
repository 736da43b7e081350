# session 5: stress the smoke() shape (24 one-iteration contributors per tile, 4 idle CTAs) through the
# phase-2 timeout / abandon paths: zero wait bound (debug 2, 3) and partial residency (SMs held)
O=gpurun_out/s5s; mkdir -p $O
for D in 2 3 18; do timeout 300 python tools/smoke_diag.py --reps 300 --debug $D >> $O/diag.jsonl 2>> $O/diag.err; done
timeout 300 python tools/smoke_diag.py --reps 100 --debug 2 --fresh-plan >> $O/diag.jsonl 2>> $O/diag.err
for H in 140 120 100 60 20; do
  SKPP_LIVENESS_SHAPE=384,256,1536 timeout 200 python tests/_liveness_worker.py partial 6 $H 21 $PWD > $O/partial_$H.log 2>&1; echo "hold $H rc=$?"; tail -2 $O/partial_$H.log
done
python - <<'PY'
import json
for l in open('gpurun_out/s5s/diag.jsonl'):
    d = json.loads(l); print(d['debug'], d['fresh_plan'], {k: (v['fails'], v['first']) for k, v in d.items() if isinstance(v, dict)})
PY
tail -3 $O/diag.err
