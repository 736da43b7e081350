# session 5: fresh-process smoke sequence in a loop (~25 min) to estimate the rate of the one-off
# fresh-box mismatch; every 10th iteration follows 15 s of GPU idle
O=gpurun_out/s5l; mkdir -p $O
end=$(( $(date +%s) + ${SMOKE_LOOP_SECONDS:-1500} ))
i=0
while [ $(date +%s) -lt $end ]; do
  i=$((i+1))
  timeout 120 python tools/smoke_cold.py >> $O/cold.jsonl 2>> $O/cold.err || echo "iter $i rc=$?" >> $O/rc.txt
  if [ $((i % 10)) -eq 0 ]; then sleep 15; fi
done
python - <<'PY'
import json
n = bad = 0
for l in open('gpurun_out/s5l/cold.jsonl'):
    d = json.loads(l); n += 1
    if not all(v['ok'] for v in d.values()):
        bad += 1; print(l.strip()[:3000])
print(f"processes {n}, with a mismatch {bad}")
PY
