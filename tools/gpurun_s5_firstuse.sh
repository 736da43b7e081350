# session 5: fresh processes — does a PDL GEMM ever read an operand before the first-use torch kernel that wrote it finished?
O=gpurun_out/s5u; mkdir -p $O
end=$(( $(date +%s) + ${LOOP:-900} ))
while [ $(date +%s) -lt $end ]; do
  timeout 120 python tools/pdl_firstuse.py >> $O/firstuse.jsonl 2>> $O/firstuse.err
done
python - <<'PY'
import json
n = 0; bad = {}
for l in open('gpurun_out/s5u/firstuse.jsonl'):
    d = json.loads(l); n += 1
    for k, v in d.items():
        if not v: bad[k] = bad.get(k, 0) + 1
print(f"processes {n}, failed events {bad}")
PY
tail -3 $O/firstuse.err
