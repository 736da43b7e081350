# session 5: try to reproduce the fresh-box smoke() mismatch — fresh processes after the GPU idles
O=gpurun_out/s5c; mkdir -p $O
for i in $(seq 1 12); do
  nvidia-smi --query-gpu=clocks.sm,pstate --format=csv,noheader >> $O/clocks.txt
  timeout 120 python tools/smoke_cold.py >> $O/cold.jsonl 2>> $O/cold.err
  sleep 20
done
python - <<'PY'
import json
for l in open('gpurun_out/s5c/cold.jsonl'):
    d = json.loads(l); print({k: v['ok'] for k, v in d.items()})
PY
