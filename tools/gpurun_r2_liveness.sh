# round 2: abandon protocol — liveness + abandon-path tests first (bounded), then the full
# GPU suite, the per-launch cost (tools/ab_coop.py: plain = protocol, coop = cooperative)
set -x
O=gpurun_out/live; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_liveness.py -q -rf -x > $O/liveness.log 2>&1; echo liveness rc=$?
tail -15 $O/liveness.log
timeout 1500 python -m pytest tests -m gpu -q -rf -x > $O/gpu_tests.log 2>&1; echo tests rc=$?
tail -3 $O/gpu_tests.log
timeout 600 python tools/ab_coop.py > $O/ab_coop.jsonl 2> $O/ab_coop.err; echo ab rc=$?
cat $O/ab_coop.jsonl
timeout 300 python tests/_liveness_worker.py partial 3 100 14 . > $O/partial.txt 2>&1; echo partial rc=$?
cat $O/partial.txt
