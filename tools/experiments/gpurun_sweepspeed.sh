# sweep host-overhead check: small grid, one tile, old vs new time_plan
for root in "" _orig; do echo "== ${root:-new}"
  PYTHONPATH=$root timeout 900 python -m paper_2408_11417_b200.sweep --out gpurun_out/ss_${root:-new} --grid paper --tiles 128x128x128 > gpurun_out/ss_${root:-new}.log 2>&1
  python -c "import json;d=json.load(open('gpurun_out/ss_${root:-new}/summary.json'));print(d['sizes'], d['sweep_seconds_max_over_ranks'], d['shape_policy_per_s'])"
done
