timeout 900 python -m cProfile -o gpurun_out/sweep.prof -m paper_2408_11417_b200.sweep --out gpurun_out/sp5 --grid paper --tiles 128x128x64,128x64x128,128x128x128,256x256x64,256x256x128 --max-gflop 0.05 > gpurun_out/sp5.log 2>&1
python -c "
import pstats; p=pstats.Stats('gpurun_out/sweep.prof'); p.sort_stats('cumulative').print_stats(25)" > gpurun_out/sweep_prof.txt 2>&1
python -c "
import pstats; p=pstats.Stats('gpurun_out/sweep.prof'); p.sort_stats('tottime').print_stats(20)" >> gpurun_out/sweep_prof.txt 2>&1
python -c "import json;d=json.load(open('gpurun_out/sp5/summary.json'));print(d['sizes'], d['sweep_seconds_max_over_ranks'])"
