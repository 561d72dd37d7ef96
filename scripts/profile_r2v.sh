#!/bin/bash
# Round-2 lines after lazy staging / retire-once / per-CTA totals / hashed
# summaries (r2v): smoke, bench lines without a profiler, iteration profiles,
# then the ncu launch list and one full capture per headline configuration.
R=${R:-r2v}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${R}_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --scale 22 --no-cpu-baseline > gpurun_out/${R}_s22_selmax.json 2> gpurun_out/${R}_s22.err
python bench.py --graph er --no-cpu-baseline > gpurun_out/${R}_er.json 2> gpurun_out/${R}_er.err
python bench.py --variant tropical --no-cpu-baseline > gpurun_out/${R}_s26_tropical.json 2> gpurun_out/${R}_s26t.err
for c in "--scale 26" "--scale 22" "--scale 26 --graph er" "--scale 26 --variant 0"; do
  python scripts/iter_profile.py $c >> gpurun_out/${R}_iterprof.jsonl 2>/dev/null
done
python scripts/k3_per_root.py > gpurun_out/${R}_s26_k3_per_root.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-validate --e2e-steps 0 > gpurun_out/${R}_ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bfs32 -s 1 -c 1 -o gpurun_out/${R}_bfs32_full \
    python scripts/prof_iter.py --iters 100 --L 2048 --root 2564265 > gpurun_out/${R}_ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:bfs32 -s 1 -c 1 -o gpurun_out/${R}_bfs32_s22_full \
    python scripts/prof_iter.py --scale 22 --iters 100 --L 2048 --g500 0 > gpurun_out/${R}_ncu_s22.log 2>&1
